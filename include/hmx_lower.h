/*
 * hmx_lower.h — C ABI of the native H-LU lowering (libhmxdag.so, host C++).
 *
 * Lowers the reference's recursive H-LU (arith.hlu, arith.py:76-140, or
 * accumulator.hlu_accu, accumulator.py:164-235, with their leaf kernels,
 * hmatrix.py:286-448) over a block table to the op program the device
 * executes (hmx_op records, include/hmx.h), and builds its execution graph.
 * The reference has no executor (SPEC.md:460-504 is absent); this is the
 * planning half of the one the build creates.  planner.py is the Python
 * statement of the same lowering; tests/test_lower_cpu.py requires equal
 * op records.
 */
#ifndef HMX_LOWER_H
#define HMX_LOWER_H

#include <stdint.h>

#include "hmx.h"
#include "hmx_dag.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hmx_prog hmx_prog;

/* Block table in uid pre-order: row / column ranges, leaf and admissible
 * flags, children (n x 4 row-major, -1 for leaves).  mode 0 = std (hlu),
 * 1 = accumulator (hlu_accu).  policy/fixed_rank/eps = TruncationPolicy
 * (HMX_POLICY_*).  rank_cap <= 0: no cap.  split_min > 0: H x H products
 * with min(m, n) >= split_min run as parallel micro-tasks.  caps: optional
 * per-uid capacity bound of low-rank leaves (-1 = none).  acc_budget > 0:
 * accumulator storage is reused by lifetime once the pool reaches that many
 * doubles (reuse ordered by extra execution edges); <= 0: one region per
 * accumulator (planner.py layout).  Returns 0; 1 bad
 * argument; 2 structural error (low-rank diagonal, non-conformal blocks);
 * 4 out of memory. */
int hmx_lower_hlu(int32_t n_blocks, const int64_t* r0, const int64_t* r1, const int64_t* c0,
                  const int64_t* c1, const int8_t* leaf, const int8_t* adm, const int32_t* kids,
                  int32_t mode, int32_t policy, int32_t fixed_rank, double eps, int64_t rank_cap,
                  int64_t split_min, const int32_t* caps, int64_t acc_budget, hmx_prog** out);
/* what: 0 tasks, 1 ops, 2 layout doubles, 3 accumulator pool doubles,
 * 4 workspace doubles, 5 workspace rank slots, 6 per-CTA scratch doubles,
 * 7 per-CTA rank slots, 8 update count, 9 execution edges (-1 before
 * hmx_prog_graph), 10 DAG edges, 11 edges beyond the DAG's. */
int64_t hmx_prog_count(const hmx_prog* prog, int32_t what);
/* Any pointer may be NULL.  ops[n_ops]; task_ops[n_tasks+1]; kind[n_tasks]
 * (hmx_dag.h kind codes, 11 = micro task); uids[n_tasks x 3] (-1 unused);
 * alpha[n_tasks]; task_scratch[n_tasks]; layout d_off/u_off/v_off/cap
 * [n_blocks]. */
int hmx_prog_export(const hmx_prog* prog, hmx_op* ops, int64_t* task_ops, int32_t* kind,
                    int32_t* uids, double* alpha, int64_t* task_scratch, int64_t* d_off,
                    int64_t* u_off, int64_t* v_off, int64_t* cap);
/* Execution graph over program tasks: mode 0 (std) = the DAG's edges plus
 * micro-task edges; mode 1 (accu) = data-flow edges of the sequential
 * program.  The DAG (hmx_dag_build of the same table, std or accu-merged)
 * must have exactly the planned tasks as nodes.  Returns 0; 1 bad
 * argument; 4 out of memory; 5 planned tasks differ from the DAG's nodes;
 * 6 an edge contradicts program order. */
int hmx_prog_graph(hmx_prog* prog, int32_t n_blocks, const int64_t* r0, const int64_t* r1,
                   const int64_t* c0, const int64_t* c1, const int8_t* leaf, const int8_t* adm,
                   const int32_t* kids, int32_t mode, const hmx_dag* dag);
/* succ_ptr[n_tasks+1], succ_idx[edges] (sorted rows). */
int hmx_prog_graph_export(const hmx_prog* prog, int64_t* succ_ptr, int32_t* succ_idx);
/* Release the per-task data-access records (kept for hmx_prog_graph). */
void hmx_prog_drop_access(hmx_prog* prog);
void hmx_prog_free(hmx_prog* prog);

#ifdef __cplusplus
}
#endif
#endif /* HMX_LOWER_H */
