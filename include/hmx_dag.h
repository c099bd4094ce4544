/*
 * hmx_dag.h — C ABI of the native task-DAG builder (libhmxdag.so, host C++).
 *
 * Replaces the refinement DAG construction of the reference
 * (hmatdag/taskgraph.py:530-665, compute_dag / build_hlu_dag, Alg. 10-12 and
 * 14-15 of arXiv 1911.07531) with the same node and edge sets (tests compare
 * them with the reference's own DAGs), optionally with the reference's edge
 * sparsification (Alg. 13, taskgraph.py:360-432).
 */
#ifndef HMX_DAG_H
#define HMX_DAG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hmx_dag hmx_dag;

/* Block table in uid pre-order (trees.py:181-199 numbering): row / column
 * ranges, leaf flags, parent uid (-1 at the root), children (n x 4, row-major
 * 2x2, -1 for leaves).  mode: 0 std, 1 accu-combined, 2 accu-merged;
 * root_op: 0 hlu (build_hlu_dag), 1 hmul, 2 htrsl, 3 htrsu (compute_dag of
 * the corresponding root task, taskgraph.py:146-180).  stop_size as in the
 * reference (0 = refine to the leaves).  Returns 0; 1 bad argument; 2
 * structural error (refining a leaf); 3 cyclic graph / edge into a
 * non-final task (the reference's CycleError). */
int hmx_dag_build(int32_t n_blocks, const int64_t* r0, const int64_t* r1, const int64_t* c0,
                  const int64_t* c1, const int8_t* leaf, const int32_t* parent,
                  const int32_t* kids, int32_t mode, int64_t stop_size, int32_t root_op,
                  hmx_dag** out);
/* hmx_dag_build plus edge sparsification per refinement round
 * (build_hlu_dag / compute_dag with sparsify=True, max_path_len,
 * taskgraph.py:530-590, 636-665): the same node set, the reference's
 * sparsified edge set.  Returns 1 for sparsify in mode 1 (the reference's
 * ValueError, taskgraph.py:652-653) or max_path_len < 1. */
int hmx_dag_build_ex(int32_t n_blocks, const int64_t* r0, const int64_t* r1, const int64_t* c0,
                     const int64_t* c1, const int8_t* leaf, const int32_t* parent,
                     const int32_t* kids, int32_t mode, int64_t stop_size, int32_t root_op,
                     int32_t sparsify, int32_t max_path_len, hmx_dag** out);
int64_t hmx_dag_nodes(const hmx_dag* dag);
int64_t hmx_dag_edges(const hmx_dag* dag);
/* Nodes in creation-sequence order (TaskGraph.nodes): kind code (0 hlu,
 * 1 htrsl, 2 htrsu, 3 hmul, 4 add_upd, 5 shift_upd, 6 apply_upd,
 * 7 leaf_factor, 8 leaf_solve_l, 9 leaf_solve_u, 10 leaf_update), matrix ids
 * (n x 3, first nm used), block uids (n x 3, first nu used), alpha; edges as
 * CSR (ptr n+1, idx sorted per node). */
int hmx_dag_export(const hmx_dag* dag, int32_t* kind, int32_t* nm, int32_t* mids, int32_t* nu,
                   int32_t* uids, double* alpha, int64_t* succ_ptr, int32_t* succ_idx);
void hmx_dag_free(hmx_dag* dag);
/* ASAP wavefronts ("levels") of any CSR graph with n nodes (ptr n+1, idx
 * ptr[n]): level[v] = longest path length from a source to v; the wave
 * schedule of the executors (engine.ExecPlan) and taskgraph.asap_levels.
 * Returns 0; 1 bad argument; 3 cyclic graph (the reference's CycleError,
 * taskgraph.py:440-441). */
int hmx_dag_levels(int64_t n, const int64_t* succ_ptr, const int32_t* succ_idx, int32_t* level);

#ifdef __cplusplus
}
#endif
#endif /* HMX_DAG_H */
