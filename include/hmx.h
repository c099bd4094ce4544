/*
 * hmx.h — C ABI of the B200-native H-LU engine (libhmx.so).
 *
 * Plain C types only: device pointers are `double*` / `int*` obtained from
 * any CUDA allocator, streams are `void*` (a cudaStream_t), sizes are
 * int64_t.  Every entry point returns an hmx_status; nothing throws across
 * the boundary.  All matrices are fp64, column-major, with explicit leading
 * dimensions.
 *
 * The reference package (hmatdag, pure Python over numpy/LAPACK) has no
 * FFI; each entry point below names the reference function whose behaviour
 * it reproduces on the device.  INTEGRATION.md shows the ctypes stub a
 * hmatdag maintainer would add to bind these.
 */
#ifndef HMX_H
#define HMX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t hmx_status;
enum {
  HMX_OK = 0,
  HMX_ERR_ARG = 1,          /* bad argument (host-side validation)            */
  HMX_ERR_CUDA = 2,         /* CUDA runtime error                              */
  HMX_ERR_PIVOT = 4,        /* |pivot| <= 1e-14*||A||_F  (arith.py:65-69)      */
  HMX_ERR_RANK_OVERFLOW = 8,/* truncation rank exceeded storage capacity       */
  HMX_ERR_NOT_CONVERGED = 16,/* Jacobi SVD hit its sweep limit                 */
  HMX_ERR_TIMEOUT = 32      /* persistent scheduler watchdog fired             */
};

/* Truncation policy codes — hmatrix.py:36-71 (TruncationPolicy.keep). */
enum { HMX_POLICY_EXACT = 0, HMX_POLICY_RANK = 1, HMX_POLICY_ACCURACY = 2 };

/* ------------------------------------------------------------------------
 * Op program (one record per device micro-op).  A task is a contiguous
 * range of ops executed in order by one CTA.  Matrix refs pack a base id
 * (bits 56..63; 15 = the executing CTA's scratch) and an element offset
 * (bits 0..55).  Dimension codes are >= 0 for constants and
 * -(1 + (base << 24 | index)) for a rank slot (base 15 = CTA-local slots).
 * ---------------------------------------------------------------------- */
typedef struct hmx_op {
  int32_t code;
  int32_t flags;
  int32_t dim[4];
  int32_t ld[4];
  int64_t ref[4];
  int32_t slot[4];
  int32_t iarg[4];
  double farg[2];
  int64_t wref;             /* workspace ref (TRUNC / D2LR)               */
} hmx_op; /* 128 bytes */

/* Workspace (doubles) behind wref that the device paths assume:
 *   OP_TRUNC (m x n, stacked capacity kb = iarg[3]):
 *       9 kb^2 + (m + n + 200) kb + 2048
 *   OP_D2LR  (m x n, l = max(m, n)):
 *       8 l + 16 l^2                 (l < 256)
 *       8 l + 3 l^2 + 2500000        (l >= 256: reflector blocks, R1^T, the
 *                                     core's scratch and a copy of the block)
 * (hmx_lower.cpp and _lib.py: trunc_scratch / d2lr_scratch use these;
 * hmx_op_workspace returns them, 0 for ops without workspace.) */
int64_t hmx_op_workspace(int32_t code, int32_t m, int32_t n, int32_t kb);

/* Library identity / capability. */
const char* hmx_version(void);
int hmx_op_size(void);

/* ------------------------------------------------------------------------
 * Batched leaf kernels (test and building-block entry points).
 * Matrices of batch entry b start at ptr + b*stride.
 * ---------------------------------------------------------------------- */

/* arith.dense_lu (arith.py:58-73): unpivoted LU, L unit-lower (with zeros
 * above the diagonal), U upper (zeros below).  info[b] = HMX_ERR_PIVOT on a
 * vanishing pivot. */
hmx_status hmx_getrf_nopiv_batched(int32_t batch, int32_t n, const double* A, int32_t lda,
                                   int64_t strideA, double* L, double* U, int64_t strideLU,
                                   int32_t* info, void* stream);

/* hm_solve_lower on a dense leaf (hmatrix.py:318-321; scipy
 * solve_triangular lower, unit_diagonal): B := L^{-1} B, B is n x c. */
hmx_status hmx_trsm_lower_unit_batched(int32_t batch, int32_t n, int32_t c, const double* L,
                                       int32_t ldl, int64_t strideL, double* B, int32_t ldb,
                                       int64_t strideB, void* stream);

/* hm_solve_upper_t on a dense leaf (hmatrix.py:331-334): B := U^{-T} B. */
hmx_status hmx_trsm_upper_trans_batched(int32_t batch, int32_t n, int32_t c, const double* U,
                                        int32_t ldu, int64_t strideU, double* B, int32_t ldb,
                                        int64_t strideB, void* stream);

/* Back substitution on a dense leaf, B := U^{-1} B (U upper, non-unit):
 * the leaf step of the solve phase with the factors (hm_solve_upper,
 * the non-transposed counterpart of hmatrix.py:331-341).
 * No reference entry point: the reference stops at the factorization. */
hmx_status hmx_trsm_upper_batched(int32_t batch, int32_t n, int32_t c, const double* U,
                                  int32_t ldu, int64_t strideU, double* B, int32_t ldb,
                                  int64_t strideB, void* stream);

/* The `@` products of hmatrix.py (dense leaf GEMM, LR apply, expansion):
 * C = beta*C + alpha*op(A)*op(B); trans flags 0/1. */
hmx_status hmx_gemm_batched(int32_t batch, int32_t m, int32_t n, int32_t k, double alpha,
                            const double* A, int32_t lda, int64_t strideA, int32_t transA,
                            const double* B, int32_t ldb, int64_t strideB, int32_t transB,
                            double beta, double* C, int32_t ldc, int64_t strideC, void* stream);

/* hmatrix.truncate (hmatrix.py:113-130): QR(U), QR(V), SVD(Ru Rv^T), keep,
 * recompose.  U is m x K, V is n x K.  Outputs Uo (m x cap), Vo (n x cap),
 * rank[b].  K == 0 passes through (rank 0, not counted). */
hmx_status hmx_truncate_batched(int32_t batch, int32_t m, int32_t n, int32_t K, const double* U,
                                const double* V, int64_t strideU, int64_t strideV,
                                int32_t policy, int32_t fixed_rank, double eps, int32_t cap,
                                double* Uo, double* Vo, int64_t strideUo, int64_t strideVo,
                                int32_t* rank, void* stream);

/* hmatrix.dense_to_lowrank (hmatrix.py:133-138): SVD of a dense m x n
 * block, keep, W_r*sigma_r and Z_r. */
hmx_status hmx_dense_to_lowrank_batched(int32_t batch, int32_t m, int32_t n, const double* M,
                                        int64_t strideM, int32_t policy, int32_t fixed_rank,
                                        double eps, int32_t cap, double* Uo, double* Vo,
                                        int64_t strideUo, int64_t strideVo, int32_t* rank,
                                        void* stream);

/* Singular values of p x q matrices by the device one-sided Jacobi SVD,
 * sorted descending (the np.linalg.svd call of hmatrix.py:126). */
hmx_status hmx_svd_values_batched(int32_t batch, int32_t p, int32_t q, const double* G,
                                  int64_t strideG, double* sigma, int64_t strideS, void* stream);

/* ------------------------------------------------------------------------
 * H-LU execution plans (arith.hlu arith.py:76-94, accumulator.hlu_accu
 * accumulator.py:164-187 executed as the refined task DAG of
 * taskgraph.build_hlu_dag taskgraph.py:636-665).  The host planner lowers
 * every DAG task to an op range; the plan owns device copies of the op
 * program, the dependency graph (CSR successors + in-degrees) and the
 * ASAP wavefronts.
 * ---------------------------------------------------------------------- */
typedef struct hmx_plan_desc {
  const hmx_op* ops;          /* host array, n_ops records                 */
  int64_t n_ops;
  const int64_t* task_ops;    /* host, n_tasks+1 prefix offsets into ops    */
  int32_t n_tasks;
  const int32_t* succ_ptr;    /* host CSR, n_tasks+1                         */
  const int32_t* succ_idx;    /* host, succ_ptr[n_tasks]                     */
  const int32_t* wave_ptr;    /* host, n_waves+1 prefix offsets             */
  const int32_t* wave_tasks;  /* host, n_tasks task ids grouped by wave      */
  int32_t n_waves;
  int64_t scratch_doubles;    /* per-CTA scratch requirement                */
  int32_t scratch_ranks;      /* per-CTA rank-slot requirement              */
  int32_t max_ctas;           /* 0 = every SM x ctas_per_sm                  */
  int32_t ctas_per_sm;        /* executor variant: 1 (160 KB shared memory,
                                 255 registers; latency) or 2 (110 KB, 128
                                 registers; batched throughput); 0 = 1     */
  /* Tiered scratch (optional; NULL / 0 = every CTA gets scratch_doubles).
   * A task whose need exceeds scratch_doubles runs in one of n_big shared
   * arenas of big_scratch_doubles, acquired with a device atomic when the
   * task starts and released when it ends (holders never wait on other
   * tasks, so acquisition cannot deadlock). */
  const int64_t* task_scratch; /* host, n_tasks: scratch need per task    */
  int64_t big_scratch_doubles;
  int32_t n_big;               /* > 0: arenas; < 0: one per -n_big CTAs    */
} hmx_plan_desc;

typedef struct hmx_plan* hmx_plan_t;

hmx_status hmx_plan_create(const hmx_plan_desc* desc, hmx_plan_t* out);
/* Bind device storage for base id 0..14 (matrix pools) and rank arrays. */
hmx_status hmx_plan_bind(hmx_plan_t plan, int32_t base_id, double* values, int32_t* ranks);
/* Execute: mode 0 = wavefront launches, 1 = wavefronts captured in a CUDA
 * graph, 2 = persistent kernel with device dependency counters (cooperative
 * launch: every CTA resident), 3 = sequential (one task per launch,
 * debugging), 4 = persistent kernel without resetting the scheduler state
 * (partitioned runs, after hmx_plan_reset on every rank). */
hmx_status hmx_plan_execute(hmx_plan_t plan, int32_t mode, void* stream);
/* Synchronise `stream` and fetch the device status word (HMX_ERR_* bits). */
hmx_status hmx_plan_status(hmx_plan_t plan, void* stream, int32_t* status_bits);
/* Counters since the last reset: [0] truncations, [1] algorithmic flops,
 * [2] algorithmic bytes, [3] tasks executed. */
hmx_status hmx_plan_counters(hmx_plan_t plan, void* stream, uint64_t out[4]);
hmx_status hmx_plan_reset_counters(hmx_plan_t plan, void* stream);
/* Per-task timeline: enable != 0 allocates a trace buffer that the
 * executors fill with (start ns, end ns, smid | cta<<32) per task, followed
 * by 16 (busy ns, count) pairs per op code and one duration word per op;
 * with out != NULL the last trace is copied to the host
 * (3*n_tasks + 32 + n_ops words). */
hmx_status hmx_plan_trace(hmx_plan_t plan, int32_t enable, uint64_t* out);
hmx_status hmx_plan_destroy(hmx_plan_t plan);

/* ------------------------------------------------------------------------
 * Block-row partitioned execution over NVLink peer memory (SURVEY.md §8e:
 * Owner(block) = owner of its row cluster; one exchange per cross-rank DAG
 * edge).  The reference has no multi-node executor; its task DAG
 * (taskgraph.py:636-665) is what gets partitioned.  A task's CTA, after the
 * task, copies the objects a task of another rank reads next into that
 * rank's storage (hmx_pub records), fences system-wide, then releases its
 * successors in their owners' scheduler state (remote atomics).
 * ---------------------------------------------------------------------- */
typedef struct hmx_pub {
  int32_t kind;      /* 0: len doubles; 1: low-rank leaf (m x rk and n x rk, rk from the rank word) */
  int32_t dst;       /* destination rank                                       */
  int32_t base;      /* matrix pool id (0..14)                                 */
  int32_t rbase;     /* rank-array id of the object's rank word                */
  int64_t src_off;   /* element offsets in the source / destination pools      */
  int64_t dst_off;
  int64_t src_off2;  /* kind 1: V factor offsets                               */
  int64_t dst_off2;
  int64_t len;       /* kind 0: doubles                                        */
  int32_t m, n;      /* kind 1: rows of U and V                                */
  int32_t src_ridx;  /* rank word index (-1: none)                             */
  int32_t dst_ridx;
} hmx_pub; /* 72 bytes */

/* Attach a partition to a plan.  rank = -1: every rank is emulated by this
 * one launch (CTA c serves rank c % nranks; the ranks' storage replicas
 * live in the bound pools at the offsets the ops and records carry).
 * rank >= 0: this process is that rank; the other ranks' storage and
 * scheduler state are attached with hmx_plan_peer.  owner[n_tasks];
 * pub_ptr[n_tasks + 1] prefix offsets into pub[n_pub]. */
hmx_status hmx_plan_partition(hmx_plan_t plan, int32_t nranks, int32_t rank, const int32_t* owner,
                              const int64_t* pub_ptr, const hmx_pub* pub, int64_t n_pub);
/* Device addresses of this plan's scheduler state (in-degrees [n_tasks],
 * ready queue [n_tasks], queue control [2]) for export to peers. */
hmx_status hmx_plan_sched_state(hmx_plan_t plan, void** indeg, void** queue, void** qctl);
/* Storage (16 pools + 16 rank arrays) and scheduler state of rank r, as
 * mapped into this process (hmx_ipc_open). */
hmx_status hmx_plan_peer(hmx_plan_t plan, int32_t r, double* const* bases, int32_t* const* rbases,
                         int32_t* indeg, int32_t* queue, int32_t* qctl);
/* Reset the scheduler state to its initial values (every rank resets and
 * synchronises before any rank launches with execute mode 4). */
hmx_status hmx_plan_reset(hmx_plan_t plan, void* stream);
/* CUDA IPC of device allocations: handle (64 bytes) of the allocation that
 * contains dptr and dptr's offset in it; open maps a peer's allocation. */
hmx_status hmx_ipc_handle(const void* dptr, void* handle, int64_t* offset);
hmx_status hmx_ipc_open(const void* handle, void** base);
hmx_status hmx_ipc_close(void* base);

/* Dense evaluation of the exponential point kernel used by the BASELINE
 * configs (problems.PointKernel problems.py:43-53 + permuted 78-81):
 * M[i,j] = scale*exp(-||x_{perm[r0+i]} - x_{perm[c0+j]}||/ell), diagonal
 * (equal original index) = diag.  points: n x dim row-major. */
hmx_status hmx_exp_kernel_blocks(int32_t nblocks, const int64_t* desc /* device, nblocks x 5:
                                 r0, m, c0, n, out_offset */, const double* points, int32_t dim,
                                 const int64_t* perm, double ell, double diag, double scale,
                                 double* out, void* stream);

/* Packed leaf transfer (wire / dump format).  Replaces the host loops of
 * HStore.upload_leaves / download_leaves over the reference's per-leaf
 * numpy arrays (hmatrix.py:141-177: D, or U and V at rank k).  Items are
 * (instance b < nrep, leaf l < nleaf) in that order; desc (device,
 * nleaf x 5 int64): uid, off0 (dense block or U offset), off_v (-1 for a
 * dense leaf), m, n; instance b's pool starts at b*pool_stride and its
 * rank words at b*rank_stride (indexed by uid).  The packed item is the
 * dense block (m*n) or U (m*k) then V (n*k), column-major, k = the rank
 * word.  offsets (device, nleaf*nrep + 1 int64) receives the exclusive scan
 * of the item sizes (offsets[last] = total doubles).  pack with
 * packed == NULL only computes offsets; pack writes at most `capacity`
 * doubles (items that would end beyond it are skipped: the caller sees
 * offsets[last] > capacity and packs again into a larger buffer). */
hmx_status hmx_pack_leaves(int32_t nleaf, int32_t nrep, const int64_t* desc, int64_t pool_stride,
                           int32_t rank_stride, const double* pool, const int32_t* ranks,
                           double* packed, int64_t capacity, int64_t* offsets, void* stream);
hmx_status hmx_unpack_leaves(int32_t nleaf, int32_t nrep, const int64_t* desc, int64_t pool_stride,
                             int32_t rank_stride, const double* packed, const int32_t* ranks,
                             double* pool, int64_t* offsets, void* stream);

/* FP64 FMA-pipe throughput probe (2*8*iters*256*blocks flops), used by
 * bench.py to measure the FP64 roofline denominator on the box. */
hmx_status hmx_fp64_fma_probe(int32_t blocks, int32_t iters, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HMX_H */
