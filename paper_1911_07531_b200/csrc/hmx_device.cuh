// hmx_device.cuh — CTA-level fp64 building blocks of the H-LU engine.
//
// Every routine here is executed cooperatively by ONE thread block of
// HMX_THREADS threads and ends with the block synchronised.  Matrices are
// column-major with explicit leading dimensions; pointers are generic (they
// may point to shared or global memory).  The reference computes the same
// quantities with numpy/LAPACK (see the per-routine citations).
#pragma once
#include <cstdint>
#include <cfloat>

#ifndef HMX_THREADS
#define HMX_THREADS 256
#endif
#define HMX_WARPS (HMX_THREADS / 32)

namespace hmx {

// ---------------------------------------------------------------------------
// reductions
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum; `red` is HMX_WARPS doubles of shared memory.  All threads
// receive the result.
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < HMX_WARPS; ++i) s += red[i];
  return s;
}

// ---------------------------------------------------------------------------
// elementwise helpers
// ---------------------------------------------------------------------------
__device__ void cta_zero(int m, int n, double* C, int ldc) {
  const int tot = m * n;
  for (int e = threadIdx.x; e < tot; e += HMX_THREADS) {
    const int i = e % m, j = e / m;
    C[i + (int64_t)j * ldc] = 0.0;
  }
}

// C (m x n) = alpha * op(A); transA: A is n x m.
__device__ void cta_copy(int m, int n, double alpha, const double* A, int lda, bool ta, double* C,
                         int ldc) {
  const int tot = m * n;
  if (!ta) {
    for (int e = threadIdx.x; e < tot; e += HMX_THREADS) {
      const int i = e % m, j = e / m;
      C[i + (int64_t)j * ldc] = alpha * A[i + (int64_t)j * lda];
    }
  } else {
    for (int e = threadIdx.x; e < tot; e += HMX_THREADS) {
      const int j = e % n, i = e / n;  // read A contiguously
      C[i + (int64_t)j * ldc] = alpha * A[j + (int64_t)i * lda];
    }
  }
}

__device__ void cta_add(int m, int n, double alpha, const double* A, int lda, double* C, int ldc) {
  const int tot = m * n;
  for (int e = threadIdx.x; e < tot; e += HMX_THREADS) {
    const int i = e % m, j = e / m;
    C[i + (int64_t)j * ldc] += alpha * A[i + (int64_t)j * lda];
  }
}

// ---------------------------------------------------------------------------
// GEMM  C = beta*C + alpha*op(A)*op(B)    (the `@` of hmatrix.py)
// 64x64 output tiles, k-chunks of 16 staged in shared memory, 4x4 register
// micro-tile per thread (rows tid%16 + 16i, cols tid/16 + 16j).
// smem: 2*16*65 doubles.
// ---------------------------------------------------------------------------
constexpr int GT = 64, GK = 16, GPAD = 65;
constexpr int GEMM_SMEM_DOUBLES = 2 * GK * GPAD;

__device__ void cta_gemm(int m, int n, int k, double alpha, const double* __restrict__ A, int lda,
                         bool ta, const double* __restrict__ B, int ldb, bool tb, bool beta1,
                         double* C, int ldc, double* sm) {
  if (m <= 0 || n <= 0) return;
  double* As = sm;              // [GK][GPAD] : As[kk*GPAD + i]
  double* Bs = sm + GK * GPAD;  // [GK][GPAD] : Bs[kk*GPAD + j]
  const int tid = threadIdx.x;
  const int tr = tid & 15, tc = tid >> 4;
  const int tiles_m = (m + GT - 1) / GT, tiles_n = (n + GT - 1) / GT;
  for (int tile = 0; tile < tiles_m * tiles_n; ++tile) {
    const int m0 = (tile % tiles_m) * GT, n0 = (tile / tiles_m) * GT;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int k0 = 0; k0 < k; k0 += GK) {
      __syncthreads();
#pragma unroll
      for (int q = 0; q < (GT * GK) / HMX_THREADS; ++q) {
        const int e = tid + q * HMX_THREADS;
        int i, kk;
        if (!ta) { i = e % GT; kk = e / GT; } else { kk = e % GK; i = e / GK; }
        const int gi = m0 + i, gk = k0 + kk;
        double v = 0.0;
        if (gi < m && gk < k) v = ta ? A[gk + (int64_t)gi * lda] : A[gi + (int64_t)gk * lda];
        As[kk * GPAD + i] = v;
        int j, kb;
        if (!tb) { kb = e % GK; j = e / GK; } else { j = e % GT; kb = e / GT; }
        const int gj = n0 + j, gkb = k0 + kb;
        double w = 0.0;
        if (gj < n && gkb < k) w = tb ? B[gj + (int64_t)gkb * ldb] : B[gkb + (int64_t)gj * ldb];
        Bs[kb * GPAD + j] = w;
      }
      __syncthreads();
      const int kc = min(GK, k - k0);
      for (int kk = 0; kk < kc; ++kk) {
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[kk * GPAD + tr + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Bs[kk * GPAD + tc + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gj = n0 + tc + 16 * j;
      if (gj >= n) continue;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int gi = m0 + tr + 16 * i;
        if (gi >= m) continue;
        double* c = C + gi + (int64_t)gj * ldc;
        *c = beta1 ? (*c + alpha * acc[i][j]) : alpha * acc[i][j];
      }
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Unpivoted dense LU — arith.dense_lu (arith.py:58-73).  The update is
// computed as a rounded product followed by a rounded subtraction
// (np.outer then -=), so on equal input the factors match the reference
// bit for bit.  W is an n x n work buffer (shared or global, ld n).
// Returns false on a vanishing pivot (|piv| <= 1e-14 * ||A||_F).
// ---------------------------------------------------------------------------
__device__ bool cta_lu(int n, const double* A, int lda, double* L, int ldl, double* U, int ldu,
                       double* W, double* lv, double* red) {
  double ss = 0.0;
  for (int e = threadIdx.x; e < n * n; e += HMX_THREADS) {
    const int i = e % n, j = e / n;
    const double v = A[i + (int64_t)j * lda];
    W[i + j * n] = v;
    ss += v * v;
  }
  const double scale = sqrt(block_sum(ss, red));
  __syncthreads();
  bool ok = true;
  for (int k = 0; k < n; ++k) {
    const double piv = W[k + k * n];
    if (fabs(piv) <= 1e-14 * scale) { ok = false; break; }
    for (int i = k + 1 + threadIdx.x; i < n; i += HMX_THREADS) lv[i] = W[i + k * n] / piv;
    __syncthreads();
    const int r = n - k - 1;
    for (int e = threadIdx.x; e < r * (r + 1); e += HMX_THREADS) {
      const int i = k + 1 + e % r, j = k + e / r;  // columns k..n-1
      if (j == k) W[i + j * n] = lv[i];             // park the multiplier (U gets 0)
      else W[i + j * n] = __dsub_rn(W[i + j * n], __dmul_rn(lv[i], W[k + j * n]));
    }
    __syncthreads();
  }
  // write out: L unit lower (zeros above), U upper (zeros below)
  for (int e = threadIdx.x; e < n * n; e += HMX_THREADS) {
    const int i = e % n, j = e / n;
    const double w = W[i + j * n];
    L[i + (int64_t)j * ldl] = (i > j) ? w : (i == j ? 1.0 : 0.0);
    U[i + (int64_t)j * ldu] = (i <= j) ? w : 0.0;
  }
  __syncthreads();
  return ok;
}

// ---------------------------------------------------------------------------
// Triangular solves on a dense leaf (hmatrix.py:318-341).
//   trsm_lower_unit : B := L^{-1} B     (L unit lower, n x n)
//   trsm_upper_trans: B := U^{-T} B     (U upper, non-unit)
// B is n x c.  Right-looking column sweep; T is the triangular factor
// staged by the caller (ld n), B in place.
// ---------------------------------------------------------------------------
__device__ void cta_trsm_lower_unit(int n, int c, const double* T, int ldt, double* B, int ldb) {
  for (int l = 0; l < n - 1; ++l) {
    const int r = n - l - 1;
    for (int e = threadIdx.x; e < r * c; e += HMX_THREADS) {
      const int i = l + 1 + e % r, j = e / r;
      B[i + (int64_t)j * ldb] -= T[i + (int64_t)l * ldt] * B[l + (int64_t)j * ldb];
    }
    __syncthreads();
  }
}

__device__ void cta_trsm_upper_trans(int n, int c, const double* T, int ldt, double* B, int ldb) {
  for (int l = 0; l < n; ++l) {
    const double d = T[l + (int64_t)l * ldt];
    for (int j = threadIdx.x; j < c; j += HMX_THREADS) B[l + (int64_t)j * ldb] /= d;
    __syncthreads();
    const int r = n - l - 1;
    for (int e = threadIdx.x; e < r * c; e += HMX_THREADS) {
      const int i = l + 1 + e % r, j = e / r;
      // (U^T)[i,l] = U[l,i]
      B[i + (int64_t)j * ldb] -= T[l + (int64_t)i * ldt] * B[l + (int64_t)j * ldb];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Householder QR (LAPACK dgeqr2 / dlarfg convention), in place on the
// m x K matrix A: R in the upper triangle, reflectors v (v0 = 1 implicit)
// below, tau[j].  np.linalg.qr (hmatrix.py:124-125) returns the same R up to
// row signs.  One warp per trailing column for the reflector application.
// ---------------------------------------------------------------------------
__device__ void cta_householder_qr(int m, int K, double* A, int lda, double* tau, double* red) {
  const int p = min(m, K);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int j = 0; j < p; ++j) {
    double* x = A + (int64_t)j * lda;
    double ss = 0.0;
    for (int i = j + 1 + threadIdx.x; i < m; i += HMX_THREADS) ss += x[i] * x[i];
    const double xn2 = block_sum(ss, red);
    const double alpha = x[j];
    double t = 0.0, beta = alpha, scal = 0.0;
    if (xn2 > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
      t = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    __syncthreads();
    if (xn2 > 0.0)
      for (int i = j + 1 + threadIdx.x; i < m; i += HMX_THREADS) x[i] *= scal;
    if (threadIdx.x == 0) { tau[j] = t; x[j] = beta; }
    __syncthreads();
    if (t != 0.0) {
      for (int c = j + 1 + w; c < K; c += HMX_WARPS) {
        double* y = A + (int64_t)c * lda;
        double d = (lane == 0) ? y[j] : 0.0;
        for (int i = j + 1 + lane; i < m; i += 32) d += x[i] * y[i];
        d = warp_sum(d) * t;
        if (lane == 0) y[j] -= d;
        for (int i = j + 1 + lane; i < m; i += 32) y[i] -= d * x[i];
      }
    }
    __syncthreads();
  }
}

// X (m x r) := Q X where Q = H_0 H_1 ... H_{p-1} from cta_householder_qr.
__device__ void cta_apply_q(int m, int p, const double* A, int lda, const double* tau, int r,
                            double* X, int ldx) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int j = p - 1; j >= 0; --j) {
    const double t = tau[j];
    if (t != 0.0) {
      const double* v = A + (int64_t)j * lda;
      for (int c = w; c < r; c += HMX_WARPS) {
        double* y = X + (int64_t)c * ldx;
        double d = (lane == 0) ? y[j] : 0.0;
        for (int i = j + 1 + lane; i < m; i += 32) d += v[i] * y[i];
        d = warp_sum(d) * t;
        if (lane == 0) y[j] -= d;
        for (int i = j + 1 + lane; i < m; i += 32) y[i] -= d * v[i];
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// One-sided (Hestenes) Jacobi SVD of the p x q matrix G (columns rotated in
// place), accumulating the q x q rotation J (initialised to I here).  On
// exit G*J_in... : G = W*Sigma (column norms sigma), J = Z.  Parallel
// round-robin ordering: each round pairs all columns disjointly, one warp
// per pair.  sigma[q] = column norms, order[q] = column indices sorted by
// descending sigma (ties by index).  Returns false if not converged.
// The high relative accuracy of one-sided Jacobi keeps singular values near
// the eps*sigma_1 cut within rounding of LAPACK's dgesdd (hmatrix.py:126).
// ---------------------------------------------------------------------------
__device__ bool cta_jacobi_svd(int p, int q, double* G, int ldg, double* J, int ldj,
                               double* sigma, int* order, int* flag) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < q * q; e += HMX_THREADS) {
    const int i = e % q, j = e / q;
    J[i + (int64_t)j * ldj] = (i == j) ? 1.0 : 0.0;
  }
  const int qq = q + (q & 1);
  const double tol = DBL_EPSILON * sqrt((double)max(p, 1));
  bool converged = (q <= 1);
  __syncthreads();
  for (int sweep = 0; sweep < 60 && !converged; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int rnd = 0; rnd < qq - 1; ++rnd) {
      for (int pr = w; pr < qq / 2; pr += HMX_WARPS) {
        // circle method: x_i = 1 + (i + rnd) % (qq-1); pairs (0,x_0), (x_pr, x_{qq-1-pr})
        int a, b;
        if (pr == 0) { a = 0; b = 1 + rnd % (qq - 1); }
        else {
          a = 1 + (pr + rnd) % (qq - 1);
          b = 1 + (qq - 1 - pr + rnd) % (qq - 1);
        }
        if (a >= q || b >= q) continue;
        if (a > b) { const int t = a; a = b; b = t; }
        double* ga = G + (int64_t)a * ldg;
        double* gb = G + (int64_t)b * ldg;
        double al = 0.0, be = 0.0, ga_gb = 0.0;
        for (int i = lane; i < p; i += 32) {
          const double x = ga[i], y = gb[i];
          al = fma(x, x, al); be = fma(y, y, be); ga_gb = fma(x, y, ga_gb);
        }
        al = warp_sum(al); be = warp_sum(be); ga_gb = warp_sum(ga_gb);
        if (al == 0.0 || be == 0.0) continue;
        if (fabs(ga_gb) <= tol * sqrt(al) * sqrt(be)) continue;
        const double zeta = (be - al) / (2.0 * ga_gb);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int i = lane; i < p; i += 32) {
          const double x = ga[i], y = gb[i];
          ga[i] = c * x - s * y;
          gb[i] = s * x + c * y;
        }
        double* ja = J + (int64_t)a * ldj;
        double* jb = J + (int64_t)b * ldj;
        for (int i = lane; i < q; i += 32) {
          const double x = ja[i], y = jb[i];
          ja[i] = c * x - s * y;
          jb[i] = s * x + c * y;
        }
        if (lane == 0) *flag = 1;
      }
      __syncthreads();
    }
    converged = (*flag == 0);
    __syncthreads();
  }
  // column norms
  for (int c = w; c < q; c += HMX_WARPS) {
    const double* g = G + (int64_t)c * ldg;
    double s = 0.0;
    for (int i = lane; i < p; i += 32) s = fma(g[i], g[i], s);
    s = warp_sum(s);
    if (lane == 0) sigma[c] = sqrt(s);
  }
  __syncthreads();
  // rank sort (descending, ties by index)
  for (int c = threadIdx.x; c < q; c += HMX_THREADS) {
    const double sc = sigma[c];
    int pos = 0;
    for (int d = 0; d < q; ++d) {
      const double sd = sigma[d];
      pos += (sd > sc) || (sd == sc && d < c);
    }
    order[pos] = c;
  }
  __syncthreads();
  return converged;
}


// ---------------------------------------------------------------------------
// Rank-revealing QR: column-pivoted Householder QR (LAPACK dgeqp3 / dlaqp2
// conventions) of the p x q matrix G, stopped after k steps as soon as the
// Frobenius norm of the trailing block G[k:, k:] is <= thr * |R_00|.
// |R_00| (the largest column norm) is a lower bound of sigma_1, so dropping
// the trailing block moves every singular value by at most thr*sigma_1
// (Weyl); the callers use thr = 1e-8 * (keep cut), far below the measured
// rank margins (SURVEY.md finding 4).  Returns k; perm[c] = original column
// of pivoted column c; tau[j] the reflector scalars; R in rows 0..k-1.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void argmax_block(double v, int i, double* red, int* ired, double& bv,
                                             int& bi) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, i, o);
    if (ov > v || (ov == v && oi >= 0 && (i < 0 || oi < i))) { v = ov; i = oi; }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) { red[w] = v; ired[w] = i; }
  __syncthreads();
  bv = red[0];
  bi = ired[0];
  for (int k = 1; k < HMX_WARPS; ++k)
    if (red[k] > bv || (red[k] == bv && ired[k] >= 0 && (bi < 0 || ired[k] < bi))) {
      bv = red[k];
      bi = ired[k];
    }
}

__device__ int cta_rrqr(int p, int q, double* G, int ldg, double* tau, int* perm, double* cn,
                        double* cn0, double thr, double* red, int* ired) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int c = w; c < q; c += HMX_WARPS) {
    const double* g = G + (int64_t)c * ldg;
    double s = 0.0;
    for (int i = lane; i < p; i += 32) s = fma(g[i], g[i], s);
    s = warp_sum(s);
    if (lane == 0) { cn[c] = s; cn0[c] = s; perm[c] = c; }
  }
  __syncthreads();
  const int kmax = min(p, q);
  double r00sq = 0.0;
  int k = 0;
  for (int j = 0; j < kmax; ++j) {
    double bv;
    int bi;
    {
      double v = -1.0;
      int idx = -1;
      for (int c = j + threadIdx.x; c < q; c += HMX_THREADS)
        if (cn[c] > v) { v = cn[c]; idx = c; }
      argmax_block(v, idx, red, ired, bv, bi);
    }
    if (j == 0) r00sq = bv;
    if (!(bv > 0.0)) break;
    // trailing-norm test (maintained norms first, exact recompute near the cut)
    double ts = 0.0;
    for (int c = j + threadIdx.x; c < q; c += HMX_THREADS) ts += cn[c];
    double tail = block_sum(ts, red);
    const double lim = thr * thr * r00sq;
    if (tail <= 4.0 * lim) {
      __syncthreads();
      for (int c = j + w; c < q; c += HMX_WARPS) {
        const double* g = G + (int64_t)c * ldg;
        double s2 = 0.0;
        for (int i = j + lane; i < p; i += 32) s2 = fma(g[i], g[i], s2);
        s2 = warp_sum(s2);
        if (lane == 0) { cn[c] = s2; cn0[c] = s2; }
      }
      __syncthreads();
      ts = 0.0;
      for (int c = j + threadIdx.x; c < q; c += HMX_THREADS) ts += cn[c];
      tail = block_sum(ts, red);
      if (tail <= lim) break;
      // re-pick the pivot from the exact norms
      double v = -1.0;
      int idx = -1;
      for (int c = j + threadIdx.x; c < q; c += HMX_THREADS)
        if (cn[c] > v) { v = cn[c]; idx = c; }
      argmax_block(v, idx, red, ired, bv, bi);
    }
    // swap columns j <-> bi
    if (bi != j) {
      double* a = G + (int64_t)j * ldg;
      double* b = G + (int64_t)bi * ldg;
      for (int i = threadIdx.x; i < p; i += HMX_THREADS) {
        const double t = a[i];
        a[i] = b[i];
        b[i] = t;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = cn[j]; cn[j] = cn[bi]; cn[bi] = t;
        t = cn0[j]; cn0[j] = cn0[bi]; cn0[bi] = t;
        const int pi = perm[j]; perm[j] = perm[bi]; perm[bi] = pi;
      }
    }
    __syncthreads();
    // Householder reflector of column j (dlarfg)
    double* x = G + (int64_t)j * ldg;
    double ss = 0.0;
    for (int i = j + 1 + threadIdx.x; i < p; i += HMX_THREADS) ss += x[i] * x[i];
    const double xn2 = block_sum(ss, red);
    const double alpha = x[j];
    double t = 0.0, beta = alpha, scal = 0.0;
    if (xn2 > 0.0) {
      beta = -copysign(sqrt(alpha * alpha + xn2), alpha);
      t = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    __syncthreads();
    if (xn2 > 0.0)
      for (int i = j + 1 + threadIdx.x; i < p; i += HMX_THREADS) x[i] *= scal;
    if (threadIdx.x == 0) { tau[j] = t; x[j] = beta; }
    __syncthreads();
    for (int c = j + 1 + w; c < q; c += HMX_WARPS) {
      double* y = G + (int64_t)c * ldg;
      if (t != 0.0) {
        double d = (lane == 0) ? y[j] : 0.0;
        for (int i = j + 1 + lane; i < p; i += 32) d += x[i] * y[i];
        d = warp_sum(d) * t;
        if (lane == 0) y[j] -= d;
        for (int i = j + 1 + lane; i < p; i += 32) y[i] -= d * x[i];
      }
      // norm downdate (dlaqp2): recompute when cancellation is severe
      __syncwarp();
      if (lane == 0) {
        const double rj = y[j];
        double nv = cn[c] - rj * rj;
        cn[c] = nv;
      }
      __syncwarp();
      if (!(cn[c] > 1e-4 * cn0[c])) {
        double s2 = 0.0;
        for (int i = j + 1 + lane; i < p; i += 32) s2 = fma(y[i], y[i], s2);
        s2 = warp_sum(s2);
        if (lane == 0) { cn[c] = s2; cn0[c] = s2; }
      }
    }
    __syncthreads();
    k = j + 1;
  }
  __syncthreads();
  return k;
}

// Number of singular values kept — TruncationPolicy.keep (hmatrix.py:62-71).
// `sig_sorted(i)` = sigma[order[i]]; size = number of singular values.
__device__ int keep_count(int policy, int fixed_k, double eps, const double* sigma,
                          const int* order, int size) {
  if (size == 0) return 0;
  const double s1 = sigma[order[0]];
  if (!(s1 > 0.0)) return 0;
  int lim = size;
  double thr;
  if (policy == 1) { lim = min(fixed_k, size); thr = 1e-14 * s1; }
  else if (policy == 2) thr = eps * s1;
  else thr = 1e-14 * s1;
  int r = 0;
  for (int i = 0; i < lim; ++i) r += (sigma[order[i]] > thr);
  return r;
}

}  // namespace hmx
