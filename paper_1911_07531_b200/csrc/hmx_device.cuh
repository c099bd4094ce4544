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
// Numerical stopping parameters of the SVD core (see cta_jacobi_svd and
// cta_rrqr for the error bounds they imply).
#ifndef HMX_JACOBI_TOL
#define HMX_JACOBI_TOL 1e-10
#endif
#ifndef HMX_JROT
#define HMX_JROT 0
#endif
#ifndef HMX_GSMALL
#define HMX_GSMALL 1
#endif
// unroll factor of the GEMM k-loop (loads of several k steps in flight)
#ifndef HMX_GUNROLL
#define HMX_GUNROLL 2
#endif
#define HMX_PRAGMA_(x) _Pragma(#x)
#define HMX_PRAGMA(x) HMX_PRAGMA_(x)
#if HMX_GUNROLL > 1
#define HMX_GEMM_UNROLL HMX_PRAGMA(unroll HMX_GUNROLL)
#else
#define HMX_GEMM_UNROLL
#endif
#ifndef HMX_RRQR_THR
#define HMX_RRQR_THR 1e-4
#endif
#define HMX_WARPS (HMX_THREADS / 32)
// 2-D loop over an m x n column-major block without integer division:
// one warp per column, lanes over rows (coalesced).
#define FOR_MN(i, j, m, n)                                                  \
  for (int j = (int)(threadIdx.x >> 5); j < (n); j += HMX_WARPS)            \
    for (int i = (int)(threadIdx.x & 31); i < (m); i += 32)

namespace hmx {

// ---------------------------------------------------------------------------
// reductions
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int G>
__device__ __forceinline__ double seg_sum(double v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
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
  FOR_MN(i, j, m, n) C[i + (int64_t)j * ldc] = 0.0;
}


// C (m x n) = alpha * op(A); transA: A is n x m.
__device__ void cta_copy(int m, int n, double alpha, const double* A, int lda, bool ta, double* C,
                         int ldc) {
  if (!ta) {
    FOR_MN(i, j, m, n) C[i + (int64_t)j * ldc] = alpha * A[i + (int64_t)j * lda];
  } else {
    FOR_MN(j, i, n, m) C[i + (int64_t)j * ldc] = alpha * A[j + (int64_t)i * lda];
  }
}

__device__ void cta_add(int m, int n, double alpha, const double* A, int lda, double* C, int ldc) {
  FOR_MN(i, j, m, n) C[i + (int64_t)j * ldc] += alpha * A[i + (int64_t)j * lda];
}

// ---------------------------------------------------------------------------
// GEMM  C = beta*C + alpha*op(A)*op(B)    (the `@` of hmatrix.py)
// Output tiles of (16*MI) x (16*MJ), MI*MJ = 16: every thread owns an
// MI x MJ register micro-tile (rows tid%16 + 16i, cols tid/16 + 16j), so
// the tile shape follows the output shape (64x64 square, 128x32 / 256x16
// for tall-skinny, 32x128 / 16x256 for short-wide) without idle threads.
// k-chunks of KC are staged in shared memory and double buffered: the
// global loads of chunk c+1 are issued into registers before the FMAs of
// chunk c (one barrier per chunk).  Each output is one thread's fma chain
// over k in increasing order, so every tile shape gives the same bits.
// Small outputs with a long reduction (<= 32 4x4 blocks, k >= 128: the
// V^T C products of blocked Householder) split k over the warps instead
// (gemm_splitk).  smem: GEMM_SMEM_DOUBLES.
// ---------------------------------------------------------------------------
constexpr int GT = 64, GK = 16, GPAD = 65;
constexpr int GEMM_SMEM_DOUBLES = 4 * GK * GPAD;  // two stages of A and B tiles

template <int MI, int MJ, int KC>
__device__ __forceinline__ void gemm_tiles(int m, int n, int k, double alpha, const double* __restrict__ A, int lda,
                           bool ta, const double* __restrict__ B, int ldb, bool tb, bool beta1,
                           double* C, int ldc, double* sm) {
  constexpr int TCOLS = HMX_THREADS / 16;  // thread columns of the 16 x TCOLS grid
  constexpr int TM = 16 * MI, TN = TCOLS * MJ, PA = TM + 1, PB = TN + 1;
  constexpr int SA = KC * PA, SB = KC * PB;
  static_assert(2 * (SA + SB) <= GEMM_SMEM_DOUBLES, "gemm staging exceeds its smem budget");
  constexpr int NLA = (TM * KC + HMX_THREADS - 1) / HMX_THREADS;
  constexpr int NLB = (TN * KC + HMX_THREADS - 1) / HMX_THREADS;
  const int tid = threadIdx.x;
  const int tr = tid & 15, tc = tid >> 4;
  const int tiles_m = (m + TM - 1) / TM, tiles_n = (n + TN - 1) / TN;
  for (int tile = 0; tile < tiles_m * tiles_n; ++tile) {
    const int m0 = (tile % tiles_m) * TM, n0 = (tile / tiles_m) * TN;
    double acc[MI][MJ];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < MJ; ++j) acc[i][j] = 0.0;
    double ra[NLA], rb[NLB];
    auto load = [&](int k0) {
#pragma unroll
      for (int q = 0; q < NLA; ++q) {
        const int e = tid + q * HMX_THREADS;
        int i, kk;
        if (!ta) { i = e % TM; kk = e / TM; } else { kk = e % KC; i = e / KC; }
        const int gi = m0 + i, gk = k0 + kk;
        ra[q] = (e < TM * KC && gi < m && gk < k)
                    ? (ta ? A[gk + (int64_t)gi * lda] : A[gi + (int64_t)gk * lda]) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < NLB; ++q) {
        const int e = tid + q * HMX_THREADS;
        int j, kb;
        if (!tb) { kb = e % KC; j = e / KC; } else { j = e % TN; kb = e / TN; }
        const int gj = n0 + j, gkb = k0 + kb;
        rb[q] = (e < TN * KC && gj < n && gkb < k)
                    ? (tb ? B[gj + (int64_t)gkb * ldb] : B[gkb + (int64_t)gj * ldb]) : 0.0;
      }
    };
    auto store = [&](int buf) {
      double* As = sm + buf * (SA + SB);
      double* Bs = As + SA;
#pragma unroll
      for (int q = 0; q < NLA; ++q) {
        const int e = tid + q * HMX_THREADS;
        int i, kk;
        if (!ta) { i = e % TM; kk = e / TM; } else { kk = e % KC; i = e / KC; }
        if (e < TM * KC) As[kk * PA + i] = ra[q];
      }
#pragma unroll
      for (int q = 0; q < NLB; ++q) {
        const int e = tid + q * HMX_THREADS;
        int j, kb;
        if (!tb) { kb = e % KC; j = e / KC; } else { j = e % TN; kb = e / TN; }
        if (e < TN * KC) Bs[kb * PB + j] = rb[q];
      }
    };
    const int nk = (k + KC - 1) / KC;
    load(0);
    store(0);
    __syncthreads();
    for (int c = 0; c < nk; ++c) {
      if (c + 1 < nk) load((c + 1) * KC);
      const double* As = sm + (c & 1) * (SA + SB);
      const double* Bs = As + SA;
      const int kc = min(KC, k - c * KC);
      HMX_GEMM_UNROLL
      for (int kk = 0; kk < kc; ++kk) {
        double a[MI], b[MJ];
#pragma unroll
        for (int i = 0; i < MI; ++i) a[i] = As[kk * PA + tr + 16 * i];
#pragma unroll
        for (int j = 0; j < MJ; ++j) b[j] = Bs[kk * PB + tc + TCOLS * j];
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < MJ; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
      }
      if (c + 1 < nk) store((c + 1) & 1);
      __syncthreads();
    }
    // epilogue: all loads of C first (one exposed latency), then the stores
    if (beta1) {
#pragma unroll
      for (int j = 0; j < MJ; ++j) {
        const int gj = n0 + tc + TCOLS * j;
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const int gi = m0 + tr + 16 * i;
          const double cv = (gi < m && gj < n) ? C[gi + (int64_t)gj * ldc] : 0.0;
          acc[i][j] = cv + alpha * acc[i][j];  // contracted to fma(alpha, acc, cv)
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < MJ; ++j)
#pragma unroll
        for (int i = 0; i < MI; ++i) acc[i][j] = alpha * acc[i][j];
    }
#pragma unroll
    for (int j = 0; j < MJ; ++j) {
      const int gj = n0 + tc + TCOLS * j;
      if (gj >= n) continue;
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int gi = m0 + tr + 16 * i;
        if (gi < m) C[gi + (int64_t)gj * ldc] = acc[i][j];
      }
    }
  }
  __syncthreads();
}

// FP64 tensor-core (DMMA, mma.sync m8n8k4) variant of the 64x64 tile path,
// for the ncu A/B against the DFMA register tiles (HMX_DMMA=1 builds use
// it for every cta_gemm).  Same k-chunk staging and double buffering as
// gemm_tiles<4,4,GK>; warp w owns rows 16*(w%4)..+16 and columns
// 32*(w/4)..+32 of the tile as 2x4 mma tiles of 8x8; per 4-wide k step a
// thread holds one A and one B element per mma row / column tile
// (fragment layout of mma.m8n8k4.f64: A[g][t], B[t][g], C[g][2t+i] with
// g = lane/4, t = lane%4).  The k-order inside one mma is the hardware's,
// so results differ from the DFMA chains in the last bits.
// 1 (default since round 2): the 64x64 tiles of cta_gemm run on the FP64
// tensor cores.  A/B on one box (profiles/r02_dmma_ab.md): 256^3 batch 10.8
// vs 9.2 TFLOP/s, 128x128x64 4.0 vs 3.6, c2 factorization 0.1990 vs 0.2053 s,
// ranks equal to the reference fixtures with both arms; half the issued
// instructions (431 M vs 887 M for the 256^3 batch).
#ifndef HMX_DMMA
#define HMX_DMMA 1
#endif
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__device__ __noinline__ void gemm_tiles_dmma(int m, int n, int k, double alpha, const double* __restrict__ A,
                                             int lda, bool ta, const double* __restrict__ B, int ldb,
                                             bool tb, bool beta1, double* C, int ldc, double* sm) {
  static_assert(HMX_THREADS == 256, "DMMA tiles assume 8 warps");
  constexpr int TM = 64, TN = 64, KC = GK, PA = TM + 1, PB = TN + 1;
  constexpr int SA = KC * PA, SB = KC * PB;
  constexpr int NL = (TM * KC) / HMX_THREADS;  // 4 loads of A and of B per thread and chunk
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int wr = (w & 3) * 16, wc = (w >> 2) * 32;
  const int tiles_m = (m + TM - 1) / TM, tiles_n = (n + TN - 1) / TN;
  for (int tile = 0; tile < tiles_m * tiles_n; ++tile) {
    const int m0 = (tile % tiles_m) * TM, n0 = (tile / tiles_m) * TN;
    double acc[2][4][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    double ra[NL], rb[NL];
    auto load = [&](int k0) {
#pragma unroll
      for (int q = 0; q < NL; ++q) {
        const int e = tid + q * HMX_THREADS;
        int i, kk;
        if (!ta) { i = e % TM; kk = e / TM; } else { kk = e % KC; i = e / KC; }
        const int gi = m0 + i, gk = k0 + kk;
        ra[q] = (gi < m && gk < k) ? (ta ? A[gk + (int64_t)gi * lda] : A[gi + (int64_t)gk * lda]) : 0.0;
        int j, kb;
        if (!tb) { kb = e % KC; j = e / KC; } else { j = e % TN; kb = e / TN; }
        const int gj = n0 + j, gkb = k0 + kb;
        rb[q] = (gj < n && gkb < k) ? (tb ? B[gj + (int64_t)gkb * ldb] : B[gkb + (int64_t)gj * ldb]) : 0.0;
      }
    };
    auto store = [&](int buf) {
      double* As = sm + buf * (SA + SB);
      double* Bs = As + SA;
#pragma unroll
      for (int q = 0; q < NL; ++q) {
        const int e = tid + q * HMX_THREADS;
        int i, kk;
        if (!ta) { i = e % TM; kk = e / TM; } else { kk = e % KC; i = e / KC; }
        As[kk * PA + i] = ra[q];
        int j, kb;
        if (!tb) { kb = e % KC; j = e / KC; } else { j = e % TN; kb = e / TN; }
        Bs[kb * PB + j] = rb[q];
      }
    };
    const int nk = (k + KC - 1) / KC;
    load(0);
    store(0);
    __syncthreads();
    for (int c = 0; c < nk; ++c) {
      if (c + 1 < nk) load((c + 1) * KC);
      const double* As = sm + (c & 1) * (SA + SB);
      const double* Bs = As + SA;
#pragma unroll
      for (int k4 = 0; k4 < KC; k4 += 4) {
        double a[2], b[4];
#pragma unroll
        for (int ri = 0; ri < 2; ++ri) a[ri] = As[(k4 + tq) * PA + wr + ri * 8 + g];
#pragma unroll
        for (int ci = 0; ci < 4; ++ci) b[ci] = Bs[(k4 + tq) * PB + wc + ci * 8 + g];
#pragma unroll
        for (int ri = 0; ri < 2; ++ri)
#pragma unroll
          for (int ci = 0; ci < 4; ++ci) dmma884(acc[ri][ci][0], acc[ri][ci][1], a[ri], b[ci]);
      }
      if (c + 1 < nk) store((c + 1) & 1);
      __syncthreads();
    }
#pragma unroll
    for (int ri = 0; ri < 2; ++ri)
#pragma unroll
      for (int ci = 0; ci < 4; ++ci)
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          const int gi = m0 + wr + ri * 8 + g, gj = n0 + wc + ci * 8 + 2 * tq + x;
          if (gi < m && gj < n) {
            double* cp = C + gi + (int64_t)gj * ldc;
            *cp = beta1 ? fma(alpha, acc[ri][ci][x], *cp) : alpha * acc[ri][ci][x];
          }
        }
  }
  __syncthreads();
}

// Split-k GEMM for at most 32 output blocks of 4x4 (lane = block) and a
// long reduction: warp w sums k in [w*k/8, (w+1)*k/8) for every block, the
// eight partial tiles meet in shared memory (8 x 32 x 16 doubles).
__device__ __forceinline__ void gemm_splitk(int m, int n, int k, double alpha, const double* __restrict__ A, int lda,
                            bool ta, const double* __restrict__ B, int ldb, bool tb, bool beta1,
                            double* C, int ldc, double* sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nbi = (m + 3) >> 2, nbj = (n + 3) >> 2, nblk = nbi * nbj;
  const int k0 = (int)(((int64_t)k * w) / HMX_WARPS), k1 = (int)(((int64_t)k * (w + 1)) / HMX_WARPS);
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  if (lane < nblk) {
    const int bi = lane % nbi, bj = lane / nbi;
    const int i0 = bi * 4, j0 = bj * 4;
    // element (i, kk) of op(A) at A[ao[i] + kk * as], (kk, j) of op(B) at B[bo[j] + kk * bs]
    int ao[4], bo[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int gi = min(i0 + i, m - 1);
      ao[i] = ta ? gi * lda : gi;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gj = min(j0 + j, n - 1);
      bo[j] = tb ? gj : gj * ldb;
    }
    const int as = ta ? 1 : lda, bs = tb ? ldb : 1;
#pragma unroll 2
    for (int kk = k0; kk < k1; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = A[ao[i] + kk * as];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = B[bo[j] + kk * bs];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
  }
  double* red = sm + (w * 32 + lane) * 16;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) red[i * 4 + j] = acc[i][j];
  __syncthreads();
  for (int e = threadIdx.x; e < nblk * 16; e += HMX_THREADS) {
    const int blk = e >> 4, ij = e & 15, i = ij >> 2, j = ij & 3;
    const int gi = (blk % nbi) * 4 + i, gj = (blk / nbi) * 4 + j;
    if (gi >= m || gj >= n) continue;
    double s = 0.0;
#pragma unroll
    for (int ww = 0; ww < HMX_WARPS; ++ww) s += sm[(ww * 32 + blk) * 16 + ij];
    double* cp = C + gi + (int64_t)gj * ldc;
    *cp = beta1 ? (*cp + alpha * s) : alpha * s;
  }
  __syncthreads();
}

// Small-output GEMM (m*n <= 4*HMX_THREADS outputs, op(A) and op(B) fit the
// shared work area): every load of op(A), op(B) and C is issued in one
// pass (batches of 8 independent loads per thread), one barrier, then each
// thread owns up to 4 outputs, each the same increasing-k fma chain as in
// gemm_tiles (and the same epilogue), so the bits are identical.  Saves the
// per-k-chunk barriers and exposed load latencies of the 64x64 tiling when
// the output is a few rank x rank or m x rank blocks.
__device__ __noinline__ void gemm_small(int m, int n, int k, double alpha, const double* __restrict__ A,
                                        int lda, bool ta, const double* __restrict__ B, int ldb, bool tb,
                                        bool beta1, double* C, int ldc, double* sm) {
  const int kb = k | 1;
  double* As = sm;          // op(A): As[i + kk*m]
  double* Bs = sm + m * k;  // op(B): Bs[kk + j*kb]
  const int tid = threadIdx.x;
  const int mk = m * k, tot = mk + n * k;
  const int mn = m * n;
  double cv[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int e = tid + r * HMX_THREADS;
    cv[r] = 0.0;
    if (beta1 && e < mn) cv[r] = C[(e % m) + (int64_t)(e / m) * ldc];
  }
  for (int e0 = tid; e0 < tot; e0 += 8 * HMX_THREADS) {
    double v[8];
    int d[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = e0 + q * HMX_THREADS;
      d[q] = -1;
      v[q] = 0.0;
      if (e < mk) {
        int i, kk;
        if (!ta) { i = e % m; kk = e / m; v[q] = A[i + (int64_t)kk * lda]; }
        else { kk = e % k; i = e / k; v[q] = A[kk + (int64_t)i * lda]; }
        d[q] = i + kk * m;
      } else if (e < tot) {
        const int f = e - mk;
        int j, kk;
        if (!tb) { kk = f % k; j = f / k; v[q] = B[kk + (int64_t)j * ldb]; }
        else { j = f % n; kk = f / n; v[q] = B[j + (int64_t)kk * ldb]; }
        d[q] = mk + kk + j * kb;
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (d[q] >= 0) sm[d[q]] = v[q];
  }
  __syncthreads();
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  int ii[4], jj[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int e = min(tid + r * HMX_THREADS, mn - 1);
    ii[r] = e % m;
    jj[r] = (e / m) * kb;
  }
  if (tid < mn) {
    for (int kk = 0; kk < k; ++kk) {
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[r] = fma(As[ii[r] + kk * m], Bs[kk + jj[r]], acc[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int e = tid + r * HMX_THREADS;
    if (e < mn) {
      // fma(alpha, acc, cv): the contraction the tiled epilogue gets
      const double o = beta1 ? fma(alpha, acc[r], cv[r]) : alpha * acc[r];
      C[ii[r] + (int64_t)(jj[r] / kb) * ldc] = o;
    }
  }
  __syncthreads();
}

// Inline GEMM of the op interpreter: the 64x64 tile shape only (every
// extra instantiation raises the register pressure of the whole persistent
// kernel).
__device__ __forceinline__ void cta_gemm(int m, int n, int k, double alpha, const double* __restrict__ A,
                                         int lda, bool ta, const double* __restrict__ B, int ldb, bool tb,
                                         bool beta1, double* C, int ldc, double* sm) {
  if (m <= 0 || n <= 0) return;
#if HMX_DMMA
  gemm_tiles_dmma(m, n, k, alpha, A, lda, ta, B, ldb, tb, beta1, C, ldc, sm);
#else
  gemm_tiles<4, 4, GK>(m, n, k, alpha, A, lda, ta, B, ldb, tb, beta1, C, ldc, sm);
#endif
}

// Shape-adaptive GEMM for the large-block paths (blocked QR / Q
// application, called from __noinline__ functions only).
__device__ void cta_gemm_wide(int m, int n, int k, double alpha, const double* __restrict__ A, int lda,
                              bool ta, const double* __restrict__ B, int ldb, bool tb, bool beta1,
                              double* C, int ldc, double* sm) {
  if (m <= 0 || n <= 0) return;
  static_assert(HMX_WARPS * 32 * 16 <= GEMM_SMEM_DOUBLES, "split-k partials exceed smem budget");
  if (k >= 128 && ((m + 3) >> 2) * ((n + 3) >> 2) <= 32) {
    gemm_splitk(m, n, k, alpha, A, lda, ta, B, ldb, tb, beta1, C, ldc, sm);
    return;
  }
  if (n <= 32 && m > 64) gemm_tiles<8, 2, 8>(m, n, k, alpha, A, lda, ta, B, ldb, tb, beta1, C, ldc, sm);
  else if (m <= 32 && n > 64) gemm_tiles<2, 8, 8>(m, n, k, alpha, A, lda, ta, B, ldb, tb, beta1, C, ldc, sm);
  else gemm_tiles<4, 4, GK>(m, n, k, alpha, A, lda, ta, B, ldb, tb, beta1, C, ldc, sm);
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
  FOR_MN(i, j, n, n) {
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
  FOR_MN(i, j, n, n) {
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
    const double rd = 1.0 / T[l + (int64_t)l * ldt];  // pivot reciprocal (OpenBLAS trsm convention)
    for (int j = threadIdx.x; j < c; j += HMX_THREADS) B[l + (int64_t)j * ldb] *= rd;
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

// Back substitution B := U^{-1} B (U upper, non-unit; the solve phase
// with the factors, hm_solve_upper below hm_solve_lower):
// pivots l = n-1 .. 0, divide row l, then eliminate it from rows 0..l-1.
__device__ void cta_trsm_upper(int n, int c, const double* T, int ldt, double* B, int ldb) {
  for (int l = n - 1; l >= 0; --l) {
    const double rd = 1.0 / T[l + (int64_t)l * ldt];
    for (int j = threadIdx.x; j < c; j += HMX_THREADS) B[l + (int64_t)j * ldb] *= rd;
    __syncthreads();
    for (int e = threadIdx.x; e < l * c; e += HMX_THREADS) {
      const int i = e % l, j = e / l;
      B[i + (int64_t)j * ldb] -= T[i + (int64_t)l * ldt] * B[l + (int64_t)j * ldb];
    }
    __syncthreads();
  }
}

// Warp-per-column-group triangular solve for n <= 128 (no block barriers):
// T is the factor staged so that the multiplier of row i at pivot l is
// T[i + l*ldt] (L itself for the unit-lower solve, U^T for the transposed
// upper solve).  Lane owns rows lane + 32q; a warp solves up to 4 columns of
// B at once, keeping them in registers; the pivot value travels by shuffle.
// Every element sees the same operations in the same order as the
// CTA-wide sweeps above (bitwise-identical results; for the non-unit
// solves T's diagonal holds the pivot reciprocals 1/u_ll).  REV addresses the
// rows of B in reverse (row n-1-i), which turns the back substitution of
// an upper solve into this forward sweep (T staged reversed by the caller).
template <bool UNIT, bool REV = false>
__device__ void warp_trsm_cols(int n, int c, const double* T, int ldt, double* B, int ldb) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int j0 = w * 4; j0 < c; j0 += HMX_WARPS * 4) {
    const int nc = min(4, c - j0);
    double b[4][4];
#pragma unroll
    for (int cc = 0; cc < 4; ++cc)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = lane + 32 * q;
        b[cc][q] = (cc < nc && i < n) ? B[(REV ? n - 1 - i : i) + (int64_t)(j0 + cc) * ldb] : 0.0;
      }
    for (int l = 0; l < n; ++l) {
      const int ql = l >> 5, ll = l & 31;
      double x[4];
      if (!UNIT) {
        // the caller stages the pivot reciprocals on the diagonal of T, so
        // the pivot step is a multiply, not an fp64 divide, on the chain
        const double rd = T[l + (int64_t)l * ldt];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q == ql && lane == ll) {
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) b[cc][q] *= rd;
          }
      }
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const double v = ql == 0 ? b[cc][0] : ql == 1 ? b[cc][1] : ql == 2 ? b[cc][2] : b[cc][3];
        x[cc] = __shfl_sync(0xffffffffu, v, ll);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = lane + 32 * q;
        if (i > l && i < n) {
          const double t = T[i + (int64_t)l * ldt];
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) b[cc][q] -= t * x[cc];
        }
      }
    }
#pragma unroll
    for (int cc = 0; cc < 4; ++cc)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = lane + 32 * q;
        if (cc < nc && i < n) B[(REV ? n - 1 - i : i) + (int64_t)(j0 + cc) * ldb] = b[cc][q];
      }
  }
}

// ---------------------------------------------------------------------------
// Householder QR (LAPACK dgeqr2 / dlarfg convention), in place on the
// m x K matrix A: R in the upper triangle, reflectors v (v0 = 1 implicit)
// below, tau[j].  np.linalg.qr (hmatrix.py:124-125) returns the same R up to
// row signs.  Per step: warp 0 builds the reflector (one barrier), then one
// warp per trailing column applies it (one barrier).  Rows are owned by
// lane (i mod 32) throughout, so no intra-warp hazards arise.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void warp_reflector(int m, int j, double* x, double* tau) {
  // x = column j; builds H_j = I - tau v v^T with v_j = 1, x[j] := beta
  const int lane = threadIdx.x & 31;
  double ss = 0.0;
  for (int i = j + 1 + ((lane - j - 1) & 31); i < m; i += 32) ss = fma(x[i], x[i], ss);
  ss = warp_sum(ss);
  const double alpha = x[j];
  double t = 0.0, beta = alpha;
  if (ss > 0.0) {
    beta = -copysign(sqrt(alpha * alpha + ss), alpha);
    t = (beta - alpha) / beta;
    const double scal = 1.0 / (alpha - beta);
    for (int i = j + 1 + ((lane - j - 1) & 31); i < m; i += 32) x[i] *= scal;
  }
  __syncwarp();
  if (lane == 0) { tau[j] = t; x[j] = beta; }
}

// y := H_j y for one column y (whole warp), lane-owned rows i = lane mod 32.
__device__ __forceinline__ void warp_apply_reflector(int m, int j, const double* v, double t,
                                                     double* y) {
  const int lane = threadIdx.x & 31;
  const int i0 = j + ((lane - j) & 31);  // first owned row >= j
  double d = 0.0;
  for (int i = i0; i < m; i += 32) d = fma(i == j ? 1.0 : v[i], y[i], d);
  d = warp_sum(d) * t;
  for (int i = i0; i < m; i += 32) y[i] -= d * (i == j ? 1.0 : v[i]);
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Lanes per column G: minimise (passes over the jobs) x (latency of one
// reflector application ~ 30 cycles per owned row + 35 per shuffle level +
// 100 fixed), measured primitive latencies of tools/probes/latency.cu.
__device__ __forceinline__ int pick_g(int m, int jobs, int nthreads) {
  int best = 32;
  long best_cost = 1L << 60;
#pragma unroll
  for (int lg = 2; lg <= 5; ++lg) {
    const int g = 1 << lg;
    const long passes = (jobs * (long)g + nthreads - 1) / nthreads;
    const long cost = passes * ((m + g - 1) / g * 30 + lg * 35 + 100);
    if (cost < best_cost) { best_cost = cost; best = g; }
  }
  return best;
}

#define HMX_G_SWITCH(g, CALL)                                   \
  do {                                                          \
    switch (g) {                                                \
      case 4: { constexpr int GG = 4; CALL; } break;            \
      case 8: { constexpr int GG = 8; CALL; } break;            \
      case 16: { constexpr int GG = 16; CALL; } break;          \
      default: { constexpr int GG = 32; CALL; } break;          \
    }                                                           \
  } while (0)

// G from the row count alone (~8 rows per lane), for fixed-structure loops.
#define HMX_G_DISPATCH(m, CALL)            \
  do {                                     \
    if ((m) <= 64) { constexpr int GG = 8; CALL; }        \
    else if ((m) <= 128) { constexpr int GG = 16; CALL; } \
    else { constexpr int GG = 32; CALL; }                 \
  } while (0)

// y := H_j y by a group of G lanes (G divides 32); lane gl owns the rows
// i = gl (mod G).  Several columns are processed concurrently by the groups
// of a warp, so each reduction is log2(G) shuffle levels deep instead of 5.
// All 32 lanes of a warp must call this (the shuffles are warp-wide).
template <int G>
__device__ __forceinline__ void grp_apply_reflector(int m, int j, const double* v, double t,
                                                    double* y, int gl, bool active) {
  // the implicit unit element v_j = 1 belongs to the lane whose first row
  // is j; it is peeled off so the loops carry no per-element select (same
  // operations in the same order as the select form: bitwise identical)
  double d = 0.0;
  const int i0 = j + ((gl - j) & (G - 1));
  if (active && i0 < m) {
    d = (i0 == j) ? y[j] : v[i0] * y[i0];
#pragma unroll 4
    for (int i = i0 + G; i < m; i += G) d = fma(v[i], y[i], d);
  }
  d = seg_sum<G>(d) * t;
  if (active && i0 < m) {
    y[i0] -= (i0 == j) ? d : d * v[i0];
#pragma unroll 4
    for (int i = i0 + G; i < m; i += G) y[i] -= d * v[i];
  }
}

// Apply reflector j (column x) to columns [c0, K) of A with `nthreads`
// threads starting at thread t0 (whole warps).
template <int G>
__device__ __forceinline__ void grp_update_cols(int m, int j, const double* x, double t, double* A,
                                                int lda, int c0, int K, int t0, int nthreads) {
  const int tid = (int)threadIdx.x - t0;
  const int grp = tid / G, gl = tid % G, ngrp = nthreads / G;
  const int njobs = K - c0;
  for (int b = 0; b < njobs; b += ngrp) {
    const int c = c0 + b + grp;
    grp_apply_reflector<G>(m, j, x, t, A + (int64_t)min(c, K - 1) * lda, gl, c < K);
  }
}

__device__ void qr_steps(int m, int K, double* A, int lda, double* tau, int wbeg, int nw, int bar) {
  const int p = min(m, K);
  const int w = (int)(threadIdx.x >> 5) - wbeg;
  for (int j = 0; j < p; ++j) {
    double* x = A + (int64_t)j * lda;
    if (w == 0) warp_reflector(m, j, x, tau);
    if (bar) named_bar(bar, nw * 32); else __syncthreads();
    const double t = tau[j];
    if (t != 0.0)  // ~8 rows per lane (measured best for the step-synchronous QR)
      HMX_G_DISPATCH(m, (grp_update_cols<GG>(m, j, x, t, A, lda, j + 1, K, wbeg * 32, nw * 32)));
    if (bar) named_bar(bar, nw * 32); else __syncthreads();
  }
}


__device__ void cta_householder_qr(int m, int K, double* A, int lda, double* tau, double* red) {
  qr_steps(m, K, A, lda, tau, 0, HMX_WARPS, 0);
}


// Householder QR by a group of nw warps [wbeg, wbeg + nw) synchronised on
// named barrier bar_id, so that two factorizations (U and V of a
// truncation) run concurrently in one CTA.
__device__ void group_householder_qr(int m, int K, double* A, int lda, double* tau, int wbeg,
                                     int nw, int bar_id) {
  qr_steps(m, K, A, lda, tau, wbeg, nw, bar_id);
}

// X (m x r) := Q X where Q = H_0 H_1 ... H_{p-1} from cta_householder_qr.
// Columns of X are independent: one lane group per column, no block
// barriers between reflectors.
template <int G>
__device__ void apply_q_cols(int m, int p, const double* A, int lda, const double* tau, int r,
                             double* X, int ldx) {
  const int grp = threadIdx.x / G, gl = threadIdx.x % G, ngrp = HMX_THREADS / G;
  for (int b = 0; b < r; b += ngrp) {
    const int c = b + grp;
    const bool act = c < r;
    double* y = X + (int64_t)min(c, max(r - 1, 0)) * ldx;
    for (int j = p - 1; j >= 0; --j) {
      const double t = tau[j];
      if (t != 0.0) grp_apply_reflector<G>(m, j, A + (int64_t)j * lda, t, y, gl, act);
    }
  }
}

__device__ void cta_apply_q(int m, int p, const double* A, int lda, const double* tau, int r,
                            double* X, int ldx) {
  if (r > 0) HMX_G_SWITCH(pick_g(m, r, HMX_THREADS), (apply_q_cols<GG>(m, p, A, lda, tau, r, X, ldx)));
  __syncthreads();
}

// ---------------------------------------------------------------------------
// One-sided (Hestenes) Jacobi SVD of the p x q matrix G (columns rotated in
// place), accumulating the q x q rotation J (initialised to I here).  On
// exit G = W*Sigma (column norms sigma) and J = Z.  Parallel round-robin
// ordering: every round pairs all columns disjointly and ALL pairs of a
// round run at once, one group of g lanes per pair (g = power of two with
// (q/2)*g <= threads, g <= 32), with segmented shuffles for the three dot
// products.  sigma[q] = column norms, order[q] = column indices by
// descending sigma (ties by index).  Returns false if not converged.
// One-sided Jacobi has high relative accuracy, so singular values near the
// eps*sigma_1 cut agree with LAPACK's dgesdd (hmatrix.py:126) to rounding.
// ---------------------------------------------------------------------------

template <int G>
__device__ void jacobi_rounds(int p, int q, double* Gm, int ldg, double* J, int ldj, double tol2,
                              int* flag) {
  const int qq = q + (q & 1);
  const int npairs = qq / 2;
  const int grp = threadIdx.x / G, gl = threadIdx.x % G;
  const int ngrp = HMX_THREADS / G;
  for (int rnd = 0; rnd < qq - 1; ++rnd) {
    for (int pr0 = 0; pr0 < npairs; pr0 += ngrp) {
      const int pr = pr0 + grp;
      // circle method: x_i = 1 + (i + rnd) mod (qq-1); pairs (0, x_0), (x_pr, x_{qq-1-pr})
      const int mq = qq - 1;
      int a, b;
      if (pr == 0) { a = 0; b = 1 + rnd; }
      else {
        a = pr + rnd; if (a >= mq) a -= mq;
        a += 1;
        b = mq - pr + rnd; if (b >= mq) b -= mq;
        b += 1;
      }
      const bool valid = pr < npairs && a < q && b < q;
      if (a > b) { const int t = a; a = b; b = t; }
      double al = 0.0, be = 0.0, ga = 0.0;
      double* x = Gm + (int64_t)a * ldg;
      double* y = Gm + (int64_t)b * ldg;
      if (valid) {
        for (int i = gl; i < p; i += G) {
          const double u = x[i], v = y[i];
          al = fma(u, u, al); be = fma(v, v, be); ga = fma(u, v, ga);
        }
      }
      al = seg_sum<G>(al); be = seg_sum<G>(be); ga = seg_sum<G>(ga);
      if (!valid || al == 0.0 || be == 0.0 || ga * ga <= tol2 * al * be) continue;
#if HMX_JROT
      // the same rotation from two reciprocal square roots (no fp64 divide
      // or sqrt on the round's critical path): with d = be - al, g = 2 ga,
      // h = |(d, g)|, cos 2theta = |d|/h, c = sqrt((1 + cos 2theta)/2),
      // s = sign(d) g / (2 c h); c^2 + s^2 = 1 exactly in exact arithmetic
      const double d = be - al, g2 = 2.0 * ga;
      const double rh = rsqrt(fma(d, d, g2 * g2));
      const double hc = fma(0.5 * fabs(d), rh, 0.5);  // c^2, in [1/2, 1]
      const double rc = rsqrt(hc);
      const double c = hc * rc;
      const double s = copysign(0.5, d) * g2 * rh * rc;
#else
      const double zeta = (be - al) / (2.0 * ga);
      const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
      const double c = rsqrt(fma(t, t, 1.0)), s = c * t;
#endif
      for (int i = gl; i < p; i += G) {
        const double u = x[i], v = y[i];
        x[i] = c * u - s * v;
        y[i] = s * u + c * v;
      }
      double* ja = J + (int64_t)a * ldj;
      double* jb = J + (int64_t)b * ldj;
      for (int i = gl; i < q; i += G) {
        const double u = ja[i], v = jb[i];
        ja[i] = c * u - s * v;
        jb[i] = s * u + c * v;
      }
      if (gl == 0) *flag = 1;
    }
    __syncthreads();
  }
}

__device__ void jacobi_sigma_order(int p, int q, const double* G, int ldg, double* sigma,
                                   int* order);

__device__ bool cta_jacobi_svd(int p, int q, double* G, int ldg, double* J, int ldj,
                               double* sigma, int* order, int* flag, int* sweeps_out = nullptr) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  FOR_MN(i, j, q, q) J[i + (int64_t)j * ldj] = (i == j) ? 1.0 : 0.0;
  // Convergence: |g_a . g_b| <= tol |g_a||g_b| for all pairs.  With
  // G^T G = D^{1/2}(I + F)D^{1/2}, |F_ab| <= tol, every singular value has
  // relative error <= q*tol/2 (relative perturbation of scaled diagonally
  // dominant matrices): tol = 1e-10 and q <= 512 give <= 2.6e-8, far below
  // the rank margins near the cut (>= 4e-5 relative, SURVEY.md finding 4).
  const double tol = HMX_JACOBI_TOL;
  const double tol2 = tol * tol;
  const int npairs = (q + (q & 1)) / 2;
  bool converged = (q <= 1);
  __syncthreads();
  int sweep = 0;
  for (; sweep < 60 && !converged; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    if (npairs * 32 <= HMX_THREADS) jacobi_rounds<32>(p, q, G, ldg, J, ldj, tol2, flag);
    else if (npairs * 16 <= HMX_THREADS) jacobi_rounds<16>(p, q, G, ldg, J, ldj, tol2, flag);
    else if (npairs * 8 <= HMX_THREADS) jacobi_rounds<8>(p, q, G, ldg, J, ldj, tol2, flag);
    else jacobi_rounds<4>(p, q, G, ldg, J, ldj, tol2, flag);
    converged = (*flag == 0);
    __syncthreads();
  }
  if (sweeps_out) *sweeps_out = sweep;
  jacobi_sigma_order(p, q, G, ldg, sigma, order);
  return converged;
}

// column norms sigma[q] of G and order[q] = columns by descending sigma
// (ties by index); whole CTA, ends synchronised.
__device__ void jacobi_sigma_order(int p, int q, const double* G, int ldg, double* sigma,
                                   int* order) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
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
}

// ---------------------------------------------------------------------------
// Rank-revealing QR: column-pivoted Householder QR (LAPACK dgeqp3 / dlaqp2
// conventions) of the p x q matrix G, stopped after k steps as soon as the
// Frobenius norm of the trailing block G[k:, k:] is <= thr * |R_00|.
// Dropping the trailing rows B = [0 R22] of R is a positive semidefinite
// change of R^T R = A^T A + B^T B, so every singular value moves by at most
// ||B||^2 / sigma_i <= thr^2 sigma_1^2 / sigma_i (|R_00| <= sigma_1).  The
// callers use thr = HMX_RRQR_THR * cut = 1e-4 * cut: singular values at the
// keep cut (cut * sigma_1) move by <= thr^2/cut^2 = 1e-8 relative (1e-3,
// i.e. 1e-6 relative, flipped one of ~46k block ranks of c3 std), below the measured rank
// margins (>= 4e-5 relative, SURVEY.md finding 4).  Returns k; perm[c] =
// original column of pivoted column c; tau[j] the reflector scalars; R in
// rows 0..k-1.
// Per step: warp 0 pivots, swaps and builds the reflector (one barrier),
// all warps apply it and downdate column norms (one barrier).
// ---------------------------------------------------------------------------
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
  int* ctl = ired;  // ctl[0]: 0 continue, 1 stop, 2 recompute norms
  for (int j = 0; j < kmax; ++j) {
    if (w == 0) {
      double v = -1.0, tail = 0.0;
      int idx = -1;
      for (int c = j + lane; c < q; c += 32) {
        const double x = cn[c];
        tail += x;
        if (x > v) { v = x; idx = c; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (ov > v || (ov == v && oi >= 0 && (idx < 0 || oi < idx))) { v = ov; idx = oi; }
      }
      tail = warp_sum(tail);
      if (j == 0) r00sq = v;
      const double lim = thr * thr * r00sq;
      int act = 0;
      if (!(v > 0.0)) act = 1;
      else if (tail <= 4.0 * lim) act = 2;
      if (lane == 0) { ctl[0] = act; ctl[1] = idx; red[0] = r00sq; }
    }
    __syncthreads();
    r00sq = red[0];
    int act = ctl[0];
    if (act == 2) {  // exact trailing norms near the cut
      for (int c = j + w; c < q; c += HMX_WARPS) {
        const double* g = G + (int64_t)c * ldg;
        double s2 = 0.0;
        for (int i = j + lane; i < p; i += 32) s2 = fma(g[i], g[i], s2);
        s2 = warp_sum(s2);
        if (lane == 0) { cn[c] = s2; cn0[c] = s2; }
      }
      __syncthreads();
      if (w == 0) {
        double v = -1.0, tail = 0.0;
        int idx = -1;
        for (int c = j + lane; c < q; c += 32) {
          const double x = cn[c];
          tail += x;
          if (x > v) { v = x; idx = c; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, v, o);
          const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
          if (ov > v || (ov == v && oi >= 0 && (idx < 0 || oi < idx))) { v = ov; idx = oi; }
        }
        tail = warp_sum(tail);
        if (lane == 0) { ctl[0] = (tail <= thr * thr * r00sq || !(v > 0.0)) ? 1 : 0; ctl[1] = idx; }
      }
      __syncthreads();
      act = ctl[0];
    }
    if (act == 1) return j;
    if (w == 0) {
      const int bi = ctl[1];
      if (bi != j) {
        double* a = G + (int64_t)j * ldg;
        double* b = G + (int64_t)bi * ldg;
        for (int i = lane; i < p; i += 32) {
          const double t = a[i];
          a[i] = b[i];
          b[i] = t;
        }
        if (lane == 0) {
          double t = cn[j]; cn[j] = cn[bi]; cn[bi] = t;
          t = cn0[j]; cn0[j] = cn0[bi]; cn0[bi] = t;
          const int pi = perm[j]; perm[j] = perm[bi]; perm[bi] = pi;
        }
        __syncwarp();
      }
      warp_reflector(p, j, G + (int64_t)j * ldg, tau);
    }
    __syncthreads();
    const double t = tau[j];
    const double* x = G + (int64_t)j * ldg;
    if (t != 0.0) HMX_G_DISPATCH(p, (grp_update_cols<GG>(p, j, x, t, G, ldg, j + 1, q, 0, HMX_THREADS)));
    __syncthreads();
    // norm downdate (dlaqp2): one warp per column; recompute on cancellation
    for (int c = j + 1 + w; c < q; c += HMX_WARPS) {
      const double* y = G + (int64_t)c * ldg;
      const double rj = y[j];
      const double nv = cn[c] - rj * rj;
      const bool rec = !(nv > 1e-4 * cn0[c]);
      if (rec) {
        double s2 = 0.0;
        for (int i = j + 1 + lane; i < p; i += 32) s2 = fma(y[i], y[i], s2);
        s2 = warp_sum(s2);
        if (lane == 0) { cn[c] = s2; cn0[c] = s2; }
      } else if (lane == 0) {
        cn[c] = nv;
      }
    }
    __syncthreads();
  }
  return kmax;
}

// ---------------------------------------------------------------------------
// Blocked Householder QR (LAPACK dgeqrf) of a tall m x K matrix A in global
// memory: panels of QR_NB columns are factored in shared memory
// (cta_householder_qr), the block reflector I - V T V^T is formed (dlarft)
// and the trailing columns are updated with two GEMMs.  V is also kept
// explicitly (unit lower, Vx m x p) with the T blocks (Tb, NB x NB each) so
// that Q can later be applied as GEMMs (cta_apply_q_blocked).
// ---------------------------------------------------------------------------
constexpr int QR_NB = 16;

// Panel width of the blocked QR for m rows: as wide as fits (panel + T +
// GEMM staging) in the shared work area, between 4 and QR_NB.
__device__ __forceinline__ int qr_nb(int m, int smcap) {
  int nb = (smcap - QR_NB * QR_NB - GEMM_SMEM_DOUBLES) / max(m, 1);
  return max(4, min(QR_NB, nb));
}

// T (jb x jb, ld QR_NB) of the block reflector from explicit V (rows x jb).
__device__ void cta_larft(int rows, int jb, const double* V, int ldv, const double* tau, double* T,
                          double* S) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int e = w; e < jb * jb; e += HMX_WARPS) {
    const int i = e % jb, j = e / jb;
    if (i >= j) continue;
    const double* vi = V + (int64_t)i * ldv;
    const double* vj = V + (int64_t)j * ldv;
    double d = 0.0;
    for (int r = j + lane; r < rows; r += 32) d = fma(vi[r], vj[r], d);
    d = warp_sum(d);
    if (lane == 0) S[i + j * QR_NB] = d;
  }
  __syncthreads();
  if (w == 0) {
    for (int j = 0; j < jb; ++j) {
      // T[0:j, j] = -tau_j * T[0:j, 0:j] * S[0:j, j];  T[j, j] = tau_j
      double v = 0.0;
      if (lane < j) {
        for (int l = lane; l < j; ++l) v = fma(T[lane + l * QR_NB], S[l + j * QR_NB], v);
        v *= -tau[j];
      }
      __syncwarp();
      if (lane < j) T[lane + j * QR_NB] = v;
      if (lane == 0) T[j + j * QR_NB] = tau[j];
      for (int i = j + 1 + lane; i < jb; i += 32) T[i + j * QR_NB] = 0.0;
      __syncwarp();
    }
  }
  __syncthreads();
}

// Y (jb x nc, ld ldy) := op(T) * Y for upper-triangular T (ld QR_NB)
__device__ void cta_trmm_small(int jb, int nc, const double* T, bool trans, double* Y, int ldy,
                               double* tmp) {
  for (int e = threadIdx.x; e < jb * nc; e += HMX_THREADS) {
    const int i = e % jb, c = e / jb;
    double v = 0.0;
    if (!trans) {
      for (int l = i; l < jb; ++l) v = fma(T[i + l * QR_NB], Y[l + (int64_t)c * ldy], v);
    } else {
      for (int l = 0; l <= i; ++l) v = fma(T[l + i * QR_NB], Y[l + (int64_t)c * ldy], v);
    }
    tmp[e] = v;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < jb * nc; e += HMX_THREADS) {
    const int i = e % jb, c = e / jb;
    Y[i + (int64_t)c * ldy] = tmp[e];
  }
  __syncthreads();
}

// ws (global): W (QR_NB x K) + tmp (QR_NB x K).  sm: shared work area of
// smcap doubles (panel staging + GEMM staging).
__device__ __noinline__ void cta_qr_blocked(int m, int K, double* A, int lda, double* tau, double* Vx, int ldv,
                               double* Tb, double* ws, double* sm, int smcap, double* red) {
  const int p = min(m, K);
  const int nb = qr_nb(m, smcap);
  double* S = sm;                      // QR_NB^2
  double* panel = sm + QR_NB * QR_NB;  // rows x jb
  double* gsm = panel;                 // GEMM staging (after the panel is written back)
  for (int j0 = 0; j0 < p; j0 += nb) {
    const int jb = min(nb, p - j0);
    const int rows = m - j0;
    double* Ap = A + j0 + (int64_t)j0 * lda;
    const bool psm = rows * jb + QR_NB * QR_NB <= smcap && GEMM_SMEM_DOUBLES + QR_NB * QR_NB <= smcap;
    double* P = psm ? panel : Ap;
    const int ldp = psm ? rows : lda;
    if (psm) {
      FOR_MN(i, c, rows, jb) P[i + c * rows] = Ap[i + (int64_t)c * lda];
      __syncthreads();
    }
    cta_householder_qr(rows, jb, P, ldp, tau + j0, red);
    double* Vp = Vx + j0 + (int64_t)j0 * ldv;
    FOR_MN(i, c, rows, jb) {
      const double v = P[i + (int64_t)c * ldp];
      Vp[i + (int64_t)c * ldv] = (i > c) ? v : (i == c ? 1.0 : 0.0);
      if (psm) Ap[i + (int64_t)c * lda] = v;
    }
    __syncthreads();
    double* T = Tb + (int64_t)(j0 / nb) * QR_NB * QR_NB;
    cta_larft(rows, jb, Vp, ldv, tau + j0, T, S);
    const int nc = K - j0 - jb;
    if (nc > 0) {
      double* C = A + j0 + (int64_t)(j0 + jb) * lda;
      double* W = ws;
      double* tmp = ws + (int64_t)QR_NB * K;
      cta_gemm_wide(jb, nc, rows, 1.0, Vp, ldv, true, C, lda, false, false, W, QR_NB, gsm);
      cta_trmm_small(jb, nc, T, true, W, QR_NB, tmp);
      cta_gemm_wide(rows, nc, jb, -1.0, Vp, ldv, false, W, QR_NB, false, true, C, lda, gsm);
    }
  }
}

// X (m x r) := Q X with Q = (I - V0 T0 V0^T)(I - V1 T1 V1^T)...
// ws: W (QR_NB x r) + tmp (QR_NB x r)
__device__ __noinline__ void cta_apply_q_blocked(int m, int p, const double* Vx, int ldv, const double* Tb,
                                    int r, double* X, int ldx, double* ws, double* gsm,
                                    int smcap) {
  if (r == 0) return;
  const int nb = qr_nb(m, smcap);
  const int nblk = (p + nb - 1) / nb;
  double* W = ws;
  double* tmp = ws + (int64_t)QR_NB * r;
  for (int b = nblk - 1; b >= 0; --b) {
    const int j0 = b * nb, jb = min(nb, p - j0), rows = m - j0;
    const double* Vp = Vx + j0 + (int64_t)j0 * ldv;
    const double* T = Tb + (int64_t)b * QR_NB * QR_NB;
    double* Xp = X + j0;
    cta_gemm_wide(jb, r, rows, 1.0, Vp, ldv, true, Xp, ldx, false, false, W, QR_NB, gsm);
    cta_trmm_small(jb, r, T, false, W, QR_NB, tmp);
    cta_gemm_wide(rows, r, jb, -1.0, Vp, ldv, false, W, QR_NB, false, true, Xp, ldx, gsm);
  }
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
