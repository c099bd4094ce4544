// hmx_ws.cuh — warp-synchronous building blocks of the truncation
// (hmatrix.truncate, hmatrix.py:113-130, and dense_to_lowrank, :133-138).
//
// The step-synchronous CTA-wide routines of hmx_device.cuh pay two block
// barriers, a warp reduction and an fp64 sqrt/divide chain per Householder
// reflector and then walk every reflector again, one by one, to apply Q.
// Here:
//  * Householder QR runs with lane = column and the rows split over the
//    warps of a group (ws_qr): per reflector one pass of inner products, ONE
//    exchange of the per-warp partial sums (named barrier), the scalar chain
//    (one sqrt, one reciprocal) computed redundantly by every lane, one
//    update pass.  No shuffles, no broadcast.
//  * Reflectors are kept unscaled: H_j = I - tp_j w_j w_j^T with
//    w_j = (0, .., 0, wd_j, a_{j+1,j}, .., a_{m-1,j}), wd_j = alpha - beta,
//    tp_j = 1 / (|beta| (|alpha| + |beta|)); the tails stay in place below
//    the diagonal of A, beta (= R_jj) on it.
//  * Q = H_0 .. H_{p-1} = I - W T W^T with T^{-1} = striu(W^T W) + diag(1/tp)
//    (compact-WY in its inverse form): applying Q to Y is  B = W^T Y,
//    a back substitution with T^{-1}, and Y -= W Z  -- three dense phases
//    instead of p dependent reflector applications (ws_smat / ws_wtb /
//    ws_trsolve / ws_wz).  striu(W^T W) overwrites the strict upper triangle
//    of A once R has been consumed.
//  * Rank-revealing QR runs with lane = column and the COLUMNS split over
//    warps (ws_rrqr): exact trailing column norms come out of the update
//    pass (no downdating), the pivot is a warp arg-max, columns are never
//    swapped (perm / pos bookkeeping instead).
//  * One-sided Jacobi rotates X = R1^T only (ws_jacobi); the left factor is
//    recovered as R1 X / sigma afterwards.
// Tall factors that do not fit shared memory are factored panel by panel
// (TSQR): every panel is a ws_qr in shared memory, the R factors are
// stacked and factored again; Q is applied level by level with the same
// three dense phases (engine: trunc_ws_panel).
#pragma once
#include "hmx_device.cuh"

#ifndef HMX_WS_JTOL
#define HMX_WS_JTOL 1e-6
#endif

namespace hmx {

// Reflector scalars from alpha = a_jj and ss = sum_{i>j} a_ij^2.
__device__ __forceinline__ void house_scalars(double alpha, double ss, double& beta, double& wd,
                                              double& tp) {
  if (!(ss > 0.0)) {  // H = I (dlarfg: tau = 0); w = 0 keeps the WY form consistent
    beta = alpha; wd = 0.0; tp = 0.0;
    return;
  }
  const double x = fma(alpha, alpha, ss);
  const double ri = rsqrt(x);
  const double nrm = x * ri;
  const double t = fabs(alpha) + nrm;
  beta = -copysign(nrm, alpha);
  wd = copysign(t, alpha);
  tp = ri * __drcp_rn(t);
}

__device__ __forceinline__ void grp_sync(int bar, int nthreads) {
  if (nthreads <= 32) __syncwarp();
  else named_bar(bar, nthreads);
}

// ---------------------------------------------------------------------------
// Householder QR of the m x K matrix A (shared memory, lda odd) by the warps
// [w0, w0 + nw) of the CTA, synchronised on named barrier `bar`.  Lane owns
// the columns lane + 32 t (t < CT, K <= 32 CT); warp gw owns a contiguous
// chunk of rows.  xch: 2 * (NW + 1) * (K + 1) doubles.  On exit: R on and above
// the diagonal, reflector tails below, tp[j], wd[j] (j < min(m, K)).
// ---------------------------------------------------------------------------
// dot product with the loads of RB elements issued before their FMAs (a
// shared-memory load costs ~70 cycles when the next instruction waits on
// it), two accumulation chains
template <int RB>
__device__ __forceinline__ double ws_dot(const double* a, int sa, const double* b, int sb, int n) {
  double s0 = 0.0, s1 = 0.0;
  int i = 0;
  for (; i + RB <= n; i += RB) {
    double x[RB], y[RB];
#pragma unroll
    for (int u = 0; u < RB; ++u) { x[u] = a[(i + u) * sa]; y[u] = b[(i + u) * sb]; }
#pragma unroll
    for (int u = 0; u < RB; u += 2) { s0 = fma(x[u], y[u], s0); s1 = fma(x[u + 1], y[u + 1], s1); }
  }
  for (; i < n; ++i) s0 = fma(a[i * sa], b[i * sb], s0);
  return s0 + s1;
}

// Rows per register block of ws_qr and the padded row count it works on:
// the caller provides lda >= ws_qr_rows(m, NW, CT) with rows m.. zero (they
// stay zero), so the row loops need no tail handling.
template <int CT>
struct WsQrRB { static constexpr int value = CT == 1 ? 8 : (CT == 2 ? 4 : 2); };
__host__ __device__ __forceinline__ int ws_qr_rows(int m, int nw, int ct) {
  const int rb = ct == 1 ? 8 : (ct == 2 ? 4 : 2);
  const int chunk = (((m + nw - 1) / nw) + rb - 1) / rb * rb;
  return chunk * nw;
}

template <int CT, int NW>
__device__ void ws_qr(int m, int K, double* A, int lda, double* tp, double* wd, double* xch, int w0,
                      int bar) {
  constexpr int RB = WsQrRB<CT>::value;
  const int lane = threadIdx.x & 31, gw = (int)(threadIdx.x >> 5) - w0;
  const int p = min(m, K);
  const int chunk = (((m + NW - 1) / NW) + RB - 1) / RB * RB;
  const int r0 = gw * chunk, r1 = r0 + chunk;  // padded rows are zero
  constexpr int nt = NW * 32;
  const int KP = K + 1;  // row of the exchange buffer: NW partials per column
  double* col[CT];
#pragma unroll
  for (int t = 0; t < CT; ++t) col[t] = A + (int64_t)min(lane + 32 * t, K - 1) * lda;
  // inner products of column 0 with every column over the rows > 0
  double acc[CT], a1[CT];
#pragma unroll
  for (int t = 0; t < CT; ++t) acc[t] = a1[t] = 0.0;
  for (int i = r0; i < r1; i += RB) {
    double v[RB], x[CT][RB];
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      v[u] = A[i + u];
#pragma unroll
      for (int t = 0; t < CT; ++t) x[t][u] = col[t][i + u];
    }
    if (i == 0) v[0] = 0.0;
#pragma unroll
    for (int t = 0; t < CT; ++t)
#pragma unroll
      for (int u = 0; u < RB; u += 2) {
        acc[t] = fma(v[u], x[t][u], acc[t]);
        a1[t] = fma(v[u + 1], x[t][u + 1], a1[t]);
      }
  }
#pragma unroll
  for (int t = 0; t < CT; ++t) acc[t] += a1[t];
  for (int j = 0; j < p; ++j) {
    const double* aj = A + (int64_t)j * lda;
    const bool hasn = j + 1 < K;
    const int jn = hasn ? j + 1 : j;
    const double* an = A + (int64_t)jn * lda;
    // exchange buffer of this step: [c][NW] partial sums, then row j
    double* px = xch + (j & 1) * (NW + 1) * KP;
    double* prow = px + NW * KP;
    const bool own = (j >= r0 && j < r1);  // this warp holds row j
#pragma unroll
    for (int t = 0; t < CT; ++t) {
      const int c = lane + 32 * t;
      if (c >= j && c < K) {
        px[c * NW + gw] = acc[t];
        if (own) prow[c] = col[t][j];
      }
    }
    grp_sync(bar, nt);
    double ss = 0.0, gn = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      ss += px[j * NW + w];
      gn += px[jn * NW + w];
    }
    const double alpha = prow[j];
    const double rown = prow[jn];
    double g[CT], rowv[CT];
    bool on[CT];
#pragma unroll
    for (int t = 0; t < CT; ++t) {
      const int c = lane + 32 * t;
      on[t] = c > j && c < K;
      const int cc = min(c, K - 1);
      g[t] = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) g[t] += px[cc * NW + w];
      rowv[t] = prow[cc];
    }
    double beta, wdj, tpj;
    house_scalars(alpha, ss, beta, wdj, tpj);
    const double fn = hasn ? tpj * fma(wdj, rown, gn) : 0.0;
    double f[CT];
#pragma unroll
    for (int t = 0; t < CT; ++t) f[t] = tpj * fma(wdj, rowv[t], g[t]);
    if (gw == 0 && lane == 0) { tp[j] = tpj; wd[j] = wdj; }
    if (own) {
#pragma unroll
      for (int t = 0; t < CT; ++t) {
        if (on[t]) col[t][j] = fma(-f[t], wdj, rowv[t]);
        if (lane + 32 * t == j) col[t][j] = beta;
      }
    }
    // one pass over the rows below j: update, and the next step's inner
    // products (of the updated column j + 1 with every updated column over
    // the rows > j + 1)
#pragma unroll
    for (int t = 0; t < CT; ++t) acc[t] = a1[t] = 0.0;
    int i = max(r0, (j + 1) / RB * RB);
    if (i <= j + 1 && i < r1) {
      // the block holding row j + 1: rows <= j keep their values, row j + 1
      // is updated but stays out of the inner products
      double v[RB], vn[RB], x[CT][RB];
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        v[u] = aj[i + u];
        vn[u] = an[i + u];
#pragma unroll
        for (int t = 0; t < CT; ++t) x[t][u] = col[t][i + u];
      }
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        if (i + u <= j) v[u] = 0.0;
        vn[u] = (i + u > j + 1) ? fma(-fn, v[u], vn[u]) : 0.0;
#pragma unroll
        for (int t = 0; t < CT; ++t) x[t][u] = fma(-f[t], v[u], x[t][u]);
      }
#pragma unroll
      for (int t = 0; t < CT; ++t)
#pragma unroll
        for (int u = 0; u < RB; u += 2) {
          acc[t] = fma(vn[u], x[t][u], acc[t]);
          a1[t] = fma(vn[u + 1], x[t][u + 1], a1[t]);
        }
      __syncwarp();  // every lane has read column j + 1 before its owner stores it
#pragma unroll
      for (int t = 0; t < CT; ++t)
        if (on[t]) {
#pragma unroll
          for (int u = 0; u < RB; ++u) col[t][i + u] = x[t][u];
        }
      i += RB;
    }
    for (; i < r1; i += RB) {
      double v[RB], vn[RB], x[CT][RB];
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        v[u] = aj[i + u];
        vn[u] = an[i + u];
#pragma unroll
        for (int t = 0; t < CT; ++t) x[t][u] = col[t][i + u];
      }
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        vn[u] = fma(-fn, v[u], vn[u]);
#pragma unroll
        for (int t = 0; t < CT; ++t) x[t][u] = fma(-f[t], v[u], x[t][u]);
      }
#pragma unroll
      for (int t = 0; t < CT; ++t)
#pragma unroll
        for (int u = 0; u < RB; u += 2) {
          acc[t] = fma(vn[u], x[t][u], acc[t]);
          a1[t] = fma(vn[u + 1], x[t][u + 1], a1[t]);
        }
      __syncwarp();
#pragma unroll
      for (int t = 0; t < CT; ++t)
        if (on[t]) {
#pragma unroll
          for (int u = 0; u < RB; ++u) col[t][i + u] = x[t][u];
        }
    }
#pragma unroll
    for (int t = 0; t < CT; ++t) acc[t] += a1[t];
  }
  grp_sync(bar, nt);
}

// number of warps as a runtime value (1, 2, 4 or 8)
template <int CT>
__device__ __forceinline__ void ws_qr_nw(int m, int K, double* A, int lda, double* tp, double* wd,
                                         double* xch, int w0, int nw, int bar) {
  if (nw == 8) ws_qr<CT, 8>(m, K, A, lda, tp, wd, xch, w0, bar);
  else if (nw == 4) ws_qr<CT, 4>(m, K, A, lda, tp, wd, xch, w0, bar);
  else if (nw == 2) ws_qr<CT, 2>(m, K, A, lda, tp, wd, xch, w0, bar);
  else ws_qr<CT, 1>(m, K, A, lda, tp, wd, xch, w0, bar);
}

// S[i, j] = w_i . w_j (i < j < p) written to A[i, j] -- the strict upper
// triangle, whose R entries must be dead.  rows = length of the reflectors.
// Reads touch only the strictly lower part: no hazard with the writes.
// One thread per (i, group of 4 columns j0..j0+3): the column-i values are
// loaded once for four inner products (the phase is shared-memory bound).
__device__ void ws_smat(int rows, int p, double* A, int lda, const double* wd, int tid, int nthr) {
  const int ngj = (p + 3) >> 2;
  for (int e = tid; e < p * ngj; e += nthr) {
    const int i = e % p, j0 = (e / p) * 4;
    if (i >= j0 + 3 || i >= p - 1) continue;  // no column of the group lies right of i
    const double* ai = A + (int64_t)i * lda;
    const double* aj[4];
#pragma unroll
    for (int x = 0; x < 4; ++x) aj[x] = A + (int64_t)min(j0 + x, p - 1) * lda;
    // rows l > j0 + 3 are common to the four products
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    const int lb = min(j0 + 4, rows);
    for (int l = lb; l < rows; l += 4) {
      double v[4], y[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int ll = min(l + u, rows - 1);
        v[u] = (l + u < rows) ? ai[ll] : 0.0;
#pragma unroll
        for (int x = 0; x < 4; ++x) y[x][u] = aj[x][ll];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int x = 0; x < 4; ++x) s[x] = fma(v[u], y[x][u], s[x]);
    }
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int j = j0 + x;
      if (j < p && j > i) {
        // head: w_j's diagonal entry, then the rows j < l < j0 + 4
        double h = wd[j] * ai[j];
        for (int l = j + 1; l < lb; ++l) h = fma(ai[l], aj[x][l], h);
        A[i + (int64_t)j * lda] = h + s[x];
      }
    }
  }
}

// B[j, t] = (W^T Y)[j, t] for j < p, t < r; Y has rowsY (<= rows of W)
// non-zero rows, column t of Y is Y[:, ymap ? ymap[t] : t].
__device__ void ws_wtb(int rowsY, int p, const double* A, int lda, const double* wd, const double* Y,
                       int ldy, const int* ymap, int r, double* B, int ldb, int tid, int nthr) {
  for (int e = tid; e < p * r; e += nthr) {
    const int j = e % p, t = e / p;
    const double* aj = A + (int64_t)j * lda;
    const double* y = Y + (int64_t)(ymap ? ymap[t] : t) * ldy;
    const double d = (j < rowsY) ? wd[j] * y[j] : 0.0;
    B[j + (int64_t)t * ldb] = d + ws_dot<8>(aj + j + 1, 1, y + j + 1, 1, max(rowsY - j - 1, 0));
  }
}

// Z = T B in place: back substitution with T^{-1} = striu(S) + diag(1/tp),
// S[i, j] = A[i, j].  One warp per right-hand side, lane owns the rows
// lane + 32 u (u < RP, p <= 32 RP) in registers; per step the new z_j
// travels by shuffle and every lane eliminates it from its rows
// (column-oriented: the loads of S do not depend on the chain).
template <int RP>
__device__ void ws_trsolve_w(int p, const double* A, int lda, const double* tp, double* B, int ldb, int r,
                             int tid, int nthr) {
  const int lane = tid & 31, wid = tid >> 5, nwp = nthr >> 5;
  for (int t = wid; t < r; t += nwp) {
    double* bt = B + (int64_t)t * ldb;
    double b[RP];
#pragma unroll
    for (int u = 0; u < RP; ++u) b[u] = (lane + 32 * u < p) ? bt[lane + 32 * u] : 0.0;
    double sc[RP], tj = 0.0;
    if (p > 0) {
      tj = tp[p - 1];
#pragma unroll
      for (int u = 0; u < RP; ++u) sc[u] = A[min(lane + 32 * u, p - 1) + (int64_t)(p - 1) * lda];
    }
    for (int j = p - 1; j >= 0; --j) {
      // prefetch the next step's column of S and scalar
      double sn[RP], tn = 0.0;
      const int jn = max(j - 1, 0);
      tn = tp[jn];
#pragma unroll
      for (int u = 0; u < RP; ++u) sn[u] = A[min(lane + 32 * u, p - 1) + (int64_t)jn * lda];
      double bj = b[0];
#pragma unroll
      for (int u = 1; u < RP; ++u) if ((j >> 5) == u) bj = b[u];
      const double zj = __shfl_sync(0xffffffffu, bj, j & 31) * tj;
#pragma unroll
      for (int u = 0; u < RP; ++u) {
        const int row = lane + 32 * u;
        if (row < j) b[u] = fma(-sc[u], zj, b[u]);
        else if (row == j) b[u] = zj;
      }
      tj = tn;
#pragma unroll
      for (int u = 0; u < RP; ++u) sc[u] = sn[u];
    }
#pragma unroll
    for (int u = 0; u < RP; ++u) if (lane + 32 * u < p) bt[lane + 32 * u] = b[u];
  }
}

__device__ void ws_trsolve(int p, const double* A, int lda, const double* tp, double* B, int ldb, int r,
                           int tid, int nthr) {
  if (p <= 32) ws_trsolve_w<1>(p, A, lda, tp, B, ldb, r, tid, nthr);
  else if (p <= 64) ws_trsolve_w<2>(p, A, lda, tp, B, ldb, r, tid, nthr);
  else ws_trsolve_w<4>(p, A, lda, tp, B, ldb, r, tid, nthr);
}

// Out[i, t] = (i < rowsY ? Y[i, t] : 0) - sum_{j < p} W[i, j] Z[j, t] for
// i < rows, t < r.  W[i, j] = A[i, j] below the diagonal, wd[j] on it, 0
// above.  Out may alias Y (each output reads only its own Y entry).  One
// warp per (32-row block, 4-column tile): lanes over rows (coalesced /
// conflict-free), Z broadcast (shared memory, ldz).
template <int CTL, int JU>
__device__ void ws_wz_t(int rows, int p, const double* A, int lda, const double* wd, const double* Y,
                        int ldy, const int* ymap, int rowsY, const double* Z, int ldz, int r, double* Out,
                        int ldo, int tid, int nthr) {
  const int lane = tid & 31, w = tid >> 5, nwp = nthr >> 5;
  const int rb = (rows + 31) >> 5, cb = (r + CTL - 1) / CTL;
  for (int tile = w; tile < rb * cb; tile += nwp) {
    const int i = (tile % rb) * 32 + lane, t0 = (tile / rb) * CTL;
    const bool act = i < rows;
    const int ii = min(i, rows - 1);
    double acc[CTL];
    const double* z[CTL];
#pragma unroll
    for (int x = 0; x < CTL; ++x) { acc[x] = 0.0; z[x] = Z + (int64_t)min(t0 + x, r - 1) * ldz; }
    const int jd = min(p, ii);  // W[i, j] = A[i, j] for j < min(p, i)
    const int jw = min(p, ((tile % rb) * 32 + 31));  // warp-uniform bound of the blocked loop
    const double* ar = A + ii;
    int j = 0;
    for (; j + JU <= jw; j += JU) {
      double wv[JU];
#pragma unroll
      for (int u = 0; u < JU; ++u) {
        wv[u] = ar[(int64_t)(j + u) * lda];
        if (j + u >= jd) wv[u] = 0.0;
      }
#pragma unroll
      for (int u = 0; u < JU; ++u)
#pragma unroll
        for (int x = 0; x < CTL; ++x) acc[x] = fma(wv[u], z[x][j + u], acc[x]);
    }
    for (; j < jd; ++j) {
      const double wv = ar[(int64_t)j * lda];
#pragma unroll
      for (int x = 0; x < CTL; ++x) acc[x] = fma(wv, z[x][j], acc[x]);
    }
    if (ii < p) {
      const double wv = wd[ii];
#pragma unroll
      for (int x = 0; x < CTL; ++x) acc[x] = fma(wv, z[x][ii], acc[x]);
    }
    if (act) {
#pragma unroll
      for (int x = 0; x < CTL; ++x) {
        const int t = t0 + x;
        if (t < r) {
          const double y0 = (i < rowsY) ? Y[i + (int64_t)(ymap ? ymap[t] : t) * ldy] : 0.0;
          Out[i + (int64_t)t * ldo] = y0 - acc[x];
        }
      }
    }
  }
}

// gsrc: A lives in global memory (more loads in flight, wider column tiles)
__device__ void ws_wz(int rows, int p, const double* A, int lda, const double* wd, const double* Y,
                      int ldy, const int* ymap, int rowsY, const double* Z, int ldz, int r, double* Out,
                      int ldo, int tid, int nthr, bool gsrc = false) {
  if (gsrc) ws_wz_t<8, 8>(rows, p, A, lda, wd, Y, ldy, ymap, rowsY, Z, ldz, r, Out, ldo, tid, nthr);
  else ws_wz_t<4, 4>(rows, p, A, lda, wd, Y, ldy, ymap, rowsY, Z, ldz, r, Out, ldo, tid, nthr);
}

// ---------------------------------------------------------------------------
// Rank-revealing (column-pivoted) Householder QR of the p x q matrix G by the
// warps [w0, w0 + nw), q <= 32 nw, one physical column per lane, stopped
// after k steps once ||G[k:, unpivoted]||_F <= thr |R_00| (the criterion of
// cta_rrqr).  Columns are not swapped: perm[j] = physical column of step j,
// pos[c] = step at which column c was chosen (INT_MAX: never).  R_1[i, c] =
// G[i, c] if pos[c] > i, rd[i] if pos[c] == i, 0 otherwise.  Reflector j:
// tail in G[j+1:, perm[j]], wd[j], tp[j].  xch: 6 * nw doubles.
// ---------------------------------------------------------------------------
__device__ int ws_rrqr(int p, int q, double* G, int ldg, double* tp, double* wd, double* rd, int* perm,
                       int* pos, double thr, double* xch, int w0, int nw, int bar) {
  constexpr int RB = 4;
  const int lane = threadIdx.x & 31, gw = (int)(threadIdx.x >> 5) - w0;
  const int c = gw * 32 + lane;
  const bool has = c < q;
  double* gc = G + (int64_t)min(c, q - 1) * ldg;
  bool active = has;
  double cn = 0.0;
  if (has) {
    cn = ws_dot<8>(gc, 1, gc, 1, p);
    pos[c] = 0x7fffffff;
  }
  const int kmax = min(p, q);
  const int nt = nw * 32;
  double r00sq = 0.0;
  int k = kmax;
  for (int j = 0; j < kmax; ++j) {
    double v = active ? cn : -1.0, tail = active ? cn : 0.0;
    int idx = active ? c : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      tail += __shfl_xor_sync(0xffffffffu, tail, o);
      if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
    }
    if (nw > 1) {
      double* px = xch + (j & 1) * 3 * nw;
      if (lane == 0) { px[3 * gw] = v; px[3 * gw + 1] = (double)idx; px[3 * gw + 2] = tail; }
      grp_sync(bar, nt);
      v = -1.0; idx = 0x7fffffff; tail = 0.0;
      for (int w = 0; w < nw; ++w) {
        const double ov = px[3 * w];
        const int oi = (int)px[3 * w + 1];
        if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
        tail += px[3 * w + 2];
      }
    } else {
      __syncwarp();
    }
    if (j == 0) r00sq = v;
    if (!(v > 0.0) || tail <= thr * thr * r00sq) { k = j; break; }
    const int pc = idx;
    const double* gp = G + (int64_t)pc * ldg;
    const double alpha = gp[j];
    const bool upd = active && c != pc;
    double ss = 0.0, ss1 = 0.0, g0 = 0.0, g1 = 0.0;
    for (int i = j + 1; i < p; i += RB) {
      double a[RB], x[RB];
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        const int ii = min(i + u, p - 1);
        a[u] = gp[ii];
        if (i + u >= p) a[u] = 0.0;
        x[u] = gc[ii];
      }
#pragma unroll
      for (int u = 0; u < RB; u += 2) {
        ss = fma(a[u], a[u], ss); ss1 = fma(a[u + 1], a[u + 1], ss1);
        g0 = fma(a[u], x[u], g0); g1 = fma(a[u + 1], x[u + 1], g1);
      }
    }
    double beta, wdj, tpj;
    house_scalars(alpha, ss + ss1, beta, wdj, tpj);
    if (has && c == pc) {
      active = false;
      pos[c] = j; perm[j] = pc; tp[j] = tpj; wd[j] = wdj; rd[j] = beta;
    }
    if (upd) {
      const double f = tpj * fma(wdj, gc[j], g0 + g1);
      gc[j] = fma(-f, wdj, gc[j]);
      double s0 = 0.0, s1 = 0.0;
      for (int i = j + 1; i < p; i += RB) {
        double a[RB], x[RB];
#pragma unroll
        for (int u = 0; u < RB; ++u) {
          const int ii = min(i + u, p - 1);
          a[u] = gp[ii];
          x[u] = gc[ii];
        }
#pragma unroll
        for (int u = 0; u < RB; ++u) {
          x[u] = (i + u < p) ? fma(-f, a[u], x[u]) : 0.0;
          if (i + u < p) gc[i + u] = x[u];
        }
#pragma unroll
        for (int u = 0; u < RB; u += 2) { s0 = fma(x[u], x[u], s0); s1 = fma(x[u + 1], x[u + 1], s1); }
      }
      cn = s0 + s1;
    }
  }
  grp_sync(bar, nt);
  return k;
}

// ---------------------------------------------------------------------------
// One-sided Jacobi on the rows x k matrix X (columns rotated in place), the
// whole CTA, one group of G lanes per column pair, all pairs of a round at
// once (round-robin ordering as in jacobi_rounds).  A lane keeps its RPL
// rows of both columns in registers between the inner products and the
// rotation (rows <= G * RPL).  The rotation comes from two reciprocal
// square roots: with d = be - al, g = 2 ga, h = |(d, g)|:
// c^2 = (1 + |d|/h)/2, s = sign(d) g / (2 c h).
// Pairs are rotated whenever their cosine exceeds 1e-14 (the inner products
// are there anyway), but only cosines above `tol` keep the iteration going:
// the last sweep then leaves the columns orthogonal to ~tol^2, which the
// recovery of the left factor as R1 X / sigma relies on.
// ---------------------------------------------------------------------------
template <int G, int RPL>
__device__ void ws_jacobi_rounds(int rows, int k, double* X, int ldx, double tol2, int* flag) {
  const int kk = k + (k & 1);
  const int npairs = kk / 2;
  const int grp = threadIdx.x / G, gl = threadIdx.x % G;
  const int ngrp = HMX_THREADS / G;
  const int mq = kk - 1;
  for (int rnd = 0; rnd < mq; ++rnd) {
    for (int pr0 = 0; pr0 < npairs; pr0 += ngrp) {
      const int pr = pr0 + grp;
      int a, b;
      if (pr == 0) { a = 0; b = 1 + rnd; }
      else {
        a = pr + rnd; if (a >= mq) a -= mq;
        a += 1;
        b = mq - pr + rnd; if (b >= mq) b -= mq;
        b += 1;
      }
      const bool valid = pr < npairs && a < k && b < k;
      if (a > b) { const int t = a; a = b; b = t; }
      double* x = X + (int64_t)(valid ? a : 0) * ldx;
      double* y = X + (int64_t)(valid ? b : 0) * ldx;
      double xr[RPL], yr[RPL];
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        const int i = gl + u * G;
        const bool in = valid && i < rows;
        xr[u] = in ? x[i] : 0.0;
        yr[u] = in ? y[i] : 0.0;
      }
      double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        al = fma(xr[u], xr[u], al); be = fma(yr[u], yr[u], be); ga = fma(xr[u], yr[u], ga);
      }
      al = seg_sum<G>(al); be = seg_sum<G>(be); ga = seg_sum<G>(ga);
      const double gg = ga * ga, ab = al * be;
      if (!valid || al == 0.0 || be == 0.0 || gg <= 1e-28 * ab) continue;
      const double d = be - al, g2 = 2.0 * ga;
      const double rh = rsqrt(fma(d, d, g2 * g2));
      const double hc = fma(0.5 * fabs(d), rh, 0.5);  // c^2 in [1/2, 1]
      const double rc = rsqrt(hc);
      const double c = hc * rc;
      const double s = copysign(0.5, d) * g2 * rh * rc;
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        const int i = gl + u * G;
        if (i < rows) {
          x[i] = c * xr[u] - s * yr[u];
          y[i] = s * xr[u] + c * yr[u];
        }
      }
      if (gl == 0 && gg > tol2 * ab) *flag = 1;
    }
    __syncthreads();
  }
}

// Returns false if not converged after 60 sweeps.  sigma / order as in
// cta_jacobi_svd.  rows <= 512.
__device__ bool ws_jacobi(int rows, int k, double* X, int ldx, double* sigma, int* order, int* flag,
                          int* sweeps_out) {
  // A sweep whose pairs all arrive with cosines <= HMX_WS_JTOL is the last
  // one: its rotations (applied down to 1e-14) leave cosines of order
  // k * HMX_WS_JTOL^2 (quadratic convergence of the cyclic method), i.e.
  // <= 1e-10 for k <= 100, the bound the step-synchronous path verifies with
  // one more sweep.
  const double tol = HMX_WS_JTOL;
  const double tol2 = tol * tol;
  const int npairs = (k + (k & 1)) / 2;
  bool converged = (k <= 1);
  __syncthreads();
  int sweep = 0;
  for (; sweep < 60 && !converged; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    // widest lane group that still covers every pair in one pass, rows in
    // at most 8 registers per column and lane
    if (npairs * 32 <= HMX_THREADS || rows > 128) {
      if (rows <= 64) ws_jacobi_rounds<32, 2>(rows, k, X, ldx, tol2, flag);
      else if (rows <= 128) ws_jacobi_rounds<32, 4>(rows, k, X, ldx, tol2, flag);
      else if (rows <= 256) ws_jacobi_rounds<32, 8>(rows, k, X, ldx, tol2, flag);
      else ws_jacobi_rounds<32, 16>(rows, k, X, ldx, tol2, flag);
    } else if (npairs * 16 <= HMX_THREADS || rows > 64) {
      if (rows <= 64) ws_jacobi_rounds<16, 4>(rows, k, X, ldx, tol2, flag);
      else ws_jacobi_rounds<16, 8>(rows, k, X, ldx, tol2, flag);
    } else {
      ws_jacobi_rounds<8, 8>(rows, k, X, ldx, tol2, flag);
    }
    converged = (*flag == 0);
    __syncthreads();
  }
  if (sweeps_out) *sweeps_out = sweep;
  jacobi_sigma_order(rows, k, X, ldx, sigma, order);
  return converged;
}

// ---------------------------------------------------------------------------
// Rank-revealing Householder QR of a p x q block G held in GLOBAL memory
// (dense_to_lowrank of large blocks: the block does not fit shared memory
// but lives in L2), whole CTA.  Lanes run over rows (coalesced), warp w
// owns the columns c = w (mod HMX_WARPS).  One pass over the trailing
// matrix per step: the pass that applies reflector j to a column also
// accumulates the column's inner product with the NEXT pivot column and
// its exact trailing norm.  The next pivot is chosen before the pass from
// the norms downdated by one step (exact norm minus r_jc^2, as dlaqp2 does
// once); the stopping test uses the exact norms the pass produces:
// stop after k steps when ||G[k:, unpivoted]||_F <= thr |R_00|, or at
// kcap.  Columns are not swapped (perm / pos as in ws_rrqr); R_1[i, c] =
// G[i, c] if pos[c] > i, rd[i] if pos[c] == i.
// Shared work arrays: tp, wd, rd (kcap), perm (kcap), pos, cn, gq, rown, fq
// (q each), wv, wn (p each), red (3 * HMX_WARPS + 8 doubles).
// ---------------------------------------------------------------------------
struct WsGqr {
  double *tp, *wd, *rd, *cn, *gq, *rown, *fq, *wv, *wn, *red;
  int *perm, *pos;
};

template <int RPLG>
__device__ int ws_gqr(int p, int q, double* G, int64_t ld, double thr, int kcap, const WsGqr& a) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  int* ired = reinterpret_cast<int*>(a.red + 3 * HMX_WARPS);
  // column norms
  for (int c = w; c < q; c += HMX_WARPS) {
    const double* x = G + (int64_t)c * ld;
    double s0 = 0.0;
#pragma unroll
    for (int u = 0; u < RPLG; ++u) {
      const int i = lane + 32 * u;
      const double v = i < p ? x[i] : 0.0;
      s0 = fma(v, v, s0);
    }
    s0 = warp_sum(s0);
    if (lane == 0) { a.cn[c] = s0; a.pos[c] = 0x7fffffff; }
  }
  __syncthreads();
  // block arg-max of cn over the unpivoted columns (+ their sum)
  auto argmax = [&](double& vmax, double& tail) -> int {
    double v = -1.0, t = 0.0;
    int idx = 0x7fffffff;
    for (int c = tid; c < q; c += HMX_THREADS)
      if (a.pos[c] == 0x7fffffff) {
        const double x = a.cn[c];
        t += x;
        if (x > v) { v = x; idx = c; }
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      t += __shfl_xor_sync(0xffffffffu, t, o);
      if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
    }
    __syncthreads();
    if (lane == 0) { a.red[3 * w] = v; a.red[3 * w + 1] = (double)idx; a.red[3 * w + 2] = t; }
    __syncthreads();
    v = -1.0; idx = 0x7fffffff; t = 0.0;
#pragma unroll
    for (int x = 0; x < HMX_WARPS; ++x) {
      const double ov = a.red[3 * x];
      const int oi = (int)a.red[3 * x + 1];
      if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
      t += a.red[3 * x + 2];
    }
    vmax = v; tail = t;
    return idx;
  };
  double vmax, tail;
  int pc = argmax(vmax, tail);
  const double r00sq = vmax;
  const int kmax = min(min(p, q), kcap);
  if (!(vmax > 0.0) || kmax == 0) return 0;
  // inner products of the first pivot column (rows > 0) with every column
  for (int i = tid; i < p; i += HMX_THREADS) a.wn[i] = i > 0 ? G[i + (int64_t)pc * ld] : 0.0;
  __syncthreads();
  for (int c = w; c < q; c += HMX_WARPS) {
    const double* x = G + (int64_t)c * ld;
    double s0 = 0.0;
#pragma unroll
    for (int u = 0; u < RPLG; ++u) {
      const int i = lane + 32 * u;
      if (i < p) s0 = fma(a.wn[i], x[i], s0);
    }
    s0 = warp_sum(s0);
    if (lane == 0) { a.gq[c] = s0; a.rown[c] = x[0]; }
  }
  __syncthreads();
  int k = kmax;
  for (int j = 0; j < kmax; ++j) {
    // reflector j from column pc; update factors, row j of R, downdated norms
    double beta, wdj, tpj;
    house_scalars(a.rown[pc], a.gq[pc], beta, wdj, tpj);
    __syncthreads();  // everyone has read rown[pc] / gq[pc]
    for (int c = tid; c < q; c += HMX_THREADS) {
      if (a.pos[c] != 0x7fffffff || c == pc) continue;
      const double f = tpj * fma(wdj, a.rown[c], a.gq[c]);
      const double rjc = fma(-f, wdj, a.rown[c]);
      a.fq[c] = f;
      G[j + (int64_t)c * ld] = rjc;
      a.cn[c] = fmax(a.cn[c] - rjc * rjc, 0.0);
    }
    if (tid == 0) { a.tp[j] = tpj; a.wd[j] = wdj; a.rd[j] = beta; a.perm[j] = pc; }
    // w_j tail (rows > j) for the pass
    for (int i = tid; i < p; i += HMX_THREADS) a.wv[i] = i > j ? G[i + (int64_t)pc * ld] : 0.0;
    __syncthreads();
    if (tid == 0) a.pos[pc] = j;
    __syncthreads();
    if (j + 1 == kmax) break;
    const int pn = argmax(vmax, tail);  // next pivot from the downdated norms
    if (pn == 0x7fffffff || !(vmax > 0.0)) { k = j + 1; break; }
    // the next pivot column first: updated, stored, its tail (rows > j+1) to wn
    __syncthreads();  // the arg-max results in red are consumed
    {
      double* x = G + (int64_t)pn * ld;
      const double f = a.fq[pn];
      double s0 = 0.0, s1 = 0.0;
      for (int i = tid; i < p; i += HMX_THREADS) {
        const double v = fma(-f, a.wv[i], x[i]);
        if (i > j) x[i] = v;
        a.wn[i] = i > j + 1 ? v : 0.0;
        if (i == j + 1) a.rown[pn] = v;
        if (i > j) s0 = fma(v, v, s0);
        if (i > j + 1) s1 = fma(v, v, s1);
      }
      s0 = warp_sum(s0); s1 = warp_sum(s1);
      if (lane == 0) { a.red[2 * w] = s0; a.red[2 * w + 1] = s1; }
      __syncthreads();
      if (tid == 0) {
        double t0 = 0.0, t1 = 0.0;
        for (int x2 = 0; x2 < HMX_WARPS; ++x2) { t0 += a.red[2 * x2]; t1 += a.red[2 * x2 + 1]; }
        a.cn[pn] = t0; a.gq[pn] = t1;
      }
    }
    // fused pass over this warp's other unpivoted columns, two at a time
    const int lj = (j + 1) & 31, uj = (j + 1) >> 5;
    for (int c0 = w; c0 < q; c0 += 2 * HMX_WARPS) {
      const int c1 = c0 + HMX_WARPS;
      const bool on0 = a.pos[c0] == 0x7fffffff && c0 != pn;
      const bool on1 = c1 < q && a.pos[c1] == 0x7fffffff && c1 != pn;
      if (!on0 && !on1) continue;
      double* x0 = G + (int64_t)c0 * ld;
      double* x1 = G + (int64_t)(on1 ? c1 : c0) * ld;
      const double f0 = on0 ? a.fq[c0] : 0.0, f1 = on1 ? a.fq[c1] : 0.0;
      double v0[RPLG], v1[RPLG];
#pragma unroll
      for (int u = 0; u < RPLG; ++u) {
        const int i = lane + 32 * u;
        v0[u] = (on0 && i < p) ? x0[i] : 0.0;
        v1[u] = (on1 && i < p) ? x1[i] : 0.0;
      }
      double g0 = 0.0, g1 = 0.0, n0 = 0.0, n1 = 0.0, r0 = 0.0, r1 = 0.0;
#pragma unroll
      for (int u = 0; u < RPLG; ++u) {
        const int i = lane + 32 * u;
        const double wvi = i < p ? a.wv[i] : 0.0, wni = i < p ? a.wn[i] : 0.0;
        v0[u] = fma(-f0, wvi, v0[u]);
        v1[u] = fma(-f1, wvi, v1[u]);
        g0 = fma(wni, v0[u], g0);
        g1 = fma(wni, v1[u], g1);
        if (i > j) { n0 = fma(v0[u], v0[u], n0); n1 = fma(v1[u], v1[u], n1); }
        if (u == uj && lane == lj) { r0 = v0[u]; r1 = v1[u]; }
        if (i > j && i < p) {
          if (on0) x0[i] = v0[u];
          if (on1) x1[i] = v1[u];
        }
      }
      g0 = warp_sum(g0); g1 = warp_sum(g1); n0 = warp_sum(n0); n1 = warp_sum(n1);
      if (lane == lj) {
        if (on0) { a.rown[c0] = r0; }
        if (on1) { a.rown[c1] = r1; }
      }
      if (lane == 0) {
        if (on0) { a.gq[c0] = g0; a.cn[c0] = n0; }
        if (on1) { a.gq[c1] = g1; a.cn[c1] = n1; }
      }
    }
    __syncthreads();
    // exact trailing norms: stop?
    {
      double t = 0.0;
      for (int c = tid; c < q; c += HMX_THREADS)
        if (a.pos[c] == 0x7fffffff) t += a.cn[c];
      t = warp_sum(t);
      if (lane == 0) a.red[w] = t;
      __syncthreads();
      if (tid == 0) {
        double tt = 0.0;
        for (int x2 = 0; x2 < HMX_WARPS; ++x2) tt += a.red[x2];
        ired[0] = (tt <= thr * thr * r00sq) ? 1 : 0;
      }
      __syncthreads();
      if (ired[0]) { k = j + 1; break; }
    }
    pc = pn;
  }
  __syncthreads();
  return k;
}

// striu(W^T W) of a reflector block in global memory (coalesced: one warp per
// pair, lanes over rows), written to the strict upper triangle.
__device__ void ws_smat_g(int rows, int p, double* A, int64_t lda, const double* wd) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int npair = p * (p - 1) / 2;
  for (int e = w; e < npair; e += HMX_WARPS) {
    int j = (int)((1.0f + sqrtf(1.0f + 8.0f * (float)e)) * 0.5f);
    while (j * (j - 1) / 2 > e) --j;
    while ((j + 1) * j / 2 <= e) ++j;
    const int i = e - j * (j - 1) / 2;
    const double* ai = A + (int64_t)i * lda;
    double* aj = A + (int64_t)j * lda;
    double s0 = 0.0, s1 = 0.0;
    int l = j + 1 + lane;
    for (; l + 32 < rows; l += 64) {
      const double x0 = ai[l], y0 = aj[l], x1 = ai[l + 32], y1 = aj[l + 32];
      s0 = fma(x0, y0, s0);
      s1 = fma(x1, y1, s1);
    }
    if (l < rows) s0 = fma(ai[l], aj[l], s0);
    s0 = warp_sum(s0 + s1);
    if (lane == 0) aj[i] = fma(wd[j], ai[j], s0);
  }
}

// ---------------------------------------------------------------------------
// Column-blocked Householder QR for factors whose K columns do not fit
// shared memory next to their rows ("fat" stacked factors, K up to 128 and
// more): blocks of nb columns are factored in shared memory by all warps
// (ws_qr) after the previous blocks have been applied to them, each block
// c in compact-WY form Q_c = I - W_c T_c W_c^T with its own T_c^{-1} =
// striu(W_c^T W_c) + diag(1/tp) (nb x nb, kept in the strict upper triangle
// of the block's diagonal block).  Q = Q_0 Q_1 ... Q_{B-1}.
// ---------------------------------------------------------------------------

// forward substitution (T^{-1})^T Z = B with L[i, j] (i > j) = Ls[i + j ldl]
// (the transposed striu(S)) and diagonal 1/tp; warp per right-hand side.
template <int RP>
__device__ void ws_trsolve_fwd_w(int p, const double* Ls, int ldl, const double* tp, double* B, int ldb,
                                 int r, int tid, int nthr) {
  const int lane = tid & 31, wid = tid >> 5, nwp = nthr >> 5;
  for (int t = wid; t < r; t += nwp) {
    double* bt = B + (int64_t)t * ldb;
    double b[RP];
#pragma unroll
    for (int u = 0; u < RP; ++u) b[u] = (lane + 32 * u < p) ? bt[lane + 32 * u] : 0.0;
    double sc[RP], tj = p > 0 ? tp[0] : 0.0;
#pragma unroll
    for (int u = 0; u < RP; ++u) sc[u] = p > 0 ? Ls[min(lane + 32 * u, p - 1)] : 0.0;
    for (int j = 0; j < p; ++j) {
      double sn[RP];
      const int jn = min(j + 1, p - 1);
      const double tn = tp[jn];
#pragma unroll
      for (int u = 0; u < RP; ++u) sn[u] = Ls[min(lane + 32 * u, p - 1) + (int64_t)jn * ldl];
      double bj = b[0];
#pragma unroll
      for (int u = 1; u < RP; ++u) if ((j >> 5) == u) bj = b[u];
      const double zj = __shfl_sync(0xffffffffu, bj, j & 31) * tj;
#pragma unroll
      for (int u = 0; u < RP; ++u) {
        const int row = lane + 32 * u;
        if (row > j) b[u] = fma(-sc[u], zj, b[u]);
        else if (row == j) b[u] = zj;
      }
      tj = tn;
#pragma unroll
      for (int u = 0; u < RP; ++u) sc[u] = sn[u];
    }
#pragma unroll
    for (int u = 0; u < RP; ++u) if (lane + 32 * u < p) bt[lane + 32 * u] = b[u];
  }
}

__device__ void ws_trsolve_fwd(int p, const double* Ls, int ldl, const double* tp, double* B, int ldb, int r,
                               int tid, int nthr) {
  if (p <= 32) ws_trsolve_fwd_w<1>(p, Ls, ldl, tp, B, ldb, r, tid, nthr);
  else if (p <= 64) ws_trsolve_fwd_w<2>(p, Ls, ldl, tp, B, ldb, r, tid, nthr);
  else ws_trsolve_fwd_w<4>(p, Ls, ldl, tp, B, ldb, r, tid, nthr);
}

// Y (rows x r, in place, any memory) := Q_c Y (trans = false) or Q_c^T Y
// (trans = true) for one reflector block in CLEAN form: W (rows x jc at A,
// lda) holds the tails below the diagonal, wd ON the diagonal and zeros
// above it, so W^T Y and W Z are plain GEMMs (cta_gemm: shared-memory
// staged tiles, any operand memory); striu(W^T W) is kept apart (Sg, jc x jc,
// ld lds).  Shared work: Sc ((jc|1) x jc), Bm ((jc|1) x r), sw (jc), gsm
// (GEMM_SMEM_DOUBLES).  Whole CTA, ends synchronised.
__device__ void ws_apply_block(int rows, int jc, const double* A, int64_t lda, const double* tp,
                               const double* Sg, int lds, bool trans, double* Y, int64_t ldy, int r,
                               double* Sc, double* Bm, double* sw, double* gsm) {
  const int tid = threadIdx.x;
  const int lb = jc | 1;
  if (jc <= 0 || r <= 0) return;
  for (int e = tid; e < jc; e += HMX_THREADS) sw[e] = tp[e];
  if (!trans) { FOR_MN(i, j, jc, jc) Sc[i + j * lb] = (i < j) ? Sg[i + (int64_t)j * lds] : 0.0; }
  else { FOR_MN(j, i, jc, jc) Sc[i + j * lb] = (i > j) ? Sg[j + (int64_t)i * lds] : 0.0; }
  __syncthreads();
  cta_gemm(jc, r, rows, 1.0, A, (int)lda, true, Y, (int)ldy, false, false, Bm, lb, gsm);
  if (!trans) ws_trsolve(jc, Sc, lb, sw, Bm, lb, r, tid, HMX_THREADS);
  else ws_trsolve_fwd(jc, Sc, lb, sw, Bm, lb, r, tid, HMX_THREADS);
  __syncthreads();
  cta_gemm(rows, r, jc, -1.0, A, (int)lda, false, Bm, lb, false, true, Y, (int)ldy, gsm);
}

// striu(W^T W) of a clean reflector block (rows x jc) into Sg (jc x jc, ld
// lds; the lower part and the diagonal receive W^T W too and are ignored).
__device__ void ws_smat_gemm(int rows, int jc, const double* A, int64_t lda, double* Sg, int lds, double* gsm) {
  cta_gemm(jc, jc, rows, 1.0, A, (int)lda, true, A, (int)lda, false, false, Sg, lds, gsm);
}

// block width for an m-row factor: the panel (m + pad rows) x nb, two
// (nb|1) x nb work blocks, the GEMM staging and the exchange buffers must
// fit `cap` doubles
__device__ __forceinline__ int ws_cb_nb(int m, int K, int64_t cap) {
  const int64_t lp = (m + 64) | 1;
  for (int nb = 64; nb >= 8; nb -= 8) {
    const int64_t need = lp * nb + 2 * (int64_t)(nb | 1) * nb + 2 * (HMX_WARPS + 1) * (nb + 1) + 4 * nb +
                         GEMM_SMEM_DOUBLES + 64;
    if (need <= cap) return min(nb, (K + 7) & ~7);
  }
  return 0;
}

// QR of the m x K factor A (global, in place; on exit the clean reflector
// blocks: tails below the diagonal, wd on it, zeros above within a block's
// diagonal block; rows above a block keep stale R entries).  Rz: R (p x K,
// ld p, zeros below the diagonal).  sc (global): tp at [0, p).  Sg (global,
// nb x nb per block, ld nb): striu(W_c^T W_c).  wk: shared work area.
__device__ void ws_cbqr(int m, int K, double* A, int64_t lda, double* Rz, double* sc, double* Sg, int nb,
                        double* wk) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int p = min(m, K);
  const int lp = (m + 64) | 1, lb = nb | 1;
  double* Ps = wk;
  double* Sc = Ps + (int64_t)lp * nb;
  double* Bm = Sc + lb * nb;
  double* xch = Bm + lb * nb;
  double* tps = xch + 2 * (HMX_WARPS + 1) * (nb + 1);
  double* wds = tps + nb;
  double* sw = wds + nb;  // nb
  double* gsm = sw + 2 * nb;
  for (int j0 = 0; j0 < K; j0 += nb) {
    const int jb = min(nb, K - j0);
    for (int c = w; c < jb; c += HMX_WARPS) {
      const double* s_ = A + (int64_t)(j0 + c) * lda;
      double* d_ = Ps + c * lp;
      for (int i = lane; i < lp; i += 128) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = (i + 32 * u < m) ? s_[i + 32 * u] : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) if (i + 32 * u < lp) d_[i + 32 * u] = v[u];
      }
    }
    __syncthreads();
    // Q_{b-1}^T ... Q_0^T applied to the new columns, first block first
    for (int c0 = 0; c0 < min(j0, p); c0 += nb) {
      const int jc = min(nb, p - c0);
      ws_apply_block(m - c0, jc, A + c0 + (int64_t)c0 * lda, lda, sc + c0, Sg + (int64_t)(c0 / nb) * nb * nb, nb,
                     true, Ps + c0, lp, jb, Sc, Bm, sw, gsm);
    }
    if (j0 < p) {
      if (jb <= 32) ws_qr<1, HMX_WARPS>(m - j0, jb, Ps + j0, lp, tps, wds, xch, 0, 0);
      else ws_qr<2, HMX_WARPS>(m - j0, jb, Ps + j0, lp, tps, wds, xch, 0, 0);
    }
    FOR_MN(i, c, p, jb) Rz[i + (int64_t)(j0 + c) * p] = (i <= j0 + c) ? Ps[i + c * lp] : 0.0;
    __syncthreads();
    if (j0 < p) {
      const int jq = min(jb, p - j0);
      ws_smat(m - j0, jq, Ps + j0, lp, wds, tid, HMX_THREADS);
      __syncthreads();
      double* Sgb = Sg + (int64_t)(j0 / nb) * nb * nb;
      FOR_MN(i, c, jq, jq) Sgb[i + c * nb] = (i < c) ? Ps[j0 + i + c * lp] : 0.0;
      // clean block: wd on the diagonal, zeros above it (columns beyond p keep R)
      for (int c = w; c < jb; c += HMX_WARPS)
        for (int i = j0 + lane; i < m; i += 32) {
          const int ii = i - j0;
          double v = Ps[i + c * lp];
          if (c < jq) v = ii > c ? v : (ii == c ? wds[c] : 0.0);
          A[i + (int64_t)(j0 + c) * lda] = v;
        }
      for (int e = tid; e < jq; e += HMX_THREADS) sc[j0 + e] = tps[e];
    }
    __syncthreads();
  }
}

}  // namespace hmx
