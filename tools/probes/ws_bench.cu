// Cycle counts of the warp-synchronous truncation building blocks
// (hmx_ws.cuh) on one CTA:  nvcc -O3 -arch=sm_100a -o ws_bench ws_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_1911_07531_b200/csrc/hmx_ws.cuh"
using namespace hmx;

__device__ double rnd(unsigned& s) { s = s * 1664525u + 1013904223u; return ((s >> 8) & 0xffff) / 65536.0 - 0.5; }

__global__ void __launch_bounds__(256, 1) k_bench(int what, int m, int K, int nw, long long* cyc, double* out, int reps) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x;
  const int lda = m | 1;
  double* A = sm;
  double* tp = A + lda * K;
  double* wd = tp + K;
  double* rd = wd + K;
  double* xch = rd + K;               // 2 * 9 * K
  double* B = xch + 2 * 9 * (K + 1) + 64;   // lda x K
  int* perm = reinterpret_cast<int*>(B + lda * K);
  int* pos = perm + K;
  int* ord = pos + K;
  double* sig = reinterpret_cast<double*>(ord + K);
  int* flag = reinterpret_cast<int*>(sig + K);
  long long t0 = 0;
  for (int rep = 0; rep < reps; ++rep) {
  unsigned s = 1234u + tid * 7919u;
  for (int e = tid; e < lda * K; e += 256) { A[e] = rnd(s) * exp(-0.3 * (e / lda)); B[e] = rnd(s); }
  __syncthreads();
  t0 = clock64();
  if (what == 0) {  // ws_qr on nw warps
    if ((tid >> 5) < nw) {
      if (K <= 32) ws_qr_nw<1>(m, K, A, lda, tp, wd, xch, 0, nw, nw == 8 ? 0 : 1);
      else ws_qr_nw<2>(m, K, A, lda, tp, wd, xch, 0, nw, nw == 8 ? 0 : 1);
    }
  } else if (what == 1) {  // rrqr m x K
    const int nwr = (K + 31) >> 5;
    if ((tid >> 5) < nwr) ws_rrqr(m, K, A, lda, tp, wd, rd, perm, pos, 1e-10, xch, 0, nwr, 1);
  } else if (what == 2) {  // jacobi m x K
    ws_jacobi(m, K, A, lda, sig, ord, flag, perm);
  } else if (what == 3) {  // smat
    ws_smat(m, min(m, K), A, lda, wd, tid, 256);
  } else if (what == 4) {  // wtb + trsolve + wz with r = K/2
    const int p = min(m, K), r = max(K / 2, 1);
    ws_wtb(p, p, A, lda, wd, B, lda, nullptr, r, B + (lda * K) / 2, lda, tid, 256);
    __syncthreads();
    long long t1 = clock64();
    ws_trsolve(p, A, lda, tp, B + (lda * K) / 2, lda, r, tid, 256);
    __syncthreads();
    long long t2 = clock64();
    ws_wz(m, p, A, lda, wd, B, lda, nullptr, p, B + (lda * K) / 2, lda, r, out + 1024, m, tid, 256);
    __syncthreads();
    long long t3 = clock64();
    if (tid == 0) { cyc[1] = t1 - t0; cyc[2] = t2 - t1; cyc[3] = t3 - t2; }
  }
  __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) { cyc[0] = t1 - t0; if (what == 2) cyc[1] = perm[0]; }
  out[tid] = A[tid % (lda * K)];
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  long long* cyc; double* out;
  cudaMallocManaged(&cyc, 64); cudaMalloc(&out, 8 << 20);
  cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct C { int what, m, K, nw; const char* name; };
  C cases[] = {
    {0, 64, 20, 4, "qr 64x20 4w"}, {0, 64, 32, 4, "qr 64x32 4w"}, {0, 64, 40, 4, "qr 64x40 4w"},
    {0, 64, 20, 1, "qr 64x20 1w"}, {0, 64, 20, 2, "qr 64x20 2w"}, {0, 64, 20, 8, "qr 64x20 8w"},
    {0, 256, 24, 4, "qr 256x24 4w"}, {0, 256, 24, 8, "qr 256x24 8w"}, {0, 384, 24, 8, "qr 384x24 8w"},
    {1, 20, 20, 1, "rrqr 20x20"}, {1, 40, 40, 2, "rrqr 40x40"}, {1, 24, 24, 1, "rrqr 24x24"},
    {2, 20, 20, 8, "jacobi 20x20"}, {2, 40, 40, 8, "jacobi 40x40"}, {2, 24, 12, 8, "jacobi 24x12"},
    {3, 64, 20, 8, "smat 64x20"}, {3, 256, 24, 8, "smat 256x24"}, {3, 384, 24, 8, "smat 384x24"},
    {4, 64, 20, 8, "apply 64x20"}, {4, 256, 24, 8, "apply 256x24"}, {4, 384, 24, 8, "apply 384x24"},
  };
  int ci = -1;
  for (auto& c : cases) {
    ++ci;
    if (only >= 0 && ci != only) continue;
    for (int rep = 0; rep < 2; ++rep) {
      cyc[1] = cyc[2] = cyc[3] = 0;
      k_bench<<<1, 256, 190 * 1024>>>(c.what, c.m, c.K, c.nw, cyc, out, only >= 0 ? 300 : 1);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("%s: %s\n", c.name, cudaGetErrorString(e)); return 1; }
    }
    printf("%-16s total %8lld cycles (%.1f us)  [%lld %lld %lld]\n", c.name, cyc[0], cyc[0] / 1965.0, cyc[1], cyc[2], cyc[3]);
  }
  return 0;
}
