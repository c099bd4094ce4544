// Latency probes (cycles) on sm_100a: dependent DFMA, DADD, 64-bit SHFL
// reduction step, shared-memory load, L2 load, __syncthreads.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(double* out, long long* cyc, const double* g, int n) {
  __shared__ double sm[1024];
  const int t = threadIdx.x;
  for (int i = t; i < 1024; i += blockDim.x) sm[i] = i * 1e-3;
  __syncthreads();
  double a = t * 1e-7, b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < 1024; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  double s = a;
  for (int i = 0; i < 1024; ++i) s += __shfl_xor_sync(0xffffffffu, s, 1);
  long long t2 = clock64();
  int idx = t & 31;
  double x = 0;
  for (int i = 0; i < 1024; ++i) { x += sm[idx]; idx = ((int)x + idx + 1) & 1023; }
  long long t3 = clock64();
  for (int i = 0; i < 256; ++i) __syncthreads();
  long long t4 = clock64();
  double y = 0; int gi = t;
  for (int i = 0; i < 256; ++i) { y += g[gi]; gi = ((int)(y * 0) + gi + 4099) & (n - 1); }
  long long t5 = clock64();
  double z = 1.0;
  for (int i = 0; i < 256; ++i) z = sqrt(z + 1.0);
  long long t6 = clock64();
  double w = 3.0;
  for (int i = 0; i < 256; ++i) w = 1.0 / (w + 1.0);
  long long t7 = clock64();
  if (t == 0) {
    cyc[0] = (t1 - t0) / 1024; cyc[1] = (t2 - t1) / 1024; cyc[2] = (t3 - t2) / 1024;
    cyc[3] = (t4 - t3) / 256; cyc[4] = (t5 - t4) / 256; cyc[5] = (t6 - t5) / 256; cyc[6] = (t7 - t6) / 256;
  }
  out[t] = a + s + x + y + z + w;
}
int main() {
  double *out, *g; long long* cyc;
  int n = 1 << 24;
  cudaMalloc(&out, 1024 * 8); cudaMalloc(&g, n * 8); cudaMemset(g, 0, n * 8);
  cudaMallocManaged(&cyc, 8 * 8);
  for (int nt : {32, 256}) {
    probe<<<1, nt>>>(out, cyc, g, n);
    cudaDeviceSynchronize();
    printf("threads=%d: DFMA dep %lld | SHFL64+DADD step %lld | LDS dep %lld | syncthreads %lld | "
           "global dep (L2/HBM) %lld | sqrt %lld | div %lld cycles\n", nt, cyc[0], cyc[1], cyc[2],
           cyc[3], cyc[4], cyc[5], cyc[6]);
  }
  return 0;
}
