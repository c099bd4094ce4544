// dependent-chain latencies of fp64 special functions and shared-memory patterns
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(double* out, long long* cyc, double seed) {
  __shared__ double sm[2048];
  const int t = threadIdx.x;
  for (int i = t; i < 2048; i += blockDim.x) sm[i] = 1.0 + i * 1e-3;
  __syncthreads();
  double z = seed;
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) z = rsqrt(z + 1.5);
  long long t1 = clock64();
  for (int i = 0; i < 256; ++i) z = __drcp_rn(z + 1.5);
  long long t2 = clock64();
  for (int i = 0; i < 256; ++i) z = 1.0 / (z + 1.5);
  long long t3 = clock64();
  for (int i = 0; i < 256; ++i) z = sqrt(z + 1.5);
  long long t4 = clock64();
  // store then load same address by another lane with syncwarp (exchange pattern)
  for (int i = 0; i < 256; ++i) { sm[t] = z; __syncwarp(); z += sm[(t + 1) & 31]; __syncwarp(); }
  long long t5 = clock64();
  // batch of 8 independent LDS then 8 dependent FMAs
  double a = z;
  for (int i = 0; i < 256; ++i) {
    double v[8];
    const int base = ((int)a) & 1023;
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = sm[base + u * 33 + (t & 31)];
#pragma unroll
    for (int u = 0; u < 8; ++u) a = fma(a, 1e-9, v[u]);
  }
  long long t6 = clock64();
  for (int i = 0; i < 256; ++i) { asm volatile("bar.sync 1, 128;"); }
  long long t7 = clock64();
  for (int i = 0; i < 256; ++i) { z = fmin(fabs(z), 3.0); z = copysign(z + 1.0, -z); }
  long long t8 = clock64();
  if (t == 0) {
    cyc[0] = (t1 - t0) / 256; cyc[1] = (t2 - t1) / 256; cyc[2] = (t3 - t2) / 256; cyc[3] = (t4 - t3) / 256;
    cyc[4] = (t5 - t4) / 256; cyc[5] = (t6 - t5) / 256; cyc[6] = (t7 - t6) / 256; cyc[7] = (t8 - t7) / 256;
  }
  out[t] = z + a;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 8 * 8);
  probe<<<1, 128>>>(out, cyc, 2.0);
  cudaDeviceSynchronize();
  printf("rsqrt %lld | drcp %lld | div %lld | sqrt %lld | STS+syncwarp+LDS+syncwarp %lld | 8xLDS+8 dep FMA %lld | bar.sync(128) %lld | abs/copysign pair %lld\n",
         cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5], cyc[6], cyc[7]);
  return 0;
}
