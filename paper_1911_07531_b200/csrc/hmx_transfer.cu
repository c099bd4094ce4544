// hmx_transfer.cu — packed leaf transfer between the device pools and a
// compact wire format (include/hmx.h: hmx_pack_leaves / hmx_unpack_leaves).
//
// A device H-matrix pool reserves `cap` columns per low-rank factor (the
// rank bound the factorization may reach); the live data of a leaf is only
// its dense block or its U (m x k) and V (n x k) at the current rank k.  The
// packed format concatenates, over instances b and leaves l (block-tree
// pre-order, hmatrix.py:214-219 `leaves`), the live columns in column-major
// order: dense m*n, or U then V.  This is the device half of
// HStore.upload_leaves / download_leaves (the reference keeps leaves as
// numpy arrays; hmatrix.py:174-177) and the H-matrix dump format of
// SURVEY.md §8f row 4.
//
// Two kernels per direction: a one-CTA exclusive scan of the item sizes
// (item = (instance, leaf); sizes depend on the ranks, which live on the
// device), then a grid-stride copy, one CTA per item, 2-wide vector moves
// where both sides are 16-byte aligned.  HBM bound: 2 * bytes moved.

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hmx.h"

namespace {

constexpr int kScanThreads = 1024;

__device__ __forceinline__ int64_t item_size(const int64_t* d, const int32_t* ranks, int64_t rank_base) {
  // d: uid, off0, off_v, m, n (off_v < 0: dense leaf)
  const int64_t m = d[3], n = d[4];
  if (d[2] < 0) return m * n;
  const int k = ranks[rank_base + d[0]];
  return (m + n) * (int64_t)(k > 0 ? k : 0);
}

// offsets[i] = sum of sizes of items < i; offsets[nitems] = total.
__global__ void __launch_bounds__(kScanThreads) k_scan_sizes(int32_t nleaf, int32_t nrep,
                                                             const int64_t* desc, int32_t rank_stride,
                                                             const int32_t* ranks, int64_t* offsets) {
  __shared__ int64_t part[kScanThreads];
  const int64_t nitems = (int64_t)nleaf * nrep;
  const int64_t per = (nitems + kScanThreads - 1) / kScanThreads;
  const int64_t b0 = threadIdx.x * per, b1 = min(nitems, b0 + per);
  int64_t s = 0;
  for (int64_t i = b0; i < b1; ++i) {
    const int64_t b = i / nleaf, l = i - b * nleaf;
    s += item_size(desc + 5 * l, ranks, b * rank_stride);
  }
  part[threadIdx.x] = s;
  __syncthreads();
  // Hillis-Steele inclusive scan over the 1024 partial sums
  for (int o = 1; o < kScanThreads; o <<= 1) {
    const int64_t v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int64_t run = threadIdx.x ? part[threadIdx.x - 1] : 0;
  for (int64_t i = b0; i < b1; ++i) {
    offsets[i] = run;
    const int64_t b = i / nleaf, l = i - b * nleaf;
    run += item_size(desc + 5 * l, ranks, b * rank_stride);
  }
  if (threadIdx.x == kScanThreads - 1) offsets[nitems] = part[kScanThreads - 1];
}

__device__ __forceinline__ void seg_copy(const double* __restrict__ src, double* __restrict__ dst,
                                         int64_t len) {
  if (len <= 0) return;
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
    const int64_t n2 = len >> 1;
    const double2* s2 = reinterpret_cast<const double2*>(src);
    double2* d2 = reinterpret_cast<double2*>(dst);
    for (int64_t i = threadIdx.x; i < n2; i += blockDim.x) d2[i] = s2[i];
    if ((len & 1) && threadIdx.x == 0) dst[len - 1] = src[len - 1];
  } else {
    for (int64_t i = threadIdx.x; i < len; i += blockDim.x) dst[i] = src[i];
  }
}

// pack: pool -> packed (dir = 0); unpack: packed -> pool (dir = 1)
// pack items that would end beyond `capacity` doubles are skipped (the
// caller sees offsets[nitems] > capacity, grows its buffer and packs again)
__global__ void __launch_bounds__(256) k_move(int32_t nleaf, int32_t nrep, const int64_t* desc,
                                              int64_t pool_stride, int32_t rank_stride,
                                              const int32_t* ranks, const int64_t* offsets,
                                              double* pool, double* packed, int dir,
                                              int64_t capacity) {
  const int64_t nitems = (int64_t)nleaf * nrep;
  for (int64_t i = blockIdx.x; i < nitems; i += gridDim.x) {
    const int64_t b = i / nleaf, l = i - b * nleaf;
    const int64_t* d = desc + 5 * l;
    const int64_t m = d[3], n = d[4];
    double* base = pool + b * pool_stride;
    if (dir == 0 && offsets[i + 1] > capacity) continue;
    double* pk = packed + offsets[i];
    if (d[2] < 0) {
      if (dir == 0) seg_copy(base + d[1], pk, m * n);
      else seg_copy(pk, base + d[1], m * n);
    } else {
      const int k = ranks[b * rank_stride + d[0]];
      if (k <= 0) continue;
      if (dir == 0) {
        seg_copy(base + d[1], pk, m * k);
        seg_copy(base + d[2], pk + m * k, n * k);
      } else {
        seg_copy(pk, base + d[1], m * k);
        seg_copy(pk + m * k, base + d[2], n * k);
      }
    }
  }
}

int grid_for(int64_t nitems) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t g = (int64_t)sms * 8;
  return (int)(nitems < g ? (nitems > 0 ? nitems : 1) : g);
}

hmx_status status_of(cudaError_t e) { return e == cudaSuccess ? HMX_OK : HMX_ERR_CUDA; }

}  // namespace

extern "C" {

hmx_status hmx_pack_leaves(int32_t nleaf, int32_t nrep, const int64_t* desc, int64_t pool_stride,
                           int32_t rank_stride, const double* pool, const int32_t* ranks,
                           double* packed, int64_t capacity, int64_t* offsets, void* stream) {
  if (nleaf < 0 || nrep < 0 || !desc || !ranks || !offsets) return HMX_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  k_scan_sizes<<<1, kScanThreads, 0, s>>>(nleaf, nrep, desc, rank_stride, ranks, offsets);
  if (packed && pool && (int64_t)nleaf * nrep > 0)
    k_move<<<grid_for((int64_t)nleaf * nrep), 256, 0, s>>>(nleaf, nrep, desc, pool_stride, rank_stride,
                                                          ranks, offsets, const_cast<double*>(pool),
                                                          packed, 0, capacity);
  return status_of(cudaGetLastError());
}

hmx_status hmx_unpack_leaves(int32_t nleaf, int32_t nrep, const int64_t* desc, int64_t pool_stride,
                             int32_t rank_stride, const double* packed, const int32_t* ranks,
                             double* pool, int64_t* offsets, void* stream) {
  if (nleaf < 0 || nrep < 0 || !desc || !ranks || !offsets || !pool || !packed) return HMX_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  k_scan_sizes<<<1, kScanThreads, 0, s>>>(nleaf, nrep, desc, rank_stride, ranks, offsets);
  if ((int64_t)nleaf * nrep > 0)
    k_move<<<grid_for((int64_t)nleaf * nrep), 256, 0, s>>>(nleaf, nrep, desc, pool_stride, rank_stride,
                                                          ranks, offsets, pool,
                                                          const_cast<double*>(packed), 1, INT64_MAX);
  return status_of(cudaGetLastError());
}

}  // extern "C"
