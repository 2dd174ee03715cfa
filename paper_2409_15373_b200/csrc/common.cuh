// common.cuh — shared device helpers for the jagged kernels (sm_100a only).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <string>

#include "jagged_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libjagged_b200 is built for sm_100a only"
#endif

namespace jg {

constexpr int kNumSMsB200 = 148;

// ---------------------------------------------------------------- host-side error plumbing
void set_error(const std::string& msg);
jg_status fail(jg_status code, const std::string& msg);
jg_status cuda_status(cudaError_t e, const char* where);
void count_launch(int n = 1);
int device_sm_count();

#define JG_CUDA(expr)                                                  \
  do {                                                                 \
    cudaError_t e_ = (expr);                                           \
    if (e_ != cudaSuccess) return ::jg::cuda_status(e_, #expr);        \
  } while (0)

#define JG_LAUNCHED(where)                                             \
  do {                                                                 \
    cudaError_t e_ = cudaGetLastError();                               \
    if (e_ != cudaSuccess) return ::jg::cuda_status(e_, where);        \
    ::jg::count_launch();                                              \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------- element types
template <typename T> struct Elem;
template <> struct Elem<float> {
  __device__ __forceinline__ static float load(const float* p) { return *p; }
  __device__ __forceinline__ static void store(float* p, float v) { *p = v; }
};
template <> struct Elem<__nv_bfloat16> {
  __device__ __forceinline__ static float load(const __nv_bfloat16* p) { return __bfloat162float(*p); }
  __device__ __forceinline__ static void store(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
};

template <typename T> __device__ __forceinline__ float ld(const T* p) { return Elem<T>::load(p); }
template <typename T> __device__ __forceinline__ void st(T* p, float v) { Elem<T>::store(p, v); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// first sample i with offsets[i+1] > row (binary search over the device offsets array)
__device__ __forceinline__ int64_t sample_of_row(const int64_t* __restrict__ off, int64_t batch,
                                                 int64_t row) {
  int64_t lo = 0, hi = batch - 1;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (off[mid + 1] <= row) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// largest i with prefix[i] <= x, prefix non-decreasing with prefix[0] = 0 (n+1 entries)
__device__ __forceinline__ int64_t upper_index(const int64_t* __restrict__ prefix, int64_t n,
                                               int64_t x) {
  int64_t lo = 0, hi = n - 1;
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= x) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Block-wide exclusive scan of one int64 per thread (blockDim.x <= 1024); *total = block sum.
__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t* total) {
  __shared__ int64_t warp_tot[32];
  __shared__ int64_t block_tot;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    int64_t t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
    int64_t s = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    warp_tot[lane] = s - t;  // exclusive warp prefix
    if (lane == 31) block_tot = s;  // lanes beyond blockDim/32 carry zeros so s is the total
  }
  __syncthreads();
  const int64_t excl = warp_tot[w] + x - v;
  *total = block_tot;
  __syncthreads();
  return excl;
}

}  // namespace jg
