// tmem_bench.cu — TMEM load/store throughput per SM (tcgen05.ld/st 32x32b.x32), diagnostic.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2409_15373_b200/csrc \
//        tools/tmem_bench.cu -o tools/tmem_bench.bin -lcuda
#include <cstdio>

#include "common.cuh"
#include "tc.cuh"

using namespace jg;
void jg::set_error(const std::string&) {}
jg_status jg::fail(jg_status c, const std::string&) { return c; }
jg_status jg::cuda_status(cudaError_t, const char*) { return JG_CUDA_ERROR; }
void jg::count_launch(int) {}
int jg::device_sm_count() { return 148; }

// MODE 0: ld x32 + wait each; 1: two ld x32 then one wait; 2: st x32 + wait each
template <int MODE>
__global__ void __launch_bounds__(512, 1) tmem_bench(int iters, unsigned long long* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::tmem_alloc<512>(&slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t la = tmem + ((uint32_t)((warp & 3) * 32) << 16) + ((warp >> 2) * 64) % 512;
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t r[32], q[32];
    if (MODE == 0) {
      tc::tmem_ld32(la, r);
      tc::tmem_wait_ld();
      acc += r[0] ^ r[31];
    } else if (MODE == 1) {
      tc::tmem_ld32(la, r);
      tc::tmem_ld32(la + 32, q);
      tc::tmem_wait_ld();
      acc += r[0] ^ q[31];
    } else {
#pragma unroll
      for (int u = 0; u < 32; ++u) r[u] = i + u;
      tc::tmem_st32(la, r);
      tc::tmem_wait_st();
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (acc == 12345) out[1] = acc;
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem);
  }
}

template <int MODE>
void run(int warps, const char* what) {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  const int iters = 2048;
  tmem_bench<MODE><<<148, warps * 32>>>(iters, d);
  tmem_bench<MODE><<<148, warps * 32>>>(iters, d);
  cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double bytes = (double)warps * iters * (MODE == 1 ? 2 : 1) * 32 * 32 * 4;
  printf("%-28s warps=%2d: %.1f cyc/iter, %.1f B/cyc/SM  (%s)\n", what, warps, (double)h / iters, bytes / h,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int w : {4, 8, 12, 16}) run<0>(w, "ld x32 + wait");
  for (int w : {4, 8, 16}) run<1>(w, "2 x ld x32 + wait");
  for (int w : {4, 8, 16}) run<2>(w, "st x32 + wait");
  return 0;
}
