// mufu_bench.cu — measures ex2.approx (MUFU) and FFMA throughput per SM on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mufu_bench.cu -o tools/mufu_bench.bin
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int MODE>
__global__ void bench(int iters, float* out, long long* cyc) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = ex2(a[i]) - 1.0f;           // MUFU + FADD
      else a[i] = fmaf(a[i], 0.999f, 1e-6f);            // FFMA
    }
  }
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 8);
  for (int mode = 0; mode < 2; ++mode)
    for (int threads : {128, 256, 512, 1024}) {
      const int iters = 4096;
      if (mode == 0) bench<0><<<148, threads>>>(iters, out, cyc);
      else bench<1><<<148, threads>>>(iters, out, cyc);
      long long h;
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      const double ops = (double)iters * 8 * threads;  // per SM
      printf("%s threads=%4d: %.2f ops/clk/SM\n", mode == 0 ? "ex2+fadd" : "ffma    ", threads, ops / (double)h);
    }
  return 0;
}
