// tma_probe.cu — loads one [64 x 2] fp32 box through make_map_lsd and prints it (diagnostic).
#include <cstdio>
#include "common.cuh"
#include "tc.cuh"
#include "tma_host.h"
using namespace jg;
void jg::set_error(const std::string&) {}
jg_status jg::fail(jg_status c, const std::string& m) { printf("fail: %s\n", m.c_str()); return c; }
jg_status jg::cuda_status(cudaError_t, const char*) { return JG_CUDA_ERROR; }
void jg::count_launch(int) {}
int jg::device_sm_count() { return 148; }

struct P { const int64_t* a; const int2* b; const int64_t* c; int64_t d; int e; float* f; void* g; void* h2; float x, y; int dbg; unsigned long long* prof; };
__global__ void probe(const __grid_constant__ CUtensorMap m0, const __grid_constant__ CUtensorMap m1,
                      const __grid_constant__ CUtensorMap m2, const __grid_constant__ CUtensorMap m3,
                      const __grid_constant__ CUtensorMap m4, const __grid_constant__ CUtensorMap m, P pp, int row, int h, float* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* buf = reinterpret_cast<float*>(smem + 229376 + 1024);
  uint64_t& bar = *reinterpret_cast<uint64_t*>(smem + 230912);
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
    tc::mbar_expect_tx(&bar, 512);
    tc::tma_load_2d(buf, &m, &bar, row, h);
    tc::mbar_wait(&bar, 0);
  }
  __syncthreads();
  out[threadIdx.x] = buf[threadIdx.x];
}

int main() {
  const int R = 636, H = 2;
  float* d;
  cudaMallocAsync(&d, 2 * H * R * 4 + 4096, 0);
  float* hbuf = new float[2 * H * R];
  for (int i = 0; i < 2 * H * R; ++i) hbuf[i] = i;
  cudaMemcpy(d, hbuf, 2 * H * R * 4, cudaMemcpyHostToDevice);
  float* o;
  cudaMalloc(&o, 512);
  CUtensorMap m;
  printf("encode rc=%d\n", (int)make_map_lsd(&m, d, R, H, 64));
  P pp{};
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 232112);
  int rows[] = {0, 5, 64, 200, 572, 573, 600, 620, 630, 635};
  for (int hh : {0, 2})
    for (int r0 : rows) {
      probe<<<1, 128, 232112>>>(m, m, m, m, m, m, pp, r0, hh, o);
      cudaError_t e = cudaDeviceSynchronize();
      printf("row %d h2 %d: %s\n", r0, hh, cudaGetErrorString(e));
      if (e != cudaSuccess) return 1;
    }
  float r[128];
  cudaMemcpy(r, o, 512, cudaMemcpyDeviceToHost);
  const unsigned long long* mw = reinterpret_cast<const unsigned long long*>(&m);
  printf("map %llx %llx\n", mw[0], mw[1]);
  printf("%g %g %g | %g %g\n", r[0], r[1], r[63], r[64], r[127]);
  return 0;
}
