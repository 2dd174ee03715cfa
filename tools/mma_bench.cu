// mma_bench.cu — calibrates single-CTA tcgen05.mma (kind::f16, bf16 -> f32) throughput on B200.
// One CTA per SM; one thread issues `iters` MMAs of shape M x N x 16 from shared memory (SS) into
// TMEM, commits, waits; reports cycles per MMA and the implied per-SM FLOP/clk.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include -I paper_2409_15373_b200/csrc tools/mma_bench.cu -o /tmp/mma_bench
#include <cstdio>

#include "common.cuh"
#include "tc.cuh"

using namespace jg;

void jg::set_error(const std::string&) {}
jg_status jg::fail(jg_status c, const std::string&) { return c; }
jg_status jg::cuda_status(cudaError_t, const char*) { return JG_CUDA_ERROR; }
void jg::count_launch(int) {}
int jg::device_sm_count() { return 148; }

// CONT: 0 none, 1 warps 4-7 stream tcgen05.ld from TMEM cols 256+, 2 warps 4-7 stream st.shared into a
// separate smem region, 3 both
template <int N, bool TWO_ACC, int CONT>
__global__ void __launch_bounds__(256, 1) mma_bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint64_t bar2;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_init(&bar2, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  if (warp >= 4 && (CONT & 3) != 0) {
    const uint32_t la = tmem + ((uint32_t)((warp - 4) * 32) << 16) + 256;
    const uint32_t sa = tc::smem_u32(smem + 128 * 128 * 2 + 256 * 128 * 2) + (threadIdx.x - 128) * 16;
    uint32_t acc = 0;
    while (!done) {
      if (CONT & 1) {
        uint32_t r[32];
        tc::tmem_ld32(la, r);
        tc::tmem_wait_ld();
        acc += r[0] + r[31];
      }
      if (CONT & 2) {
#pragma unroll
        for (int u = 0; u < 8; ++u) tc::st_shared_v4(sa + u * 2048, acc, acc + 1, acc + 2, acc + u);
      }
    }
    if (acc == 12345) out[2] = acc;
  }
  if (threadIdx.x == 0) {
    const uint32_t a = tc::smem_u32(smem), b = a + 128 * 128 * 2;
    constexpr uint32_t id = tc::idesc_bf16_f32(128, N, (CONT & 8) != 0, (CONT & 4) != 0);
    constexpr uint32_t lbo = (CONT & 12) ? 16384 : 16;
    // warm up
    for (int i = 0; i < 8; ++i)
      tc::mma_bf16_ss(tmem, tc::sw128_desc(a + (i & 3) * 32, 16, 1024), tc::sw128_desc(b + (i & 3) * 32, 16, 1024), id, i);
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = TWO_ACC ? tmem + (i & 1) * 256 : tmem;
      tc::mma_bf16_ss(d, tc::sw128_desc(a + (i & 3) * 32, lbo, 1024), tc::sw128_desc(b + (i & 3) * 32, lbo, 1024), id, 1);
      if ((CONT & 16) && (i & 7) == 7) {  // commit every 8 MMAs (to a barrier nobody waits on)
        tc::mma_commit(&bar2);
        tc::tc_fence_after();
      }
    }
    const long long t1 = clock64();
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 1);
    const long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;  // issue time
      out[1] = t2 - t0;  // completion time
    }
    done = 1;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem);
  }
}

template <int N, bool TWO, int CONT>
void run(int iters) {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  const int sm = 128 * 128 * 2 + 256 * 128 * 2 + 16384 + 1024;
  cudaFuncSetAttribute(mma_bench<N, TWO, CONT>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mma_bench<N, TWO, CONT><<<148, 256, sm>>>(iters, d);
  cudaEventRecord(e0);
  mma_bench<N, TWO, CONT><<<148, 256, sm>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double flop = 2.0 * 128 * N * 16 * iters * 148;
  printf("cont=%d M=128 N=%3d two_acc=%d: issue %.1f cyc/mma, complete %.1f cyc/mma -> %.0f FLOP/clk/SM; %.1f TFLOP/s (%s)\n", CONT, N,
         (int)TWO, (double)h[0] / iters, (double)h[1] / iters, 2.0 * 128 * N * 16 / ((double)h[1] / iters),
         flop / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<64, false, 0>(4096);
  run<128, false, 0>(4096);
  run<128, false, 1>(4096);
  run<128, false, 2>(4096);
  run<128, false, 3>(4096);
  run<128, false, 16>(4096);
  run<128, false, 17>(4096);
  return 0;
}
