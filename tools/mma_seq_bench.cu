// mma_seq_bench.cu — replays the attention backward's per-block tcgen05 MMA sequence in isolation
// (one CTA per SM, no other traffic) to separate MMA cost from pipeline/handoff cost.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include -I paper_2409_15373_b200/csrc \
//        tools/mma_seq_bench.cu -o tools/mma_seq_bench.bin -lcuda
// Per block: S^T (8 x 128x64x16, K-major A,B), dP^T (same), dQ^T (8 x 128x64x16, MN-major A,B),
// dV, dK (4 x 128x128x16 each, B MN-major). Ideal at 8192 FLOP/clk/SM: 1664 cycles (N=64 at 67%).
#include <cstdio>

#include "common.cuh"
#include "tc.cuh"

using namespace jg;

void jg::set_error(const std::string&) {}
jg_status jg::fail(jg_status c, const std::string&) { return c; }
jg_status jg::cuda_status(cudaError_t, const char*) { return JG_CUDA_ERROR; }
void jg::count_launch(int) {}
int jg::device_sm_count() { return 148; }

constexpr int kChunkKV = 128 * 128, kChunkQ = 64 * 128;
#define MMA(...) ((CONT & 8) ? tc::mma_bf16_ss_warp(__VA_ARGS__) : tc::mma_bf16_ss(__VA_ARGS__))

// MODE bit 0: S/dP part, bit 1: dQ part, bit 2: dV/dK part, bit 3: commit after each part
// CONT bit 0: warps 4-15 spin in mbarrier.try_wait on a barrier that completes only at the end;
//      bit 1: warps 4-11 stream tcgen05.ld (32 columns) from the score columns
template <int MODE, int CONT = 0>
__global__ void __launch_bounds__(512, 1) seq_bench(int blocks, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, bar2;
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
  if (warp >= 4 && (CONT & 1)) {
    tc::mbar_wait(&bar2, 1);  // bar2 never completes phase 1 unless commits (MODE & 8) run
  } else if (warp >= 4 && warp < 12 && (CONT & 2)) {
    const uint32_t la = tmem + ((uint32_t)((warp & 3) * 32) << 16) + ((warp >> 2) & 1) * 32;
    uint32_t acc = 0;
    while (!done) {
      uint32_t r[32];
      tc::tmem_ld32(la, r);
      tc::tmem_wait_ld();
      acc += r[0] + r[31];
    }
    if (acc == 12345) out[2] = acc;
  } else if (warp >= 4 && warp < 12 && (CONT & 16)) {  // softmax-like: TMEM ld, exp, TMEM st (cols 128..255)
    const uint32_t la = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 128 + ((warp >> 2) & 1) * 64;
    float acc = 0.f;
    while (!done) {
      uint32_t r[32], pk[16];
      tc::tmem_ld32(la, r);
      tc::tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 16; ++e)
        pk[e] = tc::pack_bf16(tc::ex2(__uint_as_float(r[2 * e]) * 0.1f), tc::ex2(__uint_as_float(r[2 * e + 1]) * 0.1f));
      tc::tmem_st16(la + 32, pk);
      tc::tmem_wait_st();
      acc += __uint_as_float(pk[3]);
    }
    if (acc == 12345.f) out[2] = 1;
  } else if (warp >= 4 && warp < 12 && (CONT & 4)) {  // softmax-like FFMA + MUFU stream
    float x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 0.001f + i;
    while (!done) {
#pragma unroll 4
      for (int it = 0; it < 16; ++it)
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = tc::ex2(fmaf(x[i], 0.999f, -0.5f)) * 0.5f;
    }
    float a = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) a += x[i];
    if (a == 12345.f) out[2] = 1;
  }
  if ((CONT & 8) ? warp == 0 : threadIdx.x == 0) {
    const uint32_t k_base = tc::smem_u32(smem), v_base = k_base + 2 * kChunkKV;
    const uint32_t q_base = v_base + 2 * kChunkKV, do_base = q_base + 2 * kChunkQ;
    const uint32_t p_base = do_base + 2 * kChunkQ, ds_base = p_base + kChunkKV;
    constexpr uint32_t kIdS = tc::idesc_bf16_f32(128, 64, false, false);
    constexpr uint32_t kIdKV = tc::idesc_bf16_f32(128, 128, false, true);
    constexpr uint32_t kIdQ = tc::idesc_bf16_f32(128, 64, true, true);
    const long long t0 = clock64();
    for (int j = 0; j < blocks; ++j) {
      const uint32_t col = (j & 1) * 128;
      if (MODE & 16) {  // forward-like: S = Q K^T (SS) into cols 0..127, O += P V (TS, A = cols 0..63) into 256..383
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t ka = (kk >> 2) * kChunkKV + (kk & 3) * 32;
          MMA(tmem, tc::sw128_desc(k_base + ka, 16, 1024), tc::sw128_desc(v_base + ka, 16, 1024),
              tc::idesc_bf16_f32(128, 128, false, false), kk > 0);
        }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (CONT & 8)
            tc::mma_bf16_ts_warp(tmem + 256, tmem + kk * 8, tc::sw128_desc(v_base + kk * 2048, kChunkKV, 1024),
                                 tc::idesc_bf16_f32(128, 128, false, true), 1);
          else
            MMA(tmem + 256, tc::sw128_desc(q_base + (kk >> 2) * kChunkKV + (kk & 3) * 32, 16, 1024),
                tc::sw128_desc(v_base + kk * 2048, kChunkKV, 1024), tc::idesc_bf16_f32(128, 128, false, true), 1);
        }
      }
      if (MODE & 1) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t ka = (kk >> 2) * kChunkKV + (kk & 3) * 32, kb = (kk >> 2) * kChunkQ + (kk & 3) * 32;
          MMA(tmem + col, tc::sw128_desc(k_base + ka, 16, 1024), tc::sw128_desc(q_base + kb, 16, 1024), kIdS,
                          kk > 0);
        }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t ka = (kk >> 2) * kChunkKV + (kk & 3) * 32, kb = (kk >> 2) * kChunkQ + (kk & 3) * 32;
          MMA(tmem + col + 64, tc::sw128_desc(v_base + ka, 16, 1024), tc::sw128_desc(do_base + kb, 16, 1024),
                          kIdS, kk > 0);
        }
        if (MODE & 8) tc::mma_commit(&bar2);
      }
      if (MODE & 2) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          MMA(tmem + ((j + 1) & 1) * 128, tc::sw128_desc(k_base + kk * 2048, kChunkKV, 1024),
                          tc::sw128_desc(ds_base + kk * 2048, 16, 1024), kIdQ, kk > 0);
        if (MODE & 8) tc::mma_commit(&bar2);
      }
      if (MODE & 4) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          MMA(tmem + 256, tc::sw128_desc(p_base + kk * 32, 16, 1024),
                          tc::sw128_desc(do_base + kk * 2048, kChunkQ, 1024), kIdKV, 1);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          MMA(tmem + 384, tc::sw128_desc(ds_base + kk * 32, 16, 1024),
                          tc::sw128_desc(q_base + kk * 2048, kChunkQ, 1024), kIdKV, 1);
        if (MODE & 8) tc::mma_commit(&bar2);
      }
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    const long long t2 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
    if (threadIdx.x == 0) {
      done = 1;
      if (CONT & 1) tc::mbar_arrive(&bar2);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem);
  }
}

template <int MODE, int CONT = 0>
void run(int blocks, const char* what, double ideal) {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  const int sm = 4 * kChunkKV + 4 * kChunkQ + 2 * kChunkKV + 2048;
  cudaFuncSetAttribute(seq_bench<MODE, CONT>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  seq_bench<MODE, CONT><<<148, 512, sm>>>(blocks, d);
  seq_bench<MODE, CONT><<<148, 512, sm>>>(blocks, d);
  cudaDeviceSynchronize();
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("mode=%2d cont=%d %-34s issue %7.1f  complete %7.1f cyc/block  (ideal %.0f)  %s\n", MODE, CONT, what, (double)h[0] / blocks,
         (double)h[1] / blocks, ideal, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<16, 8>(512, "fwd S(SS)+PV(TS)", 1024);
  run<16, 0>(512, "fwd S(SS)+PV(SS) 1-lane", 1024);
  run<16, 8 | 16>(512, "fwd TS + softmax-like TMEM/exp", 1024);
  run<16, 8 | 4>(512, "fwd TS + FFMA/MUFU", 1024);
  run<16, 8 | 2>(512, "fwd TS + tmem ld", 1024);
  run<1>(512, "S^T + dP^T (16 x N=64)", 768);
  run<2>(512, "dQ^T (8 x N=64, MN-major A,B)", 384);
  run<4>(512, "dV + dK (8 x N=128, MN-major B)", 512);
  run<7>(512, "full block", 1664);
  run<15>(512, "full block + 3 commits", 1664);
  run<7, 1>(512, "full block, 12 warps spin-wait", 1664);
  run<7, 2>(512, "full block, 8 warps tmem ld", 1664);
  run<7, 4>(512, "full block, 8 warps FFMA+MUFU", 1664);
  run<7, 8>(512, "warp-wide issue", 1664);
  run<7, 12>(512, "warp-wide issue, FFMA+MUFU", 1664);
  run<7, 10>(512, "warp-wide issue, tmem ld", 1664);
  return 0;
}
