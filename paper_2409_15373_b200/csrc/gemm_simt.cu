// gemm_simt.cu — grouped strided GEMM over jagged samples (fp32 FFMA, fp32 accumulation).
//
// One persistent kernel covers the whole bmm family of linalg.cpp (jagged_dense_bmm :34,
// jagged_jagged_bmm :70, jagged_jagged_bmm_jagged_out :122, array_jagged_bmm_jagged_out :161) and
// their VJPs (:283-472): per sample i it computes C_i = A_i B_i with sizes/offsets/strides given by
// the affine GemmDesc (internal.h). Tiles of 64x64 are enumerated per sample; a one-CTA prefix kernel
// turns per-sample tile counts into a device prefix array, and CTAs (grid = k x 148 SMs) walk the
// global tile index space, locating their sample by binary search — no host round trip.
// This is the fp32-mode path (1e-5 relative vs the binary64 oracle); bf16 inputs are accepted.
#include "common.cuh"
#include "internal.h"

namespace jg {

constexpr int kBM = 64, kBN = 64, kBK = 16, kGemmThreads = 256;

__global__ void __launch_bounds__(1024) gemm_prefix_kernel(GemmDesc g, const int64_t* __restrict__ off,
                                                           const int64_t* __restrict__ sq, int64_t batch, int bm,
                                                           int bn, int64_t* __restrict__ prefix) {
  const int64_t chunk = (batch + blockDim.x - 1) / blockDim.x;
  const int64_t b = (int64_t)threadIdx.x * chunk, e = min(batch, b + chunk);
  auto tiles = [&](int64_t i) -> int64_t {
    const int64_t Bi = off[i + 1] - off[i];
    const int64_t s = sq ? sq[i] : 0;
    const int64_t M = g.M.at(Bi, off[i], s, i), N = g.N.at(Bi, off[i], s, i);
    return ((M + bm - 1) / bm) * ((N + bn - 1) / bn);
  };
  int64_t local = 0;
  for (int64_t i = b; i < e; ++i) local += tiles(i);
  int64_t total;
  int64_t run = block_exclusive_scan(local, &total);
  for (int64_t i = b; i < e; ++i) {
    prefix[i] = run;
    run += tiles(i);
  }
  if (threadIdx.x == 0) prefix[batch] = total;
}

template <typename TI, typename TO>
__global__ void __launch_bounds__(kGemmThreads) grouped_gemm_kernel(GemmDesc g, const int64_t* __restrict__ off,
                                                                    const int64_t* __restrict__ sq, int64_t batch,
                                                                    const int64_t* __restrict__ prefix,
                                                                    const TI* __restrict__ A,
                                                                    const TI* __restrict__ Bm,
                                                                    TO* __restrict__ C) {
  __shared__ float As[kBK][kBM + 4];
  __shared__ float Bs[kBK][kBN + 4];
  const int64_t total = prefix[batch];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
    const int64_t i = upper_index(prefix, batch, t);
    const int64_t Bi = off[i + 1] - off[i], o = off[i], s = sq ? sq[i] : 0;
    const int64_t M = g.M.at(Bi, o, s, i), N = g.N.at(Bi, o, s, i), K = g.K.at(Bi, o, s, i);
    const int64_t tn_count = (N + kBN - 1) / kBN;
    const int64_t local = t - prefix[i];
    const int64_t m0 = (local / tn_count) * kBM, n0 = (local % tn_count) * kBN;
    const int64_t a0 = g.a0.at(Bi, o, s, i), sam = g.sam.at(Bi, o, s, i), sak = g.sak.at(Bi, o, s, i);
    const int64_t b0 = g.b0.at(Bi, o, s, i), sbk = g.sbk.at(Bi, o, s, i), sbn = g.sbn.at(Bi, o, s, i);
    const int64_t c0 = g.c0.at(Bi, o, s, i), scm = g.scm.at(Bi, o, s, i), scn = g.scn.at(Bi, o, s, i);
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
    for (int64_t k0 = 0; k0 < K; k0 += kBK) {
      // cooperative loads; the fastest-varying thread index follows the unit-stride axis
#pragma unroll
      for (int rep = 0; rep < (kBM * kBK) / kGemmThreads; ++rep) {
        const int e = rep * kGemmThreads + threadIdx.x;
        int mm, kk;
        if (sak == 1) { kk = e % kBK; mm = e / kBK; } else { mm = e % kBM; kk = e / kBM; }
        const int64_t gm = m0 + mm, gk = k0 + kk;
        As[kk][mm] = (gm < M && gk < K) ? ld(A + a0 + gm * sam + gk * sak) : 0.f;
      }
#pragma unroll
      for (int rep = 0; rep < (kBN * kBK) / kGemmThreads; ++rep) {
        const int e = rep * kGemmThreads + threadIdx.x;
        int nn, kk;
        if (sbn == 1) { nn = e % kBN; kk = e / kBN; } else { kk = e % kBK; nn = e / kBK; }
        const int64_t gn = n0 + nn, gk = k0 + kk;
        Bs[kk][nn] = (gn < N && gk < K) ? ld(Bm + b0 + gk * sbk + gn * sbn) : 0.f;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < kBK; ++kk) {
        float av[4], bv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) av[a] = As[kk][ty + 16 * a];
#pragma unroll
        for (int b = 0; b < 4; ++b) bv[b] = Bs[kk][tx + 16 * b];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(av[a], bv[b], acc[a][b]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int64_t gm = m0 + ty + 16 * a;
      if (gm >= M) continue;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int64_t gn = n0 + tx + 16 * b;
        if (gn < N) st(C + c0 + gm * scm + gn * scn, acc[a][b]);
      }
    }
  }
}

jg_status launch_gemm_prefix(const GemmDesc& g, const int64_t* off, const int64_t* sq, int64_t batch, int bm, int bn,
                             int64_t* tile_prefix, cudaStream_t st) {
  gemm_prefix_kernel<<<1, 1024, 0, st>>>(g, off, sq, batch, bm, bn, tile_prefix);
  JG_LAUNCHED("gemm_prefix_kernel");
  return JG_OK;
}

jg_status launch_grouped_gemm(const GemmDesc& g, const int64_t* off, const int64_t* sq, int64_t batch,
                              const void* A, const void* B, void* C, jg_dtype in_dt, jg_dtype out_dt,
                              int64_t* tile_prefix, cudaStream_t st) {
  if (batch == 0) return JG_OK;
  if (jg_status rc = launch_gemm_prefix(g, off, sq, batch, kBM, kBN, tile_prefix, st)) return rc;
  const int grid = 8 * device_sm_count();
  using BF = __nv_bfloat16;
  if (in_dt == JG_F32 && out_dt == JG_F32)
    grouped_gemm_kernel<float, float><<<grid, kGemmThreads, 0, st>>>(g, off, sq, batch, tile_prefix, (const float*)A, (const float*)B, (float*)C);
  else if (in_dt == JG_BF16 && out_dt == JG_BF16)
    grouped_gemm_kernel<BF, BF><<<grid, kGemmThreads, 0, st>>>(g, off, sq, batch, tile_prefix, (const BF*)A, (const BF*)B, (BF*)C);
  else if (in_dt == JG_BF16 && out_dt == JG_F32)
    grouped_gemm_kernel<BF, float><<<grid, kGemmThreads, 0, st>>>(g, off, sq, batch, tile_prefix, (const BF*)A, (const BF*)B, (float*)C);
  else
    return fail(JG_UNSUPPORTED, "bmm: unsupported (in_dtype, out_dtype) pair (no CPU fallback)");
  JG_LAUNCHED("grouped_gemm_kernel");
  return JG_OK;
}

}  // namespace jg
