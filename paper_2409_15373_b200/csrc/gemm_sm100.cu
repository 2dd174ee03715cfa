// gemm_sm100.cu — the jagged bmm family on tcgen05 tensor cores (bf16 inputs, fp32 accumulation).
//
// One persistent warp-specialized kernel, templated on the contraction, covers the four forward
// operators of linalg.cpp and, with two transposed forms, all eight contractions of their VJPs
// (linalg.cpp:283-472; per sample i, Bi = offsets[i+1] - offsets[i]):
//   JJJ  jagged_jagged_bmm_jagged_out (:122)  S_i = Q_i K_i^T      M=Bi N=Bi K=D   A,B K-major (TMA)
//   AJ   array_jagged_bmm_jagged_out  (:161)  O_i = A_i V_i        M=Bi N=D  K=Bi  A jagged^2 (manual), B MN-major
//   JJ   jagged_jagged_bmm            (:70)   Z_i = X_i^T Y_i      M=D  N=T  K=Bi  A,B MN-major (TMA)
//   JD   jagged_dense_bmm             (:34)   O_i = X_i W_i        M=Bi N=T  K=D   A K-major, B MN-major
//   JDT  O_i = X_i W_i^T, W [B, N, K]           M=Bi N=D  K=T   A,B K-major (TMA)
//        (jagged_dense_bmm dX = dO W^T, :296; jagged_jagged_bmm dX = Y dZ^T, :334)
//   AJT  O_i = A_i^T V_i (jagged^2 A)          M=Bi N=D  K=Bi  A jagged^2 transposed (manual, MN-major), B MN-major
//        (jagged_jagged_bmm_jagged_out dK = dS^T Q, :415; array_jagged_bmm_jagged_out dV = A^T dO, :458)
// The remaining VJP contractions are forward forms: jdbmm dW = X^T dO and jjbmm dY = X dZ (JJ / JD),
// jjbmm_jout dQ = dS K (AJ), ajbmm dA = dO V^T (JJJ).
// 128x128 output tiles, 64-deep K stages through a 4-stage ring (a stage skips reloading an operand block
// it already holds), accumulators double-buffered in TMEM so the epilogue of tile t overlaps the MMAs of
// tile t+1; each CTA walks a contiguous tile range with a sample cursor. TMA coordinates are global row indices
// (offsets[i] + local row), so no padding is materialised; rows of the next sample that a tail tile
// picks up are masked: never stored (M/N tails) or zeroed in smem before the MMA (K tails of JJ, where
// the reduction runs over the jagged axis). Jagged^2 A operands (row stride Bi, arbitrary 2-byte
// alignment, unusable by TMA) are first repacked by aj_repack_kernel into 64 x 64 SWIZZLE_128B sub-block
// images (zeros past Bi) that the AJ and AJT stages are assembled from with two 8 KB bulk copies
// (cp.async.bulk) — one pass of HBM traffic instead of a latency-bound per-stage gather, and one repack for a
// VJP that needs both A and A^T. AJ / AJT with D >= 256 compute 128 x 256 tiles (two column halves share each
// A stage). Warps: 0 TMA producer, 1 MMA issuer, 4-11 epilogue (TMEM -> registers -> global; lane
// quarter x column half; JJJ stages through smem and writes aligned 16-byte chunks; JD can fuse the jagged_mlp
// bias + ReLU), except JJ: 4-7 epilogue and 8-11 loader (K-tail zeroing).
#include "common.cuh"
#include "internal.h"
#include "tc.cuh"
#include "tma_host.h"

namespace jg {
namespace gm {

enum Op { JJJ = 0, AJ = 1, JJ = 2, JD = 3, JDT = 4, AJT = 5 };

#ifndef JG_GEMM_STAGES
#define JG_GEMM_STAGES 4
#endif
constexpr int BM = 128, BN = 128, BK = 64, kStages = JG_GEMM_STAGES, kThreads = 384;
constexpr int kTileBytes = 16384;  // one operand stage: 128 x 64 bf16
struct Smem {
  static constexpr int kA = 0;
  static constexpr int kB = kStages * kTileBytes;
  static constexpr int kStg = 2 * kStages * kTileBytes;        // JJJ epilogue staging: 8 warps x 32 rows x 65 fp32
  static constexpr int kBar = kStg + 8 * 32 * 65 * 4;
  static constexpr int kNumBars = 3 * kStages + 4 + 1;
  static constexpr int kKeys = (kBar + kNumBars * 8 + 16 + 15) & ~15;  // producer's operand-block keys
  static constexpr int kAlloc = kKeys + 2 * kStages * 8 + 1024;
};

struct Params {
  const int64_t* off;
  const int64_t* sq;
  const int64_t* prefix;  // tiles per sample, exclusive prefix [batch + 1]
  int64_t batch;
  int D, T;
  const __nv_bfloat16* a_j2;  // AJ: jagged^2 A values
  void* out;
  int out_f32;
  const uint8_t* a_tiles;     // AJ / AJT: repacked 64 x 64 sub-block images (8 KB each, aj_repack_kernel)
  const int64_t* a_prefix;    // AJ / AJT: 128 x 128 tiles per sample, exclusive prefix (sub-block base = 4x)
  int dbg;                    // JG_GEMM_DBG (diagnostic, results invalid): 1 = JJJ epilogue skips the stores
  const __nv_bfloat16* bias;  // JD only (jagged_mlp layer, bf16 out): out = act(acc + bias[col]), preact = acc + bias
  int relu;
  __nv_bfloat16* preact;
  int head;        // JJJ / AJ on one head of [rows, H, D] tensors (unfused jagged_attention): TMA head coordinate
  int64_t out_ld;  // AJ / JD output row pitch in elements (0: N)
};

struct Tile {
  int64_t i, b0, n, sqo;
  int M, N, K, m0, n0, nk;
};

// Each CTA owns a contiguous range of tiles (equal counts; tiles of one op cost about the same), so the
// owning sample advances monotonically: a cursor replaces the per-tile binary search over the prefix
// (ten dependent L2 round trips per tile, which capped the producer's tile rate).
struct TileCursor {
  int64_t i = -1, lo = 0, hi = 0;  // current sample, its tile range [lo, hi)
};

__device__ __forceinline__ void tile_range(const Params& p, int64_t& t0, int64_t& t1) {
  const int64_t n = p.prefix[p.batch];
  t0 = n * blockIdx.x / gridDim.x;
  t1 = n * (blockIdx.x + 1) / gridDim.x;
}

template <int OP, int TN = BN>
__device__ __forceinline__ Tile tile_of(const Params& p, int64_t t, TileCursor& c) {
  if (c.i < 0) {
    c.i = upper_index(p.prefix, p.batch, t);
    c.lo = p.prefix[c.i];
    c.hi = p.prefix[c.i + 1];
  }
  while (t >= c.hi) {  // skips empty samples (zero tiles)
    ++c.i;
    c.lo = c.hi;
    c.hi = p.prefix[c.i + 1];
  }
  Tile r;
  r.i = c.i;
  r.b0 = p.off[r.i];
  r.n = p.off[r.i + 1] - r.b0;
  r.sqo = p.sq ? p.sq[r.i] : 0;
  const int Bi = (int)r.n;
  if (OP == JJJ) { r.M = Bi; r.N = Bi; r.K = p.D; }
  if (OP == AJ) { r.M = Bi; r.N = p.D; r.K = Bi; }
  if (OP == JJ) { r.M = p.D; r.N = p.T; r.K = Bi; }
  if (OP == JD) { r.M = Bi; r.N = p.T; r.K = p.D; }
  if (OP == JDT) { r.M = Bi; r.N = p.D; r.K = p.T; }
  if (OP == AJT) { r.M = Bi; r.N = p.D; r.K = Bi; }
  const int tn = (r.N + TN - 1) / TN;
  const int64_t local = t - c.lo;
  r.m0 = (int)(local / tn) * BM;
  r.n0 = (int)(local % tn) * TN;
  r.nk = (r.K + BK - 1) / BK;
  return r;
}

// smem A operand is K-major for JJJ/AJ/JD/JDT ([128 m rows x 64 k]) and MN-major for JJ/AJT ([64 k rows x 128 m]
// in two 64-wide chunks); B is K-major for JJJ/JDT ([128 n rows x 64 k]) and MN-major otherwise.
template <int OP> struct Layout {
  static constexpr bool a_mn = OP == JJ || OP == AJT;
  static constexpr bool b_mn = OP != JJJ && OP != JDT;
  static constexpr bool loader = OP == JJ;  // stages pass through the loader warpgroup (K-tail zeroing)
};

__device__ __forceinline__ void bulk_load_hint(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                               uint64_t policy) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                   tc::smem_u32(sdst)),
               "l"(gsrc), "r"(bytes), "r"(tc::smem_u32(bar)), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tc::smem_u32(sdst)),
               "l"(gsrc), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}

// Jagged^2 A-operand repack (AJ and AJT): sample i's Bi x Bi block (row stride Bi, arbitrary 2-byte alignment,
// unusable by TMA) becomes a grid of nb x nb images of 64 x 64 sub-blocks, nb = 2 ceil(Bi/128), each the exact
// 8 KB SWIZZLE_128B image of 64 rows x 128 B (zeros past Bi). Both GEMM forms read the SAME images: an AJ stage
// ([128 m x 64 k] K-major) is sub-blocks (m0/64, kb) and (m0/64 + 1, kb) stacked; an AJT stage (A^T's block as
// two MN-major 64-wide chunks of 64 k rows) is sub-blocks (kb, m0/64) and (kb, m0/64 + 1) — so a VJP that needs
// A and A^T (jagged_jagged_bmm_jagged_out: dQ = dS K, dK = dS^T Q) repacks once. Sub-block base of sample i:
// 4 tile128_prefix[i] (nb^2 = 4 ceil(Bi/128)^2). One CTA per sub-block; thread u builds 16-byte units from two
// aligned 16-byte loads realigned with funnel shifts.
__device__ __forceinline__ int64_t aj_block(const int64_t* pref128, int64_t i, int Bi, int br, int bc) {
  const int nb = 2 * ((Bi + 127) / 128);
  return 4 * pref128[i] + (int64_t)br * nb + bc;
}
__global__ void __launch_bounds__(256) aj_repack_kernel(const int64_t* __restrict__ off, const int64_t* __restrict__ sq,
                                                        const int64_t* __restrict__ pref128, int64_t batch,
                                                        const __nv_bfloat16* __restrict__ a, uint8_t* __restrict__ blocks) {
  const int64_t n_blocks = 4 * pref128[batch];
  const char* base = reinterpret_cast<const char*>(a);
  // each CTA takes a contiguous range of sub-blocks and walks it with a sample cursor (one search per CTA)
  const int64_t t0 = n_blocks * blockIdx.x / gridDim.x, t1 = n_blocks * (blockIdx.x + 1) / gridDim.x;
  if (t0 >= t1) return;
  int64_t i = upper_index(pref128, batch, t0 >> 2), lo = 4 * pref128[i], hi = 4 * pref128[i + 1];
  int Bi = (int)(off[i + 1] - off[i]);
  int64_t sqo = sq[i];
  for (int64_t t = t0; t < t1; ++t) {
    while (t >= hi) {  // next sample with sub-blocks
      ++i;
      lo = hi;
      hi = 4 * pref128[i + 1];
      Bi = (int)(off[i + 1] - off[i]);
      sqo = sq[i];
    }
    const int nb = 2 * ((Bi + 127) / 128);
    const int64_t local = t - lo;
    const int br = (int)(local / nb), bc = (int)(local % nb);
    uint8_t* dst = blocks + t * (kTileBytes / 2);
#pragma unroll
    for (int rep = 0; rep < 2; ++rep) {
      const int u = rep * 256 + threadIdx.x;  // 16-byte unit: row u/8, column chunk u%8
      const int row = u >> 3, c16 = u & 7;
      const int m = br * 64 + row, kb0 = bc * 64 + c16 * 8;
      const int nval = (m < Bi && kb0 < Bi) ? (Bi - kb0 < 8 ? Bi - kb0 : 8) : 0;
      uint4 lo = make_uint4(0, 0, 0, 0), hi = make_uint4(0, 0, 0, 0);
      int sh = 0;
      if (nval > 0) {
        // an aligned 16-byte chunk holding at least one valid byte lies in that byte's page: no fault
        // absolute addresses: the A base itself need not be 16-byte aligned (e.g. a slice of a larger buffer)
        const uintptr_t byte0 = reinterpret_cast<uintptr_t>(base) + (uintptr_t)((sqo + (int64_t)m * Bi + kb0) * 2);
        const uintptr_t al = byte0 & ~uintptr_t(15);
        sh = (int)(byte0 - al);
        lo = __ldg(reinterpret_cast<const uint4*>(al));
        if (sh != 0 && byte0 + 2 * nval > al + 16) hi = __ldg(reinterpret_cast<const uint4*>(al + 16));
      }
      const int ws = sh >> 2;
      const bool half = (sh & 2) != 0;
      const uint32_t w0 = lo.x, w1 = lo.y, w2 = lo.z, w3 = lo.w, w4 = hi.x, w5 = hi.y, w6 = hi.z, w7 = hi.w;
      const uint32_t x0 = ws == 0 ? w0 : ws == 1 ? w1 : ws == 2 ? w2 : w3;
      const uint32_t x1 = ws == 0 ? w1 : ws == 1 ? w2 : ws == 2 ? w3 : w4;
      const uint32_t x2 = ws == 0 ? w2 : ws == 1 ? w3 : ws == 2 ? w4 : w5;
      const uint32_t x3 = ws == 0 ? w3 : ws == 1 ? w4 : ws == 2 ? w5 : w6;
      const uint32_t x4 = ws == 0 ? w4 : ws == 1 ? w5 : ws == 2 ? w6 : w7;
      uint32_t o[4];
      o[0] = half ? __funnelshift_r(x0, x1, 16) : x0;
      o[1] = half ? __funnelshift_r(x1, x2, 16) : x1;
      o[2] = half ? __funnelshift_r(x2, x3, 16) : x2;
      o[3] = half ? __funnelshift_r(x3, x4, 16) : x3;
      if (nval < 8) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (2 * q >= nval) o[q] = 0;
          else if (2 * q + 1 >= nval) o[q] &= 0xFFFFu;
        }
      }
      *reinterpret_cast<uint4*>(dst + tc::sw128_offset(row, c16)) = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

template <int OP, bool W = false>
__global__ void __launch_bounds__(kThreads, 1) gemm_sm100_kernel(const __grid_constant__ CUtensorMap tm_a,
                                                                 const __grid_constant__ CUtensorMap tm_b, Params p) {
  using Ly = Layout<OP>;
  constexpr int TN = W ? 2 * BN : BN;  // output tile width (TMEM columns per accumulator)
  static_assert(!W || OP == AJ || OP == AJT, "wide tiles: AJ / AJT only");
  static_assert(!W || Smem::kBar - Smem::kStg >= kStages * kTileBytes, "second-half B stages need the staging region");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Smem::kBar);
  uint64_t* ready = full + kStages;
  uint64_t* empty = ready + kStages;
  uint64_t* acc_full = empty + kStages;  // [2]
  uint64_t* acc_empty = acc_full + 2;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(full + s, 1);
      tc::mbar_init(ready + s, 4);
      tc::mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(acc_full + b, 1);
      tc::mbar_init(acc_empty + b, OP == JJ ? 4 : 8);
    }
    tc::fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tm_a);
    tc::tma_prefetch(&tm_b);
  }
  if (warp == 1) tc::tmem_alloc<2 * TN>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  int64_t t_begin, t_end;
  tile_range(p, t_begin, t_end);

  if (warp == 0) {
    // ============================================ TMA producer
    if (lane == 0) {
      // A stage whose A (or B) operand block is the one it already holds is not reloaded: one-segment JD (the
      // jagged_mlp layers: every CTA would otherwise re-read the same weight block from one L2 slice), per-
      // sample JD weights across a sample's row tiles, JJJ query panels across a row of tiles. Keys identify
      // the operand block; JJ stages are rewritten by the loader (K-tail zeroing), so they always reload.
      uint64_t* key = reinterpret_cast<uint64_t*>(smem + Smem::kKeys);  // [2][kStages], producer-private
      const uint64_t pol_first = tc::l2_policy_evict_first(), pol_last = tc::l2_policy_evict_last();
      for (int s = 0; s < 2 * kStages; ++s) key[s] = ~0ull;
      uint32_t cnt = 0;
      TileCursor cur;
      for (int64_t t = t_begin; t < t_end; ++t) {
        const Tile tl = tile_of<OP, TN>(p, t, cur);
        for (int kb = 0; kb < tl.nk; ++kb, ++cnt) {
          const uint32_t s = cnt % kStages;
          tc::mbar_wait(empty + s, ((cnt / kStages) & 1) ^ 1);
          uint8_t* sa = smem + Smem::kA + s * kTileBytes;
          uint8_t* sb = smem + Smem::kB + s * kTileBytes;
          const int k0 = kb * BK;
          uint64_t ka = ~0ull, kbk = ~0ull;  // ~0: always load
          if (OP == JJJ || OP == JD || OP == JDT) ka = (uint64_t)(tl.b0 + tl.m0) * 65536u + (uint64_t)kb;
          if (OP == JJJ) kbk = (uint64_t)(tl.b0 + tl.n0) * 65536u + (uint64_t)kb;
          if (OP == JDT) kbk = ((uint64_t)tl.i * p.D + tl.n0) * 65536u + (uint64_t)kb;
          if (OP == JD) kbk = ((uint64_t)tl.i * p.D + k0) * 65536u + (uint64_t)(tl.n0 / BN);
          if ((OP == AJ || OP == AJT) && !W) kbk = (uint64_t)(tl.b0 + k0) * 65536u + (uint64_t)(tl.n0 / BN);
          const bool half2 = W && tl.n0 + BN < tl.N;  // wide tile: the second 128-column half exists
          const bool load_a = ka == ~0ull || key[s] != ka, load_b = kbk == ~0ull || key[kStages + s] != kbk;
          key[s] = ka;
          key[kStages + s] = kbk;
          tc::mbar_expect_tx(full + s, (load_a || OP == AJ || OP == AJT ? kTileBytes : 0) + (load_b ? kTileBytes : 0) +
                                           (half2 ? kTileBytes : 0));
          if (OP == AJ || OP == AJT) {  // two 8 KB sub-block images: rows m0..+63 / m0+64..+127 (AJ), chunks (AJT)
            for (int c = 0; c < 2; ++c) {
              const int64_t blk = OP == AJ ? aj_block(p.a_prefix, tl.i, (int)tl.n, tl.m0 / 64 + c, kb)
                                           : aj_block(p.a_prefix, tl.i, (int)tl.n, kb, tl.m0 / 64 + c);
              // the sub-block images are read once: evict-first, so they do not push V (re-read by every row
              // block of its sample) out of L2
              bulk_load_hint(sa + c * (kTileBytes / 2), p.a_tiles + blk * (kTileBytes / 2), kTileBytes / 2, full + s,
                             pol_first);
            }
          }
          if ((OP == JJJ || OP == JD || OP == JDT) && load_a)
            tc::tma_load_3d(sa, &tm_a, full + s, k0, p.head, (int)(tl.b0 + tl.m0));
          if (OP == JDT && load_b) tc::tma_load_3d(sb, &tm_b, full + s, k0, 0, (int)(tl.i * p.D + tl.n0));
          if (OP == JJ)
            for (int c = 0; c < 2; ++c)
              tc::tma_load_3d(sa + c * 8192, &tm_a, full + s, tl.m0 + 64 * c, 0, (int)(tl.b0 + k0));
          if (OP == JJJ && load_b) tc::tma_load_3d(sb, &tm_b, full + s, k0, p.head, (int)(tl.b0 + tl.n0));
          if ((OP == AJ || OP == AJT) && load_b)
            for (int c = 0; c < 2; ++c)
              tc::tma_load_3d_hint(sb + c * 8192, &tm_b, full + s, tl.n0 + 64 * c, p.head, (int)(tl.b0 + k0), pol_last);
          if (OP == JJ)
            for (int c = 0; c < 2; ++c) tc::tma_load_3d(sb + c * 8192, &tm_b, full + s, tl.n0 + 64 * c, 0, (int)(tl.b0 + k0));
          if (half2)
            for (int c = 0; c < 2; ++c)
              tc::tma_load_3d_hint(smem + Smem::kStg + s * kTileBytes + c * 8192, &tm_b, full + s, tl.n0 + BN + 64 * c,
                                   p.head, (int)(tl.b0 + k0), pol_last);
          if (OP == JD && load_b)
            for (int c = 0; c < 2; ++c)
              tc::tma_load_3d(sb + c * 8192, &tm_b, full + s, tl.n0 + 64 * c, 0, (int)(tl.i * p.D + k0));
        }
      }
    }
  } else if (warp == 1) {
    // ============================================ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16_f32(BM, BN, Ly::a_mn, Ly::b_mn);
      uint32_t cnt = 0, tcount = 0;
      TileCursor cur;
      for (int64_t t = t_begin; t < t_end; ++t, ++tcount) {
        const Tile tl = tile_of<OP, TN>(p, t, cur);
        const int ab = tcount & 1;
        tc::mbar_wait(acc_empty + ab, ((tcount >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        for (int kb = 0; kb < tl.nk; ++kb, ++cnt) {
          const uint32_t s = cnt % kStages;
          if (Ly::loader) tc::mbar_wait(ready + s, (cnt / kStages) & 1);
          if (!Ly::loader) tc::mbar_wait(full + s, (cnt / kStages) & 1);
          tc::tc_fence_after();
          const uint32_t sa = tc::smem_u32(smem + Smem::kA + s * kTileBytes);
          const uint32_t sb = tc::smem_u32(smem + Smem::kB + s * kTileBytes);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t da = Ly::a_mn ? tc::sw128_desc(sa + kk * 2048, 8192, 1024) : tc::sw128_desc(sa + kk * 32, 16, 1024);
            const uint64_t db = Ly::b_mn ? tc::sw128_desc(sb + kk * 2048, 8192, 1024) : tc::sw128_desc(sb + kk * 32, 16, 1024);
            tc::mma_bf16_ss(tmem + ab * TN, da, db, idesc, (kb > 0 || kk > 0));
            if (W && tl.n0 + BN < tl.N) {
              const uint32_t sb2 = tc::smem_u32(smem + Smem::kStg + s * kTileBytes);
              tc::mma_bf16_ss(tmem + ab * TN + BN, da, tc::sw128_desc(sb2 + kk * 2048, 8192, 1024), idesc, (kb > 0 || kk > 0));
            }
          }
          tc::mma_commit(empty + s);
        }
        tc::mma_commit(acc_full + ab);  // with no k blocks this arrives at once (epilogue writes zeros)
      }
    }
  } else if (OP == JJJ && warp >= 4 && warp < 12) {
    // ============================================ JJJ epilogue (8 warps: TMEM lane quarter x column half)
    // jagged^2 output rows have stride Bi and arbitrary 2-byte alignment: each warp stages its 32 rows x 64
    // columns in smem (row pitch 65 floats, conflict-free) and writes every row segment as 16-byte aligned
    // chunks (one lane each) plus at most 7 leading / 7 trailing elements. (A per-row bulk-copy variant —
    // realigned bf16 row images + cp.async.bulk global<-shared — measured slower: 690 vs 605 us on the table1
    // shape.)
    const int wq = warp & 3, hf = (warp - 4) >> 2;
    // derived from smem_raw by pointer arithmetic so the compiler keeps the shared address space (LDS/STS)
    float* stg = reinterpret_cast<float*>(smem_raw + (smem - smem_raw) + Smem::kStg) + (warp - 4) * 32 * 65;
    uint32_t tcount = 0;
    TileCursor cur;
    for (int64_t t = t_begin; t < t_end; ++t, ++tcount) {
      const Tile tl = tile_of<OP, TN>(p, t, cur);
      const int ab = tcount & 1;
      tc::mbar_wait(acc_full + ab, (tcount >> 1) & 1);
      tc::tc_fence_after();
      const int ncols = tl.N - tl.n0 < BN ? tl.N - tl.n0 : BN;
      const int nc = ncols - 64 * hf < 64 ? ncols - 64 * hf : 64;
      const int nrows = tl.M - tl.m0 - wq * 32 < 32 ? tl.M - tl.m0 - wq * 32 : 32;
      const int64_t row0 = tl.sqo + (int64_t)(tl.m0 + wq * 32) * tl.n + tl.n0 + 64 * hf;
      const int n32 = (int)tl.n;
      uint32_t* img = reinterpret_cast<uint32_t*>(stg);
      // bf16 output: absolute 16-byte alignment of the warp's first output element (the base need only be
      // element-aligned); row r starts sh_r = (a0 + r * Bi) & 7 elements into its 16-byte chunk
      const int a0 = (int)((reinterpret_cast<uintptr_t>(reinterpret_cast<__nv_bfloat16*>(p.out) + row0) >> 1) & 7);
      {
        uint32_t v0[32], v1[32];  // both column chunks in flight before one wait
        tc::tmem_ld32(tmem + ((uint32_t)(wq * 32) << 16) + ab * BN + hf * 64, v0);
        tc::tmem_ld32(tmem + ((uint32_t)(wq * 32) << 16) + ab * BN + hf * 64 + 32, v1);
        tc::tmem_wait_ld();
        if (p.out_f32) {
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            stg[lane * 65 + e] = tl.nk == 0 ? 0.f : __uint_as_float(v0[e]);
            stg[lane * 65 + 32 + e] = tl.nk == 0 ? 0.f : __uint_as_float(v1[e]);
          }
        } else {
          // The lane's row becomes a bf16 image already in its output's 16-byte phase: image element sh + j
          // holds column j, rows 36 words apart (16-byte aligned quads). Odd phases shift by one element
          // (funnel shift of the packed pairs); the image then leaves as aligned 16-byte chunks.
          const int sh = (a0 + lane * n32) & 7;
          const uint32_t fs = (sh & 1) ? 16u : 32u;  // 32: funnelshift_rc returns the high word (no shift)
          uint32_t* row = img + lane * 36 + (sh >> 1);
          uint32_t prev = 0;
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const uint32_t* v = k < 16 ? v0 : v1;
            const int e = (k & 15) * 2;
            const uint32_t w = tl.nk == 0 ? 0u : tc::pack_bf16(__uint_as_float(v[e]), __uint_as_float(v[e + 1]));
            row[k] = __funnelshift_rc(prev, w, fs);
            prev = w;
          }
          row[32] = __funnelshift_rc(prev, 0u, fs);
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(acc_empty + ab);  // TMEM drained; the stores below overlap the next tile
      auto store_img = [&]() {
        // 8 lanes per row (one 16-byte chunk each), 4 rows per step; all image reads before any store. The
        // partial chunks at the row ends (at most 7 elements each) are 2-byte stores.
        __nv_bfloat16* base = reinterpret_cast<__nv_bfloat16*>(p.out) + row0;
        const uint16_t* img16 = reinterpret_cast<const uint16_t*>(img);
        const int sub = lane >> 3, li = lane & 7;
        uint4 body[8];
        uint16_t lead[8], trail[8];
        int cpos[8], lpos[8], tpos[8];
        uint32_t okm = 0, lm = 0, tm = 0;
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int rr = sub + it * 4;
          const int s0 = rr * n32, sh = (a0 + s0) & 7, end = sh + nc;
          const bool live = rr < nrows;
          const int qf = sh ? 1 : 0, ql = end >> 3;  // full chunks: image quads [qf, ql)
          const int q = qf + li;
          const bool okc = live && q < ql;
          const int le = end < 8 ? end : 8, ts = 8 * ql > 8 * qf ? 8 * ql : 8 * qf;
          const bool okl = live && sh > 0 && sh + li < le, okt = live && ts + li < end;
          body[it] = *reinterpret_cast<const uint4*>(img + rr * 36 + 4 * (okc ? q : 0));
          lead[it] = img16[rr * 72 + (okl ? sh + li : 0)];
          trail[it] = img16[rr * 72 + (okt ? ts + li : 0)];
          cpos[it] = s0 - sh + 8 * q;
          lpos[it] = s0 + li;
          tpos[it] = s0 - sh + ts + li;
          okm |= (uint32_t)okc << it;
          lm |= (uint32_t)okl << it;
          tm |= (uint32_t)okt << it;
        }
        uint16_t* base16 = reinterpret_cast<uint16_t*>(base);
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          if (okm >> it & 1) *reinterpret_cast<uint4*>(base + cpos[it]) = body[it];
          if (lm >> it & 1) base16[lpos[it]] = lead[it];
          if (tm >> it & 1) base16[tpos[it]] = trail[it];
        }
      };
      auto store_rows = [&](auto tag) {
        using E = decltype(tag);
        constexpr int CE = 16 / sizeof(E);      // elements per 16-byte chunk
        constexpr int LPR = 64 / CE;            // lanes per row
        constexpr int RPS = 32 / LPR;           // rows per step
        constexpr int NIT = 32 / RPS;           // steps to cover the warp's 32 staged rows
        constexpr int NE = (CE - 1 + LPR - 1) / LPR;  // edge elements per lane (at most CE - 1 per row end)
        // Per-row positions are 32-bit offsets from the tile's first element (rr * Bi + 64 < 2^31); chunk
        // alignment is absolute, so a0 = misalignment of that first element (the output base need only be
        // element-aligned). All staging reads are issued before any global store (the generic output pointer
        // could alias shared memory, so an interleaved loop serialises every LDS behind the previous STG), and
        // the edge elements are predicated stores rather than divergent branches.
        E* base = reinterpret_cast<E*>(p.out) + row0;
        const int a0 = (int)((reinterpret_cast<uintptr_t>(base) / sizeof(E)) & (CE - 1));
        const int sub = lane / LPR, li = lane % LPR, n32 = (int)tl.n;
        uint4 body[NIT];
        float lead[NIT][NE], trail[NIT][NE];
        int cpos[NIT], s0s[NIT], t0s[NIT];
        uint32_t okm = 0, lm = 0, tm = 0;  // bit it * NE + k: edge element li + k * LPR of step it
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
          const int rr = sub + it * RPS;
          const int s0 = rr * n32;                                  // row start (tile-relative)
          const int hd = (CE - ((a0 + s0) & (CE - 1))) & (CE - 1);  // elements before the first aligned chunk
          const int tl0 = (a0 + s0 + nc) & (CE - 1);                // elements after the last aligned chunk
          const int nh = hd < nc ? hd : nc;
          const int body_n = nc - nh - tl0;                        // aligned body length (may be < 0)
          const int c = hd + li * CE;                               // row-relative chunk start
          const bool live = rr < nrows;
          const bool okc = live && c + CE <= hd + (body_n > 0 ? body_n : 0);
          const int t0 = body_n > 0 ? nc - tl0 : nh;               // row-relative tail start
          const float* rs = stg + rr * 65;
          const int cb = okc ? c : 0;
          float f[8];
#pragma unroll
          for (int e = 0; e < CE; ++e) f[e] = rs[cb + e];
          if constexpr (sizeof(E) == 4) {
            body[it] = make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
          } else {
            body[it] = make_uint4(tc::pack_bf16(f[0], f[1]), tc::pack_bf16(f[2], f[3]), tc::pack_bf16(f[4], f[5]),
                                  tc::pack_bf16(f[6], f[7]));
          }
#pragma unroll
          for (int k = 0; k < NE; ++k) {
            const int x = li + k * LPR;
            const bool okl = live && x < nh, okt = live && x < nc - t0;
            lead[it][k] = rs[okl ? x : 0];
            trail[it][k] = rs[okt ? t0 + x : 0];
            lm |= (uint32_t)okl << (it * NE + k);
            tm |= (uint32_t)okt << (it * NE + k);
          }
          cpos[it] = s0 + c;
          s0s[it] = s0;
          t0s[it] = s0 + t0;
          okm |= (uint32_t)okc << it;
        }
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
          if (okm >> it & 1) *reinterpret_cast<uint4*>(base + cpos[it]) = body[it];
#pragma unroll
          for (int k = 0; k < NE; ++k) {
            if (lm >> (it * NE + k) & 1) base[s0s[it] + li + k * LPR] = E(lead[it][k]);
            if (tm >> (it * NE + k) & 1) base[t0s[it] + li + k * LPR] = E(trail[it][k]);
          }
        }
      };
      if (nc > 0 && !(p.dbg & 1)) {
        if (p.out_f32) store_rows(float{});
        else store_img();
      }
      __syncwarp();
    }
  } else if (warp >= 4 && warp < (Ly::loader ? 8 : 12)) {
    // ============================================ epilogue: thread = output row of the tile
    // JD / AJ: 8 warps (TMEM lane quarter x column half, two 32-column chunks each); JJ: 4 warps (warps 8-11
    // are its loader)
    constexpr int kHalves = Ly::loader ? 1 : 2, kChunks = TN / 32 / kHalves;
    const int wq = warp & 3, hf = (warp - 4) >> 2, r = wq * 32 + lane;
    uint32_t tcount = 0;
    TileCursor cur;
    for (int64_t t = t_begin; t < t_end; ++t, ++tcount) {
      const Tile tl = tile_of<OP, TN>(p, t, cur);
      const int ab = tcount & 1;
      tc::mbar_wait(acc_full + ab, (tcount >> 1) & 1);
      tc::tc_fence_after();
      const int m = tl.m0 + r;
      const bool row_ok = m < tl.M;
      const int ncols = tl.N - tl.n0 < TN ? tl.N - tl.n0 : TN;
      int64_t base;  // element index of (m, n0) in the output
      if (OP == JJJ) base = tl.sqo + (int64_t)m * tl.n + tl.n0;
      else if (OP == JJ) base = tl.i * (int64_t)p.D * p.T + (int64_t)m * p.T + tl.n0;
      else base = (tl.b0 + m) * (p.out_ld ? p.out_ld : (int64_t)tl.N) + tl.n0;
      const bool vec_tile = OP != JJJ && ncols == TN;
      // 32-byte alignment of every row start: N (or T) a multiple of 16 bf16 / 8 fp32 elements
      const bool vec32_ok = ((OP == JJ ? p.T : (p.out_ld ? p.out_ld : tl.N)) % (p.out_f32 ? 8 : 16)) == 0 &&
                            (reinterpret_cast<uintptr_t>(p.out) & 31) == 0;
#pragma unroll
      for (int cc = 0; cc < kChunks; ++cc) {
        const int c = hf * kChunks + cc;
        if (W && c * 32 >= ncols) continue;  // wide tile without its second half
        const bool vec = vec_tile || (W && OP != JJJ && (c + 1) * 32 <= ncols);
        uint32_t v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(wq * 32) << 16) + ab * TN + c * 32, v);
        tc::tmem_wait_ld();
        if (tl.nk == 0) {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = 0u;
        }
        if (!row_ok) continue;
        const bool vec32 = vec && vec32_ok;
        if (p.out_f32) {
          float* o = reinterpret_cast<float*>(p.out) + base + c * 32;
          if (vec32) {
#pragma unroll
            for (int u = 0; u < 8; u += 2)  // 32-byte sectors (STG.256)
              tc::st_global_v8(o + u * 4, make_uint4(v[u * 4], v[u * 4 + 1], v[u * 4 + 2], v[u * 4 + 3]),
                               make_uint4(v[u * 4 + 4], v[u * 4 + 5], v[u * 4 + 6], v[u * 4 + 7]));
          } else if (vec) {
#pragma unroll
            for (int u = 0; u < 8; ++u)
              *reinterpret_cast<uint4*>(o + u * 4) = make_uint4(v[u * 4], v[u * 4 + 1], v[u * 4 + 2], v[u * 4 + 3]);
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (c * 32 + e < ncols) o[e] = __uint_as_float(v[e]);
          }
        } else {
          __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) + base + c * 32;
          if (OP == JD && p.bias && !(p.dbg & 2)) {  // fused jagged_mlp layer epilogue (= bias_act_kernel)
            __nv_bfloat16* pre = p.preact ? p.preact + base + c * 32 : nullptr;
            // the chunk's 32 bias values: four 16-byte loads (the same address in every lane: one broadcast
            // transaction each) instead of 32 dependent 2-byte loads
            uint32_t bw[16];
            if (vec) {
              const uint4* bp = reinterpret_cast<const uint4*>(p.bias + tl.n0 + c * 32);
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const uint4 q = __ldg(bp + u);
                bw[u * 4] = q.x, bw[u * 4 + 1] = q.y, bw[u * 4 + 2] = q.z, bw[u * 4 + 3] = q.w;
              }
            } else {
#pragma unroll
              for (int u = 0; u < 16; ++u) {
                const int col = tl.n0 + c * 32 + 2 * u;
                const uint32_t lo = col < tl.N ? __bfloat16_as_ushort(p.bias[col]) : 0u;
                const uint32_t hi = col + 1 < tl.N ? __bfloat16_as_ushort(p.bias[col + 1]) : 0u;
                bw[u] = lo | (hi << 16);
              }
            }
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              const float bv = __uint_as_float((e & 1) ? (bw[e >> 1] & 0xffff0000u) : (bw[e >> 1] << 16));
              const float x = __uint_as_float(v[e]) + bv;
              if (pre && c * 32 + e < ncols) pre[e] = __float2bfloat16_rn(x);
              v[e] = __float_as_uint(p.relu ? fmaxf(x, 0.f) : x);
            }
          }
          if (vec) {
            uint4 w[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              w[u].x = tc::pack_bf16(__uint_as_float(v[u * 8 + 0]), __uint_as_float(v[u * 8 + 1]));
              w[u].y = tc::pack_bf16(__uint_as_float(v[u * 8 + 2]), __uint_as_float(v[u * 8 + 3]));
              w[u].z = tc::pack_bf16(__uint_as_float(v[u * 8 + 4]), __uint_as_float(v[u * 8 + 5]));
              w[u].w = tc::pack_bf16(__uint_as_float(v[u * 8 + 6]), __uint_as_float(v[u * 8 + 7]));
            }
            if (vec32) {  // 32-byte sectors (STG.256)
              tc::st_global_v8(o, w[0], w[1]);
              tc::st_global_v8(o + 16, w[2], w[3]);
            } else {
#pragma unroll
              for (int u = 0; u < 4; ++u) *reinterpret_cast<uint4*>(o + u * 8) = w[u];
            }
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (c * 32 + e < ncols) o[e] = __float2bfloat16_rn(__uint_as_float(v[e]));
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(acc_empty + ab);
    }
  } else if (warp >= 8 && Ly::loader) {
    // ============================================ loader warpgroup
    const int wq = warp - 8;
    uint32_t cnt = 0;
    TileCursor cur;
    for (int64_t t = t_begin; t < t_end; ++t) {
      const Tile tl = tile_of<OP, TN>(p, t, cur);
      for (int kb = 0; kb < tl.nk; ++kb, ++cnt) {
        const uint32_t s = cnt % kStages;
        uint8_t* sa = smem + Smem::kA + s * kTileBytes;
        const int k0 = kb * BK;
        {
          // JJ: zero the A (and B) rows of the K tail that belong to the next sample
          tc::mbar_wait(full + s, (cnt / kStages) & 1);
          const int rem = tl.K - k0;
          if (rem < BK) {
            uint8_t* sb = smem + Smem::kB + s * kTileBytes;
            for (int idx = wq * 32 + lane; idx < 2 * 2 * BK * 8; idx += 128) {
              const int which = idx / (2 * BK * 8), rest = idx % (2 * BK * 8);
              const int chunk = rest / (BK * 8), row = (rest / 8) % BK, u = rest % 8;
              if (row >= rem)
                *reinterpret_cast<uint4*>((which ? sb : sa) + chunk * 8192 + row * 128 + u * 16) = make_uint4(0, 0, 0, 0);
            }
          }
        }
        tc::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(ready + s);
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<2 * TN>(tmem);
  }
}

// 2-D view [rows, cols] bf16 as a 3-D map (cols, 1, rows) with box (64, 1, box_rows), SWIZZLE_128B
static jg_status map2d(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int box_rows) {
  return make_map(m, ptr, rows, 1, (int)cols, box_rows);
}

template <int OP, bool W = false>
static jg_status run(const Params& p, const CUtensorMap& ma, const CUtensorMap& mb, cudaStream_t st) {
  if (jg_status rc = ensure_smem_attr((const void*)gemm_sm100_kernel<OP, W>, Smem::kAlloc, "gemm_sm100_kernel")) return rc;
  gemm_sm100_kernel<OP, W><<<device_sm_count(), kThreads, Smem::kAlloc, st>>>(ma, mb, p);
  JG_LAUNCHED("gemm_sm100_kernel");
  return JG_OK;
}

}  // namespace gm

bool gemm_sm100_supported(int op, int64_t D, int64_t T, jg_dtype in_dt) {
  if (in_dt != JG_BF16) return false;
  switch (op) {
    case gm::JJJ: return D % 64 == 0;
    case gm::AJ: case gm::AJT: return D % 64 == 0;
    case gm::JJ: case gm::JD: case gm::JDT: return D % 64 == 0 && T % 64 == 0;
  }
  return false;
}

// Repack a jagged^2 operand into 64 x 64 sub-block images (aj_repack_kernel) for AJ / AJT GEMMs; the buffer is sized
// from the host-known sum Bi^2 (sum 4 ceil(Bi/128)^2 <= sum_sq / 4096 + total_rows / 16 + 4 batch + 4), or with one
// stream-synchronising read of the block count when it is unknown (sum_sq < 0).
jg_status aj_repack(const int64_t* off, const int64_t* sq, int64_t batch, int64_t total_rows, int64_t sum_sq,
                    const void* a, AjBlocks* out, cudaStream_t st) {
  *out = AjBlocks{};
  if (batch == 0) return JG_OK;
  auto ok = [](cudaError_t e, const char* where) { return e == cudaSuccess ? JG_OK : cuda_status(e, where); };
  if (jg_status rc = ok(cudaMallocAsync(&out->prefix, sizeof(int64_t) * (batch + 1), st), "aj prefix")) return rc;
  out->prefix_bytes = (int64_t)sizeof(int64_t) * (batch + 1);
  scratch_note(out->prefix_bytes);
  GemmDesc ga;
  Lin bi;
  bi.bi = 1;
  ga.M = bi;
  ga.N = bi;
  jg_status rc = launch_gemm_prefix(ga, off, sq, batch, 128, 128, out->prefix, st);
  int64_t n = 0;
  if (sum_sq >= 0) {
    n = sum_sq / 4096 + total_rows / 16 + 4 * batch + 4;
  } else if (!rc) {
    rc = ok(cudaMemcpyAsync(&n, out->prefix + batch, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "aj block count");
    if (!rc) rc = ok(cudaStreamSynchronize(st), "aj block count");
    n *= 4;
  }
  out->n_blocks = n;
  if (!rc && n > 0) {
    rc = ok(cudaMallocAsync(&out->blocks, (size_t)n * (gm::kTileBytes / 2), st), "aj blocks");
    if (!rc) {
      out->blocks_bytes = n * (gm::kTileBytes / 2);
      scratch_note(out->blocks_bytes);
      const unsigned rgrid = (unsigned)std::min<int64_t>(n, 32LL * device_sm_count());
      gm::aj_repack_kernel<<<rgrid, 256, 0, st>>>(off, sq, out->prefix, batch, (const __nv_bfloat16*)a, out->blocks);
      rc = ok(cudaGetLastError(), "aj_repack_kernel");
      count_launch();
    }
  }
  if (rc) aj_release(out, st);
  return rc;
}

void aj_release(AjBlocks* b, cudaStream_t st) {
  if (b->blocks) {
    cudaFreeAsync(b->blocks, st);
    scratch_note(-b->blocks_bytes);
  }
  if (b->prefix) {
    cudaFreeAsync(b->prefix, st);
    scratch_note(-b->prefix_bytes);
  }
  *b = AjBlocks{};
}

// A/B roles per op: JJJ (q, k), AJ / AJT (a_j2, v), JJ (x, y), JD (x, w [B, D, T]), JDT (x [rows, T], w [B, D, T])
jg_status launch_gemm_sm100(int op, const int64_t* off, const int64_t* sq, int64_t batch, int64_t total_rows, int64_t D,
                            int64_t T, const void* a, const void* b, void* out, jg_dtype out_dt, int64_t* tile_prefix,
                            cudaStream_t st, const void* bias, int relu, void* preact, int heads, int head,
                            int64_t sum_sq, const AjBlocks* pre) {
  // tile prefix over samples with the op's (M, N)
  GemmDesc g;
  Lin bi;
  bi.bi = 1;
  if (op == gm::JJJ) { g.M = bi; g.N = bi; }
  if (op == gm::AJ) { g.M = bi; g.N = L_const(D); }
  if (op == gm::JJ) { g.M = L_const(D); g.N = L_const(T); }
  if (op == gm::JD) { g.M = bi; g.N = L_const(T); }
  if (op == gm::JDT || op == gm::AJT) { g.M = bi; g.N = L_const(D); }
  // AJ / AJT with D >= 256: 128 x 256 output tiles (the jagged^2 A stages are shared by both column halves)
  const bool wide = (op == gm::AJ || op == gm::AJT) && D >= 256;
  if (jg_status rc = launch_gemm_prefix(g, off, sq, batch, 128, wide ? 256 : 128, tile_prefix, st)) return rc;
  gm::Params p{off, sq, tile_prefix, batch, (int)D, (int)T, (const __nv_bfloat16*)a, out, out_dt == JG_F32,
               nullptr, nullptr, std::getenv("JG_GEMM_DBG") ? std::atoi(std::getenv("JG_GEMM_DBG")) : 0,
               (const __nv_bfloat16*)bias, relu, (__nv_bfloat16*)preact, head,
               heads > 1 && (op == gm::AJ || op == gm::AJT) ? (int64_t)heads * D : 0};
  if (bias && (op != gm::JD || out_dt != JG_BF16)) return fail(JG_UNSUPPORTED, "gemm_sm100: fused bias only for JD bf16");
  CUtensorMap ma{}, mb{};
  const int64_t rows = total_rows > 0 ? total_rows : 1;
  switch (op) {
    case gm::JJJ:
      if (jg_status rc = make_map(&ma, a, rows, heads, (int)D, 128)) return rc;
      if (jg_status rc = make_map(&mb, b, rows, heads, (int)D, 128)) return rc;
      return gm::run<gm::JJJ>(p, ma, mb, st);
    case gm::AJ:
    case gm::AJT: {
      if (jg_status rc = make_map(&mb, b, rows, heads, (int)D, 64)) return rc;
      AjBlocks own;
      const AjBlocks* blk = pre;
      if (!blk) {
        if (jg_status rc = aj_repack(off, sq, batch, total_rows, sum_sq, a, &own, st)) return rc;
        blk = &own;
      }
      p.a_tiles = blk->blocks;
      p.a_prefix = blk->prefix;
      jg_status rc = JG_OK;
      if (blk->n_blocks > 0) {
        if (wide) rc = op == gm::AJ ? gm::run<gm::AJ, true>(p, mb, mb, st) : gm::run<gm::AJT, true>(p, mb, mb, st);
        else rc = op == gm::AJ ? gm::run<gm::AJ>(p, mb, mb, st) : gm::run<gm::AJT>(p, mb, mb, st);
      }
      if (!pre) aj_release(&own, st);
      return rc;
    }
    case gm::JJ:
      if (jg_status rc = gm::map2d(&ma, a, rows, D, 64)) return rc;
      if (jg_status rc = gm::map2d(&mb, b, rows, T, 64)) return rc;
      return gm::run<gm::JJ>(p, ma, mb, st);
    case gm::JD:
      if (jg_status rc = gm::map2d(&ma, a, rows, D, 128)) return rc;
      if (jg_status rc = gm::map2d(&mb, b, batch * D > 0 ? batch * D : 1, T, 64)) return rc;
      return gm::run<gm::JD>(p, ma, mb, st);
    case gm::JDT:  // A [rows, T] and the per-sample W [B*D rows, T] both K-major, [128 x 64] boxes
      if (jg_status rc = gm::map2d(&ma, a, rows, T, 128)) return rc;
      if (jg_status rc = gm::map2d(&mb, b, batch * D > 0 ? batch * D : 1, T, 128)) return rc;
      return gm::run<gm::JDT>(p, ma, mb, st);
  }
  return fail(JG_UNSUPPORTED, "gemm_sm100: unknown op");
}

}  // namespace jg
