// attn_bwd_sm100.cu — Jagged Flash Attention backward on tcgen05 tensor cores (bf16, head_dim 128).
//
// Semantics: attention.cpp:227-289 (jagged_flash_attention_backward): recompute P = exp(S/sqrt(D) - lse)
// from (q, k, lse), Delta = rowsum(dO * O), dV = P^T dO, dS = P * (dP - Delta) with dP = dO V^T,
// dQ = dS K / sqrt(D), dK = dS^T Q / sqrt(D). Per segment only; no padding materialised.
//
// Three launches:
//   1. prologue: Delta[h, r] = sum_d dO*O (fp32) and zero the dQ accumulator             (HBM-bound)
//   2. main persistent kernel, key-stationary: a CTA owns 128 key rows of one (sample, head) and
//      streams the sample's queries in 64-row blocks:
//        S^T = K Q_j^T, dP^T = V dO_j^T                      (tcgen05, M=128 keys, N=64 queries)
//        P^T and dS^T (bf16) back into TMEM over S^T, dS^T also -> smem   (softmax warps, thread = key row)
//        dV += P^T dO_j, dK += dS^T Q_j (TS: A from TMEM; accumulated in TMEM across all j)
//        dQ_j^T = K^T dS^T                                    (M = head_dim, N = 64 queries)
//      dQ_j^T is drained by a second warpgroup through smem and added into the accumulator with TMA
//      tensor reduce-adds (cp.reduce.async.bulk.tensor .add, two alternating staging buffers). The key tiles of
//      a sample add into one query block in whatever order they finish, so:
//        deterministic (default, the reference's fixed order attention.cpp:252-254): each
//          partial is first rounded to a per-head grid u_h (a power of two) with one FFMA2 against a magic
//          constant, so every fp32 add of the reduction is EXACT — multiples of u_h summing to less than
//          2^24 u_h — and the result is bit-identical for every arrival order, grid and schedule. u_h comes
//          from a rigorous bound on every partial sum: |sum_{k in any key subset} dS_qk K_kd| / sqrt(D)
//          <= 2 max|K| max||V|| max||dO|| / sqrt(D) = T_h (|dS_qk| <= P_qk 2 ||dO_q|| max||V||, sum_k P_qk = 1);
//          with B = 2 T_h in [2^e, 2^(e+1)), u_h = 2^(e-22): |partials| <= T_h < 2^22 u_h (the magic rounding's
//          range) and |sums| < 2^24 u_h. The per-head maxima come from the prologue (which then also reads K
//          and V). The rounding error, at most u_h / 2 per key tile, is ~2^-24 of the head's dQ bound;
//        fast: plain fp32 adds, order-dependent rounding in the last bits.
//      Both reduce fp32 [16 q x D] boxes (the same HBM/L2 traffic and convert pass).
//      Work items are taken dynamically in LPT order.
//   3. epilogue: dQ (bf16) = accumulator                                                 (HBM-bound)
// Warps: 0 TMA producer, 1-2 MMA issuers, 4-11 softmax/dS (two warps per TMEM lane
// quarter, 32 query columns each), 12-15 dQ drain + dK/dV epilogue.
// TMEM columns: two score buffers b at [128b, 128b+128) = S^T (64) + dP^T (64); P^T_j and dS^T_j (16 packed
// columns per 32 queries each, interleaved) are written over the S^T slot and dQ_j^T into the dP^T slot of buffer
// j&1 once its scores are consumed; dV [256,384), dK [384,512). S_{j+1} is issued before
// dV_j/dK_j/dQ_j so the softmax warpgroup works on block j+1 while the tensor core finishes block j.
#include "common.cuh"
#include "internal.h"
#include "tc.cuh"
#include "tma_host.h"

namespace jg {
namespace fb {

constexpr int BKV = 128;  // key rows per CTA tile
constexpr int BQ = 64;    // query rows per streamed block
constexpr int kThreads = 512;
constexpr int kSmWarp0 = 4, kDqWarp0 = 12;
constexpr int kSmWarps = 8;  // two warps per TMEM lane quarter, each owning 32 of the 64 query columns
// Dynamic work distribution: the producer takes items from a global counter (in LPT order) and hands
// them to the other roles through a small smem ring; every other warp consumes each entry once.
constexpr int kItemSlots = 4;
constexpr int kItemConsumers = 2 + kSmWarps + 4;  // S and G issuers, softmax warps, drain warps
constexpr float kLog2e = 1.4426950408889634f;
#ifndef JG_BWD_QD_STAGES
#define JG_BWD_QD_STAGES 3
#endif
constexpr int kQdStages = JG_BWD_QD_STAGES;  // (Q_j, dO_j) smem ring depth: 3 stages + 4 dQ staging buffers measured
                                             // ~2.5% faster on cfg3 and ~4% at L=4096 than 4 stages + 2 buffers
constexpr int kPdsBufs = 1;   // dS^T smem buffers
// deterministic dQ: the magic constant 1.5 * 2^23 * u of the grid u = 2^(e - 22), B in [2^e, 2^(e+1)) the bound
// (see the header): fma(x, scale, M) - M rounds x * scale to a multiple of u. Degenerate bounds give 0 (B = 0:
// dQ is exactly 0; not finite: no rounding).
__device__ __forceinline__ float grid_magic(float bound) {
  if (!(bound > 0.f) || !(bound <= 1.0e37f)) return 0.f;
  int e = (int)((__float_as_uint(bound) >> 23) & 0xff) + 1;  // biased exponent of 2^(e + 1), M = 1.5 * 2^(e + 1)
  if (e < 2) e = 2;                                            // (denormal bounds: the smallest normal grid)
  return __uint_as_float(((unsigned)e << 23) | 0x400000u);
}

template <int D, bool DET = false>
struct Smem {
  static constexpr int kChunkKV = BKV * 128;  // [128 rows x 64] bf16 = 16 KB
  static constexpr int kChunkQ = BQ * 128;    // [64 rows x 64] bf16 = 8 KB
  static constexpr int kTileKV = (D / 64) * kChunkKV;
  static constexpr int kTileQ = (D / 64) * kChunkQ;
  static constexpr int kStages = kQdStages;
  static constexpr int kK = 0;
  static constexpr int kV = kK + kTileKV;
  static constexpr int kQD = kV + kTileKV;                  // stages of (Q_j, dO_j)
  static constexpr int kDS = kQD + kStages * 2 * kTileQ;    // kPdsBufs x dS^T [128 keys x 64 q] bf16 (P^T is in TMEM)
  static constexpr int kStg = kDS + kPdsBufs * BKV * 128;   // dQ staging: kStgBufs x [kStgRows q x D] fp32 | int64
  static constexpr int kAccBytes = 4;                       // fp32 accumulator element
  static constexpr int kStgRows = 16;                       // dQ rows per TMA reduce (four per block; 8-row boxes
                                                            // measured slower: the TMA op rate binds)
  static constexpr int kStgBufs = kQdStages > 3 ? 2 : 4;    // fill one while the TMA reads the others
  static constexpr int kLsdBytes = 2 * BQ * 4;              // per stage: 64 -lse*log2(e) + 64 -Delta, fp32
  // the dK/dV epilogue reuses the staging region as four 4 KB warp slices (32 rows x 128 B)
  static constexpr int kStgBytes = kStgBufs * kStgRows * D * kAccBytes > 4 * 4096 ? kStgBufs * kStgRows * D * kAccBytes
                                                                                 : 4 * 4096;
  static constexpr int kLse = kStg + kStgBytes;  // kStages x kLsdBytes, loaded with (Q_j, dO_j)
  static constexpr int kBar = kLse + kStages * kLsdBytes;
  static constexpr int kNumBars = 4 + 2 * kStages + 4 + 1 + kPdsBufs + 4 + 2 + 2 * kItemSlots;
  static constexpr int kItemRing = (kBar + kNumBars * 8 + 16 + 15) & ~15;  // kItemSlots x 32-byte descriptors
  static constexpr int kMaxMagicHeads = 64;                   // deterministic: per-head magic constants in smem
  static constexpr int kMagic = kItemRing + kItemSlots * 32;
  static constexpr int kBytes = kMagic + (DET ? kMaxMagicHeads * 4 : 0);
  // no alignment slack: the dynamic smem base is 1024-aligned (declared so; checked at kernel entry)
  static constexpr int kAlloc = kBytes;
  static_assert(kAlloc <= 232448, "exceeds the 227 KB dynamic shared memory limit");
};

struct Params {
  const int64_t* off;
  const int2* items;
  const int64_t* n_items;
  int64_t total_rows;
  int H;
  const float* lsd;  // [2][H][total_rows]: -lse * log2(e), -Delta (written by the prologue), then [3][H] max|K|,
                     // max||V||^2, max||dO||^2 per head (deterministic mode)
  void* dq_acc;  // fp32 [total_rows, H, D]
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  float scale_log2;
  float scale;
  int dbg;                   // JG_BWD_DBG diagnostic bits (results invalid when set): 1 skip the dQ reduce,
                             // 4 skip the P/dS smem stores, 8 skip the dK/dV stores, 64 skip the main kernel, 128 sync + report after it
  unsigned long long* work_counter;  // [2] self-resetting (internal.h work_counters_exit); items beyond the first round
  unsigned long long* prof;  // JG_WAIT_PROF counters (producer 0-7, MMA 8-15, softmax 16-23, drain 24-31)
  const int64_t* valid;      // padded mode: per-sample valid length <= segment length (nullptr: jagged). Keys and
                             // queries past it get P = dS = 0, so their dQ/dK/dV rows come out zero.
};

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bulk_reduce_add_f32(float* gdst, uint32_t ssrc, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(gdst), "r"(ssrc),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tensor_reduce_add_3d(const CUtensorMap* map, uint32_t ssrc, int c0, int c1, int c2) {
  asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(ssrc), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
// the grid magic of head h: B = 4 max|K| max||V|| max||dO|| / sqrt(D) (kvb = [3][H] max|K|, max||V||^2, max||dO||^2)
__device__ __forceinline__ float head_magic(const float* kvb, int H, int h, float inv_sqrt_d) {
  return grid_magic(4.f * kvb[h] * sqrtf(kvb[H + h]) * sqrtf(kvb[2 * H + h]) * inv_sqrt_d);
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }


template <int D, bool DET>
__global__ void __launch_bounds__(kThreads, 1)
    jfa_bwd_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                         const __grid_constant__ CUtensorMap tm_dq, Params p) {
  using L = Smem<D, DET>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (threadIdx.x == 0 && (tc::smem_u32(smem) & 1023) != 0) __trap();  // SWIZZLE_128B tiles need 1 KB alignment
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* k_full = bars + 0;
  uint64_t* k_empty = bars + 1;  // S issuer after its last S^T, G issuer after its last dQ^T
  uint64_t* v_full = bars + 2;
  uint64_t* v_empty = bars + 3;  // S issuer after its last dP^T: the next item's V loads while G finishes
  uint64_t* qd_full = bars + 4;
  uint64_t* qd_empty = qd_full + L::kStages;
  uint64_t* st_full = qd_empty + L::kStages;  // [2] per TMEM score buffer
  uint64_t* pt_free = st_full + 2;            // [2] dV / dK finished reading P^T / dS^T from TMEM buffer b
  uint64_t* p_full = pt_free + 2;
  uint64_t* pds_empty = p_full + 1;            // [kPdsBufs]
  uint64_t* dq_full = pds_empty + kPdsBufs;          // [2] one per score buffer: a single barrier could complete
                                              // twice before the drain warps wait (no S fill between dQ_{n-2}, dQ_{n-1})
  uint64_t* dq_empty = dq_full + 2;           // [2] dQ^T_j lives in score buffer j&1
  uint64_t* dkv_full = dq_empty + 2;
  uint64_t* dkv_empty = dkv_full + 1;
  uint64_t* item_full = dkv_empty + 1;        // [kItemSlots]
  uint64_t* item_empty = item_full + kItemSlots;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(item_empty + kItemSlots);
  // ring slot: (sample, key tile, head, end) (b0 lo, b0 hi, n lo, n hi) — the producer's decoded item, so
  // the other roles never touch the work list or the offsets
  const uint32_t item_ring = tc::smem_u32(smem + L::kItemRing);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    tc::mbar_init(k_full, 1);
    tc::mbar_init(k_empty, 2);
    tc::mbar_init(v_full, 1);
    tc::mbar_init(v_empty, 1);
    for (int s = 0; s < L::kStages; ++s) {
      tc::mbar_init(qd_full + s, 1 + 32);  // TMA expect_tx arrival + 32 cp.async (lse/Delta) arrivals
      tc::mbar_init(qd_empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(st_full + b, 1);
      tc::mbar_init(pt_free + b, 1);
      tc::mbar_init(dq_empty + b, 4);
    }
    tc::mbar_init(p_full, kSmWarps);
    for (int b = 0; b < kPdsBufs; ++b) tc::mbar_init(pds_empty + b, 1);
    tc::mbar_init(dq_full, 1);
    tc::mbar_init(dq_full + 1, 1);
    tc::mbar_init(dkv_full, 1);
    tc::mbar_init(dkv_empty, 4);
    for (int s = 0; s < kItemSlots; ++s) {
      tc::mbar_init(item_full + s, 1);
      tc::mbar_init(item_empty + s, kItemConsumers);
    }
    tc::fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tm_q);
    tc::tma_prefetch(&tm_k);
    tc::tma_prefetch(&tm_v);
    tc::tma_prefetch(&tm_do);
    tc::tma_prefetch(&tm_dq);
  }
  tc::cta_time_mark(p.prof, 0);
  if (warp == 1) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int H = p.H;
  const int64_t n_work = *p.n_items * H;
  // a consumer warp's next work index (the producer publishes n_work as the end marker)
  struct Work {
    int2 it;
    int h;
    int64_t b0, n, nv;  // nv: valid keys/queries (== n except in padded mode)
  };
  auto take_item = [&](uint32_t ic, Work& wk) -> bool {
    const uint32_t s = ic % kItemSlots;
    tc::mbar_wait(item_full + s, (ic / kItemSlots) & 1);
    const uint4 a = tc::ld_shared_v4u(item_ring + s * 32), c = tc::ld_shared_v4u(item_ring + s * 32 + 16);
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(item_empty + s);
    wk.it = make_int2((int)a.x, (int)a.y);
    wk.h = (int)a.z;
    wk.b0 = (int64_t)(((uint64_t)c.y << 32) | c.x);
    wk.n = (int64_t)c.z;
    wk.nv = (int64_t)c.w;
    return a.w == 0;
  };

  if (warp == 0) {
    // ===================================================== producer warp
    // Lane 0 issues the TMA loads; all 32 lanes stage the block's 64 lse and 64 Delta values with 4-byte
    // cp.async copies (rows start anywhere, so a TMA tensor box is not aligned) that arrive on the same
    // qd_full barrier as the (Q_j, dO_j) tiles.
    tc::WaitProf wp;
    wp.init(lane == 0 ? p.prof : nullptr, 0);
    const long long t_role = clock64();
    uint32_t item_cnt = 0, qd_cnt = 0;
    int64_t w_next = blockIdx.x;  // first round static, then the global counter (LPT order)
    for (;; ++item_cnt) {
      const int64_t w = w_next < n_work ? w_next : n_work;
      int2 it = make_int2(0, 0);
      int64_t b0 = 0, n = 0, nv = 0;
      if (w < n_work) {
        it = p.items[w / H];
        b0 = p.off[it.x];
        n = p.off[it.x + 1] - b0;
        nv = p.valid ? (p.valid[it.x] < n ? p.valid[it.x] : n) : n;
      }
      const int h = (int)(w % H);
      {  // publish the decoded item to the consumer warps
        const uint32_t s = item_cnt % kItemSlots;
        wp.wait_warp(item_empty + s, ((item_cnt / kItemSlots) & 1) ^ 1, 3);
        if (lane == 0) {
          tc::st_shared_v4(item_ring + s * 32, (uint32_t)it.x, (uint32_t)it.y, (uint32_t)h, w >= n_work ? 1u : 0u);
          tc::st_shared_v4(item_ring + s * 32 + 16, (uint32_t)b0, (uint32_t)((uint64_t)b0 >> 32), (uint32_t)n,
                           (uint32_t)nv);
          tc::mbar_arrive(item_full + s);
        }
      }
      if (w >= n_work) break;
      if (lane == 0) w_next = (int64_t)gridDim.x + (int64_t)atomicAdd(p.work_counter, 1ull);
      w_next = __shfl_sync(0xffffffffu, w_next, 0);
      const int nq = (int)((n + BQ - 1) / BQ);
      const int kv_row = (int)(b0 + (int64_t)it.y * BKV);
      const float* lse_h = p.lsd + (int64_t)h * p.total_rows;
      const float* del_h = p.lsd + ((int64_t)H + h) * p.total_rows;
      wp.wait_warp(v_empty, (item_cnt & 1) ^ 1, 2);
      if (lane == 0) {
        tc::mbar_expect_tx(v_full, L::kTileKV);
        for (int c = 0; c < D / 64; ++c)
          tc::tma_load_3d(smem + L::kV + c * L::kChunkKV, &tm_v, v_full, c * 64, h, kv_row);
      }
      wp.wait_warp(k_empty, (item_cnt & 1) ^ 1, 0);
      if (lane == 0) {
        tc::mbar_expect_tx(k_full, L::kTileKV);
        for (int c = 0; c < D / 64; ++c)
          tc::tma_load_3d(smem + L::kK + c * L::kChunkKV, &tm_k, k_full, c * 64, h, kv_row);
        if (wp.g) wp.trace(50);
      }
      for (int j = 0; j < nq; ++j, ++qd_cnt) {
        const uint32_t s = qd_cnt % L::kStages;
        const int64_t q_row = b0 + (int64_t)j * BQ;
        wp.wait_warp(qd_empty + s, ((qd_cnt / L::kStages) & 1) ^ 1, 1);
        // lse/Delta: rows past the sample are masked by the softmax; rows past the tensor are not copied
        const uint32_t ls = tc::smem_u32(smem + L::kLse + s * L::kLsdBytes);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int t = lane + 32 * u;
          if (q_row + t < p.total_rows) {
            tc::cp_async_4(ls + t * 4, lse_h + q_row + t);
            tc::cp_async_4(ls + (BQ + t) * 4, del_h + q_row + t);
          }
        }
        tc::cp_async_arrive_noinc(qd_full + s);
        if (lane == 0) {
          tc::mbar_expect_tx(qd_full + s, 2 * L::kTileQ);
          uint8_t* qs = smem + L::kQD + s * 2 * L::kTileQ;
          for (int c = 0; c < D / 64; ++c) {
            tc::tma_load_3d(qs + c * L::kChunkQ, &tm_q, qd_full + s, c * 64, h, (int)q_row);
            tc::tma_load_3d(qs + L::kTileQ + c * L::kChunkQ, &tm_do, qd_full + s, c * 64, h, (int)q_row);
          }
        }
      }
    }
    wp.add(7, clock64() - t_role);
    wp.flush();
  } else if (warp == 1 || warp == 2) {
    // ===================================================== MMA issuers
    // Two issuing threads feed the tensor core (each tcgen05.mma blocks its issuer for about one MMA
    // duration, so a single issuer exposes every barrier wait as tensor idle time):
    //   warp 1: S^T_j = K Q_j^T and dP^T_j = V dO_j^T into TMEM score buffer j&1, up to two blocks ahead
    //   warp 2: dV += P^T_j dO_j, dK += dS^T_j Q_j, dQ^T_j = K^T dS^T_j once the softmax published block j
    // They touch disjoint TMEM columns except dQ^T_j, which reuses buffer j&1 only after the softmax
    // consumed it (p_full) and is drained before warp 1 refills that buffer (dq_empty).
    // The whole warp runs the issue loop with warp-uniform operands (they stay in uniform registers);
    // one elected lane issues each MMA / commit. A single-lane loop needs R2UR moves per MMA, which the
    // softmax warps' FFMA/MUFU traffic on the same SM sub-partition slows by ~25% (tools/mma_seq_bench.cu).
    {
      constexpr uint32_t kIdS = tc::idesc_bf16_f32(BKV, BQ, false, false);  // S^T, dP^T
      constexpr uint32_t kIdKV = tc::idesc_bf16_f32(BKV, D, false, true);   // dV, dK
      // dQ^T: M = head_dim rows, run at M = 128 (for D = 64 the upper 64 rows read the next smem chunk and are
      // never drained)
      constexpr uint32_t kIdQ = tc::idesc_bf16_f32(128, BQ, true, true);
      const uint32_t k_base = tc::smem_u32(smem + L::kK), v_base = tc::smem_u32(smem + L::kV);
      const uint32_t ds_base = tc::smem_u32(smem + L::kDS);
      const uint32_t qd_base = tc::smem_u32(smem + L::kQD);
      auto stage_of = [&](uint32_t cnt) { return qd_base + (cnt % L::kStages) * 2 * L::kTileQ; };
      tc::WaitProf wp;
      wp.init(lane == 0 ? p.prof : nullptr, warp == 1 ? 8 : 32);
      const long long t_role = clock64();
      // per-buffer phase parities live in bit b of a register (a runtime-indexed [2] array goes to local memory)
      uint32_t item_cnt = 0, qd_cnt = 0, p_cnt = 0, fill_par = 0;
      Work wk;
      for (bool more = take_item(item_cnt, wk); more; more = take_item(++item_cnt, wk)) {
        const int2 it = wk.it;
        const int64_t n = wk.n;
        const int nq = (int)((n + BQ - 1) / BQ);
        if (warp == 1) {
          wp.wait_warp(k_full, item_cnt & 1, 0);
          wp.wait_warp(v_full, item_cnt & 1, 1);
          for (int j = 0; j < nq; ++j, ++qd_cnt) {
            const int b = j & 1;
            const uint32_t s = qd_cnt % L::kStages;
            wp.wait_warp(qd_full + s, (qd_cnt / L::kStages) & 1, 2);
            wp.wait_warp(pt_free + b, ((fill_par >> b) & 1) ^ 1, 3);  // dV / dK of the block that used b are done
            wp.wait_warp(dq_empty + b, ((fill_par >> b) & 1) ^ 1, 4);  // dQ^T previously written here was drained
            fill_par ^= 1u << b;
            tc::tc_fence_after();
            if (wp.g) wp.trace(56);
            const uint32_t q_base = stage_of(qd_cnt), do_base = q_base + L::kTileQ;
            const uint32_t col = b * 128;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t ka = (kk >> 2) * L::kChunkKV + (kk & 3) * 32;
              const uint32_t kb = (kk >> 2) * L::kChunkQ + (kk & 3) * 32;
              tc::mma_bf16_ss_warp(tmem + col, tc::sw128_desc(k_base + ka, 16, 1024),
                              tc::sw128_desc(q_base + kb, 16, 1024), kIdS, kk > 0);
            }
            if (wp.g) wp.trace(57);
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t ka = (kk >> 2) * L::kChunkKV + (kk & 3) * 32;
              const uint32_t kb = (kk >> 2) * L::kChunkQ + (kk & 3) * 32;
              tc::mma_bf16_ss_warp(tmem + col + 64, tc::sw128_desc(v_base + ka, 16, 1024),
                              tc::sw128_desc(do_base + kb, 16, 1024), kIdS, kk > 0);
            }
            tc::mma_commit_warp(st_full + b);
            if (wp.g) wp.trace(58);
          }
          tc::mma_commit_warp(v_empty);  // this issuer's reads of K and V are done
          tc::mma_commit_warp(k_empty);
        } else {
          wp.wait_warp(dkv_empty, (item_cnt & 1) ^ 1, 1);
          for (int j = 0; j < nq; ++j, ++qd_cnt) {
            wp.wait_warp(p_full, p_cnt & 1, 5);
            const uint32_t pb = p_cnt % kPdsBufs;
            const uint32_t ds_cur = ds_base + pb * (BKV * 128);
            ++p_cnt;
            tc::tc_fence_after();
            const uint32_t q_base = stage_of(qd_cnt), do_base = q_base + L::kTileQ;
            const uint32_t col = (j & 1) * 128;
            if (wp.g) wp.trace(83);
            // dV += P^T dO_j first (TS: A = P^T from TMEM; K-step kk covers queries 16kk..16kk+15, which the
            // softmax half kk/2 packed at columns col + 32(kk/2) + 8(kk&1)), so buffer j&1 frees early
#pragma unroll
            for (int kk = 0; kk < BQ / 16; ++kk)
              tc::mma_bf16_ts_warp(tmem + 256, tmem + col + 32 * (kk >> 1) + 8 * (kk & 1),
                                   tc::sw128_desc(do_base + kk * 2048, L::kChunkQ, 1024), kIdKV, (j > 0 || kk > 0));
            // dQ_j^T = K^T dS^T into the consumed dP^T slot of buffer j&1 (B = dS^T from smem)
#pragma unroll
            for (int kk = 0; kk < BKV / 16; ++kk)
              tc::mma_bf16_ss_warp(tmem + col + 64, tc::sw128_desc(k_base + kk * 2048, L::kChunkKV, 1024),
                                   tc::sw128_desc(ds_cur + kk * 2048, 16, 1024), kIdQ, kk > 0);
            tc::mma_commit_warp(dq_full + (j & 1));
            tc::mma_commit_warp(pds_empty + pb);  // the smem dS^T's only reader is done
            if (j == nq - 1) tc::mma_commit_warp(k_empty);  // the item's last read of K: reload during dK
            if (wp.g) wp.trace(84);
            // dK += dS^T Q_j (TS: A = dS^T from TMEM, packed by the softmax into the S^T columns P^T leaves free:
            // col + 32(kk/2) + 16 + 8(kk&1); B MN-major [64 q x D])
#pragma unroll
            for (int kk = 0; kk < BQ / 16; ++kk)
              tc::mma_bf16_ts_warp(tmem + 384, tmem + col + 32 * (kk >> 1) + 16 + 8 * (kk & 1),
                                   tc::sw128_desc(q_base + kk * 2048, L::kChunkQ, 1024), kIdKV, (j > 0 || kk > 0));
            tc::mma_commit_warp(pt_free + (j & 1));  // P^T and dS^T of buffer j&1 are consumed
            // Q_j, dO_j are no longer needed (warp 1's S/dP_j completed before the softmax published P_j)
            tc::mma_commit_warp(qd_empty + (qd_cnt % L::kStages));
            if (wp.g) wp.trace(82);
          }
          tc::mma_commit_warp(dkv_full);
        }
      }
      wp.add(7, clock64() - t_role);
      wp.flush();
    }
  } else if (warp >= kSmWarp0 && warp < kSmWarp0 + kSmWarps) {
    // ===================================================== P^T / dS^T warps (thread = key row x 32 queries)
    const int tid = threadIdx.x - kSmWarp0 * 32;
    const int wq = warp & 3;                       // TMEM lane quarter
    const int row = wq * 32 + lane;                // key row within the tile
    const int half = (warp - kSmWarp0) >> 2;       // query columns [32 half, 32 half + 32)
    const uint32_t lane_addr = tmem + ((uint32_t)(wq * 32) << 16);
    const uint32_t ds_base = tc::smem_u32(smem + L::kDS);
    const uint32_t lsd = tc::smem_u32(smem + L::kLse);
    uint32_t cons_par = 0, pds_cnt = 0, qd_cnt = 0;  // bit b: phase parity of st_full[b]
    tc::WaitProf wp;
    wp.init(tid == 0 ? p.prof : nullptr, 16);
    const long long t_role = clock64();
    uint32_t ic = 0;
    Work wk;
    for (bool more = take_item(ic, wk); more; more = take_item(++ic, wk)) {
      const int2 it = wk.it;
      const int64_t n = wk.n;
      const int nq = (int)((n + BQ - 1) / BQ);
      const bool row_valid = (int64_t)it.y * BKV + row < wk.nv;
      for (int j = 0; j < nq; ++j, ++qd_cnt) {
        const int b = j & 1;
        const uint32_t s = qd_cnt % L::kStages;
        wp.wait_warp(st_full + b, (cons_par >> b) & 1, 1);
        cons_par ^= 1u << b;
        tc::tc_fence_after();
        uint32_t sr[32], dr[32];
        tc::tmem_ld32(lane_addr + b * 128 + half * 32, sr);
        tc::tmem_ld32(lane_addr + b * 128 + 64 + half * 32, dr);
        // lse/Delta of block j arrived with (Q_j, dO_j); the stage stays valid until p_full (the issuer's
        // qd_empty commit follows the MMAs that consume P_j)
        wp.wait_warp(qd_full + s, (qd_cnt / L::kStages) & 1, 0);
        const uint32_t lb = lsd + (s * 2 * BQ + half * 32) * 4;
        // queries past the sample end (rows of the next sample in the Q tile) and key rows past it get P = 0
        const int64_t qrem = wk.nv - (int64_t)j * BQ - half * 32;
        const int qlim = qrem < 32 ? (qrem > 0 ? (int)qrem : 0) : 32;
        const bool full = __all_sync(0xffffffffu, row_valid && qlim == 32);
        tc::tmem_wait_ld();
        uint32_t pk[16], dk2[16];
        auto body = [&](auto masked) {
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            const float4 l4 = tc::ld_shared_f4(lb + e * 4);
            const float4 d4 = tc::ld_shared_f4(lb + (BQ + e) * 4);
            // lsd holds -lse*log2(e) and -Delta, so each pair is one FFMA2 / FADD2 / FMUL2
            const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
            const float2 x01 = tc::ffma2(make_float2(__uint_as_float(sr[e + 0]), __uint_as_float(sr[e + 1])), sc2,
                                         make_float2(l4.x, l4.y));
            const float2 x23 = tc::ffma2(make_float2(__uint_as_float(sr[e + 2]), __uint_as_float(sr[e + 3])), sc2,
                                         make_float2(l4.z, l4.w));
            float p0 = tc::ex2(x01.x), p1 = tc::ex2(x01.y), p2 = tc::ex2(x23.x), p3 = tc::ex2(x23.y);
            const float2 g01 = tc::fadd2(make_float2(__uint_as_float(dr[e + 0]), __uint_as_float(dr[e + 1])),
                                         make_float2(d4.x, d4.y));
            const float2 g23 = tc::fadd2(make_float2(__uint_as_float(dr[e + 2]), __uint_as_float(dr[e + 3])),
                                         make_float2(d4.z, d4.w));
            const float2 s01 = tc::fmul2(make_float2(p0, p1), g01), s23 = tc::fmul2(make_float2(p2, p3), g23);
            float s0 = s01.x, s1 = s01.y, s2 = s23.x, s3 = s23.y;
            if constexpr (decltype(masked)::value) {  // after the products: masked lanes may hold stale inf/nan
              if (!row_valid || e + 0 >= qlim) p0 = s0 = 0.f;
              if (!row_valid || e + 1 >= qlim) p1 = s1 = 0.f;
              if (!row_valid || e + 2 >= qlim) p2 = s2 = 0.f;
              if (!row_valid || e + 3 >= qlim) p3 = s3 = 0.f;
            }
            pk[e >> 1] = tc::pack_bf16(p0, p1);
            pk[(e >> 1) + 1] = tc::pack_bf16(p2, p3);
            dk2[e >> 1] = tc::pack_bf16(s0, s1);
            dk2[(e >> 1) + 1] = tc::pack_bf16(s2, s3);
          }
        };
        if (full)
          body(std::false_type{});
        else
          body(std::true_type{});
        // P^T (bf16) back over the S^T columns this thread read: the A operand of the dV MMA
        tc::tmem_st16(lane_addr + b * 128 + half * 32, pk);
        tc::tmem_st16(lane_addr + b * 128 + half * 32 + 16, dk2);  // dS^T for the TS-form dK MMA
        const uint32_t pb = pds_cnt % kPdsBufs;
        wp.wait_warp(pds_empty + pb, ((pds_cnt / kPdsBufs) & 1) ^ 1, 2);
        ++pds_cnt;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (p.dbg & 4) break;
          const uint32_t o = tc::sw128_offset(row, half * 4 + u);
          tc::st_shared_v4(ds_base + pb * (BKV * 128) + o, dk2[u * 4], dk2[u * 4 + 1], dk2[u * 4 + 2], dk2[u * 4 + 3]);
        }
        tc::fence_proxy_async_smem();
        tc::tmem_wait_st();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(p_full);
        if (wp.g) wp.trace(66);
      }
    }
    wp.add(7, clock64() - t_role);
    wp.flush();
  } else if (warp >= kDqWarp0) {
    // ===================================================== dQ drain + dK/dV epilogue
    const int tid = threadIdx.x - kDqWarp0 * 32;  // == TMEM lane: head-dim row of dQ^T, key row of dK/dV
    const int wq = warp - kDqWarp0;
    const uint32_t lane_addr = tmem + ((uint32_t)(wq * 32) << 16);
    float* stg = reinterpret_cast<float*>(smem + L::kStg);
    const uint32_t stg_base = tc::smem_u32(stg);
    uint32_t item_cnt = 0, dq_par = 0;  // bit b: phase parity of dq_full[b]
    tc::WaitProf wp;
    wp.init(tid == 0 ? p.prof : nullptr, 24);
    const long long t_role = clock64();
    Work wk;
    const float* kvb = p.lsd + 2 * (int64_t)H * p.total_rows;  // deterministic: per-head maxima
    const uint32_t magic_s = tc::smem_u32(smem + L::kMagic);
    if (DET && H <= L::kMaxMagicHeads) {
      for (int hh = tid; hh < H; hh += 128) tc::st_shared_f32(magic_s + hh * 4, head_magic(kvb, H, hh, p.scale));
      named_bar(2, 128);
    }
    for (bool more = take_item(item_cnt, wk); more; more = take_item(++item_cnt, wk)) {
      const int2 it = wk.it;
      const int h = wk.h;
      const int64_t b0 = wk.b0, n = wk.n;
      const int nq = (int)((n + BQ - 1) / BQ);
      const float mgc = !DET ? 0.f : (H <= L::kMaxMagicHeads ? tc::ld_shared_f32(magic_s + h * 4) : head_magic(kvb, H, h, p.scale));
      for (int j = 0; j < nq; ++j) {
        const int b = j & 1;
        wp.wait_warp(dq_full + b, (dq_par >> b) & 1, 0);
        dq_par ^= 1u << b;
        tc::tc_fence_after();
        const long long t_ld = clock64();
        uint32_t a[32], c2[32];
        tc::tmem_ld32(lane_addr + b * 128 + 64, a);
        tc::tmem_ld32(lane_addr + b * 128 + 96, c2);
        tc::tmem_wait_ld();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(dq_empty + b);
        wp.add(6, clock64() - t_ld);
        // [kStgRows q x D] boxes through two alternating staging buffers, one TMA tensor reduce-add each (the
        // drain fills one buffer while the TMA unit reads the other); rows of padded queries are exactly zero
        // (P = 0 there), so adding them into the next sample's rows is a no-op
        static_assert((BQ / L::kStgRows) % L::kStgBufs == 0, "buffer index must be static per sub-block");
#pragma unroll
        for (int hh = 0; hh < BQ / L::kStgRows; ++hh) {
          const uint32_t sb = stg_base + (hh % L::kStgBufs) * (L::kStgRows * D * L::kAccBytes);
          const long long tb = clock64();
          if (tid == 0) bulk_wait_read<L::kStgBufs - 1>();  // the reduction issued from this buffer has read it
          named_bar(2, 128);
          wp.add(1, clock64() - tb);
#pragma unroll
          for (int q = 0; q < L::kStgRows; q += 2) {  // two rows per paired FFMA2 (+ FADD2 in deterministic mode)
            const int qq = hh * L::kStgRows + q;
            const float2 v = make_float2(__uint_as_float(qq < 32 ? a[qq & 31] : c2[qq & 31]),
                                         __uint_as_float(qq + 1 < 32 ? a[(qq + 1) & 31] : c2[(qq + 1) & 31]));
            float2 x = tc::ffma2(v, make_float2(p.scale, p.scale), make_float2(mgc, mgc));
            if constexpr (DET) x = tc::fadd2(x, make_float2(-mgc, -mgc));  // exact: x on the head's grid
            if (tid < D) {
              tc::st_shared_f32(sb + (q * D + tid) * 4, x.x);
              tc::st_shared_f32(sb + ((q + 1) * D + tid) * 4, x.y);
            }
          }
          tc::fence_proxy_async_smem();
          named_bar(2, 128);
          if (tid == 0 && !(p.dbg & 1)) {
            tensor_reduce_add_3d(&tm_dq, sb, 0, h, (int)(b0 + (int64_t)j * BQ + L::kStgRows * hh));
            bulk_commit();
          }
        }
      }
      // dK / dV for this key tile. A thread holds one key row; rows are 1 KB apart in HBM, so each warp
      // transposes its 32 rows x 64 columns through a private 4 KB slice of the (now idle) dQ staging
      // buffer and writes them back as whole 128-byte lines (four rows per instruction). Per-thread 16-byte
      // row stores would leave every sector half-written and flood the SM's outbound path exactly when the
      // next item's K/V/Q loads are issued.
      wp.wait_warp(dkv_full, item_cnt & 1, 2);
      tc::tc_fence_after();
      {
        const long long tb = clock64();
        if (tid == 0) bulk_wait_read0();  // the last dQ reductions have read the staging buffers
        named_bar(2, 128);
        wp.add(3, clock64() - tb);
        if (wp.g) wp.trace(75);
      }
      const uint32_t xs = stg_base + wq * 4096;  // this warp's [32 rows x 128 B] slice, 16-byte chunks XOR row&7
      const int64_t tile0 = (int64_t)it.y * BKV + wq * 32;  // first key row of this warp (sample-local)
#pragma unroll 1
      for (int which = 0; which < 2; ++which) {
        const uint32_t col = which == 0 ? 256 : 384;
        const float sc = which == 0 ? 1.f : p.scale;
        __nv_bfloat16* dst = (which == 0 ? p.dv : p.dk) + ((b0 + tile0) * H + h) * D;  // this warp's first row
#pragma unroll 1
        for (int half = 0; half < D / 64; ++half) {
#pragma unroll
          for (int g = 0; g < 2; ++g) {  // 32 columns at a time (register budget)
            uint32_t o[32];
            const long long t4 = clock64();
            tc::tmem_ld32(lane_addr + col + half * 64 + g * 32, o);
            tc::tmem_wait_ld();
            wp.add(4, clock64() - t4);
#pragma unroll
            for (int uu = 0; uu < 4; ++uu) {
              const int u = g * 4 + uu;
#define JG_EPI(k) __uint_as_float(o[uu * 8 + (k)]) * sc
              tc::st_shared_v4(xs + lane * 128 + ((u ^ (lane & 7)) << 4), tc::pack_bf16(JG_EPI(0), JG_EPI(1)),
                               tc::pack_bf16(JG_EPI(2), JG_EPI(3)), tc::pack_bf16(JG_EPI(4), JG_EPI(5)),
                               tc::pack_bf16(JG_EPI(6), JG_EPI(7)));
#undef JG_EPI
            }
          }
          __syncwarp();
          const long long t5 = clock64();
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = i * 4 + (lane >> 3), c = lane & 7;  // row within the warp's 32, 16-byte chunk
            const uint4 v = tc::ld_shared_v4u(xs + r * 128 + ((c ^ (r & 7)) << 4));
            if (tile0 + r < n && !(p.dbg & 8)) *reinterpret_cast<uint4*>(dst + (uint32_t)(r * H * D + half * 64 + c * 8)) = v;
          }
          __syncwarp();
          wp.add(5, clock64() - t5);
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(dkv_empty);
      if (wp.g) wp.trace(74);
    }
    if (tid == 0) bulk_wait0();
    wp.add(7, clock64() - t_role);
    wp.flush();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem);
  }
  if (threadIdx.x == 0) work_counters_exit(p.work_counter);
  tc::cta_time_mark(p.prof, 1);
}

// Delta = rowsum(dO * O) per (row, head), zero the dQ accumulator, and write -lse*log2(e) and -Delta into
// lsd[2][H][total_rows] (staged per query block by the main kernel's producer with cp.async; negated so the
// softmax needs one paired FFMA2 / FADD2 per two scores). Deterministic mode (DET) also reads K and V for the
// per-head maxima max|K|, max||V||^2 and max||dO||^2 (lsd tail [3][H], zeroed before the launch) that bound the
// grid-rounded dQ partials.
#ifndef JG_PRO_LD
#define JG_PRO_LD __ldcs
#endif
template <int D, bool DET>
__global__ void __launch_bounds__(256) bwd_prologue_kernel(const __nv_bfloat16* __restrict__ go,
                                                           const __nv_bfloat16* __restrict__ o,
                                                           const __nv_bfloat16* __restrict__ kk,
                                                           const __nv_bfloat16* __restrict__ vv, int64_t units,
                                                           int H, int64_t total_rows, const float* __restrict__ lse,
                                                           float* __restrict__ lsd, void* __restrict__ dq_acc) {
  // LPU lanes per (row, head) unit, 16 bytes of dO and of O per lane; a warp covers UPW units per step and
  // unrolls two steps with every load issued before the reductions (the streaming read is latency-bound
  // with one dependent unit per warp)
  constexpr int LPU = D / 8, UPW = 32 / LPU, kUnroll = 2;
  extern __shared__ unsigned kv_max[];  // DET: [3][H] block-local max|K|, max||V||^2, max||dO||^2 (float bits, >= 0)
  if (DET) {
    for (int i = threadIdx.x; i < 3 * H; i += blockDim.x) kv_max[i] = 0u;
    __syncthreads();
  }
  const int lane = threadIdx.x & 31, sub = lane / LPU, li = lane % LPU;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * (UPW * kUnroll); u0 < units;
       u0 += warps * UPW * kUnroll) {
    uint4 a[kUnroll], b[kUnroll], ka[kUnroll], va[kUnroll];
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
      const int64_t u = u0 + k * UPW + sub;
      a[k] = b[k] = ka[k] = va[k] = make_uint4(0u, 0u, 0u, 0u);
      if (u < units) {
        a[k] = JG_PRO_LD(reinterpret_cast<const uint4*>(go + u * D) + li);  // streamed once
        b[k] = JG_PRO_LD(reinterpret_cast<const uint4*>(o + u * D) + li);
        if (DET) {
          ka[k] = __ldg(reinterpret_cast<const uint4*>(kk + u * D) + li);  // the main kernel reads K, V next
          va[k] = __ldg(reinterpret_cast<const uint4*>(vv + u * D) + li);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) {
      const int64_t u = u0 + k * UPW + sub;
      const __nv_bfloat162* ha = reinterpret_cast<const __nv_bfloat162*>(&a[k]);
      const __nv_bfloat162* hb = reinterpret_cast<const __nv_bfloat162*>(&b[k]);
      float acc = 0.f, nn = 0.f, km = 0.f, vn = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 x = __bfloat1622float2(ha[e]), y = __bfloat1622float2(hb[e]);
        acc = fmaf(x.x, y.x, fmaf(x.y, y.y, acc));
        if (DET) {
          nn = fmaf(x.x, x.x, fmaf(x.y, x.y, nn));
          const float2 kx = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(&ka[k])[e]);
          const float2 vx = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(&va[k])[e]);
          km = fmaxf(km, fmaxf(fabsf(kx.x), fabsf(kx.y)));
          vn = fmaf(vx.x, vx.x, fmaf(vx.y, vx.y, vn));
        }
      }
#pragma unroll
      for (int m = LPU / 2; m > 0; m >>= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, m);
        if (DET) {
          nn += __shfl_xor_sync(0xffffffffu, nn, m);
          km = fmaxf(km, __shfl_xor_sync(0xffffffffu, km, m));
          vn += __shfl_xor_sync(0xffffffffu, vn, m);
        }
      }
      if (u < units) {
        // 8 fp32 / int32 zeros per lane: one 32-byte sector store
        tc::st_global_v8(reinterpret_cast<float*>(dq_acc) + u * D + li * 8, make_uint4(0u, 0u, 0u, 0u),
                         make_uint4(0u, 0u, 0u, 0u));
        if (li == 0) {
          const int64_t r = u / H, h = u - r * H;
          lsd[h * total_rows + r] = -lse[h * total_rows + r] * kLog2e;  // negated: one FFMA2 per pair downstream
          lsd[(H + h) * total_rows + r] = -acc;
          if (DET) {
            atomicMax(kv_max + h, __float_as_uint(km));
            atomicMax(kv_max + H + h, __float_as_uint(vn));
            atomicMax(kv_max + 2 * H + h, __float_as_uint(nn));
          }
        }
      }
    }
  }
  if (DET) {
    __syncthreads();
    unsigned* g = reinterpret_cast<unsigned*>(lsd + 2 * (int64_t)H * total_rows);
    for (int i = threadIdx.x; i < 3 * H; i += blockDim.x)
      if (kv_max[i]) atomicMax(g + i, kv_max[i]);
  }
}

__global__ void __launch_bounds__(256) dq_convert_kernel(const float* __restrict__ acc, __nv_bfloat16* __restrict__ dq,
                                                         int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = reinterpret_cast<const float4*>(acc)[i];
    uint2 r;
    r.x = tc::pack_bf16(v.x, v.y);
    r.y = tc::pack_bf16(v.z, v.w);
    reinterpret_cast<uint2*>(dq)[i] = r;
  }
}

}  // namespace fb

bool attn_sm100_bwd_supported(int head_dim, jg_dtype dt) { return dt == JG_BF16 && (head_dim == 128 || head_dim == 64); }

template <int kD, bool kDet>
static jg_status bwd_launch(const int64_t* off, int64_t total_rows, int H, const void* q, const void* k, const void* v,
                            const void* go, const void* o, const float* lse, void* dq, void* dk, void* dv,
                            float* delta, void* dq_acc, const int2* items, const int64_t* n_items, int64_t max_items,
                            const int64_t* valid, unsigned long long* counters, cudaStream_t st) {
  using L = fb::Smem<kD, kDet>;
  const int sms = device_sm_count();
  const int64_t units = total_rows * H;
  if (kDet) JG_CUDA(cudaMemsetAsync(delta + 2 * (int64_t)H * total_rows, 0, 3 * H * sizeof(float), st));
  fb::bwd_prologue_kernel<kD, kDet><<<(int)std::min<int64_t>((units + 8 * (256 / kD) * 2 - 1) / (8 * (256 / kD) * 2), 32 * sms), 256,
                                      kDet ? 3 * H * sizeof(unsigned) : 0, st>>>(
      (const __nv_bfloat16*)go, (const __nv_bfloat16*)o, (const __nv_bfloat16*)k, (const __nv_bfloat16*)v, units, H,
      total_rows, lse, delta, dq_acc);
  JG_LAUNCHED("bwd_prologue_kernel");
  CUtensorMap mq, mk, mv, mdo;
  if (jg_status rc = make_map(&mq, q, total_rows, H, kD, fb::BQ)) return rc;
  if (jg_status rc = make_map(&mk, k, total_rows, H, kD, fb::BKV)) return rc;
  if (jg_status rc = make_map(&mv, v, total_rows, H, kD, fb::BKV)) return rc;
  if (jg_status rc = make_map(&mdo, go, total_rows, H, kD, fb::BQ)) return rc;
  CUtensorMap mdq;
  if (jg_status rc = make_map_f32(&mdq, dq_acc, total_rows, H, kD, L::kStgRows))
    return rc;
  if (jg_status rc = ensure_smem_attr((const void*)fb::jfa_bwd_sm100_kernel<kD, kDet>, L::kAlloc, "jfa_bwd_sm100_kernel"))
    return rc;
  fb::Params p{off, items, n_items, total_rows, H, delta, dq_acc, (__nv_bfloat16*)dk, (__nv_bfloat16*)dv,
               1.4426950408889634f / sqrtf((float)kD), 1.0f / sqrtf((float)kD), std::getenv("JG_BWD_DBG") ? std::atoi(std::getenv("JG_BWD_DBG")) : 0,
               counters, wait_prof_begin(st), valid};
  int64_t grid = std::min<int64_t>(sms, max_items * H);
  // JG_BWD_MAX_CTAS (tests): a smaller persistent grid changes which CTA runs which item and when
  if (const char* cap = std::getenv("JG_BWD_MAX_CTAS")) grid = std::min<int64_t>(grid, std::atoi(cap));
  grid = std::max<int64_t>(1, grid);
  if (!(p.dbg & 64)) fb::jfa_bwd_sm100_kernel<kD, kDet><<<(int)grid, fb::kThreads, L::kAlloc, st>>>(mq, mk, mv, mdo, mdq, p);
  if (p.dbg & 128) {
    cudaError_t e = cudaStreamSynchronize(st);
    std::fprintf(stderr, "[bwd dbg] main kernel: %s\n", cudaGetErrorString(e));
  }
  JG_LAUNCHED("jfa_bwd_sm100_kernel");
  wait_prof_end(p.prof, st, "bwd",
                {"P.k_empty", "P.qd_empty", "P.v_empty", "P.item_empty", "", "", "", "P.total", "M.k_full", "M.v_full", "M.qd_full",
                 "M.pt_free", "M.dq_empty", "", "", "M.total", "S.qd_full", "S.st_full", "S.pds_empty", "",
                 "", "", "", "S.total", "D.dq_full", "D.stage_bar", "D.dkv_full", "D.epi_read0", "D.epi_tmem", "D.epi_out", "D.tmem_ld", "D.total", "G.unused", "G.dkv_empty", "", "", "", "G.p_full", "", "G.total"});
  const int64_t n4 = units * kD / 4;
  const int cgrid = (int)std::min<int64_t>((n4 + 255) / 256, 32 * sms);
  fb::dq_convert_kernel<<<cgrid, 256, 0, st>>>((const float*)dq_acc, (__nv_bfloat16*)dq, n4);
  JG_LAUNCHED("dq_convert_kernel");
  return JG_OK;
}

jg_status launch_attn_bwd_sm100(const int64_t* off, int64_t batch, int64_t total_rows, int H, int D, const void* q,
                                const void* k, const void* v, const void* go, const void* o, const float* lse,
                                void* dq, void* dk, void* dv, float* delta, void* dq_acc, bool deterministic,
                                const int2* items, const int64_t* n_items, int64_t max_items, const int64_t* valid,
                                unsigned long long* counters, cudaStream_t st) {
  (void)batch;
#define JG_BWD(DD, DET)                                                                                              \
  return bwd_launch<DD, DET>(off, total_rows, H, q, k, v, go, o, lse, dq, dk, dv, delta, dq_acc, items, n_items,   \
                             max_items, valid, counters, st)
  if (D == 128 && deterministic) JG_BWD(128, true);
  if (D == 128) JG_BWD(128, false);
  if (D == 64 && deterministic) JG_BWD(64, true);
  if (D == 64) JG_BWD(64, false);
#undef JG_BWD
  return fail(JG_UNSUPPORTED, "tcgen05 attention backward: head_dim must be 64 or 128");
}

}  // namespace jg
