// attn_sm100.cu — Jagged Flash Attention forward on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Semantics: attention.cpp:172-225 (jagged_flash_attention_forward): per segment, scores
// S = Q_i K_i^T / sqrt(D) over the segment's own keys only, streaming online softmax, O = acc / l,
// lse = m + log l. No padding is materialised: Q/K/V tiles are TMA-loaded straight from row
// offsets[i] + 128*t of the flat [total_rows, H, D] buffers (3-D tensor map D x H x rows, SWIZZLE_128B);
// rows past a segment end belong to the next sample and are masked (keys) or never stored (queries).
//
// Persistent kernel, one CTA per SM, taking (sample, 256-query tile pair) x head items from the device LPT
// work list (layout.cu) through a global counter (the first round is static). A work item holds two 128-row query tiles A and B of
// the same sample (B absent when the sample has an odd number of 128-row tiles); they share every
// K/V block, and their softmax warpgroups ping-pong with the tensor core (FlashAttention-4 style):
//     tensor core:  PV_A(j) S_A(j+1) | PV_B(j) S_B(j+1) | PV_A(j+1) S_A(j+2) | ...
//     softmax A  :          ^ works on S_A(j+1) while the tensor core runs PV_B(j), S_B(j+1)
// Warp roles (10 warps):
//   warps 0-3   softmax warpgroup A (thread = query row = TMEM lane), warps 4-7 warpgroup B:
//               tcgen05.ld S, mask, running max (FMNMX3), exp2 (MUFU + 2 of 8 on the FMA pipe, paired
//               FFMA2/FADD2), P -> TMEM over S (bf16; the A operand of the TS-form PV MMA), lazy O rescale
//               in TMEM (only when the max grows by > 2^8), epilogue O / l -> global (32-byte sector stores)
//               (padded dense_flash_attention mode: keys/rows past each sample's valid length masked)
//   warp 8      TMA producer: Q tiles, then K_0, V_0, K_1, V_1, ... through a ring of smem stages;
//               claims work items and publishes decoded descriptors through an smem ring
//   warp 9      MMA issuer (warp-collective, one elected lane issues)
// TMEM (512 cols): S_A [0,128), O_A [128,256), S_B [256,384), O_B [384,512).
// tcgen05 operations of one thread complete in issue order, so S_X(j+1) completing implies PV_X(j)
// completed: the softmax needs no separate "PV done" barrier inside the key loop.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "internal.h"
#include "tc.cuh"
#include "tma_host.h"

namespace jg {

namespace fa {

constexpr int BM = 128;          // query rows per tile (two tiles per work item)
constexpr int BN = 128;          // keys per block
constexpr int kThreads = 320;    // 10 warps
constexpr int kProducerWarp = 8, kMmaWarp = 9;
// Dynamic work distribution: the producer takes items from a global counter (in LPT order) and hands them
// to the MMA warp and the 8 softmax warps through a small smem ring.
constexpr int kItemSlots = 4;
constexpr int kItemConsumers = 1 + 8;
#ifndef JG_FWD_POLY_EXP
#define JG_FWD_POLY_EXP 2
#endif
constexpr int kPolyExp = JG_FWD_POLY_EXP;  // of every 8 exponentials, this many run on the FMA pipe (ex2_poly)
constexpr float kRescaleThreshold = 8.0f;  // log2 units: rescale O only when the max grows by > 2^8

template <int D>
struct Smem {
  static constexpr int kChunk = BM * 128;               // one [128 rows x 64] bf16 SW128 chunk = 16 KB
  static constexpr int kChunks = D / 64;
  static constexpr int kTile = kChunks * kChunk;        // 128 x D bf16
  static constexpr int kStages = D == 128 ? 5 : 8;      // K/V ring (P lives in TMEM, not smem)
  static constexpr int kQ = 0;                           // Q_A, Q_B
  static constexpr int kKV = kQ + 2 * kTile;
  static constexpr int kBar = kKV + kStages * kTile;
  // q_full, q_empty, kv_full[S], kv_empty[S], s_full[2], p_full[2], o_done[2], o_empty[2], tmem slot
  static constexpr int kNumBars = 2 + 2 * kStages + 8 + 1 + 2 * kItemSlots;
  static constexpr int kItemRing = (kBar + kNumBars * 8 + 16 + 15) & ~15;  // kItemSlots x 48-byte descriptors
  static constexpr int kBytes = kItemRing + kItemSlots * 48;
  static constexpr int kAlloc = kBytes + 1024;          // manual 1 KB alignment
  static_assert(kAlloc <= 232448, "exceeds the 227 KB dynamic shared memory limit");
};

struct Params {
  const int64_t* off;
  const int2* items;  // (sample, tile pair) LPT list
  const int64_t* n_items;
  int64_t batch, total_rows;
  int H;
  __nv_bfloat16* out;
  float* lse;
  float scale_log2;
  unsigned long long* prof;  // JG_WAIT_PROF counters (producer 0-7, MMA 8-15, softmax 16-23)
  unsigned long long* work_counter;  // [2] self-resetting (internal.h work_counters_exit); items beyond the first round
  int dbg;                   // JG_FWD_DBG (diagnostic, results invalid): 1 = softmax publishes P without computing
  const int64_t* valid;      // padded mode (dense_flash_attention): per-sample valid length <= segment length, or
                             // nullptr. Keys past it are masked, rows past it get zeros and lse = -inf.
  const int64_t* q_off;      // cross mode (fused feature_interaction): query segments [q_off[i], q_off[i+1]) over
                             // the keys of sample i (`off`), or nullptr (self-attention). Samples without keys
                             // produce zero rows. total_rows then counts query rows; lse may be nullptr.
};

struct Item {
  int64_t b0, n;      // key segment
  int h, nkv, q_row;  // q_row: first row of tile A
  int nv;             // valid keys (== n except in padded mode)
  int store_end;      // query rows [q_row, store_end) are written ...
  int valid_end;      // ... and those below valid_end hold attention (the others zero, lse = -inf)
  bool has_b;
  int pk_i0, pk_cnt;  // packed item (jagged mode): samples [pk_i0, pk_i0 + pk_cnt) share tile A and key block 0,
                      // each query row attending only its own sample's keys; pk_cnt = 0 otherwise
};

__device__ __forceinline__ Item load_item(const Params& p, int64_t w) {
  const int2 it = p.items[w / p.H];
  Item r;
  r.h = (int)(w % p.H);
  r.pk_i0 = r.pk_cnt = 0;
  if (it.y < 0) {  // (first sample, -count): consecutive short samples inside one 128-row window (layout.cu)
    r.pk_i0 = it.x;
    r.pk_cnt = -it.y;
    r.b0 = p.off[it.x];
    r.n = p.off[it.x + r.pk_cnt] - r.b0;  // <= 128
    r.nkv = 1;
    r.nv = (int)r.n;
    r.q_row = (int)r.b0;
    r.has_b = false;
    r.store_end = r.valid_end = (int)(r.b0 + r.n);
    return r;
  }
  r.b0 = p.off[it.x];
  r.n = p.off[it.x + 1] - r.b0;
  r.nkv = (int)((r.n + BN - 1) / BN);
  r.nv = (int)(p.valid ? (p.valid[it.x] < r.n ? p.valid[it.x] : r.n) : r.n);
  if (it.y & (1 << 30)) {  // single 128-row query tile (short batches: layout.cu work list)
    const int t = it.y & ~(1 << 30);
    r.q_row = (int)(r.b0 + (int64_t)t * BM);
    r.has_b = false;
    r.store_end = (int)(r.b0 + r.n);
    r.valid_end = (int)(r.b0 + r.nv);
  } else if (p.q_off) {
    const int64_t qb0 = p.q_off[it.x], nq = p.q_off[it.x + 1] - qb0;
    r.q_row = (int)(qb0 + (int64_t)it.y * 2 * BM);
    r.has_b = (int64_t)it.y * 2 * BM + BM < nq;
    r.store_end = (int)(qb0 + nq);
    r.valid_end = r.n > 0 ? r.store_end : 0;
  } else {
    r.q_row = (int)(r.b0 + (int64_t)it.y * 2 * BM);
    r.has_b = (int64_t)it.y * 2 * BM + BM < r.n;
    r.store_end = (int)(r.b0 + r.n);
    r.valid_end = (int)(r.b0 + r.nv);
  }
  return r;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    jfa_fwd_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v, Params p) {
  using L = Smem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* kv_full = bars + 2;
  uint64_t* kv_empty = kv_full + L::kStages;
  uint64_t* s_full = kv_empty + L::kStages;  // [2] per tile
  uint64_t* p_full = s_full + 2;             // [2]
  uint64_t* o_done = p_full + 2;             // [2] last PV of an item
  uint64_t* o_empty = o_done + 2;            // [2] epilogue drained O
  uint64_t* item_full = o_empty + 2;  // [kItemSlots]
  uint64_t* item_empty = item_full + kItemSlots;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(item_empty + kItemSlots);
  // ring slot: (b0 lo, b0 hi, n, q_row) (h, nkv, has_b, end) — the producer's decoded item, so the other
  // roles never touch the work list or the offsets
  const uint32_t item_ring = tc::smem_u32(smem + L::kItemRing);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    tc::mbar_init(q_full, 1);
    tc::mbar_init(q_empty, 1);
    for (int s = 0; s < L::kStages; ++s) {
      tc::mbar_init(kv_full + s, 1);
      tc::mbar_init(kv_empty + s, 1);
    }
    for (int t = 0; t < 2; ++t) {
      tc::mbar_init(s_full + t, 1);
      tc::mbar_init(p_full + t, 4);
      tc::mbar_init(o_done + t, 1);
      tc::mbar_init(o_empty + t, 4);
    }
    for (int s = 0; s < kItemSlots; ++s) {
      tc::mbar_init(item_full + s, 1);
      tc::mbar_init(item_empty + s, kItemConsumers);
    }
    tc::fence_barrier_init();
  }
  if (warp == kProducerWarp && lane == 0) {
    tc::tma_prefetch(&tm_q);
    tc::tma_prefetch(&tm_k);
    tc::tma_prefetch(&tm_v);
  }
  tc::cta_time_mark(p.prof, 0);
  if (warp == kMmaWarp) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t n_work = *p.n_items * p.H;
  // a consumer warp's next work index (the producer publishes n_work as the end marker)
  auto take_item = [&](uint32_t ic, Item& it) -> bool {
    const uint32_t s = ic % kItemSlots;
    tc::mbar_wait(item_full + s, (ic / kItemSlots) & 1);
    const uint4 a = tc::ld_shared_v4u(item_ring + s * 48), b = tc::ld_shared_v4u(item_ring + s * 48 + 16),
                c = tc::ld_shared_v4u(item_ring + s * 48 + 32);
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(item_empty + s);
    it.b0 = (int64_t)(((uint64_t)a.y << 32) | a.x);
    it.n = (int)a.z;
    it.q_row = (int)a.w;
    it.h = (int)b.x;
    it.nkv = (int)b.y;
    it.has_b = (b.z & 1) != 0;
    it.nv = (int)b.w;
    it.store_end = (int)c.x;
    it.valid_end = (int)c.y;
    it.pk_i0 = (int)c.z;
    it.pk_cnt = (int)c.w;
    return (b.z >> 1) == 0;
  };

  if (warp == kProducerWarp) {
    // ===================================================== TMA producer
    if (lane == 0) {
      tc::WaitProf wp;
      wp.init(p.prof, 0);
      const long long t_role = clock64();
      uint32_t kv_cnt = 0, item_cnt = 0, q_cnt = 0;  // q_cnt: items with keys (cross mode may have none)
      int64_t w_next = blockIdx.x;  // first round static, then the global counter (LPT order)
      for (;; ++item_cnt) {
        const int64_t w = w_next < n_work ? w_next : n_work;
        Item it{};
        if (w < n_work) it = load_item(p, w);
        const uint32_t slot = item_cnt % kItemSlots;
        wp.wait(item_empty + slot, ((item_cnt / kItemSlots) & 1) ^ 1, 2);
        tc::st_shared_v4(item_ring + slot * 48, (uint32_t)it.b0, (uint32_t)((uint64_t)it.b0 >> 32), (uint32_t)it.n,
                         (uint32_t)it.q_row);
        tc::st_shared_v4(item_ring + slot * 48 + 16, (uint32_t)it.h, (uint32_t)it.nkv,
                         (it.has_b ? 1u : 0u) | (w >= n_work ? 2u : 0u), (uint32_t)it.nv);
        tc::st_shared_v4(item_ring + slot * 48 + 32, (uint32_t)it.store_end, (uint32_t)it.valid_end, (uint32_t)it.pk_i0,
                         (uint32_t)it.pk_cnt);
        tc::mbar_arrive(item_full + slot);
        if (w >= n_work) break;
        // the next item is claimed once this item's loads are issued (the ring blocks the producer until the
        // consumers are within a few stages of the item's end), not when it starts: with about one item per CTA
        // (short batches) an early claim hands the second-round items to CTAs still busy with long first items
        if (it.nkv == 0) {  // cross mode, sample without keys: the softmax warps write zeros
          w_next = (int64_t)gridDim.x + (int64_t)atomicAdd(p.work_counter, 1ull);
          continue;
        }
        wp.wait(q_empty, (q_cnt++ & 1) ^ 1, 0);
        tc::mbar_expect_tx(q_full, (it.has_b ? 2 : 1) * L::kTile);
        for (int t = 0; t < (it.has_b ? 2 : 1); ++t)
          for (int c = 0; c < L::kChunks; ++c)
            tc::tma_load_3d(smem + L::kQ + t * L::kTile + c * L::kChunk, &tm_q, q_full, c * 64, it.h,
                            it.q_row + t * BM);
        for (int j = 0; j < 2 * it.nkv; ++j) {  // K_0, V_0, K_1, V_1, ...
          const uint32_t s = kv_cnt % L::kStages;
          wp.wait(kv_empty + s, ((kv_cnt / L::kStages) & 1) ^ 1, 1);
          tc::mbar_expect_tx(kv_full + s, L::kTile);
          uint8_t* dst = smem + L::kKV + s * L::kTile;
          const int row = (int)(it.b0 + (int64_t)(j >> 1) * BN);
          const CUtensorMap* tm = (j & 1) ? &tm_v : &tm_k;
          for (int c = 0; c < L::kChunks; ++c) tc::tma_load_3d(dst + c * L::kChunk, tm, kv_full + s, c * 64, it.h, row);
          ++kv_cnt;
        }
        w_next = (int64_t)gridDim.x + (int64_t)atomicAdd(p.work_counter, 1ull);
      }
      wp.add(7, clock64() - t_role);
      wp.flush();
    }
  } else if (warp == kMmaWarp) {
    // ===================================================== MMA issuer
    // warp-collective: operands stay warp-uniform (uniform registers) and one elected lane issues; a
    // single-lane loop pays per-MMA R2UR moves that the softmax warps' traffic slows (tools/mma_seq_bench.cu)
    {
      constexpr uint32_t kIdescS = tc::idesc_bf16_f32(BM, BN, false, false);
      constexpr uint32_t kIdescO = tc::idesc_bf16_f32(BM, D, false, true);
      const uint32_t q_base = tc::smem_u32(smem + L::kQ);
      const uint32_t kv_base = tc::smem_u32(smem + L::kKV);
      tc::WaitProf wp;
      wp.init(lane == 0 ? p.prof : nullptr, 8);
      const long long t_role = clock64();
      uint32_t kv_cnt = 0, item_cnt = 0, q_cnt = 0, p_cnt[2] = {0, 0}, o_use[2] = {0, 0};
      auto next_stage = [&]() {
        const uint32_t s = kv_cnt % L::kStages;
        wp.wait_warp(kv_full + s, (kv_cnt / L::kStages) & 1, 2);
        ++kv_cnt;
        tc::tc_fence_after();
        return s;
      };
      auto issue_s = [&](int t, uint32_t k_stage) {
        const long long t0 = clock64();
        const uint32_t qa = q_base + t * L::kTile, ka = kv_base + k_stage * L::kTile;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t koff = (kk >> 2) * L::kChunk + (kk & 3) * 32;
          tc::mma_bf16_ss_warp(tmem + t * 256, tc::sw128_desc(qa + koff, 16, 1024), tc::sw128_desc(ka + koff, 16, 1024),
                          kIdescS, kk > 0);
        }
        wp.add(5, clock64() - t0);
        wp.add(6, D / 16);
        tc::mma_commit_warp(s_full + t);
      };
      auto issue_pv = [&](int t, uint32_t v_stage, int j) {
        const long long t0 = clock64();
        const uint32_t va = kv_base + v_stage * L::kTile;
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
          // A = P_t from TMEM (bf16 packed two per column over S_t's first 64 columns: keys 16kk.. at
          // column 8kk); B = V [128 keys x D] MN-major (LBO = next 64-wide D chunk)
          tc::mma_bf16_ts_warp(tmem + t * 256 + 128, tmem + t * 256 + kk * 8,
                               tc::sw128_desc(va + kk * 16 * 128, L::kChunk, 1024), kIdescO, (j > 0 || kk > 0));
        }
        wp.add(5, clock64() - t0);
        wp.add(6, BN / 16);
      };
      Item it;
      for (bool more = take_item(item_cnt, it); more; more = take_item(++item_cnt, it)) {
        const long long t_li = clock64();
        const int nt = it.has_b ? 2 : 1;
        wp.add(1, clock64() - t_li);
        if (it.nkv == 0) continue;
        wp.wait_warp(q_full, q_cnt++ & 1, 0);
        uint32_t ks = next_stage();  // K_0
        for (int t = 0; t < nt; ++t) issue_s(t, ks);
        tc::mma_commit_warp(kv_empty + ks);
        if (it.nkv == 1) tc::mma_commit_warp(q_empty);  // Q is only read by S MMAs: the next Q loads now
        for (int j = 0; j < it.nkv; ++j) {
          const uint32_t vs = next_stage();  // V_j
          const bool more = j + 1 < it.nkv;
          uint32_t kn = 0;
          for (int t = 0; t < nt; ++t) {
            wp.wait_warp(p_full + t, p_cnt[t] & 1, 4);  // softmax t wrote P_t(j) (and finished reading S_t(j))
            ++p_cnt[t];
            if (j == 0) {  // the previous item that used tile t has drained O_t
              wp.wait_warp(o_empty + t, (o_use[t] & 1) ^ 1, 3);
              ++o_use[t];
            }
            tc::tc_fence_after();
            issue_pv(t, vs, j);
            if (!more) tc::mma_commit_warp(o_done + t);
            if (more) {
              if (t == 0) kn = next_stage();  // K_{j+1}
              issue_s(t, kn);
            }
          }
          tc::mma_commit_warp(kv_empty + vs);
          if (more) tc::mma_commit_warp(kv_empty + kn);
          if (j + 2 == it.nkv) tc::mma_commit_warp(q_empty);  // after the item's last S MMAs
        }
      }
      wp.add(7, clock64() - t_role);
      wp.flush();
    }
  } else {
    // ===================================================== softmax warpgroups A (warps 0-3), B (4-7)
    const int t = warp >> 2;                    // tile
    const int wq = warp & 3;                    // TMEM lane quarter
    const int row = wq * 32 + lane;             // query row within the tile == TMEM lane
    const uint32_t s_addr = tmem + ((uint32_t)(wq * 32) << 16) + t * 256;
    const uint32_t o_addr = s_addr + 128;
    uint32_t s_cnt = 0, done_cnt = 0;
    tc::WaitProf wp;
    wp.init(row == 0 && t == 0 ? p.prof : nullptr, 16);
    const long long t_role = clock64();
    uint32_t ic = 0;
    Item it;
    for (bool more = take_item(ic, it); more; more = take_item(++ic, it)) {
      if (t == 1 && !it.has_b) continue;
      if (it.nkv == 0) {  // cross mode, sample without keys: zero rows (no TMEM or barrier traffic)
        const int arow = it.q_row + t * BM + row;
        if (arow < it.store_end) {
          uint4* orow = reinterpret_cast<uint4*>(p.out + ((int64_t)arow * p.H + it.h) * D);
#pragma unroll
          for (int c = 0; c < D / 8; ++c) orow[c] = make_uint4(0u, 0u, 0u, 0u);
          if (p.lse) p.lse[(int64_t)it.h * p.total_rows + arow] = -INFINITY;
        }
        continue;
      }
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < it.nkv; ++j) {
        wp.wait(s_full + t, s_cnt & 1, 0);
        ++s_cnt;
        tc::tc_fence_after();
        const long long t_sm = clock64();
        if (p.dbg & 1) {
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(p_full + t);
          continue;
        }
        const int64_t rem = (int64_t)it.nv - (int64_t)j * BN;  // valid keys left (<= 0: block fully masked)
        // warp-uniform: a segment's last key block (or padded-mode masked blocks, or a packed item)
        const bool partial = rem < BN || it.pk_cnt > 0;
        // pass 1: raw-score row max over TMEM in 32-column chunks, 8 independent chains
        float m8[8] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY};
        if (!partial) {
          // two 32-column loads in flight per wait
#pragma unroll
          for (int c = 0; c < BN / 32; c += 2) {
            uint32_t r[2][32];
            tc::tmem_ld32(s_addr + c * 32, r[0]);
            tc::tmem_ld32(s_addr + c * 32 + 32, r[1]);
            tc::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 64; e += 2)  // FMNMX3: two scores per instruction
              m8[(e >> 1) & 7] = tc::fmax3(m8[(e >> 1) & 7], __uint_as_float(r[e >> 5][e & 31]),
                                           __uint_as_float(r[e >> 5][(e & 31) + 1]));
          }
        } else {
          // last key block of the segment: write -inf over the keys of the next sample back into TMEM so
          // the exp pass needs no masking (exp2(-inf) = 0); keys [lo, hi) stay
          int lo = 0, hi = rem > 0 ? (int)rem : 0;
          if (it.pk_cnt > 0) {
            // packed item (one key block): this row's own sample's keys (block-diagonal mask). The pack's
            // offsets are read once per warp and scanned with shuffles; rows past the pack keep [0, n).
            int k = 0;
            for (int c0 = 1; c0 <= it.pk_cnt; c0 += 32) {
              const int ov = c0 + lane <= it.pk_cnt ? (int)(p.off[it.pk_i0 + c0 + lane] - it.b0) : 0x7fffffff;
#pragma unroll 8
              for (int jj = 0; jj < 32; ++jj) k += __shfl_sync(0xffffffffu, ov, jj) <= row ? 1 : 0;
            }
            if (k < it.pk_cnt) {
              lo = (int)(p.off[it.pk_i0 + k] - it.b0);
              hi = (int)(p.off[it.pk_i0 + k + 1] - it.b0);
            } else {
              hi = (int)it.n;
            }
          }
#pragma unroll
          for (int c = 0; c < BN / 32; ++c) {
            uint32_t r[32];
            tc::tmem_ld32(s_addr + c * 32, r);
            tc::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              r[e] = (c * 32 + e >= lo && c * 32 + e < hi) ? r[e] : __float_as_uint(-INFINITY);
              m8[e & 7] = fmaxf(m8[e & 7], __uint_as_float(r[e]));
            }
            tc::tmem_st32(s_addr + c * 32, r);
          }
          tc::tmem_wait_st();
        }
        const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                               fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7]))) * p.scale_log2;
        float alpha = 1.f;
        const bool rescale = j > 0 && mx > m + kRescaleThreshold;
        if (j == 0 || rescale) {
          alpha = j == 0 ? 0.f : tc::ex2(m - mx);
          m = mx;
        }
        // O_t is stable here: PV_t(j-1) completed before S_t(j) (in-order tcgen05 completion). Warp-uniform
        // (tcgen05.ld/st are .sync.aligned, so every lane takes part): rows without a rescale scale by 1
        if (__any_sync(0xffffffffu, rescale)) {
          const float a = rescale ? alpha : 1.f;
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            tc::tmem_ld32(o_addr + c * 32, o);
            tc::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * a);
            tc::tmem_st32(o_addr + c * 32, o);
          }
          tc::tmem_wait_st();
        }
        // pass 2: P = exp2(S*scale - m) as bf16 back into TMEM over S_t's first 64 columns (the A operand of
        // the PV MMA): chunk c (keys 32c..32c+31) packs into columns 16c..16c+15, which this thread has
        // already read (they belong to chunks <= c)
        float r8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        // software-pipelined: chunk c+1's TMEM load is in flight while chunk c is exponentiated
        uint32_t r[2][32];
        tc::tmem_ld32(s_addr, r[0]);
        tc::tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
          if (c + 1 < BN / 32) tc::tmem_ld32(s_addr + (c + 1) * 32, r[(c + 1) & 1]);
          uint32_t pk[16];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            float pv[8];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {  // FFMA2 / FADD2: two scores per instruction
              const float2 x = tc::ffma2(make_float2(__uint_as_float(r[c & 1][u * 8 + e]),
                                                     __uint_as_float(r[c & 1][u * 8 + e + 1])),
                                         make_float2(p.scale_log2, p.scale_log2), make_float2(-m, -m));
              if (e + 2 <= 8 - kPolyExp) {
                pv[e] = tc::ex2(x.x);
                pv[e + 1] = tc::ex2(x.y);
              } else {
                const float2 y = tc::ex2_poly2(x);
                pv[e] = y.x;
                pv[e + 1] = y.y;
              }
              const float2 acc = tc::fadd2(make_float2(r8[e], r8[e + 1]), make_float2(pv[e], pv[e + 1]));
              r8[e] = acc.x;
              r8[e + 1] = acc.y;
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) pk[u * 4 + e] = tc::pack_bf16(pv[2 * e], pv[2 * e + 1]);
          }
          tc::tmem_st16(s_addr + c * 16, pk);
          if (c + 1 < BN / 32) tc::tmem_wait_ld();
        }
        l = l * alpha + (((r8[0] + r8[1]) + (r8[2] + r8[3])) + ((r8[4] + r8[5]) + (r8[6] + r8[7])));
        tc::tmem_wait_st();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(p_full + t);
        wp.add(3, clock64() - t_sm);
        wp.add(4, 1);
      }
      // epilogue: last PV of the item, normalise, store
      wp.wait(o_done + t, done_cnt & 1, 2);
      ++done_cnt;
      tc::tc_fence_after();
      const int64_t arow = (int64_t)it.q_row + t * BM + row;  // absolute query row
      const bool store = arow < it.store_end;
      const bool row_ok = arow < it.valid_end;  // padded mode: rows past the valid length are zero, lse = -inf
      const float inv_l = row_ok ? 1.f / l : 0.f;  // with o zeroed below: exact zeros even when l is NaN
      __nv_bfloat16* orow = p.out + (arow * p.H + it.h) * D;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o[32];
        tc::tmem_ld32(o_addr + c * 32, o);
        tc::tmem_wait_ld();
        if (!row_ok) {  // NaN-safe zeros (a segment with no valid key has m = -inf)
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = 0u;
        }
        if (store) {
          uint4 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            v[u].x = tc::pack_bf16(__uint_as_float(o[u * 8 + 0]) * inv_l, __uint_as_float(o[u * 8 + 1]) * inv_l);
            v[u].y = tc::pack_bf16(__uint_as_float(o[u * 8 + 2]) * inv_l, __uint_as_float(o[u * 8 + 3]) * inv_l);
            v[u].z = tc::pack_bf16(__uint_as_float(o[u * 8 + 4]) * inv_l, __uint_as_float(o[u * 8 + 5]) * inv_l);
            v[u].w = tc::pack_bf16(__uint_as_float(o[u * 8 + 6]) * inv_l, __uint_as_float(o[u * 8 + 7]) * inv_l);
          }
          tc::st_global_v8(orow + c * 32, v[0], v[1]);  // whole 32-byte sectors (rows are 1 KB apart)
          tc::st_global_v8(orow + c * 32 + 16, v[2], v[3]);
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(o_empty + t);
      if (store && p.lse)
        p.lse[(int64_t)it.h * p.total_rows + arow] = row_ok ? (m + __log2f(l)) * 0.6931471805599453f : -INFINITY;
    }
    wp.add(7, clock64() - t_role);
    wp.flush();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem);
  }
  if (threadIdx.x == 0) work_counters_exit(p.work_counter);
  tc::cta_time_mark(p.prof, 1);
}

}  // namespace fa

// ------------------------------------------------------------------ host side
bool attn_sm100_supported(int head_dim, jg_dtype dt) {
  return dt == JG_BF16 && (head_dim == 64 || head_dim == 128);
}

template <int D>
static jg_status fwd_launch(const int64_t* off, int64_t batch, int64_t total_rows, int H, const void* q, const void* k,
                            const void* v, void* out, float* lse, const int2* items, const int64_t* n_items,
                            int64_t max_items, const int64_t* valid, const int64_t* q_off, int64_t q_rows,
                            unsigned long long* counter, cudaStream_t st) {
  using L = fa::Smem<D>;
  CUtensorMap mq, mk, mv;
  if (jg_status rc = make_map(&mq, q, q_off ? q_rows : total_rows, H, D, 128)) return rc;
  if (jg_status rc = make_map(&mk, k, total_rows, H, D, 128)) return rc;
  if (jg_status rc = make_map(&mv, v, total_rows, H, D, 128)) return rc;
  if (jg_status rc = ensure_smem_attr((const void*)fa::jfa_fwd_sm100_kernel<D>, L::kAlloc, "jfa_fwd_sm100_kernel"))
    return rc;
  fa::Params p{off, items, n_items, batch, q_off ? q_rows : total_rows, H, (__nv_bfloat16*)out, lse,
               1.4426950408889634f / sqrtf((float)D), wait_prof_begin(st), counter,
               std::getenv("JG_FWD_DBG") ? std::atoi(std::getenv("JG_FWD_DBG")) : 0, valid, q_off};
  const int64_t work = max_items * H;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(device_sm_count(), work));
  fa::jfa_fwd_sm100_kernel<D><<<grid, fa::kThreads, L::kAlloc, st>>>(mq, mk, mv, p);
  const cudaError_t launch_err = cudaGetLastError();
  if (launch_err != cudaSuccess) return cuda_status(launch_err, "jfa_fwd_sm100_kernel");
  count_launch();
  wait_prof_end(p.prof, st, "fwd",
                {"P.q_empty", "P.kv_empty", "P.item_empty", "", "", "", "", "P.total", "M.q_full", "M.load_item", "M.kv_full", "M.o_empty",
                 "M.p_full", "M.issue_cyc", "M.n_mma(x1e-2%)", "M.total", "S.s_full", "", "S.o_done", "S.compute", "S.blocks(x1e-2%)", "", "", "S.total"});
  return JG_OK;
}

// items: (sample, 256-row tile pair) LPT work list (schedule tile 256)
jg_status launch_attn_fwd_sm100(const int64_t* off, int64_t batch, int64_t total_rows, int H, int D, const void* q,
                                const void* k, const void* v, void* out, float* lse, const int2* items,
                                const int64_t* n_items, int64_t max_items, const int64_t* valid,
                                unsigned long long* counters, cudaStream_t st, const int64_t* q_off, int64_t q_rows) {
  if (D == 128)
    return fwd_launch<128>(off, batch, total_rows, H, q, k, v, out, lse, items, n_items, max_items, valid, q_off, q_rows,
                           counters, st);
  if (D == 64)
    return fwd_launch<64>(off, batch, total_rows, H, q, k, v, out, lse, items, n_items, max_items, valid, q_off, q_rows,
                          counters, st);
  return fail(JG_UNSUPPORTED, "tcgen05 attention: head_dim must be 64 or 128");
}

}  // namespace jg
