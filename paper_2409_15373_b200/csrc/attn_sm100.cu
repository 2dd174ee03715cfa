// attn_sm100.cu — Jagged Flash Attention forward on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Semantics: attention.cpp:172-225 (jagged_flash_attention_forward): per segment, scores
// S = Q_i K_i^T / sqrt(D) over the segment's own keys only, streaming online softmax, O = acc / l,
// lse = m + log l. No padding is materialised: Q/K/V tiles are TMA-loaded straight from row
// offsets[i] + 128*t of the flat [total_rows, H, D] buffers (3-D tensor map D x H x rows, SWIZZLE_128B);
// rows past a segment end belong to the next sample and are masked (keys) or never stored (queries).
//
// Persistent kernel, one CTA per SM, walking the device LPT work list (layout.cu) of
// (sample, 128-query tile) items x heads. Warp roles:
//   warp 0      TMA producer: Q tile, then K_0, K_1, V_0, K_2, V_1, ... through a ring of smem stages
//               (exactly the order the MMA warp consumes them)
//   warp 1      MMA issuer (one thread): S_j = Q K_j^T into one of two TMEM score buffers, O += P_j V_j
//   warps 4-7   softmax warpgroup (thread = query row = TMEM lane): tcgen05.ld S_j, mask, running max,
//               exp2, P_j -> smem (bf16, SWIZZLE_128B K-major), lazy O rescale in TMEM (only when the
//               max grows by > 2^8), epilogue O / l -> global bf16 and lse -> global fp32.
// TMEM: S buffer 0 at col 0, S buffer 1 at col 128, O at col 256 (D fp32 columns).
// Overlap: S_{j+1} runs on the tensor core while the softmax warps work on S_j.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "internal.h"
#include "tc.cuh"
#include "tma_host.h"

namespace jg {

namespace fa {

constexpr int BM = 128;          // query rows per tile
constexpr int BN = 128;          // keys per block
constexpr int kThreads = 256;    // 8 warps
constexpr int kSoftmaxWarp0 = 4; // warps 4..7
constexpr float kRescaleThreshold = 8.0f;  // log2 units: rescale O only when the max grows by > 2^8

template <int D>
struct Smem {
  static constexpr int kChunk = BM * 64 * 2;            // one [128 x 64] bf16 SW128 chunk = 16 KB
  static constexpr int kChunks = D / 64;
  static constexpr int kTile = kChunks * kChunk;        // 128 x D bf16
  static constexpr int kStages = D == 128 ? 4 : 8;      // K/V ring
  static constexpr int kQ = 0;
  static constexpr int kP = kQ + kTile;                  // 128 x 128 bf16 = 32 KB
  static constexpr int kKV = kP + 2 * kChunk;
  static constexpr int kBar = kKV + kStages * kTile;
  // barriers: q_full, q_empty, kv_full[S], kv_empty[S], s_full[2], s_empty[2], p_full, o_done, o_empty, tmem slot
  static constexpr int kNumBars = 2 + 2 * kStages + 4 + 3;
  static constexpr int kBytes = kBar + kNumBars * 8 + 16;
  static constexpr int kAlloc = kBytes + 1024;          // manual 1 KB alignment
};

struct Params {
  const int64_t* off;
  const int2* items;
  const int64_t* n_items;
  int64_t batch, total_rows;
  int H;
  __nv_bfloat16* out;
  float* lse;
  float scale_log2;
  unsigned long long* prof;  // JG_WAIT_PROF counters (producer 0-7, MMA 8-15, softmax 16-23)
};

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
  uint64_t* s_full = kv_empty + L::kStages;  // [2]
  uint64_t* s_empty = s_full + 2;            // [2]
  uint64_t* p_full = s_empty + 2;
  uint64_t* o_done = p_full + 1;
  uint64_t* o_empty = o_done + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    tc::mbar_init(q_full, 1);
    tc::mbar_init(q_empty, 1);
    for (int s = 0; s < L::kStages; ++s) {
      tc::mbar_init(kv_full + s, 1);
      tc::mbar_init(kv_empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(s_full + b, 1);
      tc::mbar_init(s_empty + b, 4);
    }
    tc::mbar_init(p_full, 4);
    tc::mbar_init(o_done, 1);
    tc::mbar_init(o_empty, 4);
    tc::fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tm_q);
    tc::tma_prefetch(&tm_k);
    tc::tma_prefetch(&tm_v);
  }
  if (warp == 1) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int64_t n_items = *p.n_items * p.H;
  const int H = p.H;

  if (warp == 0) {
    // ===================================================== TMA producer
    if (lane == 0) {
      uint32_t kv_cnt = 0, item_cnt = 0;
      tc::WaitProf wp;
      wp.init(p.prof, 0);
      const long long t_role = clock64();
      for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x, ++item_cnt) {
        const int2 it = p.items[w / H];
        const int h = (int)(w % H);
        const int64_t b0 = p.off[it.x], n = p.off[it.x + 1] - b0;
        const int nkv = (int)((n + BN - 1) / BN);
        const int q_row = (int)(b0 + (int64_t)it.y * BM);
        wp.wait(q_empty, (item_cnt & 1) ^ 1, 0);
        tc::mbar_expect_tx(q_full, L::kTile);
        for (int c = 0; c < L::kChunks; ++c)
          tc::tma_load_3d(smem + L::kQ + c * L::kChunk, &tm_q, q_full, c * 64, h, q_row);
        // consumption order: K0, K1, V0, K2, V1, ..., K_{n-1}, V_{n-2}, V_{n-1}
        auto load = [&](const CUtensorMap* tm, int blk) {
          const uint32_t s = kv_cnt % L::kStages;
          wp.wait(kv_empty + s, ((kv_cnt / L::kStages) & 1) ^ 1, 1);
          tc::mbar_expect_tx(kv_full + s, L::kTile);
          uint8_t* dst = smem + L::kKV + s * L::kTile;
          const int row = (int)(b0 + (int64_t)blk * BN);
          for (int c = 0; c < L::kChunks; ++c) tc::tma_load_3d(dst + c * L::kChunk, tm, kv_full + s, c * 64, h, row);
          ++kv_cnt;
        };
        load(&tm_k, 0);
        if (nkv > 1) load(&tm_k, 1);
        for (int j = 0; j < nkv; ++j) {
          load(&tm_v, j);
          if (j + 2 < nkv) load(&tm_k, j + 2);
        }
      }
      wp.add(7, clock64() - t_role);
      wp.flush();
    }
  } else if (warp == 1) {
    // ===================================================== MMA issuer
    if (lane == 0) {
      constexpr uint32_t kIdescS = tc::idesc_bf16_f32(BM, BN, false, false);
      constexpr uint32_t kIdescO = tc::idesc_bf16_f32(BM, D, false, true);
      const uint32_t q_base = tc::smem_u32(smem + L::kQ);
      const uint32_t p_base = tc::smem_u32(smem + L::kP);
      const uint32_t kv_base = tc::smem_u32(smem + L::kKV);
      uint32_t kv_cnt = 0, item_cnt = 0, s_use[2] = {0, 0}, p_cnt = 0;
      tc::WaitProf wp;
      wp.init(p.prof, 8);
      const long long t_role = clock64();
      auto next_stage = [&]() {
        const uint32_t s = kv_cnt % L::kStages;
        wp.wait(kv_full + s, (kv_cnt / L::kStages) & 1, 2);
        ++kv_cnt;
        return s;
      };
      auto issue_s = [&](int buf) {
        wp.wait(s_empty + buf, (s_use[buf] & 1) ^ 1, 1);
        ++s_use[buf];
        const uint32_t s = next_stage();
        tc::tc_fence_after();
        const uint32_t k_base = kv_base + s * L::kTile;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t koff = (kk >> 2) * L::kChunk + (kk & 3) * 32;
          tc::mma_bf16_ss(tmem + buf * BN, tc::sw128_desc(q_base + koff, 16, 1024),
                          tc::sw128_desc(k_base + koff, 16, 1024), kIdescS, kk > 0);
        }
        tc::mma_commit(kv_empty + s);
        tc::mma_commit(s_full + buf);
      };
      for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x, ++item_cnt) {
        const int2 it = p.items[w / H];
        const int64_t n = p.off[it.x + 1] - p.off[it.x];
        const int nkv = (int)((n + BN - 1) / BN);
        wp.wait(q_full, item_cnt & 1, 0);
        issue_s(0);
        if (nkv > 1) issue_s(1);
        wp.wait(o_empty, (item_cnt & 1) ^ 1, 3);  // previous epilogue has drained O
        for (int j = 0; j < nkv; ++j) {
          wp.wait(p_full, p_cnt & 1, 4);
          ++p_cnt;
          const uint32_t s = next_stage();  // V_j
          tc::tc_fence_after();
          const uint32_t v_base = kv_base + s * L::kTile;
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk) {
            // A = P [128 x 128 keys] K-major; B = V [128 keys x D] MN-major (LBO = next 64-wide D chunk)
            const uint32_t aoff = (kk >> 2) * L::kChunk + (kk & 3) * 32;
            const uint32_t boff = kk * 16 * 128;
            tc::mma_bf16_ss(tmem + 2 * BN, tc::sw128_desc(p_base + aoff, 16, 1024),
                            tc::sw128_desc(v_base + boff, L::kChunk, 1024), kIdescO, (j > 0 || kk > 0));
          }
          tc::mma_commit(kv_empty + s);
          tc::mma_commit(o_done);
          if (j + 2 < nkv) issue_s(j & 1);
        }
        tc::mma_commit(q_empty);
      }
      wp.add(7, clock64() - t_role);
      wp.flush();
    }
  } else if (warp >= kSoftmaxWarp0) {
    // ===================================================== softmax / correction / epilogue
    const int wq = warp - kSoftmaxWarp0;        // TMEM lane quarter
    const int row = wq * 32 + lane;             // query row within the tile == TMEM lane
    const uint32_t lane_addr = tmem + ((uint32_t)(wq * 32) << 16);
    const uint32_t p_base = tc::smem_u32(smem + L::kP);
    uint32_t s_cons[2] = {0, 0}, pv_cnt = 0;
    tc::WaitProf wp;
    wp.init(row == 0 ? p.prof : nullptr, 16);
    const long long t_role = clock64();
    for (int64_t w = blockIdx.x; w < n_items; w += gridDim.x) {
      const int2 it = p.items[w / H];
      const int h = (int)(w % H);
      const int64_t b0 = p.off[it.x], n = p.off[it.x + 1] - b0;
      const int nkv = (int)((n + BN - 1) / BN);
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < nkv; ++j) {
        const int buf = j & 1;
        wp.wait(s_full + buf, s_cons[buf] & 1, 0);
        ++s_cons[buf];
        tc::tc_fence_after();
        uint32_t sr[BN];
#pragma unroll
        for (int c = 0; c < BN / 32; ++c)
          tc::tmem_ld32(lane_addr + buf * BN + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
        tc::tmem_wait_ld();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(s_empty + buf);
        // mask keys past the segment end (only the last block has any)
        const int64_t rem = n - (int64_t)j * BN;
        const int valid = rem < BN ? (int)rem : BN;
        float s[BN];
#pragma unroll
        for (int c = 0; c < BN; ++c) s[c] = __uint_as_float(sr[c]) * p.scale_log2;
        if (valid < BN) {  // warp-uniform: only a segment's last key block is partial
#pragma unroll
          for (int c = 0; c < BN; ++c) s[c] = c < valid ? s[c] : -INFINITY;
        }
        // 8 independent max chains (a single 128-long fmax chain costs ~512 cycles of latency)
        float m8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) m8[k] = s[k];
#pragma unroll
        for (int c = 8; c < BN; ++c) m8[c & 7] = fmaxf(m8[c & 7], s[c]);
        const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                               fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        float alpha = 1.f;
        bool rescale = false;
        if (mx > m + kRescaleThreshold || j == 0) {
          alpha = (j == 0) ? 0.f : tc::ex2(m - mx);
          rescale = j > 0;
          m = mx;
        }
        float r8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c = 0; c < BN; ++c) {
          s[c] = tc::ex2(s[c] - m);
          r8[c & 7] += s[c];
        }
        const float rs = ((r8[0] + r8[1]) + (r8[2] + r8[3])) + ((r8[4] + r8[5]) + (r8[6] + r8[7]));
        l = l * alpha + rs;
        // PV_{j-1} must be complete before P is overwritten or O is rescaled
        if (j > 0) {
          wp.wait(o_done, pv_cnt & 1, 1);
          ++pv_cnt;
          tc::tc_fence_after();
        }
        if (rescale) {
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            tc::tmem_ld32(lane_addr + 2 * BN + c * 32, o);
            tc::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            tc::tmem_st32(lane_addr + 2 * BN + c * 32, o);
          }
          tc::tmem_wait_st();
        }
        // P_j -> smem as bf16, SWIZZLE_128B K-major [128 rows x 128 keys] (two 64-key chunks)
#pragma unroll
        for (int u = 0; u < BN / 8; ++u) {
          const uint32_t addr = p_base + (u >> 3) * L::kChunk + tc::sw128_offset(row, u & 7);
          tc::st_shared_v4(addr, tc::pack_bf16(s[u * 8 + 0], s[u * 8 + 1]), tc::pack_bf16(s[u * 8 + 2], s[u * 8 + 3]),
                           tc::pack_bf16(s[u * 8 + 4], s[u * 8 + 5]), tc::pack_bf16(s[u * 8 + 6], s[u * 8 + 7]));
        }
        tc::fence_proxy_async_smem();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(p_full);
      }
      // epilogue: wait for the last PV, normalise, store
      wp.wait(o_done, pv_cnt & 1, 2);
      ++pv_cnt;
      tc::tc_fence_after();
      const int64_t q_local = (int64_t)it.y * BM + row;
      const bool store = q_local < n;
      const float inv_l = 1.f / l;
      __nv_bfloat16* orow = p.out + ((b0 + q_local) * H + h) * D;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o[32];
        tc::tmem_ld32(lane_addr + 2 * BN + c * 32, o);
        tc::tmem_wait_ld();
        if (store) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint4 v;
            v.x = tc::pack_bf16(__uint_as_float(o[u * 8 + 0]) * inv_l, __uint_as_float(o[u * 8 + 1]) * inv_l);
            v.y = tc::pack_bf16(__uint_as_float(o[u * 8 + 2]) * inv_l, __uint_as_float(o[u * 8 + 3]) * inv_l);
            v.z = tc::pack_bf16(__uint_as_float(o[u * 8 + 4]) * inv_l, __uint_as_float(o[u * 8 + 5]) * inv_l);
            v.w = tc::pack_bf16(__uint_as_float(o[u * 8 + 6]) * inv_l, __uint_as_float(o[u * 8 + 7]) * inv_l);
            *reinterpret_cast<uint4*>(orow + c * 32 + u * 8) = v;
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(o_empty);
      if (store) p.lse[(int64_t)h * p.total_rows + b0 + q_local] = (m + __log2f(l)) * 0.6931471805599453f;
    }
    wp.add(7, clock64() - t_role);
    wp.flush();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem);
  }
}

}  // namespace fa

// ------------------------------------------------------------------ host side
bool attn_sm100_supported(int head_dim, jg_dtype dt) {
  return dt == JG_BF16 && (head_dim == 64 || head_dim == 128);
}

template <int D>
static jg_status fwd_launch(const int64_t* off, int64_t batch, int64_t total_rows, int H, const void* q, const void* k,
                            const void* v, void* out, float* lse, const int2* items, const int64_t* n_items,
                            int64_t max_items, cudaStream_t st) {
  using L = fa::Smem<D>;
  CUtensorMap mq, mk, mv;
  if (jg_status rc = make_map(&mq, q, total_rows, H, D, 128)) return rc;
  if (jg_status rc = make_map(&mk, k, total_rows, H, D, 128)) return rc;
  if (jg_status rc = make_map(&mv, v, total_rows, H, D, 128)) return rc;
  static bool attr_set = false;
  if (!attr_set) {
    JG_CUDA(cudaFuncSetAttribute(fa::jfa_fwd_sm100_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kAlloc));
    attr_set = true;
  }
  fa::Params p{off, items, n_items, batch, total_rows, H, (__nv_bfloat16*)out, lse,
               1.4426950408889634f / sqrtf((float)D), wait_prof_begin(st)};
  const int64_t work = max_items * H;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(device_sm_count(), work));
  fa::jfa_fwd_sm100_kernel<D><<<grid, fa::kThreads, L::kAlloc, st>>>(mq, mk, mv, p);
  JG_LAUNCHED("jfa_fwd_sm100_kernel");
  wait_prof_end(p.prof, st, "fwd", {"P.q_empty", "P.kv_empty", "", "", "", "", "", "P.total", "M.q_full", "M.s_empty", "M.kv_full", "M.o_empty", "M.p_full", "", "", "M.total", "S.s_full", "S.o_done", "S.o_done_epi", "", "", "", "", "S.total"});
  return JG_OK;
}

jg_status launch_attn_fwd_sm100(const int64_t* off, int64_t batch, int64_t total_rows, int H, int D, const void* q,
                                const void* k, const void* v, void* out, float* lse, const int2* items,
                                const int64_t* n_items, int64_t max_items, cudaStream_t st) {
  if (D == 128) return fwd_launch<128>(off, batch, total_rows, H, q, k, v, out, lse, items, n_items, max_items, st);
  if (D == 64) return fwd_launch<64>(off, batch, total_rows, H, q, k, v, out, lse, items, n_items, max_items, st);
  return fail(JG_UNSUPPORTED, "tcgen05 attention: head_dim must be 64 or 128");
}



}  // namespace jg
