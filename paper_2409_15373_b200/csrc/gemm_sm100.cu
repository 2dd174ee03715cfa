// gemm_sm100.cu — the jagged bmm family on tcgen05 tensor cores (bf16 inputs, fp32 accumulation).
//
// One persistent warp-specialized kernel, templated on the contraction, covers the four forward
// operators of linalg.cpp (per sample i, Bi = offsets[i+1] - offsets[i]):
//   JJJ  jagged_jagged_bmm_jagged_out (:122)  S_i = Q_i K_i^T      M=Bi N=Bi K=D   A,B K-major (TMA)
//   AJ   array_jagged_bmm_jagged_out  (:161)  O_i = A_i V_i        M=Bi N=D  K=Bi  A jagged^2 (manual), B MN-major
//   JJ   jagged_jagged_bmm            (:70)   Z_i = X_i^T Y_i      M=D  N=T  K=Bi  A,B MN-major (TMA)
//   JD   jagged_dense_bmm             (:34)   O_i = X_i W_i        M=Bi N=T  K=D   A K-major, B MN-major
// 128x128 output tiles, 64-deep K stages through a 4-stage ring, accumulators double-buffered in TMEM
// so the epilogue of tile t overlaps the MMAs of tile t+1. TMA coordinates are global row indices
// (offsets[i] + local row), so no padding is materialised; rows of the next sample that a tail tile
// picks up are masked: never stored (M/N tails) or zeroed in smem before the MMA (K tails of JJ, where
// the reduction runs over the jagged axis). Jagged^2 A operands (row stride Bi, not 16-byte aligned,
// unusable by TMA) are gathered by a loader warpgroup into the swizzled layout with zeros past Bi.
// Warps: 0 TMA producer, 1 MMA issuer, 4-7 epilogue (TMEM -> registers -> global), 8-11 loader.
#include "common.cuh"
#include "internal.h"
#include "tc.cuh"
#include "tma_host.h"

namespace jg {
namespace gm {

enum Op { JJJ = 0, AJ = 1, JJ = 2, JD = 3 };

constexpr int BM = 128, BN = 128, BK = 64, kStages = 4, kThreads = 384;
constexpr int kTileBytes = 16384;  // one operand stage: 128 x 64 bf16
struct Smem {
  static constexpr int kA = 0;
  static constexpr int kB = kStages * kTileBytes;
  static constexpr int kStg = 2 * kStages * kTileBytes;        // JJJ epilogue staging, 32 rows x 128 fp32 per warp
  static constexpr int kBar = kStg + 4 * 32 * 128 * 4;
  static constexpr int kNumBars = 3 * kStages + 4 + 1;
  static constexpr int kAlloc = kBar + kNumBars * 8 + 16 + 1024;
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
};

struct Tile {
  int64_t i, b0, n, sqo;
  int M, N, K, m0, n0, nk;
};

template <int OP>
__device__ __forceinline__ Tile tile_of(const Params& p, int64_t t) {
  Tile r;
  r.i = upper_index(p.prefix, p.batch, t);
  r.b0 = p.off[r.i];
  r.n = p.off[r.i + 1] - r.b0;
  r.sqo = p.sq ? p.sq[r.i] : 0;
  const int Bi = (int)r.n;
  if (OP == JJJ) { r.M = Bi; r.N = Bi; r.K = p.D; }
  if (OP == AJ) { r.M = Bi; r.N = p.D; r.K = Bi; }
  if (OP == JJ) { r.M = p.D; r.N = p.T; r.K = Bi; }
  if (OP == JD) { r.M = Bi; r.N = p.T; r.K = p.D; }
  const int tn = (r.N + BN - 1) / BN;
  const int64_t local = t - p.prefix[r.i];
  r.m0 = (int)(local / tn) * BM;
  r.n0 = (int)(local % tn) * BN;
  r.nk = (r.K + BK - 1) / BK;
  return r;
}

// smem A operand is K-major for JJJ/AJ/JD ([128 m rows x 64 k]) and MN-major for JJ ([64 k rows x 128 m]
// in two 64-wide chunks); B is K-major for JJJ ([128 n rows x 64 k]) and MN-major otherwise.
template <int OP> struct Layout {
  static constexpr bool a_mn = OP == JJ;
  static constexpr bool b_mn = OP != JJJ;
  static constexpr bool loader = OP == AJ || OP == JJ;  // stages pass through the loader warpgroup
};

template <int OP>
__global__ void __launch_bounds__(kThreads, 1) gemm_sm100_kernel(const __grid_constant__ CUtensorMap tm_a,
                                                                 const __grid_constant__ CUtensorMap tm_b, Params p) {
  using Ly = Layout<OP>;
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
      tc::mbar_init(acc_empty + b, 4);
    }
    tc::fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tm_a);
    tc::tma_prefetch(&tm_b);
  }
  if (warp == 1) tc::tmem_alloc<256>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t n_tiles = p.prefix[p.batch];

  if (warp == 0) {
    // ============================================ TMA producer
    if (lane == 0) {
      uint32_t cnt = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const Tile tl = tile_of<OP>(p, t);
        for (int kb = 0; kb < tl.nk; ++kb, ++cnt) {
          const uint32_t s = cnt % kStages;
          tc::mbar_wait(empty + s, ((cnt / kStages) & 1) ^ 1);
          uint8_t* sa = smem + Smem::kA + s * kTileBytes;
          uint8_t* sb = smem + Smem::kB + s * kTileBytes;
          const int k0 = kb * BK;
          const int bytes = (OP == AJ ? 1 : 2) * kTileBytes;
          tc::mbar_expect_tx(full + s, bytes);
          if (OP == JJJ || OP == JD)
            tc::tma_load_3d(sa, &tm_a, full + s, k0, 0, (int)(tl.b0 + tl.m0));
          if (OP == JJ)
            for (int c = 0; c < 2; ++c)
              tc::tma_load_3d(sa + c * 8192, &tm_a, full + s, tl.m0 + 64 * c, 0, (int)(tl.b0 + k0));
          if (OP == JJJ) tc::tma_load_3d(sb, &tm_b, full + s, k0, 0, (int)(tl.b0 + tl.n0));
          if (OP == AJ || OP == JJ)
            for (int c = 0; c < 2; ++c)
              tc::tma_load_3d(sb + c * 8192, &tm_b, full + s, tl.n0 + 64 * c, 0, (int)(tl.b0 + k0));
          if (OP == JD)
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
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tcount) {
        const Tile tl = tile_of<OP>(p, t);
        const int ab = tcount & 1;
        tc::mbar_wait(acc_empty + ab, ((tcount >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        for (int kb = 0; kb < tl.nk; ++kb, ++cnt) {
          const uint32_t s = cnt % kStages;
          if (Ly::loader) tc::mbar_wait(ready + s, (cnt / kStages) & 1);
          if (OP == JJJ || OP == JD || OP == AJ) tc::mbar_wait(full + s, (cnt / kStages) & 1);
          tc::tc_fence_after();
          const uint32_t sa = tc::smem_u32(smem + Smem::kA + s * kTileBytes);
          const uint32_t sb = tc::smem_u32(smem + Smem::kB + s * kTileBytes);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t da = Ly::a_mn ? tc::sw128_desc(sa + kk * 2048, 8192, 1024) : tc::sw128_desc(sa + kk * 32, 16, 1024);
            const uint64_t db = Ly::b_mn ? tc::sw128_desc(sb + kk * 2048, 8192, 1024) : tc::sw128_desc(sb + kk * 32, 16, 1024);
            tc::mma_bf16_ss(tmem + ab * BN, da, db, idesc, (kb > 0 || kk > 0));
          }
          tc::mma_commit(empty + s);
        }
        tc::mma_commit(acc_full + ab);  // with no k blocks this arrives at once (epilogue writes zeros)
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ============================================ epilogue: thread = output row of the tile
    const int wq = warp - 4, r = wq * 32 + lane;
    uint32_t tcount = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tcount) {
      const Tile tl = tile_of<OP>(p, t);
      const int ab = tcount & 1;
      tc::mbar_wait(acc_full + ab, (tcount >> 1) & 1);
      tc::tc_fence_after();
      const int m = tl.m0 + r;
      const bool row_ok = m < tl.M;
      const int ncols = tl.N - tl.n0 < BN ? tl.N - tl.n0 : BN;
      int64_t base;  // element index of (m, n0) in the output
      if (OP == JJJ) base = tl.sqo + (int64_t)m * tl.n + tl.n0;
      else if (OP == JJ) base = tl.i * (int64_t)p.D * p.T + (int64_t)m * p.T + tl.n0;
      else base = (tl.b0 + m) * (int64_t)tl.N + tl.n0;
      const bool vec = OP != JJJ && ncols == BN;
      if (OP == JJJ) {
        // jagged^2 rows (stride Bi, arbitrary alignment): stage this warp's 32 rows in smem (row pitch 129
        // floats, conflict-free) and write each row with the lanes along its columns (coalesced)
        float* stg = reinterpret_cast<float*>(smem + Smem::kStg) + wq * 32 * 129;
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t v[32];
          tc::tmem_ld32(tmem + ((uint32_t)(wq * 32) << 16) + ab * BN + c * 32, v);
          tc::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) stg[lane * 129 + c * 32 + e] = __uint_as_float(v[e]);
        }
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(acc_empty + ab);  // TMEM drained; the stores below overlap the next tile
        const int nrows = tl.M - tl.m0 - wq * 32 < 32 ? tl.M - tl.m0 - wq * 32 : 32;
        for (int rr = 0; rr < nrows; ++rr) {
          const int64_t rb = tl.sqo + (int64_t)(tl.m0 + wq * 32 + rr) * tl.n + tl.n0;
#pragma unroll
          for (int h = 0; h < BN / 32; ++h) {
            const int col = lane + 32 * h;
            if (col < ncols) {
              const float x = stg[rr * 129 + col];
              if (p.out_f32) reinterpret_cast<float*>(p.out)[rb + col] = x;
              else reinterpret_cast<__nv_bfloat16*>(p.out)[rb + col] = __float2bfloat16_rn(x);
            }
          }
        }
        __syncwarp();
        continue;
      }
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(wq * 32) << 16) + ab * BN + c * 32, v);
        tc::tmem_wait_ld();
        if (tl.nk == 0) {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = 0u;
        }
        if (!row_ok) continue;
        if (p.out_f32) {
          float* o = reinterpret_cast<float*>(p.out) + base + c * 32;
          if (vec) {
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
          if (vec) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              uint4 w;
              w.x = tc::pack_bf16(__uint_as_float(v[u * 8 + 0]), __uint_as_float(v[u * 8 + 1]));
              w.y = tc::pack_bf16(__uint_as_float(v[u * 8 + 2]), __uint_as_float(v[u * 8 + 3]));
              w.z = tc::pack_bf16(__uint_as_float(v[u * 8 + 4]), __uint_as_float(v[u * 8 + 5]));
              w.w = tc::pack_bf16(__uint_as_float(v[u * 8 + 6]), __uint_as_float(v[u * 8 + 7]));
              *reinterpret_cast<uint4*>(o + u * 8) = w;
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
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const Tile tl = tile_of<OP>(p, t);
      for (int kb = 0; kb < tl.nk; ++kb, ++cnt) {
        const uint32_t s = cnt % kStages;
        uint8_t* sa = smem + Smem::kA + s * kTileBytes;
        const int k0 = kb * BK;
        if (OP == AJ) {
          // gather A[m0 + r][k0 .. k0+63] (row stride Bi, arbitrary 2-byte alignment) into the [128 rows x 64 k]
          // SWIZZLE_128B K-major stage: 8 lanes per row, each producing one 16-byte unit from two aligned
          // 16-byte loads realigned with funnel shifts; zeros past the sample (k >= Bi or m >= Bi).
          // All 16 loads of a lane are issued before the stage is free and before any is consumed.
          const char* base = reinterpret_cast<const char*>(p.a_j2);
          const int u = lane & 7;
          uint4 lo[8], hi[8];
          int shv[8], nval[8];
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int row = wq * 32 + it * 4 + (lane >> 3), m = tl.m0 + row;
            const int kb0 = k0 + u * 8;  // first element of this 16-byte unit
            nval[it] = (m < tl.M && kb0 < tl.K) ? (tl.K - kb0 < 8 ? tl.K - kb0 : 8) : 0;
            lo[it] = hi[it] = make_uint4(0, 0, 0, 0);
            shv[it] = 0;
            if (nval[it] > 0) {
              // an aligned 16-byte chunk holding at least one valid byte lies in the same page as that
              // byte, so these over-reads never fault; hi is read only if valid elements reach into it
              const int64_t byte0 = (tl.sqo + (int64_t)m * tl.n + kb0) * 2;
              const int64_t al = byte0 & ~int64_t(15);
              shv[it] = (int)(byte0 - al);
              lo[it] = __ldg(reinterpret_cast<const uint4*>(base + al));
              if (shv[it] != 0 && byte0 + 2 * nval[it] > al + 16) hi[it] = __ldg(reinterpret_cast<const uint4*>(base + al + 16));
            }
          }
          tc::mbar_wait(empty + s, ((cnt / kStages) & 1) ^ 1);
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int row = wq * 32 + it * 4 + (lane >> 3);
            const int sh = shv[it], ws = sh >> 2;
            const bool half = (sh & 2) != 0;
            const uint32_t w0 = lo[it].x, w1 = lo[it].y, w2 = lo[it].z, w3 = lo[it].w;
            const uint32_t w4 = hi[it].x, w5 = hi[it].y, w6 = hi[it].z, w7 = hi[it].w;
            // x_k = word (ws + k) of the 32-byte window (register selects, no local memory)
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
            const int valid = nval[it];
            if (valid < 8) {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                if (2 * q >= valid) o[q] = 0;
                else if (2 * q + 1 >= valid) o[q] &= 0xFFFFu;
              }
            }
            *reinterpret_cast<uint4*>(sa + tc::sw128_offset(row, u)) = make_uint4(o[0], o[1], o[2], o[3]);
          }
        } else {
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
    tc::tmem_dealloc<256>(tmem);
  }
}

// 2-D view [rows, cols] bf16 as a 3-D map (cols, 1, rows) with box (64, 1, box_rows), SWIZZLE_128B
static jg_status map2d(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int box_rows) {
  return make_map(m, ptr, rows, 1, (int)cols, box_rows);
}

template <int OP>
static jg_status run(const Params& p, const CUtensorMap& ma, const CUtensorMap& mb, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    JG_CUDA(cudaFuncSetAttribute(gemm_sm100_kernel<OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem::kAlloc));
    attr = true;
  }
  gemm_sm100_kernel<OP><<<device_sm_count(), kThreads, Smem::kAlloc, st>>>(ma, mb, p);
  JG_LAUNCHED("gemm_sm100_kernel");
  return JG_OK;
}

}  // namespace gm

bool gemm_sm100_supported(int op, int64_t D, int64_t T, jg_dtype in_dt) {
  if (in_dt != JG_BF16) return false;
  switch (op) {
    case gm::JJJ: return D % 64 == 0;
    case gm::AJ: return D % 64 == 0;
    case gm::JJ: return D % 64 == 0 && T % 64 == 0;
    case gm::JD: return D % 64 == 0 && T % 64 == 0;
  }
  return false;
}

// A/B roles per op: JJJ (q, k), AJ (a_j2, v), JJ (x, y), JD (x, w)
jg_status launch_gemm_sm100(int op, const int64_t* off, const int64_t* sq, int64_t batch, int64_t total_rows, int64_t D,
                            int64_t T, const void* a, const void* b, void* out, jg_dtype out_dt, int64_t* tile_prefix,
                            cudaStream_t st) {
  // tile prefix over samples with the op's (M, N)
  GemmDesc g;
  Lin bi;
  bi.bi = 1;
  if (op == gm::JJJ) { g.M = bi; g.N = bi; }
  if (op == gm::AJ) { g.M = bi; g.N = L_const(D); }
  if (op == gm::JJ) { g.M = L_const(D); g.N = L_const(T); }
  if (op == gm::JD) { g.M = bi; g.N = L_const(T); }
  if (jg_status rc = launch_gemm_prefix(g, off, sq, batch, 128, 128, tile_prefix, st)) return rc;
  gm::Params p{off, sq, tile_prefix, batch, (int)D, (int)T, (const __nv_bfloat16*)a, out, out_dt == JG_F32};
  CUtensorMap ma{}, mb{};
  const int64_t rows = total_rows > 0 ? total_rows : 1;
  switch (op) {
    case gm::JJJ:
      if (jg_status rc = gm::map2d(&ma, a, rows, D, 128)) return rc;
      if (jg_status rc = gm::map2d(&mb, b, rows, D, 128)) return rc;
      return gm::run<gm::JJJ>(p, ma, mb, st);
    case gm::AJ:
      if (jg_status rc = gm::map2d(&mb, b, rows, D, 64)) return rc;
      return gm::run<gm::AJ>(p, mb, mb, st);
    case gm::JJ:
      if (jg_status rc = gm::map2d(&ma, a, rows, D, 64)) return rc;
      if (jg_status rc = gm::map2d(&mb, b, rows, T, 64)) return rc;
      return gm::run<gm::JJ>(p, ma, mb, st);
    case gm::JD:
      if (jg_status rc = gm::map2d(&ma, a, rows, D, 128)) return rc;
      if (jg_status rc = gm::map2d(&mb, b, batch * D > 0 ? batch * D : 1, T, 64)) return rc;
      return gm::run<gm::JD>(p, ma, mb, st);
  }
  return fail(JG_UNSUPPORTED, "gemm_sm100: unknown op");
}

}  // namespace jg
