// attn_x3_sm100.cu — fp32 Jagged Flash Attention forward + backward on tcgen05 tensor cores (split emulation).
//
// Two splits: the default fp16 two-piece kernels (x2h, further below: per-tensor power-of-two scales, three MMAs per
// product) and the bf16 three-piece kernels described first (JG_FP32_X3=1: no scales, six MMAs per product).
//
// Semantics: attention.cpp:172-289 in fp32 mode (the reference's float instantiation, attention.cpp:311-331),
// same outputs as the tiled FFMA kernels in attn_simt.cu up to fp32 rounding.
//
// tcgen05 has no fp32 MMA. Every fp32 operand x is split into three bf16 pieces x = x1 + x2 + x3 (x1 = bf16(x),
// x2 = bf16(x - x1), x3 = bf16(x - x1 - x2); the residual is below 2^-26 |x|), and a product a*b is the sum of
// the piece products with i + j <= 4: a1b1 + a1b2 + a2b1 + a1b3 + a2b2 + a3b1 (the dropped terms are below
// 2^-24 |ab|), all accumulated in fp32 in TMEM — fp32-level scores for the softmax. P in [0, 1] is split the same
// way (two pieces leave a 2^-17 relative error per P that the cancellation in sum_k P V amplifies past 1e-5).
// That is 6 bf16 MMAs for S and 6 for P V per block: 6x the tensor work of the bf16 kernel. The small products
// go first: the tensor core's fp32 accumulation truncates each addend to the running sum's exponent, so adding
// the cross terms into an accumulator that already holds a1b1 would cost ~2^-23 |ab| per MMA; this order leaves
// only the D/16 k-steps of a1b1 at that magnitude (the difference shows in dS = P (dP - Delta), which cancels).
//
// Forward: one CTA (8 warps) per (sample, 128-row query tile, head) item of the schedule's LPT list (persistent,
// round-robin); Q's pieces sit in TMEM [0, 3D/2) (split on the fly per item); keys stream in 64-row blocks through
// two-stage K and V rings of bf16 pieces (SWIZZLE_128B; K K-major, V MN-major) split on the fly from fp32 (no
// scratch). The warp roles and the pipeline are described at attn_fwd_x3_kernel; the backward's two passes at
// BwdLay. Epilogues write fp32 straight to global; padded mode masks keys / rows past `valid`.
#include <cuda_fp16.h>

#include "common.cuh"
#include "internal.h"
#include "tc.cuh"

namespace jg {
namespace x3 {

constexpr int BM = 128, BN = 64, kThreads = 256;
constexpr float kLog2e = 1.4426950408889634f, kLn2 = 0.6931471805599453f;

template <int D>
struct Lay {
  static constexpr int kKChunk = BN * 128;             // [64 rows x 64] bf16
  static constexpr int kKPiece = (D / 64) * kKChunk;
  static constexpr int kKStage = 3 * kKPiece;          // K1 K2 K3 (or V1 V2 V3) of one 64-key block
  static constexpr int kK = 0;                         // K ring: 2 stages
  static constexpr int kV = kK + 2 * kKStage;          // V ring: 2 stages
  static constexpr int kBar = kV + 2 * kKStage;        // 10 mbarriers + tmem slot
  static constexpr int kAlpha = kBar + 128;            // float[2][128] (block maxima of the two key halves)
  static constexpr int kL = kAlpha + 2 * 4 * BM;       // float[2][128]
  static constexpr int kBytes = kL + 2 * 4 * BM;
  static constexpr int kAlloc = kBytes + 1024;         // + alignment slack
  // TMEM: Q1 Q2 Q3 [0, 3D/2) | S0 | S1 (64 each) | O (D) | P3_0 | P3_1 (32 each)
  static constexpr int kTmemCols = 512;
};
constexpr int kFwdThreads = 256;  // 8 warps (warp 0 also issues the MMAs)


// one paired conversion (cvt.rn.bf16x2) per piece; the pieces' fp32 values are the packed halves shifted into place
__device__ __forceinline__ void split3(float a, float b, uint32_t& w1, uint32_t& w2, uint32_t& w3) {
  w1 = tc::pack_bf16(a, b);
  const float ra = a - __uint_as_float(w1 << 16), rb = b - __uint_as_float(w1 & 0xffff0000u);  // exact
  w2 = tc::pack_bf16(ra, rb);
  w3 = tc::pack_bf16(ra - __uint_as_float(w2 << 16), rb - __uint_as_float(w2 & 0xffff0000u));
}

// rows [r0, r0 + ROWS) of a fp32 [*, H, D] tensor (rows >= n zero) as three bf16 pieces, each [ROWS x D] in
// SWIZZLE_128B 64-column chunks of ROWS x 128 B at base + piece * piece_bytes + chunk * ROWS * 128
// (threads [T0, T0 + NT) of the CTA take part)
template <int D, int ROWS, int T0 = 0, int NT = kThreads, int kMaxBatch = 4>
__device__ __forceinline__ void stage_split3(const float* __restrict__ src, int64_t b0, int64_t r0, int64_t n,
                                             int64_t rs, uint32_t base) {
  constexpr int kUnits = D / 8;  // 8 floats = one 16-byte bf16 unit per piece
  constexpr int kPiece = (D / 64) * ROWS * 128;
  constexpr int kTotal = ROWS * kUnits;
  constexpr int kIter = (kTotal + NT - 1) / NT;
  constexpr int kBatch = kIter < kMaxBatch ? kIter : kMaxBatch;  // loads of a batch in flight before its stores
  const int t = (int)threadIdx.x - T0;
#pragma unroll
  for (int i0 = 0; i0 < kIter; i0 += kBatch) {
    float4 a[kBatch], b[kBatch];
#pragma unroll
    for (int i = 0; i < kBatch; ++i) {
      const int e = t + (i0 + i) * NT, r = e / kUnits, u = e % kUnits;
      a[i] = b[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (e < kTotal && r0 + r < n) {
        const float4* p = reinterpret_cast<const float4*>(src + (b0 + r0 + r) * rs + u * 8);
        a[i] = __ldg(p);
        b[i] = __ldg(p + 1);
      }
    }
#pragma unroll
    for (int i = 0; i < kBatch; ++i) {
      const int e = t + (i0 + i) * NT, r = e / kUnits, u = e % kUnits;
      if (e >= kTotal) continue;
      uint32_t w1[4], w2[4], w3[4];
      split3(a[i].x, a[i].y, w1[0], w2[0], w3[0]);
      split3(a[i].z, a[i].w, w1[1], w2[1], w3[1]);
      split3(b[i].x, b[i].y, w1[2], w2[2], w3[2]);
      split3(b[i].z, b[i].w, w1[3], w2[3], w3[3]);
      const uint32_t off = (u >> 3) * (ROWS * 128) + tc::sw128_offset(r, u & 7);
      tc::st_shared_v4(base + off, w1[0], w1[1], w1[2], w1[3]);
      tc::st_shared_v4(base + kPiece + off, w2[0], w2[1], w2[2], w2[3]);
      tc::st_shared_v4(base + 2 * kPiece + off, w3[0], w3[1], w3[2], w3[3]);
    }
  }
}


// A moving block held in registers between its global loads and its split into smem: the loads go out while the
// tensor core still reads the block's buffer, the split + stores once it is free.
template <int D, int ROWS, int NT = kThreads>
struct Pre {
  static constexpr int kUnits = D / 8, kTotal = ROWS * kUnits, kIter = kTotal / NT;
  static constexpr int kPiece = (D / 64) * ROWS * 128;
  float4 a[kIter], b[kIter];
  __device__ __forceinline__ void load(const float* __restrict__ src, int64_t b0, int64_t r0, int64_t n, int64_t rs,
                                       int t) {
#pragma unroll
    for (int i = 0; i < kIter; ++i) {
      const int e = t + i * NT, r = e / kUnits, u = e % kUnits;
      a[i] = b[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r0 + r < n) {
        const float4* p = reinterpret_cast<const float4*>(src + (b0 + r0 + r) * rs + u * 8);
        a[i] = __ldg(p);
        b[i] = __ldg(p + 1);
      }
    }
  }
  __device__ __forceinline__ void store(uint32_t base, int t) const {
#pragma unroll
    for (int i = 0; i < kIter; ++i) {
      const int e = t + i * NT, r = e / kUnits, u = e % kUnits;
      uint32_t w1[4], w2[4], w3[4];
      split3(a[i].x, a[i].y, w1[0], w2[0], w3[0]);
      split3(a[i].z, a[i].w, w1[1], w2[1], w3[1]);
      split3(b[i].x, b[i].y, w1[2], w2[2], w3[2]);
      split3(b[i].z, b[i].w, w1[3], w2[3], w3[3]);
      const uint32_t off = (u >> 3) * (ROWS * 128) + tc::sw128_offset(r, u & 7);
      tc::st_shared_v4(base + off, w1[0], w1[1], w1[2], w1[3]);
      tc::st_shared_v4(base + kPiece + off, w2[0], w2[1], w2[2], w2[3]);
      tc::st_shared_v4(base + 2 * kPiece + off, w3[0], w3[1], w3[2], w3[3]);
    }
  }
};

// This thread's half (columns [half*D/2, +D/2)) of row `row` of a fp32 [*, H, D] tensor, split into bf16 pieces:
// pieces 0 .. NT-1 into TMEM (piece p at column t_base + p*D/2, packed two per column), piece 2 (when kS3)
// into the K-major SWIZZLE_128B smem tile at s3 ([128 rows x D], chunks of 128 x 128 B).
template <int D, int NT, bool kS3 = false>
__device__ __forceinline__ void stage_row_tmem(const float* __restrict__ src, bool in, uint32_t t_base,
                                               uint32_t lane_off, int half, int row, uint32_t s3) {
  constexpr int kCols = D / 4;  // packed columns per half per piece
  float4 xs[D / 8];             // the whole half row in flight before any store
#pragma unroll
  for (int g = 0; g < D / 8; ++g) {
    xs[g] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (in) xs[g] = __ldg(reinterpret_cast<const float4*>(src + half * (D / 2) + 4 * g));
  }
#pragma unroll
  for (int c0 = 0; c0 < kCols; c0 += 8) {  // 16 elements -> 8 packed columns per step
    uint32_t w[3][8];
    const int e0 = half * (D / 2) + 2 * c0;  // first element
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const float4 x = xs[c0 / 2 + g];
      split3(x.x, x.y, w[0][2 * g], w[1][2 * g], w[2][2 * g]);
      split3(x.z, x.w, w[0][2 * g + 1], w[1][2 * g + 1], w[2][2 * g + 1]);
    }
#pragma unroll
    for (int p = 0; p < NT; ++p) {
      const uint32_t ta = t_base + p * (D / 2) + half * kCols + c0 + lane_off;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta),
                   "r"(w[p][0]), "r"(w[p][1]), "r"(w[p][2]), "r"(w[p][3]), "r"(w[p][4]), "r"(w[p][5]), "r"(w[p][6]),
                   "r"(w[p][7])
                   : "memory");
    }
    if (kS3) {  // two 16-byte units (8 elements each) of the third piece
#pragma unroll
      for (int uu = 0; uu < 2; ++uu) {
        const int u = e0 / 8 + uu;
        tc::st_shared_v4(s3 + (u >> 3) * (BM * 128) + tc::sw128_offset(row, u & 7), w[2][4 * uu], w[2][4 * uu + 1],
                         w[2][4 * uu + 2], w[2][4 * uu + 3]);
      }
    }
  }
}

// Forward (pipelined; attention.cpp:172-225). Two TMEM score buffers and two-stage K / V rings let the tensor core
// run PV_j and S_{j+2} back to back while the warps work on block j+1. Every warp does every phase on its share:
// warp half h takes keys [32h, 32h + 32) of the softmax (the two halves of a row exchange block maxima through
// shared memory; their sums combine at the end) and output columns [h D/2, (h + 1) D/2) of O (registers), and all
// 256 threads split K_{j+2} (under PV_j, once S_j released the stage) and V_{j+2} (once PV_j released its stage).
// Warp 0 also issues the MMAs: S_0, S_1, then per block PV_j (after every P_j and the previous O read-out) and
// S_{j+2} into the score buffer P_j occupied (in-order tcgen05 execution orders the overwrite).
template <int D>
__global__ void __launch_bounds__(kFwdThreads, 1) attn_fwd_x3_kernel(
    const int64_t* __restrict__ off, const int2* __restrict__ items, const int64_t* __restrict__ n_items, int H,
    int64_t total_rows, const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
    float* __restrict__ out, float* __restrict__ lse, float scale_log2, const int64_t* __restrict__ valid) {
  using L = Lay<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = tc::smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* bar_s = bars;        // [2] score MMAs of the buffer done (commit)
  uint64_t* bar_o = bars + 2;    // PV_j done (commit)
  uint64_t* p_ready = bars + 3;  // P_j written (256 arrivals)
  uint64_t* o_free = bars + 4;   // O read out (256 arrivals)
  uint64_t* k_ready = bars + 5;  // [2] K stage split (256 arrivals)
  uint64_t* v_ready = bars + 7;  // [2] V stage split (256 arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);
  float* mx_s = reinterpret_cast<float*>(smem + L::kAlpha);  // [2][128] block maxima of the two key halves
  float* l_s = reinterpret_cast<float*>(smem + L::kL);       // [2][128] final row sums of the two halves
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane;
  if (tid == 0) {
    for (int i = 0; i < 3; ++i) tc::mbar_init(bars + i, 1);
    for (int i = 3; i < 9; ++i) tc::mbar_init(bars + i, 256);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc<L::kTmemCols>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_q = tmem, t_s0 = tmem + 3 * D / 2, t_o = t_s0 + 128, t_p30 = t_o + D;
  const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
  constexpr uint32_t kIdescS = tc::idesc_bf16_f32(BM, BN, false, false);
  constexpr uint32_t kIdescO = tc::idesc_bf16_f32(BM, D, false, true);
  const int64_t rs = (int64_t)H * D;
  const int64_t n_work = *n_items * H;
  // barrier use counters (each role tracks the completions it waits for; all are CTA-global across items)
  // (per-parity counters as scalars: a dynamically indexed pair would live in local memory)
  uint32_t cs0 = 0, cs1 = 0, c_o = 0, c_p = 0, c_of = 0, ck0 = 0, ck1 = 0, cv0 = 0, cv1 = 0;
  auto take = [](uint32_t& c0, uint32_t& c1, int b) {  // parity of the next completion of buffer b's barrier
    const uint32_t v = b ? c1 : c0;
    if (b) ++c1; else ++c0;
    return v & 1u;
  };
  for (int64_t w = blockIdx.x; w < n_work; w += gridDim.x) {
    const int2 it = items[w / H];
    const int h = (int)(w % H);
    const int64_t hd = (int64_t)h * D;
    const int64_t b0 = off[it.x], seg = off[it.x + 1] - b0;
    const int64_t nv = valid ? (valid[it.x] < seg ? valid[it.x] : seg) : seg;
    const int q0 = it.y * BM;
    const int nblk = q0 < nv ? (int)((nv + BN - 1) / BN) : 0;  // an all-padding tile attends nothing
    __syncthreads();  // the previous item's TMEM / smem reads are done
    if (nblk > 0) {  // Q pieces -> TMEM; blocks 0 and 1 -> stages 0 and 1
      stage_row_tmem<D, 3>(q + (b0 + q0 + row) * rs + hd, q0 + row < seg, t_q, lane_off, half, row, 0);
      for (int j = 0; j < 2 && j < nblk; ++j) {
        stage_split3<D, BN>(k + hd, b0, (int64_t)j * BN, nv, rs, sbase + L::kK + j * L::kKStage);
        stage_split3<D, BN>(v + hd, b0, (int64_t)j * BN, nv, rs, sbase + L::kV + j * L::kKStage);
      }
    }
    tc::tmem_wait_st();
    tc::fence_proxy_async_smem();
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    // warp 0 doubles as the MMA issuer (a ninth warp would not fit the per-SMSP register file at this size)
    auto issue_s = [&](int j) {  // S = Q3K1 + Q2K2 + Q1K3 + Q2K1 + Q1K2 + Q1K1 (small terms first)
      constexpr int kQi[6] = {2, 1, 0, 1, 0, 0}, kKj[6] = {0, 1, 2, 0, 1, 0};
      const uint32_t kst = sbase + L::kK + (j & 1) * L::kKStage, ts = t_s0 + (j & 1) * 64;
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        const uint32_t ka = kst + kKj[c] * L::kKPiece;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          tc::mma_bf16_ts_warp(ts, t_q + kQi[c] * (D / 2) + kk * 8,
                               tc::sw128_desc(ka + (kk >> 2) * L::kKChunk + (kk & 3) * 32, 16, 1024), kIdescS,
                               (c > 0 || kk > 0) ? 1u : 0u);
      }
      tc::mma_commit_warp(bar_s + (j & 1));
    };
    auto issue_pv = [&](int j) {  // O_j = P3V1 + P2V2 + P1V3 + P2V1 + P1V2 + P1V1 (V MN-major)
      constexpr int kPi[6] = {2, 1, 0, 1, 0, 0}, kVj[6] = {0, 1, 2, 0, 1, 0};
      const int b = j & 1;
      const uint32_t vst = sbase + L::kV + b * L::kKStage, ts = t_s0 + b * 64, tp3 = t_p30 + b * 32;
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        const uint32_t va = vst + kVj[c] * L::kKPiece;
        const uint32_t pa = kPi[c] == 2 ? tp3 : ts + kPi[c] * 32;
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk)
          tc::mma_bf16_ts_warp(t_o, pa + kk * 8, tc::sw128_desc(va + kk * 16 * 128, L::kKChunk, 1024), kIdescO,
                               (c > 0 || kk > 0) ? 1u : 0u);
      }
      tc::mma_commit_warp(bar_o);
    };
    if (warp == 0)
      for (int j = 0; j < 2 && j < nblk; ++j) issue_s(j);
    // ===================================================== all 8 warps: warp half h owns keys [32h, 32h + 32) of
    // each block and output columns [h D/2, (h + 1) D/2) of its lane quarter's rows (thread = query row)
    float m = -INFINITY, l = 0.f;  // running max (both halves agree), this half's running sum
    float o[D / 2];
#pragma unroll
    for (int jj = 0; jj < D / 2; ++jj) o[jj] = 0.f;
    for (int j = 0; j < nblk; ++j) {
      const int b = j & 1;
      const int64_t k0 = (int64_t)j * BN;
      tc::mbar_wait(bar_s + b, take(cs0, cs1, b));
      tc::tc_fence_after();
      const uint32_t ts = t_s0 + b * 64;
      uint32_t sr[32];
      tc::tmem_ld32(ts + lane_off + 32 * half, sr);
      tc::tmem_wait_ld();
      float s[32];
      float mx = -INFINITY;
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) {
        s[jj] = (k0 + 32 * half + jj < nv) ? __uint_as_float(sr[jj]) * scale_log2 : -INFINITY;
        mx = fmaxf(mx, s[jj]);
      }
      mx_s[half * BM + row] = mx;
      asm volatile("bar.sync 1, 256;" ::: "memory");  // both halves' maxima; every S column is read before P lands
      const float mn = fmaxf(m, fmaxf(mx, mx_s[(half ^ 1) * BM + row]));  // finite: the block has a valid key
      const float alpha = (m == -INFINITY) ? 0.f : exp2f(m - mn);
      float ps = 0.f;
      uint32_t p1[16], p2[16], p3[16];
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        const float a = exp2f(s[2 * jj] - mn), bb = exp2f(s[2 * jj + 1] - mn);
        ps += a + bb;
        split3(a, bb, p1[jj], p2[jj], p3[jj]);
      }
      l = l * alpha + ps;
      m = mn;
      tc::tmem_st16(ts + lane_off + 16 * half, p1);               // P1: keys 2c, 2c+1 at column c
      tc::tmem_st16(ts + lane_off + 32 + 16 * half, p2);          // P2 at columns [32, 64)
      tc::tmem_st16(t_p30 + b * 32 + lane_off + 16 * half, p3);   // P3 in its own slot
      tc::tmem_wait_st();
      tc::tc_fence_before();
      tc::mbar_arrive(p_ready);
      if (warp == 0) {  // issuer: PV_j once every P_j is in and O is free
        tc::mbar_wait(p_ready, c_p++ & 1);
        if (j >= 1) tc::mbar_wait(o_free, c_of++ & 1);
        if (j >= 2) tc::mbar_wait(v_ready + b, take(cv0, cv1, b));
        tc::tc_fence_after();
        issue_pv(j);
      }
      if (j + 2 < nblk) {  // K_j is consumed (S_j done): split K_{j+2} into its stage under PV_j
        stage_split3<D, BN>(k + hd, b0, (int64_t)(j + 2) * BN, nv, rs, sbase + L::kK + b * L::kKStage);
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(k_ready + b);
        if (warp == 0) {
          tc::mbar_wait(k_ready + b, take(ck0, ck1, b));
          tc::tc_fence_after();
          issue_s(j + 2);
        }
      }
      tc::mbar_wait(bar_o, c_o++ & 1);
      tc::tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < D / 2; c0 += 32) {
        uint32_t pv[32];
        tc::tmem_ld32(t_o + lane_off + half * (D / 2) + c0, pv);
        tc::tmem_wait_ld();
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) o[c0 + jj] = fmaf(o[c0 + jj], alpha, __uint_as_float(pv[jj]));
      }
      tc::tc_fence_before();
      tc::mbar_arrive(o_free);
      if (j + 2 < nblk) {  // V_j is consumed (PV_j done)
        stage_split3<D, BN>(v + hd, b0, (int64_t)(j + 2) * BN, nv, rs, sbase + L::kV + b * L::kKStage);
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(v_ready + b);
      }
    }
    if (warp == 0 && nblk > 0) tc::mbar_wait(o_free, c_of++ & 1);  // last O read-out: TMEM free next item
    l_s[half * BM + row] = l;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    {
      const float lt = l + l_s[(half ^ 1) * BM + row];
      const int64_t r = q0 + row;
      if (r < seg) {
        const bool ok = r < nv && nblk > 0;
        const float inv = ok ? 1.0f / lt : 0.f;
        float4* dst = reinterpret_cast<float4*>(out + (b0 + r) * rs + hd + half * (D / 2));
#pragma unroll
        for (int jj = 0; jj < D / 2; jj += 4)
          dst[jj / 4] = make_float4(o[jj] * inv, o[jj + 1] * inv, o[jj + 2] * inv, o[jj + 3] * inv);
        if (half == 0) lse[(int64_t)h * total_rows + b0 + r] = ok ? (m + log2f(lt)) * kLn2 : -INFINITY;
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<L::kTmemCols>(tmem);
}


// ------------------------------------------------------------------ fp16 two-piece variant (x2h)
// x = x1 + x2 with x1 = fp16(x s), x2 = fp16(x s - x1) for a power-of-two operand scale s (max |x s| <= 2^14 keeps
// both pieces inside fp16's normal range for all but tiny elements): 11-bit significands leave ~2^-22, so three
// products (x2y1, x1y2, x1y1) give ~5e-7 per product — half the MMAs of the bf16 three-piece split. P <= 1 is scaled
// by 2^14; every scale is undone in fp32 (scores in the softmax's exponent scale, O at the end). V keeps three pieces
// (P V = P1V3 + P2V1 + P1V2 + P1V1) so that a one-key row reproduces its V row exactly, as the reference does.
constexpr float kPScale = 16384.f;
__host__ __device__ constexpr uint32_t idesc_f16_f32(uint32_t M, uint32_t N, bool a_mn_major, bool b_mn_major) {
  return (1u << 4)  // D f32; A, B f16 (format 0)
         | ((a_mn_major ? 1u : 0u) << 15) | ((b_mn_major ? 1u : 0u) << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ float pow2_scale(float amax) {  // 2^(14 - e) with amax < 2^e; 1 for amax == 0
  if (!(amax > 0.f) || !(amax < 3.0e38f)) return 1.f;
  int e;
  frexpf(amax, &e);
  return ldexpf(1.f, 14 - e);
}
__device__ __forceinline__ uint32_t pack_f16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float2 unpack_f16(uint32_t w) {
  return __half22float2(*reinterpret_cast<const __half2*>(&w));
}
__device__ __forceinline__ void split2h(float a, float b, uint32_t& w1, uint32_t& w2) {
  w1 = pack_f16(a, b);
  const float2 h = unpack_f16(w1);
  w2 = pack_f16(a - h.x, b - h.y);  // the residuals are exact in fp32
}
__device__ __forceinline__ void split3h(float a, float b, uint32_t& w1, uint32_t& w2, uint32_t& w3) {
  w1 = pack_f16(a, b);
  const float2 h = unpack_f16(w1);
  const float ra = a - h.x, rb = b - h.y;
  w2 = pack_f16(ra, rb);
  const float2 m = unpack_f16(w2);
  w3 = pack_f16(ra - m.x, rb - m.y);  // x1 + x2 + x3 reproduces x exactly (33 significand bits >= 24)
}
template <int D, int ROWS, int NP, int T0 = 0, int NT = kThreads, int kMaxBatch = 4>
__device__ __forceinline__ void stage_splith(const float* __restrict__ src, int64_t b0, int64_t r0, int64_t n,
                                              int64_t rs, uint32_t base, float mul) {
  constexpr int kUnits = D / 8;
  constexpr int kPiece = (D / 64) * ROWS * 128;
  constexpr int kTotal = ROWS * kUnits;
  constexpr int kIter = (kTotal + NT - 1) / NT;
  constexpr int kBatch = kIter < kMaxBatch ? kIter : kMaxBatch;
  const int t = (int)threadIdx.x - T0;
#pragma unroll
  for (int i0 = 0; i0 < kIter; i0 += kBatch) {
    float4 a[kBatch], b[kBatch];
#pragma unroll
    for (int i = 0; i < kBatch; ++i) {
      const int e = t + (i0 + i) * NT, r = e / kUnits, u = e % kUnits;
      a[i] = b[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (e < kTotal && r0 + r < n) {
        const float4* p = reinterpret_cast<const float4*>(src + (b0 + r0 + r) * rs + u * 8);
        a[i] = __ldg(p);
        b[i] = __ldg(p + 1);
      }
    }
#pragma unroll
    for (int i = 0; i < kBatch; ++i) {
      const int e = t + (i0 + i) * NT, r = e / kUnits, u = e % kUnits;
      if (e >= kTotal) continue;
      uint32_t w1[4], w2[4], w3[4];
      const float x[8] = {a[i].x, a[i].y, a[i].z, a[i].w, b[i].x, b[i].y, b[i].z, b[i].w};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (NP == 3) split3h(x[2 * c] * mul, x[2 * c + 1] * mul, w1[c], w2[c], w3[c]);
        else split2h(x[2 * c] * mul, x[2 * c + 1] * mul, w1[c], w2[c]);
      }
      const uint32_t off = (u >> 3) * (ROWS * 128) + tc::sw128_offset(r, u & 7);
      tc::st_shared_v4(base + off, w1[0], w1[1], w1[2], w1[3]);
      tc::st_shared_v4(base + kPiece + off, w2[0], w2[1], w2[2], w2[3]);
      if (NP == 3) tc::st_shared_v4(base + 2 * kPiece + off, w3[0], w3[1], w3[2], w3[3]);
    }
  }
}
// this thread's half row, two fp16 pieces into TMEM (piece p at t_base + p*D/2)
template <int D>
__device__ __forceinline__ void stage_row_tmem2h(const float* __restrict__ src, bool in, uint32_t t_base,
                                                 uint32_t lane_off, int half, float mul) {
  constexpr int kCols = D / 4;
  float4 xs[D / 8];
#pragma unroll
  for (int g = 0; g < D / 8; ++g) {
    xs[g] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (in) xs[g] = __ldg(reinterpret_cast<const float4*>(src + half * (D / 2) + 4 * g));
  }
#pragma unroll
  for (int c0 = 0; c0 < kCols; c0 += 8) {
    uint32_t w[2][8];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const float4 x = xs[c0 / 2 + g];
      split2h(x.x * mul, x.y * mul, w[0][2 * g], w[1][2 * g]);
      split2h(x.z * mul, x.w * mul, w[0][2 * g + 1], w[1][2 * g + 1]);
    }
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const uint32_t ta = t_base + p * (D / 2) + half * kCols + c0 + lane_off;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta),
                   "r"(w[p][0]), "r"(w[p][1]), "r"(w[p][2]), "r"(w[p][3]), "r"(w[p][4]), "r"(w[p][5]), "r"(w[p][6]),
                   "r"(w[p][7])
                   : "memory");
    }
  }
}
template <int D>
struct Lay2 {
  static constexpr int kKChunk = BN * 128;
  static constexpr int kKPiece = (D / 64) * kKChunk;
  static constexpr int kKStage = 2 * kKPiece;          // K1 K2 of one 64-key block
  static constexpr int kVStage = 3 * kKPiece;          // V1 V2 V3 (three pieces: P = 1 reproduces V exactly)
  static constexpr int kK = 0;
  static constexpr int kV = kK + 2 * kKStage;
  static constexpr int kBar = kV + 2 * kVStage;
  static constexpr int kAlpha = kBar + 128;
  static constexpr int kL = kAlpha + 2 * 4 * BM;
  static constexpr int kBytes = kL + 2 * 4 * BM;
  static constexpr int kAlloc = kBytes + 1024;
  // TMEM: Q1 Q2 [0, D) | S0 | S1 (64 each; P1 | P2 land over them) | O (D)
  static constexpr int kTmemCols = D == 128 ? 512 : 256;
};

// Delta = rowsum(dO * O) in fp64 (as attn_delta_kernel) fused with max |dO| into amax_go (the x2h scales)
__global__ void delta_amax_kernel(int64_t units, int D, const float* __restrict__ go, const float* __restrict__ o,
                                  int H, int64_t total_rows, float* __restrict__ delta, unsigned* __restrict__ amax_go) {
  const int lane = threadIdx.x & 31;
  float mx = 0.f;
  for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < units;
       u += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t r = u / H;
    const int h = (int)(u - r * H);
    const int64_t base = u * D;
    double acc = 0.0;
    for (int d = lane; d < D; d += 32) {
      const float g = go[base + d];
      mx = fmaxf(mx, fabsf(g));
      acc = fma((double)g, (double)o[base + d], acc);
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
    if (lane == 0) delta[(int64_t)h * total_rows + r] = (float)acc;
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, s));
  if (lane == 0 && mx > 0.f) atomicMax(amax_go, __float_as_uint(mx));
}

// max |x| of up to three fp32 tensors of n elements (n % 4 == 0) into amax[0..2] (zeroed; floats as ordered ints)
__global__ void absmax3_kernel(const float4* __restrict__ a, const float4* __restrict__ b, const float4* __restrict__ c,
                               int64_t n4, unsigned* __restrict__ amax) {
  const float4* src[3] = {a, b, c};
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    if (!src[t]) continue;
    float m = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
      const float4 x = __ldg(src[t] + i);
      m = fmaxf(m, fmaxf(fmaxf(fabsf(x.x), fabsf(x.y)), fmaxf(fabsf(x.z), fabsf(x.w))));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(amax + t, __float_as_uint(m));
  }
}

template <int D>
__global__ void __launch_bounds__(kFwdThreads, 1) attn_fwd_x2h_kernel(
    const int64_t* __restrict__ off, const int2* __restrict__ items, const int64_t* __restrict__ n_items, int H,
    int64_t total_rows, const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
    float* __restrict__ out, float* __restrict__ lse, float scale_log2, const int64_t* __restrict__ valid,
    const float* __restrict__ amax) {
  using L = Lay2<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = tc::smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* bar_s = bars;        // [2] score MMAs of the buffer done (commit)
  uint64_t* bar_o = bars + 2;    // PV_j done (commit)
  uint64_t* p_ready = bars + 3;  // P_j written (256 arrivals)
  uint64_t* o_free = bars + 4;   // O read out (256 arrivals)
  uint64_t* k_ready = bars + 5;  // [2] K stage split (256 arrivals)
  uint64_t* v_ready = bars + 7;  // [2] V stage split (256 arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);
  float* mx_s = reinterpret_cast<float*>(smem + L::kAlpha);  // [2][128] block maxima of the two key halves
  float* l_s = reinterpret_cast<float*>(smem + L::kL);       // [2][128] final row sums of the two halves
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane;
  if (tid == 0) {
    for (int i = 0; i < 3; ++i) tc::mbar_init(bars + i, 1);
    for (int i = 3; i < 9; ++i) tc::mbar_init(bars + i, 256);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc<L::kTmemCols>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_q = tmem, t_s0 = tmem + D, t_o = t_s0 + 128;
  // power-of-two operand scales (fp16 range: max |x s| <= 2^14), P scaled by 2^14
  const float sq = pow2_scale(amax[0]), sk = pow2_scale(amax[1]), sv = pow2_scale(amax[2]);
  const float s_log2 = scale_log2 / (sq * sk);
  const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
  constexpr uint32_t kIdescS = idesc_f16_f32(BM, BN, false, false);
  constexpr uint32_t kIdescO = idesc_f16_f32(BM, D, false, true);
  const int64_t rs = (int64_t)H * D;
  const int64_t n_work = *n_items * H;
  // barrier use counters (each role tracks the completions it waits for; all are CTA-global across items)
  // (per-parity counters as scalars: a dynamically indexed pair would live in local memory)
  uint32_t cs0 = 0, cs1 = 0, c_o = 0, c_p = 0, c_of = 0, ck0 = 0, ck1 = 0, cv0 = 0, cv1 = 0;
  auto take = [](uint32_t& c0, uint32_t& c1, int b) {  // parity of the next completion of buffer b's barrier
    const uint32_t v = b ? c1 : c0;
    if (b) ++c1; else ++c0;
    return v & 1u;
  };
  for (int64_t w = blockIdx.x; w < n_work; w += gridDim.x) {
    const int2 it = items[w / H];
    const int h = (int)(w % H);
    const int64_t hd = (int64_t)h * D;
    const int64_t b0 = off[it.x], seg = off[it.x + 1] - b0;
    const int64_t nv = valid ? (valid[it.x] < seg ? valid[it.x] : seg) : seg;
    const int q0 = it.y * BM;
    const int nblk = q0 < nv ? (int)((nv + BN - 1) / BN) : 0;  // an all-padding tile attends nothing
    __syncthreads();  // the previous item's TMEM / smem reads are done
    if (nblk > 0) {  // Q pieces -> TMEM; blocks 0 and 1 -> stages 0 and 1
      stage_row_tmem2h<D>(q + (b0 + q0 + row) * rs + hd, q0 + row < seg, t_q, lane_off, half, sq);
      for (int j = 0; j < 2 && j < nblk; ++j) {
        stage_splith<D, BN, 2>(k + hd, b0, (int64_t)j * BN, nv, rs, sbase + L::kK + j * L::kKStage, sk);
        stage_splith<D, BN, 3>(v + hd, b0, (int64_t)j * BN, nv, rs, sbase + L::kV + j * L::kVStage, sv);
      }
    }
    tc::tmem_wait_st();
    tc::fence_proxy_async_smem();
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    // warp 0 doubles as the MMA issuer (a ninth warp would not fit the per-SMSP register file at this size)
    auto issue_s = [&](int j) {  // S = Q2K1 + Q1K2 + Q1K1 (small terms first)
      constexpr int kQi[3] = {1, 0, 0}, kKj[3] = {0, 1, 0};
      const uint32_t kst = sbase + L::kK + (j & 1) * L::kKStage, ts = t_s0 + (j & 1) * 64;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const uint32_t ka = kst + kKj[c] * L::kKPiece;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          tc::mma_bf16_ts_warp(ts, t_q + kQi[c] * (D / 2) + kk * 8,
                               tc::sw128_desc(ka + (kk >> 2) * L::kKChunk + (kk & 3) * 32, 16, 1024), kIdescS,
                               (c > 0 || kk > 0) ? 1u : 0u);
      }
      tc::mma_commit_warp(bar_s + (j & 1));
    };
    auto issue_pv = [&](int j) {  // O_j = P1V3 + P2V1 + P1V2 + P1V1 (V MN-major; small terms first)
      constexpr int kPi[4] = {0, 1, 0, 0}, kVj[4] = {2, 0, 1, 0};
      const int b = j & 1;
      const uint32_t vst = sbase + L::kV + b * L::kVStage, ts = t_s0 + b * 64;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t va = vst + kVj[c] * L::kKPiece;
        const uint32_t pa = ts + kPi[c] * 32;
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk)
          tc::mma_bf16_ts_warp(t_o, pa + kk * 8, tc::sw128_desc(va + kk * 16 * 128, L::kKChunk, 1024), kIdescO,
                               (c > 0 || kk > 0) ? 1u : 0u);
      }
      tc::mma_commit_warp(bar_o);
    };
    if (warp == 0)
      for (int j = 0; j < 2 && j < nblk; ++j) issue_s(j);
    // ===================================================== all 8 warps: warp half h owns keys [32h, 32h + 32) of
    // each block and output columns [h D/2, (h + 1) D/2) of its lane quarter's rows (thread = query row)
    float m = -INFINITY, l = 0.f;  // running max (both halves agree), this half's running sum
    float o[D / 2];
#pragma unroll
    for (int jj = 0; jj < D / 2; ++jj) o[jj] = 0.f;
    for (int j = 0; j < nblk; ++j) {
      const int b = j & 1;
      const int64_t k0 = (int64_t)j * BN;
      tc::mbar_wait(bar_s + b, take(cs0, cs1, b));
      tc::tc_fence_after();
      const uint32_t ts = t_s0 + b * 64;
      uint32_t sr[32];
      tc::tmem_ld32(ts + lane_off + 32 * half, sr);
      tc::tmem_wait_ld();
      float s[32];
      float mx = -INFINITY;
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) {
        s[jj] = (k0 + 32 * half + jj < nv) ? __uint_as_float(sr[jj]) * s_log2 : -INFINITY;
        mx = fmaxf(mx, s[jj]);
      }
      mx_s[half * BM + row] = mx;
      asm volatile("bar.sync 1, 256;" ::: "memory");  // both halves' maxima; every S column is read before P lands
      const float mn = fmaxf(m, fmaxf(mx, mx_s[(half ^ 1) * BM + row]));  // finite: the block has a valid key
      const float alpha = (m == -INFINITY) ? 0.f : exp2f(m - mn);
      float ps = 0.f;
      uint32_t p1[16], p2[16];
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        const float a = exp2f(s[2 * jj] - mn), bb = exp2f(s[2 * jj + 1] - mn);
        ps += a + bb;
        split2h(a * kPScale, bb * kPScale, p1[jj], p2[jj]);
      }
      l = l * alpha + ps;
      m = mn;
      tc::tmem_st16(ts + lane_off + 16 * half, p1);               // P1: keys 2c, 2c+1 at column c
      tc::tmem_st16(ts + lane_off + 32 + 16 * half, p2);          // P2 at columns [32, 64)
      tc::tmem_wait_st();
      tc::tc_fence_before();
      tc::mbar_arrive(p_ready);
      if (warp == 0) {  // issuer: PV_j once every P_j is in and O is free
        tc::mbar_wait(p_ready, c_p++ & 1);
        if (j >= 1) tc::mbar_wait(o_free, c_of++ & 1);
        if (j >= 2) tc::mbar_wait(v_ready + b, take(cv0, cv1, b));
        tc::tc_fence_after();
        issue_pv(j);
      }
      if (j + 2 < nblk) {  // K_j is consumed (S_j done): split K_{j+2} into its stage under PV_j
        stage_splith<D, BN, 2>(k + hd, b0, (int64_t)(j + 2) * BN, nv, rs, sbase + L::kK + b * L::kKStage, sk);
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(k_ready + b);
        if (warp == 0) {
          tc::mbar_wait(k_ready + b, take(ck0, ck1, b));
          tc::tc_fence_after();
          issue_s(j + 2);
        }
      }
      tc::mbar_wait(bar_o, c_o++ & 1);
      tc::tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < D / 2; c0 += 32) {
        uint32_t pv[32];
        tc::tmem_ld32(t_o + lane_off + half * (D / 2) + c0, pv);
        tc::tmem_wait_ld();
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) o[c0 + jj] = fmaf(o[c0 + jj], alpha, __uint_as_float(pv[jj]));
      }
      tc::tc_fence_before();
      tc::mbar_arrive(o_free);
      if (j + 2 < nblk) {  // V_j is consumed (PV_j done)
        stage_splith<D, BN, 3>(v + hd, b0, (int64_t)(j + 2) * BN, nv, rs, sbase + L::kV + b * L::kVStage, sv);
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(v_ready + b);
      }
    }
    if (warp == 0 && nblk > 0) tc::mbar_wait(o_free, c_of++ & 1);  // last O read-out: TMEM free next item
    l_s[half * BM + row] = l;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    {
      const float lt = l + l_s[(half ^ 1) * BM + row];
      const int64_t r = q0 + row;
      if (r < seg) {
        const bool ok = r < nv && nblk > 0;
        const float inv = ok ? 1.0f / (lt * kPScale * sv) : 0.f;
        float4* dst = reinterpret_cast<float4*>(out + (b0 + r) * rs + hd + half * (D / 2));
#pragma unroll
        for (int jj = 0; jj < D / 2; jj += 4)
          dst[jj / 4] = make_float4(o[jj] * inv, o[jj + 1] * inv, o[jj + 2] * inv, o[jj + 3] * inv);
        if (half == 0) lse[(int64_t)h * total_rows + b0 + r] = ok ? (m + log2f(lt)) * kLn2 : -INFINITY;
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<L::kTmemCols>(tmem);
}

template <int D>
static jg_status fwd_x3(const int64_t* off, int64_t total_rows, int H, const void* q, const void* k, const void* v,
                        void* out, float* lse, const int2* items, const int64_t* n_items, int64_t max_items,
                        const int64_t* valid, cudaStream_t st) {
  static const bool bf16x3 = std::getenv("JG_FP32_X3") != nullptr;  // A/B knob: the bf16 three-piece kernels
  if (!bf16x3) {  // fp16 two-piece kernels with per-tensor power-of-two scales from one max pass
    const int smem2 = Lay2<D>::kAlloc;
    if (jg_status rc = ensure_smem_attr((const void*)attn_fwd_x2h_kernel<D>, std::max(smem2, 120 * 1024),
                                        "attn_fwd_x2h_kernel"))
      return rc;
    unsigned* amax = nullptr;
    JG_CUDA(cudaMallocAsync(&amax, 16, st));
    scratch_note(16);
    JG_CUDA(cudaMemsetAsync(amax, 0, 16, st));
    const int64_t n4 = total_rows * H * D / 4;
    absmax3_kernel<<<(int)std::max<int64_t>(1, std::min<int64_t>((n4 + 255) / 256, 4 * device_sm_count())), 256, 0,
                     st>>>((const float4*)q, (const float4*)k, (const float4*)v, n4, amax);
    JG_LAUNCHED("absmax3_kernel");
    const int grid2 = (int)std::max<int64_t>(1, std::min<int64_t>(max_items * H, (int64_t)device_sm_count()));
    attn_fwd_x2h_kernel<D><<<grid2, kFwdThreads, std::max(smem2, 120 * 1024), st>>>(
        off, items, n_items, H, total_rows, (const float*)q, (const float*)k, (const float*)v, (float*)out, lse,
        kLog2e / sqrtf((float)D), valid, (const float*)amax);
    JG_LAUNCHED("attn_fwd_x2h_kernel");
    cudaFreeAsync(amax, st);
    scratch_note(-16);
    return JG_OK;
  }
  const int smem = Lay<D>::kAlloc;
  if (jg_status rc = ensure_smem_attr((const void*)attn_fwd_x3_kernel<D>, std::max(smem, 120 * 1024),
                                      "attn_fwd_x3_kernel"))
    return rc;
  // one CTA per SM (all 512 TMEM columns)
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(max_items * H, (int64_t)device_sm_count()));
  attn_fwd_x3_kernel<D><<<grid, kFwdThreads, std::max(smem, 120 * 1024), st>>>(off, items, n_items, H, total_rows, (const float*)q,
                                                       (const float*)k, (const float*)v, (float*)out, lse,
                                                       kLog2e / sqrtf((float)D), valid);
  JG_LAUNCHED("attn_fwd_x3_kernel");
  return JG_OK;
}

// ------------------------------------------------------------------ backward (attention.cpp:227-289)
// Two deterministic passes, like the FFMA kernels: query-stationary dQ, key-stationary dK / dV; every product is
// the six-MMA split-bf16 sum. Operands are split on the fly from fp32 (no scratch beyond the backward workspace: the
// SPEC.md:316 peak-intermediate bound); the stationary operand of the TS-form score MMAs lives in TMEM.
//   dQ pass   TMEM: Q1 Q2 Q3 [0, 3D/2) | S [3D/2, +64) | dP [+64) | dQ [+D) ; smem: dO pieces, K_j, V_j pieces
//             S = Q K_j^T (TS), dP = dO V_j^T (SS); dS = P (dP - Delta) -> TMEM over S / dP; dQ += dS K_j (TS,
//             K_j read MN-major from the same staging). dS is formed on both warpgroups (32 keys each); V_{j+1}
//             is split under the dQ MMA, K_{j+1} after it.
//   dK/dV pass TMEM: K1 K2 [0, D) | S^T [D, +64) | dP^T [+64) | dV [+D) | dK [+D) ; smem: K3, V pieces, Q_j, dO_j
//             S^T = K Q_j^T (TS for K1, K2; SS for K3), dP^T = V dO_j^T (SS); P^T -> TMEM, dV += P^T dO_j;
//             dS^T -> TMEM, dK += dS^T Q_j. The elementwise work runs on both warpgroups (32 queries each); dO_{j+1}
//             is split under the dK MMA, Q_{j+1} after it.
template <int D, bool KV>
struct BwdLay {
  static constexpr int kXChunk = BM * 128, kYChunk = BN * 128;
  static constexpr int kXPiece = (D / 64) * kXChunk, kYPiece = (D / 64) * kYChunk;
  // dQ pass: X = dO (3 pieces); dK/dV pass: X = K3 then V1 V2 V3 (stationary)
  static constexpr int kX = 0;
  static constexpr int kXn = KV ? 4 : 3;
  static constexpr int kYa = kX + kXn * kXPiece;        // K_j (dQ pass) or Q_j (dK/dV pass), 3 pieces
  static constexpr int kYb = kYa + 3 * kYPiece;         // V_j or dO_j, 3 pieces
  static constexpr int kBar = kYb + 3 * kYPiece;        // bar_s, bar_o, tmem slot
  static constexpr int kLs = kBar + 64;                 // float[64] lse*log2e of the moving block (dK/dV pass)
  static constexpr int kDs = kLs + 4 * BN;              // float[64] Delta
  static constexpr int kBytes = kDs + 4 * BN;
  static constexpr int kAlloc = kBytes + 1024;
};

// The backward's gradient accumulators restart in TMEM every kFlush moving blocks and are added into the fp32
// output rows (owned by this item: no races, fixed order) — the tensor core's truncating fp32 accumulation would
// otherwise lose ~2^-23 of the running sum per MMA over thousands of MMAs (measured 5e-6 norm-wise at 1,500 rows).
constexpr int kFlush = 4;
constexpr int kFlushQ = 16;  // x2h dQ pass: two alternating accumulators, each flushed after 8 of its blocks
constexpr int kFlushH = 8;  // fp16 two-piece kernels: 3 MMAs per product, so twice the blocks per flush for the same drift

// tcgen05.ld is warp-collective (.sync.aligned): every lane loads, only rows inside the segment store.
// dst (+)= scale * acc (add = false: the first flush of the item stores).
template <int D>
__device__ __forceinline__ void ld_half_flush(uint32_t t_acc, uint32_t lane_off, int half, float* __restrict__ dst,
                                              float scale, bool add, bool store) {
  float4* d4 = reinterpret_cast<float4*>(dst + half * (D / 2));
  float4 y[D / 8];  // the previous partial sums: every load in flight before any store
#pragma unroll
  for (int q = 0; q < D / 8; ++q) y[q] = (add && store) ? d4[q] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int c0 = 0; c0 < D / 2; c0 += 32) {
    uint32_t r[32];
    tc::tmem_ld32(t_acc + lane_off + half * (D / 2) + c0, r);
    tc::tmem_wait_ld();
    if (!store) continue;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int jj = 4 * q;
      const float4 o = y[c0 / 4 + q];
      d4[c0 / 4 + q] = make_float4(fmaf(__uint_as_float(r[jj]), scale, o.x), fmaf(__uint_as_float(r[jj + 1]), scale, o.y),
                                   fmaf(__uint_as_float(r[jj + 2]), scale, o.z), fmaf(__uint_as_float(r[jj + 3]), scale, o.w));
    }
  }
}

// dst (+)= scale * (acc0 + acc1) (acc1 only when it was written in this flush group)
template <int D>
__device__ __forceinline__ void ld_half_flush2(uint32_t t_a, uint32_t t_b, bool use_b, uint32_t lane_off, int half,
                                               float* __restrict__ dst, float scale, bool add, bool store) {
  float4* d4 = reinterpret_cast<float4*>(dst + half * (D / 2));
  float4 y[D / 8];
#pragma unroll
  for (int q = 0; q < D / 8; ++q) y[q] = (add && store) ? d4[q] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int c0 = 0; c0 < D / 2; c0 += 32) {
    uint32_t ra[32], rb[32];
    tc::tmem_ld32(t_a + lane_off + half * (D / 2) + c0, ra);
    tc::tmem_ld32(t_b + lane_off + half * (D / 2) + c0, rb);
    tc::tmem_wait_ld();
    if (!store) continue;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int jj = 4 * q;
      float v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        v[e] = __uint_as_float(ra[jj + e]) + (use_b ? __uint_as_float(rb[jj + e]) : 0.f);
      const float4 o = y[c0 / 4 + q];
      d4[c0 / 4 + q] = make_float4(fmaf(v[0], scale, o.x), fmaf(v[1], scale, o.y), fmaf(v[2], scale, o.z),
                                   fmaf(v[3], scale, o.w));
    }
  }
}

// zero rows (an item whose rows all lie past the valid length)
template <int D>
__device__ __forceinline__ void zero_half(float* __restrict__ dst, int half) {
  float4* d4 = reinterpret_cast<float4*>(dst + half * (D / 2));
#pragma unroll
  for (int j = 0; j < D / 8; ++j) d4[j] = make_float4(0.f, 0.f, 0.f, 0.f);
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1) attn_bwd_x3_dq_kernel(
    const int64_t* __restrict__ off, const int2* __restrict__ items, const int64_t* __restrict__ n_items, int H,
    int64_t total_rows, const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
    const float* __restrict__ go, const float* __restrict__ lse, const float* __restrict__ delta,
    float* __restrict__ dq, float scale_log2, float scale, const int64_t* __restrict__ valid) {
  using L = BwdLay<D, false>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = tc::smem_u32(smem);
  uint64_t* bar_s = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* bar_o = bar_s + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_s + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane;
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) tc::mbar_init(bar_s + i, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_q = tmem, t_s = tmem + 3 * D / 2, t_dp = t_s + 64, t_dq = t_dp + 64;
  const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
  constexpr uint32_t kIdescS = tc::idesc_bf16_f32(BM, BN, false, false);
  constexpr uint32_t kIdescQ = tc::idesc_bf16_f32(BM, D, false, true);
  constexpr int kPa[6] = {2, 1, 0, 1, 0, 0}, kPb[6] = {0, 1, 2, 0, 1, 0};
  const int64_t rs = (int64_t)H * D;
  const int64_t n_work = *n_items * H;
  uint32_t ph = 0;
  for (int64_t w = blockIdx.x; w < n_work; w += gridDim.x) {
    const int2 it = items[w / H];
    const int h = (int)(w % H);
    const int64_t hd = (int64_t)h * D, hr = (int64_t)h * total_rows;
    const int64_t b0 = off[it.x], seg = off[it.x + 1] - b0;
    const int64_t nv = valid ? (valid[it.x] < seg ? valid[it.x] : seg) : seg;
    const int q0 = it.y * BM;
    const int64_t r = q0 + row;
    const bool rin = r < nv;
    const int nblk = q0 < nv ? (int)((nv + BN - 1) / BN) : 0;
    float lr = 0.f, dr = 0.f;
    if (rin) {
      lr = lse[hr + b0 + r] * kLog2e;
      dr = delta[hr + b0 + r];
    }
    __syncthreads();  // previous item: TMEM dQ read, smem free
    if (nblk > 0) {  // Q pieces -> TMEM; dO pieces, K_0, V_0 -> smem (K_0 / V_0 loads in flight throughout)
      Pre<D, BN> k0p, v0p;
      k0p.load(k + hd, b0, 0, nv, rs, tid);
      v0p.load(v + hd, b0, 0, nv, rs, tid);
      stage_row_tmem<D, 3>(q + (b0 + r) * rs + hd, rin, t_q, lane_off, half, row, 0);
      stage_split3<D, BM, 0, kThreads, 8>(go + hd, b0, q0, nv, rs, sbase + L::kX);
      k0p.store(sbase + L::kYa, tid);
      v0p.store(sbase + L::kYb, tid);
    }
    for (int j = 0; j < nblk; ++j) {
      const int64_t k0 = (int64_t)j * BN;
      tc::tmem_wait_st();
      tc::fence_proxy_async_smem();
      tc::tc_fence_before();
      __syncthreads();
      tc::tc_fence_after();
      if (warp == 0) {
#pragma unroll
        for (int c = 0; c < 6; ++c) {  // S = sum Qa Kb^T (A = Q pieces in TMEM)
          const uint32_t kb = sbase + L::kYa + kPb[c] * L::kYPiece;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            tc::mma_bf16_ts_warp(t_s, t_q + kPa[c] * (D / 2) + kk * 8,
                                 tc::sw128_desc(kb + (kk >> 2) * L::kYChunk + (kk & 3) * 32, 16, 1024), kIdescS,
                                 (c > 0 || kk > 0) ? 1u : 0u);
        }
#pragma unroll
        for (int c = 0; c < 6; ++c) {  // dP = sum dOa Vb^T
          const uint32_t xa = sbase + L::kX + kPa[c] * L::kXPiece, vb = sbase + L::kYb + kPb[c] * L::kYPiece;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            tc::mma_bf16_ss_warp(t_dp, tc::sw128_desc(xa + (kk >> 2) * L::kXChunk + (kk & 3) * 32, 16, 1024),
                                 tc::sw128_desc(vb + (kk >> 2) * L::kYChunk + (kk & 3) * 32, 16, 1024), kIdescS,
                                 (c > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit_warp(bar_s);
      }
      tc::mbar_wait(bar_s, ph);
      tc::tc_fence_after();
      {  // dS = P (dP - Delta) on both warpgroups: warp half h takes keys [32h, 32h + 32) of its lane quarter
        uint32_t sr[32], pr[32];
        tc::tmem_ld32(t_s + lane_off + 32 * half, sr);
        tc::tmem_ld32(t_dp + lane_off + 32 * half, pr);
        tc::tmem_wait_ld();
        asm volatile("bar.sync 1, 256;" ::: "memory");  // every S / dP column is read before the pieces overwrite them
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
          const bool in = rin && (k0 + 32 * half + jj < nv);
          const float p = in ? exp2f(__uint_as_float(sr[jj]) * scale_log2 - lr) : 0.f;
          sr[jj] = __float_as_uint(p * (__uint_as_float(pr[jj]) - dr));
        }
        // dS1 over S [0, 32), dS2 over S [32, 64), dS3 over dP [0, 32): keys 32h.. packed at column 16h
        uint32_t w1[16], w2[16], w3[16];
#pragma unroll
        for (int jj = 0; jj < 32; jj += 2)
          split3(__uint_as_float(sr[jj]), __uint_as_float(sr[jj + 1]), w1[jj / 2], w2[jj / 2], w3[jj / 2]);
        tc::tmem_st16(t_s + lane_off + 16 * half, w1);
        tc::tmem_st16(t_s + lane_off + 32 + 16 * half, w2);
        tc::tmem_st16(t_dp + lane_off + 16 * half, w3);
        tc::tmem_wait_st();
      }
      tc::tc_fence_before();
      __syncthreads();
      tc::tc_fence_after();
      if (warp == 0) {  // dQ += sum dSa Kb (B = K_j MN-major: key rows, 64-wide D chunks)
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          const uint32_t pa = kPa[c] == 2 ? t_dp : t_s + kPa[c] * 32;
          const uint32_t kb = sbase + L::kYa + kPb[c] * L::kYPiece;
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk)
            tc::mma_bf16_ts_warp(t_dq, pa + kk * 8, tc::sw128_desc(kb + kk * 16 * 128, L::kYChunk, 1024), kIdescQ,
                                 (j % kFlush != 0 || c > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit_warp(bar_o);
      }
      Pre<D, BN> kpre;
      if (j + 1 < nblk) {  // under dQ_j: split V_{j+1} (V_j is free) and load K_{j+1}
        stage_split3<D, BN>(v + hd, b0, k0 + BN, nv, rs, sbase + L::kYb);
        kpre.load(k + hd, b0, k0 + BN, nv, rs, tid);
      }
      tc::mbar_wait(bar_o, ph);
      tc::tc_fence_after();
      if (j + 1 < nblk) kpre.store(sbase + L::kYa, tid);  // K_j is free
      if (j % kFlush == kFlush - 1 || j + 1 == nblk)
        ld_half_flush<D>(t_dq, lane_off, half, dq + (b0 + r) * rs + hd, scale, j >= kFlush, r < seg);
      tc::tc_fence_before();
      ph ^= 1;
    }
    if (nblk == 0 && r < seg) zero_half<D>(dq + (b0 + r) * rs + hd, half);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}


// fp16-piece variants of the backward's staging (x2h)
template <int D, int ROWS, int NP, int NT = kThreads>
struct PreH {
  static constexpr int kUnits = D / 8, kTotal = ROWS * kUnits, kIter = kTotal / NT;
  static constexpr int kPiece = (D / 64) * ROWS * 128;
  float4 a[kIter], b[kIter];
  __device__ __forceinline__ void load(const float* __restrict__ src, int64_t b0, int64_t r0, int64_t n, int64_t rs,
                                       int t) {
#pragma unroll
    for (int i = 0; i < kIter; ++i) {
      const int e = t + i * NT, r = e / kUnits, u = e % kUnits;
      a[i] = b[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r0 + r < n) {
        const float4* p = reinterpret_cast<const float4*>(src + (b0 + r0 + r) * rs + u * 8);
        a[i] = __ldg(p);
        b[i] = __ldg(p + 1);
      }
    }
  }
  __device__ __forceinline__ void store(uint32_t base, int t, float mul) const {
#pragma unroll
    for (int i = 0; i < kIter; ++i) {
      const int e = t + i * NT, r = e / kUnits, u = e % kUnits;
      uint32_t w1[4], w2[4], w3[4];
      const float x[8] = {a[i].x, a[i].y, a[i].z, a[i].w, b[i].x, b[i].y, b[i].z, b[i].w};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (NP == 3) split3h(x[2 * c] * mul, x[2 * c + 1] * mul, w1[c], w2[c], w3[c]);
        else split2h(x[2 * c] * mul, x[2 * c + 1] * mul, w1[c], w2[c]);
      }
      const uint32_t off = (u >> 3) * (ROWS * 128) + tc::sw128_offset(r, u & 7);
      tc::st_shared_v4(base + off, w1[0], w1[1], w1[2], w1[3]);
      tc::st_shared_v4(base + kPiece + off, w2[0], w2[1], w2[2], w2[3]);
      if (NP == 3) tc::st_shared_v4(base + 2 * kPiece + off, w3[0], w3[1], w3[2], w3[3]);
    }
  }
};
template <int D, bool KV>
struct BwdLay2 {
  static constexpr int kXChunk = BM * 128, kYChunk = BN * 128;
  static constexpr int kXPiece = (D / 64) * kXChunk, kYPiece = (D / 64) * kYChunk;
  static constexpr int kX = 0;                          // dQ pass: dO1 dO2; dK/dV pass: V1 V2 (stationary)
  // two stages of the moving block: [Ya: K_j (dQ pass) or Q_j (dK/dV pass) | Yb: V_j or dO_j], 2 pieces each
  static constexpr int kYa = kX + 2 * kXPiece;
  static constexpr int kYb = kYa + 2 * kYPiece;
  static constexpr int kYStage = 4 * kYPiece;
  static constexpr int kBar = kYa + 2 * kYStage;
  static constexpr int kLs = kBar + 64;
  static constexpr int kDs = kLs + 4 * BN;
  static constexpr int kBytes = kDs + 4 * BN;
  static constexpr int kAlloc = kBytes + 1024;
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1) attn_bwd_x2h_dq_kernel(
    const int64_t* __restrict__ off, const int2* __restrict__ items, const int64_t* __restrict__ n_items, int H,
    int64_t total_rows, const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
    const float* __restrict__ go, const float* __restrict__ lse, const float* __restrict__ delta,
    float* __restrict__ dq, float scale_log2, float scale, const int64_t* __restrict__ valid,
    const float* __restrict__ amax) {
  using L = BwdLay2<D, false>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = tc::smem_u32(smem);
  uint64_t* bar_s = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* bar_o = bar_s + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_s + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane;
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) tc::mbar_init(bar_s + i, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // two dQ accumulators alternate by block (each sees half the MMAs between flushes: half the truncation drift)
  const uint32_t t_q = tmem, t_s = tmem + D, t_dp = t_s + 64, t_dq = t_dp + 64;
  const float sq = pow2_scale(amax[0]), sk = pow2_scale(amax[1]), sv = pow2_scale(amax[2]), sdo = pow2_scale(amax[3]);
  const float sds = pow2_scale(2.f * D * amax[3] * amax[2]);  // |dS| <= 2 max||dO|| max||V||
  const float s_log2 = scale_log2 / (sq * sk), ipd = 1.f / (sdo * sv), fl_scale = scale / (sds * sk);
  const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
  constexpr uint32_t kIdescS = idesc_f16_f32(BM, BN, false, false);
  constexpr uint32_t kIdescQ = idesc_f16_f32(BM, D, false, true);
  constexpr int kPa[3] = {1, 0, 0}, kPb[3] = {0, 1, 0};
  const int64_t rs = (int64_t)H * D;
  const int64_t n_work = *n_items * H;
  uint32_t ph = 0;
  for (int64_t w = blockIdx.x; w < n_work; w += gridDim.x) {
    const int2 it = items[w / H];
    const int h = (int)(w % H);
    const int64_t hd = (int64_t)h * D, hr = (int64_t)h * total_rows;
    const int64_t b0 = off[it.x], seg = off[it.x + 1] - b0;
    const int64_t nv = valid ? (valid[it.x] < seg ? valid[it.x] : seg) : seg;
    const int q0 = it.y * BM;
    const int64_t r = q0 + row;
    const bool rin = r < nv;
    const int nblk = q0 < nv ? (int)((nv + BN - 1) / BN) : 0;
    float lr = 0.f, dr = 0.f;
    if (rin) {
      lr = lse[hr + b0 + r] * kLog2e;
      dr = delta[hr + b0 + r];
    }
    __syncthreads();  // previous item: TMEM dQ read, smem free
    if (nblk > 0) {  // Q pieces -> TMEM; dO pieces, K_0, V_0 -> smem (K_0 / V_0 loads in flight throughout)
      PreH<D, BN, 2> k0p, v0p;
      k0p.load(k + hd, b0, 0, nv, rs, tid);
      v0p.load(v + hd, b0, 0, nv, rs, tid);
      stage_row_tmem2h<D>(q + (b0 + r) * rs + hd, rin, t_q, lane_off, half, sq);
      stage_splith<D, BM, 2, 0, kThreads, 8>(go + hd, b0, q0, nv, rs, sbase + L::kX, sdo);
      k0p.store(sbase + L::kYa, tid, sk);
      v0p.store(sbase + L::kYb, tid, sv);
    }
    for (int j = 0; j < nblk; ++j) {
      const int64_t k0 = (int64_t)j * BN;
      const uint32_t ya = sbase + L::kYa + (j & 1) * L::kYStage, yb = sbase + L::kYb + (j & 1) * L::kYStage;
      tc::tmem_wait_st();
      tc::fence_proxy_async_smem();
      tc::tc_fence_before();
      __syncthreads();
      tc::tc_fence_after();
      if (warp == 0) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {  // S = Q2K1 + Q1K2 + Q1K1 (A = Q pieces in TMEM)
          const uint32_t kb = ya + kPb[c] * L::kYPiece;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            tc::mma_bf16_ts_warp(t_s, t_q + kPa[c] * (D / 2) + kk * 8,
                                 tc::sw128_desc(kb + (kk >> 2) * L::kYChunk + (kk & 3) * 32, 16, 1024), kIdescS,
                                 (c > 0 || kk > 0) ? 1u : 0u);
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {  // dP = dO2V1 + dO1V2 + dO1V1
          const uint32_t xa = sbase + L::kX + kPa[c] * L::kXPiece, vb = yb + kPb[c] * L::kYPiece;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            tc::mma_bf16_ss_warp(t_dp, tc::sw128_desc(xa + (kk >> 2) * L::kXChunk + (kk & 3) * 32, 16, 1024),
                                 tc::sw128_desc(vb + (kk >> 2) * L::kYChunk + (kk & 3) * 32, 16, 1024), kIdescS,
                                 (c > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit_warp(bar_s);
      }
      if (j + 1 < nblk) {  // under S_j / dP_j: split K_{j+1}, V_{j+1} into the other stage (dQ_{j-1} released it)
        const uint32_t na = sbase + L::kYa + ((j + 1) & 1) * L::kYStage, nb = na + 2 * L::kYPiece;
        PreH<D, BN, 2> vp;
        vp.load(v + hd, b0, k0 + BN, nv, rs, tid);
        stage_splith<D, BN, 2>(k + hd, b0, k0 + BN, nv, rs, na, sk);
        vp.store(nb, tid, sv);
      }
      tc::mbar_wait(bar_s, ph);
      tc::tc_fence_after();
      {  // dS = P (dP - Delta) on both warpgroups: warp half h takes keys [32h, 32h + 32) of its lane quarter
        uint32_t sr[32], pr[32];
        tc::tmem_ld32(t_s + lane_off + 32 * half, sr);
        tc::tmem_ld32(t_dp + lane_off + 32 * half, pr);
        tc::tmem_wait_ld();
        asm volatile("bar.sync 1, 256;" ::: "memory");  // every S / dP column is read before the pieces overwrite them
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
          const bool in = rin && (k0 + 32 * half + jj < nv);
          const float p = in ? exp2f(__uint_as_float(sr[jj]) * s_log2 - lr) : 0.f;
          sr[jj] = __float_as_uint(p * (__uint_as_float(pr[jj]) * ipd - dr) * sds);
        }
        // dS1 over S [0, 32), dS2 over S [32, 64): keys 32h.. packed at column 16h
        uint32_t w1[16], w2[16];
#pragma unroll
        for (int jj = 0; jj < 32; jj += 2)
          split2h(__uint_as_float(sr[jj]), __uint_as_float(sr[jj + 1]), w1[jj / 2], w2[jj / 2]);
        tc::tmem_st16(t_s + lane_off + 16 * half, w1);
        tc::tmem_st16(t_s + lane_off + 32 + 16 * half, w2);
        tc::tmem_wait_st();
      }
      tc::tc_fence_before();
      __syncthreads();
      tc::tc_fence_after();
      if (warp == 0) {  // dQ += sum dSa Kb (B = K_j MN-major: key rows, 64-wide D chunks)
#pragma unroll
        for (int c = 0; c < 3; ++c) {  // dQ += dS2K1 + dS1K2 + dS1K1
          const uint32_t pa = t_s + kPa[c] * 32;
          const uint32_t kb = ya + kPb[c] * L::kYPiece;
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk)
            tc::mma_bf16_ts_warp(t_dq + (j & 1) * D, pa + kk * 8, tc::sw128_desc(kb + kk * 16 * 128, L::kYChunk, 1024),
                                 kIdescQ, (j % kFlushQ >= 2 || c > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit_warp(bar_o);
      }
      tc::mbar_wait(bar_o, ph);
      tc::tc_fence_after();
      if (j % kFlushQ == kFlushQ - 1 || j + 1 == nblk)
        ld_half_flush2<D>(t_dq, t_dq + D, j % kFlushQ >= 1, lane_off, half, dq + (b0 + r) * rs + hd, fl_scale,
                          j >= kFlushQ, r < seg);
      tc::tc_fence_before();
      ph ^= 1;
    }
    if (nblk == 0 && r < seg) zero_half<D>(dq + (b0 + r) * rs + hd, half);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}


template <int D>
__global__ void __launch_bounds__(kThreads, 1) attn_bwd_x3_dkdv_kernel(
    const int64_t* __restrict__ off, const int2* __restrict__ items, const int64_t* __restrict__ n_items, int H,
    int64_t total_rows, const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
    const float* __restrict__ go, const float* __restrict__ lse, const float* __restrict__ delta,
    float* __restrict__ dk, float* __restrict__ dv, float scale_log2, float scale, const int64_t* __restrict__ valid) {
  using L = BwdLay<D, true>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = tc::smem_u32(smem);
  uint64_t* bar_s = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* bar_o = bar_s + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_s + 2);
  float* ls = reinterpret_cast<float*>(smem + L::kLs);
  float* dls = reinterpret_cast<float*>(smem + L::kDs);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane;  // key row in the tile
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) tc::mbar_init(bar_s + i, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_k = tmem, t_s = tmem + D, t_dp = t_s + 64, t_dv = t_dp + 64, t_dk = t_dv + D;
  const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
  constexpr uint32_t kIdescS = tc::idesc_bf16_f32(BM, BN, false, false);
  constexpr uint32_t kIdescO = tc::idesc_bf16_f32(BM, D, false, true);
  constexpr int kPa[6] = {2, 1, 0, 1, 0, 0}, kPb[6] = {0, 1, 2, 0, 1, 0};
  const uint32_t s_k3 = sbase + L::kX, s_v = s_k3 + L::kXPiece;
  const int64_t rs = (int64_t)H * D;
  const int64_t n_work = *n_items * H;
  uint32_t ph_s = 0, ph_o = 0;
  for (int64_t w = blockIdx.x; w < n_work; w += gridDim.x) {
    const int2 it = items[w / H];
    const int h = (int)(w % H);
    const int64_t hd = (int64_t)h * D, hr = (int64_t)h * total_rows;
    const int64_t b0 = off[it.x], seg = off[it.x + 1] - b0;
    const int64_t nv = valid ? (valid[it.x] < seg ? valid[it.x] : seg) : seg;
    const int x0 = it.y * BM;
    const int64_t r = x0 + row;
    const bool rin = r < nv;
    const int nblk = x0 < nv ? (int)((nv + BN - 1) / BN) : 0;
    __syncthreads();
    if (nblk > 0) {  // K1, K2 -> TMEM and K3 -> smem; V pieces, Q_0, dO_0 -> smem (Q_0 / dO_0 loads in flight)
      Pre<D, BN> q0p, g0p;
      q0p.load(q + hd, b0, 0, nv, rs, tid);
      g0p.load(go + hd, b0, 0, nv, rs, tid);
      stage_row_tmem<D, 2, true>(k + (b0 + r) * rs + hd, rin, t_k, lane_off, half, row, s_k3);
      stage_split3<D, BM, 0, kThreads, 8>(v + hd, b0, x0, nv, rs, s_v);
      q0p.store(sbase + L::kYa, tid);
      g0p.store(sbase + L::kYb, tid);
    }
    for (int j = 0; j < nblk; ++j) {
      const int64_t y0 = (int64_t)j * BN;
      if (tid < BN) {
        const bool in = y0 + tid < nv;
        ls[tid] = in ? lse[hr + b0 + y0 + tid] * kLog2e : 0.f;
        dls[tid] = in ? delta[hr + b0 + y0 + tid] : 0.f;
      }
      tc::tmem_wait_st();
      tc::fence_proxy_async_smem();
      tc::tc_fence_before();
      __syncthreads();
      tc::tc_fence_after();
      if (warp == 0) {
#pragma unroll
        for (int c = 0; c < 6; ++c) {  // S^T = sum Ka Qb^T (K1, K2 from TMEM; K3 from smem)
          const uint32_t qb = sbase + L::kYa + kPb[c] * L::kYPiece;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t bdesc = tc::sw128_desc(qb + (kk >> 2) * L::kYChunk + (kk & 3) * 32, 16, 1024);
            const uint32_t acc = (c > 0 || kk > 0) ? 1u : 0u;
            if (kPa[c] < 2)
              tc::mma_bf16_ts_warp(t_s, t_k + kPa[c] * (D / 2) + kk * 8, bdesc, kIdescS, acc);
            else
              tc::mma_bf16_ss_warp(t_s, tc::sw128_desc(s_k3 + (kk >> 2) * L::kXChunk + (kk & 3) * 32, 16, 1024),
                                   bdesc, kIdescS, acc);
          }
        }
#pragma unroll
        for (int c = 0; c < 6; ++c) {  // dP^T = sum Va dOb^T
          const uint32_t va = s_v + kPa[c] * L::kXPiece, ob = sbase + L::kYb + kPb[c] * L::kYPiece;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            tc::mma_bf16_ss_warp(t_dp, tc::sw128_desc(va + (kk >> 2) * L::kXChunk + (kk & 3) * 32, 16, 1024),
                                 tc::sw128_desc(ob + (kk >> 2) * L::kYChunk + (kk & 3) * 32, 16, 1024), kIdescS,
                                 (c > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit_warp(bar_s);
      }
      // P^T and dS^T on both warpgroups: warp half h takes queries [32h, 32h + 32) of its key quarter
      float dsv[32];  // dS^T, split into TMEM once P^T's MMAs are done
      tc::mbar_wait(bar_s, ph_s);
      tc::tc_fence_after();
      {
        uint32_t sr[32], pr[32];
        tc::tmem_ld32(t_s + lane_off + 32 * half, sr);
        tc::tmem_ld32(t_dp + lane_off + 32 * half, pr);
        tc::tmem_wait_ld();
        asm volatile("bar.sync 1, 256;" ::: "memory");  // every S^T / dP^T column is read before the pieces land
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
          const int qc = 32 * half + jj;
          const bool in = rin && (y0 + qc < nv);
          const float p = in ? exp2f(__uint_as_float(sr[jj]) * scale_log2 - ls[qc]) : 0.f;
          dsv[jj] = p * (__uint_as_float(pr[jj]) - dls[qc]);
          sr[jj] = __float_as_uint(p);
        }
        // P1 [0, 32), P2 [32, 64), P3 [64, 96) of t_s; queries 32h.. packed at column 16h
        uint32_t p1[16], p2[16], p3[16];
#pragma unroll
        for (int jj = 0; jj < 32; jj += 2)
          split3(__uint_as_float(sr[jj]), __uint_as_float(sr[jj + 1]), p1[jj / 2], p2[jj / 2], p3[jj / 2]);
        tc::tmem_st16(t_s + lane_off + 16 * half, p1);
        tc::tmem_st16(t_s + lane_off + 32 + 16 * half, p2);
        tc::tmem_st16(t_s + lane_off + 64 + 16 * half, p3);
        tc::tmem_wait_st();
      }
      tc::tc_fence_before();
      __syncthreads();
      tc::tc_fence_after();
      if (warp == 0) {  // dV += sum P^T_a dO_b (B = dO_j MN-major)
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          const uint32_t ob = sbase + L::kYb + kPb[c] * L::kYPiece;
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk)
            tc::mma_bf16_ts_warp(t_dv, t_s + kPa[c] * 32 + kk * 8, tc::sw128_desc(ob + kk * 16 * 128, L::kYChunk, 1024),
                                 kIdescO, (j % kFlush != 0 || c > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit_warp(bar_o);
      }
      tc::mbar_wait(bar_o, ph_o);  // (all threads) the P^T pieces and dO_j are consumed
      tc::tc_fence_after();
      {
        uint32_t d1[16], d2[16], d3[16];
#pragma unroll
        for (int jj = 0; jj < 32; jj += 2) split3(dsv[jj], dsv[jj + 1], d1[jj / 2], d2[jj / 2], d3[jj / 2]);
        tc::tmem_st16(t_s + lane_off + 16 * half, d1);
        tc::tmem_st16(t_s + lane_off + 32 + 16 * half, d2);
        tc::tmem_st16(t_s + lane_off + 64 + 16 * half, d3);
        tc::tmem_wait_st();
      }
      ph_o ^= 1;
      tc::tc_fence_before();
      __syncthreads();
      tc::tc_fence_after();
      if (warp == 0) {  // dK += sum dS^T_a Q_b (B = Q_j MN-major)
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          const uint32_t qb = sbase + L::kYa + kPb[c] * L::kYPiece;
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk)
            tc::mma_bf16_ts_warp(t_dk, t_s + kPa[c] * 32 + kk * 8, tc::sw128_desc(qb + kk * 16 * 128, L::kYChunk, 1024),
                                 kIdescO, (j % kFlush != 0 || c > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit_warp(bar_o);
      }
      Pre<D, BN> qpre;
      if (j + 1 < nblk) {  // under dK_j: split dO_{j+1} (dO_j is free) and load Q_{j+1}
        stage_split3<D, BN>(go + hd, b0, y0 + BN, nv, rs, sbase + L::kYb);
        qpre.load(q + hd, b0, y0 + BN, nv, rs, tid);
      }
      tc::mbar_wait(bar_o, ph_o);
      tc::tc_fence_after();
      if (j + 1 < nblk) qpre.store(sbase + L::kYa, tid);  // Q_j is free
      if (j % kFlush == kFlush - 1 || j + 1 == nblk) {
        ld_half_flush<D>(t_dv, lane_off, half, dv + (b0 + r) * rs + hd, 1.f, j >= kFlush, r < seg);
        ld_half_flush<D>(t_dk, lane_off, half, dk + (b0 + r) * rs + hd, scale, j >= kFlush, r < seg);
      }
      tc::tc_fence_before();
      ph_o ^= 1;
      ph_s ^= 1;
    }
    if (nblk == 0 && r < seg) {
      zero_half<D>(dv + (b0 + r) * rs + hd, half);
      zero_half<D>(dk + (b0 + r) * rs + hd, half);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1) attn_bwd_x2h_dkdv_kernel(
    const int64_t* __restrict__ off, const int2* __restrict__ items, const int64_t* __restrict__ n_items, int H,
    int64_t total_rows, const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
    const float* __restrict__ go, const float* __restrict__ lse, const float* __restrict__ delta,
    float* __restrict__ dk, float* __restrict__ dv, float scale_log2, float scale, const int64_t* __restrict__ valid,
    const float* __restrict__ amax) {
  using L = BwdLay2<D, true>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = tc::smem_u32(smem);
  uint64_t* bar_s = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* bar_o = bar_s + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_s + 2);
  float* ls = reinterpret_cast<float*>(smem + L::kLs);
  float* dls = reinterpret_cast<float*>(smem + L::kDs);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane;  // key row in the tile
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) tc::mbar_init(bar_s + i, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_k = tmem, t_s = tmem + D, t_dp = t_s + 64, t_dv = t_dp + 64, t_dk = t_dv + D;
  const float sq = pow2_scale(amax[0]), sk = pow2_scale(amax[1]), sv = pow2_scale(amax[2]), sdo = pow2_scale(amax[3]);
  const float sds = pow2_scale(2.f * D * amax[3] * amax[2]);  // |dS| <= 2 max||dO|| max||V||
  const float s_log2 = scale_log2 / (sk * sq), ipd = 1.f / (sv * sdo);
  const float fl_dv = 1.f / (kPScale * sdo), fl_dk = scale / (sds * sq);
  const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
  constexpr uint32_t kIdescS = idesc_f16_f32(BM, BN, false, false);
  constexpr uint32_t kIdescO = idesc_f16_f32(BM, D, false, true);
  constexpr int kPa[3] = {1, 0, 0}, kPb[3] = {0, 1, 0};
  const uint32_t s_v = sbase + L::kX;
  const int64_t rs = (int64_t)H * D;
  const int64_t n_work = *n_items * H;
  uint32_t ph_s = 0, ph_o = 0;
  for (int64_t w = blockIdx.x; w < n_work; w += gridDim.x) {
    const int2 it = items[w / H];
    const int h = (int)(w % H);
    const int64_t hd = (int64_t)h * D, hr = (int64_t)h * total_rows;
    const int64_t b0 = off[it.x], seg = off[it.x + 1] - b0;
    const int64_t nv = valid ? (valid[it.x] < seg ? valid[it.x] : seg) : seg;
    const int x0 = it.y * BM;
    const int64_t r = x0 + row;
    const bool rin = r < nv;
    const int nblk = x0 < nv ? (int)((nv + BN - 1) / BN) : 0;
    __syncthreads();
    if (nblk > 0) {  // K1, K2 -> TMEM and K3 -> smem; V pieces, Q_0, dO_0 -> smem (Q_0 / dO_0 loads in flight)
      PreH<D, BN, 2> q0p, g0p;
      q0p.load(q + hd, b0, 0, nv, rs, tid);
      g0p.load(go + hd, b0, 0, nv, rs, tid);
      stage_row_tmem2h<D>(k + (b0 + r) * rs + hd, rin, t_k, lane_off, half, sk);
      stage_splith<D, BM, 2, 0, kThreads, 8>(v + hd, b0, x0, nv, rs, s_v, sv);
      q0p.store(sbase + L::kYa, tid, sq);
      g0p.store(sbase + L::kYb, tid, sdo);
    }
    for (int j = 0; j < nblk; ++j) {
      const int64_t y0 = (int64_t)j * BN;
      const uint32_t ya = sbase + L::kYa + (j & 1) * L::kYStage, yb = sbase + L::kYb + (j & 1) * L::kYStage;
      if (tid < BN) {
        const bool in = y0 + tid < nv;
        ls[tid] = in ? lse[hr + b0 + y0 + tid] * kLog2e : 0.f;
        dls[tid] = in ? delta[hr + b0 + y0 + tid] : 0.f;
      }
      tc::tmem_wait_st();
      tc::fence_proxy_async_smem();
      tc::tc_fence_before();
      __syncthreads();
      tc::tc_fence_after();
      if (warp == 0) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {  // S^T = K2Q1 + K1Q2 + K1Q1 (K pieces in TMEM)
          const uint32_t qb = ya + kPb[c] * L::kYPiece;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            tc::mma_bf16_ts_warp(t_s, t_k + kPa[c] * (D / 2) + kk * 8,
                                 tc::sw128_desc(qb + (kk >> 2) * L::kYChunk + (kk & 3) * 32, 16, 1024), kIdescS,
                                 (c > 0 || kk > 0) ? 1u : 0u);
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {  // dP^T = V2dO1 + V1dO2 + V1dO1
          const uint32_t va = s_v + kPa[c] * L::kXPiece, ob = yb + kPb[c] * L::kYPiece;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            tc::mma_bf16_ss_warp(t_dp, tc::sw128_desc(va + (kk >> 2) * L::kXChunk + (kk & 3) * 32, 16, 1024),
                                 tc::sw128_desc(ob + (kk >> 2) * L::kYChunk + (kk & 3) * 32, 16, 1024), kIdescS,
                                 (c > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit_warp(bar_s);
      }
      if (j + 1 < nblk) {  // under S^T_j / dP^T_j: split Q_{j+1}, dO_{j+1} into the other stage (dK_{j-1} released it)
        const uint32_t na = sbase + L::kYa + ((j + 1) & 1) * L::kYStage, nb = na + 2 * L::kYPiece;
        PreH<D, BN, 2> gp;
        gp.load(go + hd, b0, y0 + BN, nv, rs, tid);
        stage_splith<D, BN, 2>(q + hd, b0, y0 + BN, nv, rs, na, sq);
        gp.store(nb, tid, sdo);
      }
      // P^T and dS^T on both warpgroups: warp half h takes queries [32h, 32h + 32) of its key quarter
      float dsv[32];  // dS^T, split into TMEM once P^T's MMAs are done
      tc::mbar_wait(bar_s, ph_s);
      tc::tc_fence_after();
      {
        uint32_t sr[32], pr[32];
        tc::tmem_ld32(t_s + lane_off + 32 * half, sr);
        tc::tmem_ld32(t_dp + lane_off + 32 * half, pr);
        tc::tmem_wait_ld();
        asm volatile("bar.sync 1, 256;" ::: "memory");  // every S^T / dP^T column is read before the pieces land
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
          const int qc = 32 * half + jj;
          const bool in = rin && (y0 + qc < nv);
          const float p = in ? exp2f(__uint_as_float(sr[jj]) * s_log2 - ls[qc]) : 0.f;
          dsv[jj] = p * (__uint_as_float(pr[jj]) * ipd - dls[qc]) * sds;
          sr[jj] = __float_as_uint(p * kPScale);
        }
        // P1 [0, 32), P2 [32, 64) of t_s; queries 32h.. packed at column 16h
        uint32_t p1[16], p2[16];
#pragma unroll
        for (int jj = 0; jj < 32; jj += 2)
          split2h(__uint_as_float(sr[jj]), __uint_as_float(sr[jj + 1]), p1[jj / 2], p2[jj / 2]);
        tc::tmem_st16(t_s + lane_off + 16 * half, p1);
        tc::tmem_st16(t_s + lane_off + 32 + 16 * half, p2);
        tc::tmem_wait_st();
      }
      tc::tc_fence_before();
      __syncthreads();
      tc::tc_fence_after();
      if (warp == 0) {  // dV += P2dO1 + P1dO2 + P1dO1 (B = dO_j MN-major)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const uint32_t ob = yb + kPb[c] * L::kYPiece;
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk)
            tc::mma_bf16_ts_warp(t_dv, t_s + kPa[c] * 32 + kk * 8, tc::sw128_desc(ob + kk * 16 * 128, L::kYChunk, 1024),
                                 kIdescO, (j % kFlushH != 0 || c > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit_warp(bar_o);
      }
      tc::mbar_wait(bar_o, ph_o);  // (all threads) the P^T pieces and dO_j are consumed
      tc::tc_fence_after();
      {
        uint32_t d1[16], d2[16];
#pragma unroll
        for (int jj = 0; jj < 32; jj += 2) split2h(dsv[jj], dsv[jj + 1], d1[jj / 2], d2[jj / 2]);
        tc::tmem_st16(t_s + lane_off + 16 * half, d1);
        tc::tmem_st16(t_s + lane_off + 32 + 16 * half, d2);
        tc::tmem_wait_st();
      }
      ph_o ^= 1;
      tc::tc_fence_before();
      __syncthreads();
      tc::tc_fence_after();
      if (warp == 0) {  // dK += dS2Q1 + dS1Q2 + dS1Q1 (B = Q_j MN-major)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const uint32_t qb = ya + kPb[c] * L::kYPiece;
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk)
            tc::mma_bf16_ts_warp(t_dk, t_s + kPa[c] * 32 + kk * 8, tc::sw128_desc(qb + kk * 16 * 128, L::kYChunk, 1024),
                                 kIdescO, (j % kFlushH != 0 || c > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit_warp(bar_o);
      }
      tc::mbar_wait(bar_o, ph_o);
      tc::tc_fence_after();
      if (j % kFlushH == kFlushH - 1 || j + 1 == nblk) {
        ld_half_flush<D>(t_dv, lane_off, half, dv + (b0 + r) * rs + hd, fl_dv, j >= kFlushH, r < seg);
        ld_half_flush<D>(t_dk, lane_off, half, dk + (b0 + r) * rs + hd, fl_dk, j >= kFlushH, r < seg);
      }
      tc::tc_fence_before();
      ph_o ^= 1;
      ph_s ^= 1;
    }
    if (nblk == 0 && r < seg) {
      zero_half<D>(dv + (b0 + r) * rs + hd, half);
      zero_half<D>(dk + (b0 + r) * rs + hd, half);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}


template <int D>
static jg_status bwd_x3(const int64_t* off, int64_t total_rows, int H, const void* q, const void* k, const void* v,
                        const void* go, const void* o, const float* lse, float* delta, void* dq, void* dk, void* dv,
                        const int2* items, const int64_t* n_items, int64_t max_items, const int64_t* valid,
                        cudaStream_t st) {
  static const bool bf16x3 = std::getenv("JG_FP32_X3") != nullptr;  // A/B knob: the bf16 three-piece kernels
  // Delta = rowsum(dO * O) (fp64 accumulation) fused with the max |dO| the fp16 scales need
  unsigned* amax = nullptr;
  JG_CUDA(cudaMallocAsync(&amax, 16, st));
  scratch_note(16);
  JG_CUDA(cudaMemsetAsync(amax, 0, 16, st));
  {
    const int64_t units = total_rows * H;
    delta_amax_kernel<<<(int)std::min<int64_t>((units + 7) / 8, 16 * device_sm_count()), 256, 0, st>>>(
        units, D, (const float*)go, (const float*)o, H, total_rows, delta, amax + 3);
    JG_LAUNCHED("delta_amax_kernel");
  }
  struct FreeAmax {
    unsigned* p;
    cudaStream_t s;
    ~FreeAmax() {
      cudaFreeAsync(p, s);
      scratch_note(-16);
    }
  } free_amax{amax, st};
  if (!bf16x3) {  // fp16 two-piece kernels with per-tensor power-of-two scales (one max pass over q, k, v)
    const int sm_q2 = std::max<int>(BwdLay2<D, false>::kAlloc, 120 * 1024);
    const int sm_kv2 = std::max<int>(BwdLay2<D, true>::kAlloc, 120 * 1024);
    if (jg_status rc = ensure_smem_attr((const void*)attn_bwd_x2h_dq_kernel<D>, sm_q2, "attn_bwd_x2h_dq_kernel"))
      return rc;
    if (jg_status rc = ensure_smem_attr((const void*)attn_bwd_x2h_dkdv_kernel<D>, sm_kv2, "attn_bwd_x2h_dkdv_kernel"))
      return rc;
    const int64_t n4 = total_rows * H * D / 4;
    const int mg = (int)std::max<int64_t>(1, std::min<int64_t>((n4 + 255) / 256, 4 * device_sm_count()));
    absmax3_kernel<<<mg, 256, 0, st>>>((const float4*)q, (const float4*)k, (const float4*)v, n4, amax);
    JG_LAUNCHED("absmax3_kernel");
    const int grid2 = (int)std::max<int64_t>(1, std::min<int64_t>(max_items * H, (int64_t)device_sm_count()));
    const float scale2 = 1.0f / sqrtf((float)D);
    attn_bwd_x2h_dq_kernel<D><<<grid2, kThreads, sm_q2, st>>>(
        off, items, n_items, H, total_rows, (const float*)q, (const float*)k, (const float*)v, (const float*)go, lse,
        delta, (float*)dq, kLog2e * scale2, scale2, valid, (const float*)amax);
    JG_LAUNCHED("attn_bwd_x2h_dq_kernel");
    attn_bwd_x2h_dkdv_kernel<D><<<grid2, kThreads, sm_kv2, st>>>(
        off, items, n_items, H, total_rows, (const float*)q, (const float*)k, (const float*)v, (const float*)go, lse,
        delta, (float*)dk, (float*)dv, kLog2e * scale2, scale2, valid, (const float*)amax);
    JG_LAUNCHED("attn_bwd_x2h_dkdv_kernel");
    return JG_OK;
  }
  // at least half the SM's shared memory: one CTA per SM, since each allocates all 512 TMEM columns
  const int sm_q = std::max<int>(BwdLay<D, false>::kAlloc, 120 * 1024);
  const int sm_kv = std::max<int>(BwdLay<D, true>::kAlloc, 120 * 1024);
  if (jg_status rc = ensure_smem_attr((const void*)attn_bwd_x3_dq_kernel<D>, sm_q, "attn_bwd_x3_dq_kernel")) return rc;
  if (jg_status rc = ensure_smem_attr((const void*)attn_bwd_x3_dkdv_kernel<D>, sm_kv, "attn_bwd_x3_dkdv_kernel"))
    return rc;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(max_items * H, (int64_t)device_sm_count()));
  const float scale = 1.0f / sqrtf((float)D), scale_log2 = kLog2e * scale;
  attn_bwd_x3_dq_kernel<D><<<grid, kThreads, sm_q, st>>>(off, items, n_items, H, total_rows, (const float*)q,
                                                          (const float*)k, (const float*)v, (const float*)go, lse,
                                                          delta, (float*)dq, scale_log2, scale, valid);
  JG_LAUNCHED("attn_bwd_x3_dq_kernel");
  attn_bwd_x3_dkdv_kernel<D><<<grid, kThreads, sm_kv, st>>>(off, items, n_items, H, total_rows, (const float*)q,
                                                             (const float*)k, (const float*)v, (const float*)go, lse,
                                                             delta, (float*)dk, (float*)dv, scale_log2, scale, valid);
  JG_LAUNCHED("attn_bwd_x3_dkdv_kernel");
  return JG_OK;
}

}  // namespace x3

bool attn_x3_supported(int head_dim, jg_dtype dt) {
  static const bool off_ = std::getenv("JG_FP32_SIMT") != nullptr;  // A/B knob: the tiled FFMA kernels
  return !off_ && dt == JG_F32 && (head_dim == 64 || head_dim == 128);
}

jg_status launch_attn_fwd_x3(const int64_t* off, int64_t total_rows, int H, int D, const void* q, const void* k,
                             const void* v, void* out, float* lse, const int2* items, const int64_t* n_items,
                             int64_t max_items, const int64_t* valid, cudaStream_t st) {
  if (total_rows == 0) return JG_OK;
  if (D == 64) return x3::fwd_x3<64>(off, total_rows, H, q, k, v, out, lse, items, n_items, max_items, valid, st);
  if (D == 128) return x3::fwd_x3<128>(off, total_rows, H, q, k, v, out, lse, items, n_items, max_items, valid, st);
  return fail(JG_UNSUPPORTED, "jagged_flash_attention_forward: split-bf16 path needs head_dim 64 or 128");
}

jg_status launch_attn_bwd_x3(const int64_t* off, int64_t total_rows, int H, int D, const void* q, const void* k,
                             const void* v, const void* go, const void* o, const float* lse, float* delta, void* dq, void* dk,
                             void* dv, const int2* items, const int64_t* n_items, int64_t max_items,
                             const int64_t* valid, cudaStream_t st) {
  if (total_rows == 0) return JG_OK;
  if (D == 64)
    return x3::bwd_x3<64>(off, total_rows, H, q, k, v, go, o, lse, delta, dq, dk, dv, items, n_items, max_items, valid,
                          st);
  if (D == 128)
    return x3::bwd_x3<128>(off, total_rows, H, q, k, v, go, o, lse, delta, dq, dk, dv, items, n_items, max_items, valid,
                           st);
  return fail(JG_UNSUPPORTED, "jagged_flash_attention_backward: split-bf16 path needs head_dim 64 or 128");
}

}  // namespace jg
