// attn_simt.cu — jagged flash attention on CUDA cores (fp32 FFMA), the fp32-mode path.
//
// Forward (attention.cpp:172-225): one warp per (query row, head); keys stream in blocks of 32,
// one key per lane for the scores, online softmax (running max m and sum l, rescale by
// exp(m - m_new) exactly as attention.cpp:205-214), then P·V with lanes over head_dim.
// Backward (attention.cpp:227-289) without atomics: Δ = rowsum(dO∘O) prologue, then a
// query-stationary pass for dQ and a key-stationary pass for dK/dV, each recomputing
// P = exp(S/√D − lse) — every output element has one writer, so results are deterministic.
// Layout: [total_rows, H, D] for q/k/v/o/grads, lse float32 [H, total_rows].
#include "common.cuh"
#include "internal.h"

namespace jg {

constexpr float kLog2eA = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr int kMaxDPL = 8;  // head_dim <= 256
constexpr int kAttnWarps = 4;

template <typename T>
__device__ __forceinline__ float dot_smem_row(const float* __restrict__ a, const T* __restrict__ b, int D) {
  float acc = 0.f;
  for (int d = 0; d < D; ++d) acc = fmaf(a[d], ld(b + d), acc);
  return acc;
}

template <typename T>
__global__ void __launch_bounds__(kAttnWarps * 32) attn_fwd_simt_kernel(
    const int64_t* __restrict__ off, int64_t batch, int64_t total_rows, int H, int D,
    const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v, T* __restrict__ out,
    float* __restrict__ lse, float scale_log2, const int64_t* __restrict__ valid) {
  extern __shared__ float smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* qs = smem + w * D;
  const int64_t units = total_rows * H;
  for (int64_t u = blockIdx.x * (int64_t)kAttnWarps + w; u < units; u += (int64_t)gridDim.x * kAttnWarps) {
    const int64_t r = u / H;
    const int h = (int)(u - r * H);
    const int64_t i = sample_of_row(off, batch, r);
    const int64_t b0 = off[i], seg = off[i + 1] - b0;
    const int64_t rs = (int64_t)H * D;  // row stride
    // padded mode: only the first `valid` keys attend; rows past it are zero with lse = -inf
    const int64_t n = valid ? (valid[i] < seg ? valid[i] : seg) : seg;
    if (r - b0 >= n) {
      for (int d = lane; d < D; d += 32) st(out + r * rs + (int64_t)h * D + d, 0.f);
      if (lane == 0) lse[(int64_t)h * total_rows + r] = -INFINITY;
      continue;
    }
    __syncwarp();
    for (int d = lane; d < D; d += 32) qs[d] = ld(q + r * rs + (int64_t)h * D + d);
    __syncwarp();
    float m = -INFINITY, l = 0.f, acc[kMaxDPL];
#pragma unroll
    for (int j = 0; j < kMaxDPL; ++j) acc[j] = 0.f;
    for (int64_t c0 = 0; c0 < n; c0 += 32) {
      const int64_t c = c0 + lane;
      float s = -INFINITY;
      if (c < n) s = dot_smem_row(qs, k + (b0 + c) * rs + (int64_t)h * D, D) * scale_log2;
      const float m_new = fmaxf(m, warp_max(s));
      const float alpha = (m == -INFINITY) ? 0.f : exp2f(m - m_new);
      const float p = (c < n) ? exp2f(s - m_new) : 0.f;
      l = l * alpha + warp_sum(p);
#pragma unroll
      for (int j = 0; j < kMaxDPL; ++j) acc[j] *= alpha;
      const int nj = (int)(n - c0 < 32 ? n - c0 : 32);
      for (int j = 0; j < nj; ++j) {
        const float pj = __shfl_sync(0xffffffffu, p, j);
        const T* vr = v + (b0 + c0 + j) * rs + (int64_t)h * D;
#pragma unroll
        for (int jd = 0; jd < kMaxDPL; ++jd) {
          const int d = lane + 32 * jd;
          if (d < D) acc[jd] = fmaf(pj, ld(vr + d), acc[jd]);
        }
      }
      m = m_new;
    }
    const float inv = 1.0f / l;
#pragma unroll
    for (int jd = 0; jd < kMaxDPL; ++jd) {
      const int d = lane + 32 * jd;
      if (d < D) st(out + r * rs + (int64_t)h * D + d, acc[jd] * inv);
    }
    if (lane == 0) lse[(int64_t)h * total_rows + r] = (m + log2f(l)) * kLn2;
  }
}

// ------------------------------------------------------------------ tiled kernels (fp32 FFMA)
// One CTA (256 threads) per (sample, 128-row tile, head) work item from the schedule's LPT list (persistent,
// round-robin); the other side's rows stream through shared memory in blocks. Operands of the score-shaped
// products are staged transposed ([d][row]) so a thread's 4 rows and its 4 or 8 columns are float4 loads; the
// row-major products (P V, dS K, P^T dO, dS^T Q) read P / dS^T from shared memory and the right operand row by
// row. Roughly 40x the row-per-warp kernels above on cfg3-sized inputs; same results up to fp32 reassociation.
namespace ft {
constexpr int BQ = 128, BK = 64, kThreads = 256;  // forward: 128 query rows x 64-key blocks
constexpr int BM = 128, BN = 32;                    // backward: 128 stationary rows x 32-row moving blocks
template <int D>
struct FwdLay {
  static constexpr int kQt = 0;                       // [D][BQ + 4]
  static constexpr int kKt = kQt + D * (BQ + 4);      // [D][BK + 4]
  static constexpr int kV = kKt + D * (BK + 4);       // [BK][D + 4]
  static constexpr int kPt = kV + BK * (D + 4);       // [BK][BQ + 4]
  static constexpr int kFloats = kPt + BK * (BQ + 4);
};
// MODE 0 (dQ): X = Q | dO (stationary, transposed), Y = K | V (moving, transposed) + K row-major
// MODE 1 (dK, dV): X = K | V (stationary, transposed), Y = Q | dO (moving, transposed) + Q, dO row-major
template <int D, int MODE>
struct BwdLay {
  static constexpr int kXa = 0;                        // [D][BM + 4]
  static constexpr int kXb = kXa + D * (BM + 4);       // [D][BM + 4]
  static constexpr int kYa = kXb + D * (BM + 4);       // [D][BN + 4]
  static constexpr int kYb = kYa + D * (BN + 4);       // [D][BN + 4]
  static constexpr int kR1 = kYb + D * (BN + 4);       // [BN][D + 4]: K (MODE 0) or Q (MODE 1)
  static constexpr int kR2 = kR1 + BN * (D + 4);       // [BN][D + 4]: dO (MODE 1 only)
  static constexpr int kPs = kR2 + (MODE ? BN * (D + 4) : 0);  // [BN][BM + 4]: P^T / dS^T
  static constexpr int kLs = kPs + BN * (BM + 4);      // [BN] lse*log2e, [BN] Delta of the moving block (MODE 1)
  static constexpr int kFloats = kLs + 2 * BN;
};

template <typename T>
__device__ __forceinline__ float4 ld4(const T* p);
template <>
__device__ __forceinline__ float4 ld4<float>(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
template <>
__device__ __forceinline__ float4 ld4<__nv_bfloat16>(const __nv_bfloat16* p) {
  const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}

// rows [r0, r0 + ROWS) of a [*, H, D] tensor (rows >= n are zero) into dst[d][row] (pitch ROWS + 4) and, when
// ROWMAJ, also into rowm[row][d] (pitch D + 4). Consecutive threads take consecutive rows: conflict-free stores.
template <typename T, int D, int ROWS, bool ROWMAJ>
__device__ __forceinline__ void stage_rows(const T* __restrict__ src, int64_t b0, int64_t r0, int64_t n,
                                           int64_t rs, float* __restrict__ dst, float* __restrict__ rowm) {
  for (int e = threadIdx.x; e < ROWS * (D / 4); e += kThreads) {
    const int r = e % ROWS, d4 = (e / ROWS) * 4;
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r0 + r < n) x = ld4(src + (b0 + r0 + r) * rs + d4);
    dst[(d4 + 0) * (ROWS + 4) + r] = x.x;
    dst[(d4 + 1) * (ROWS + 4) + r] = x.y;
    dst[(d4 + 2) * (ROWS + 4) + r] = x.z;
    dst[(d4 + 3) * (ROWS + 4) + r] = x.w;
    if (ROWMAJ) *reinterpret_cast<float4*>(rowm + r * (D + 4) + d4) = x;
  }
}

// acc[i][j] += sum_d A[d][4ty + i] * B[d][C*tx + j]  (transposed operands, pitches PA / PB)
template <int D, int C, int PA, int PB>
__device__ __forceinline__ void tile_tn(const float* __restrict__ A, const float* __restrict__ B, int ty, int tx,
                                        float (&acc)[4][C]) {
#pragma unroll 4
  for (int d = 0; d < D; ++d) {
    const float4 a = *reinterpret_cast<const float4*>(A + d * PA + 4 * ty);
    float bv[C];
#pragma unroll
    for (int j = 0; j < C; j += 4) {
      const float4 b = *reinterpret_cast<const float4*>(B + d * PB + C * tx + j);
      bv[j] = b.x; bv[j + 1] = b.y; bv[j + 2] = b.z; bv[j + 3] = b.w;
    }
    const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < C; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
  }
}

// acc[i][c] += sum_{kk < kn} P[kk][4ty + i] * R[kk][DC*tx + c]  (P pitch PP, R pitch D + 4)
template <int D, int PP>
__device__ __forceinline__ void tile_pr(const float* __restrict__ P, const float* __restrict__ R, int kn, int ty,
                                        int tx, float (&acc)[4][D / 8]) {
  constexpr int DC = D / 8;
#pragma unroll 2
  for (int kk = 0; kk < kn; ++kk) {
    const float4 a = *reinterpret_cast<const float4*>(P + kk * PP + 4 * ty);
    const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int j4 = 0; j4 < DC; j4 += 4) {
      const float4 b = *reinterpret_cast<const float4*>(R + kk * (D + 4) + tx * DC + j4);
      const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc[i][j4 + jj] = fmaf(av[i], bv[jj], acc[i][j4 + jj]);
    }
  }
}
}  // namespace ft

template <typename T, int D>
__global__ void __launch_bounds__(ft::kThreads, 1) attn_fwd_tiled_kernel(
    const int64_t* __restrict__ off, const int2* __restrict__ items, const int64_t* __restrict__ n_items, int H,
    int64_t total_rows, const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
    T* __restrict__ out, float* __restrict__ lse, float scale_log2, const int64_t* __restrict__ valid) {
  using namespace ft;
  using L = FwdLay<D>;
  constexpr int DC = D / 8;  // output columns per thread
  extern __shared__ float4 sm4[];
  float* sm = reinterpret_cast<float*>(sm4);
  float* Qt = sm + L::kQt;
  float* Kt = sm + L::kKt;
  float* Vs = sm + L::kV;
  float* Pt = sm + L::kPt;
  const int tid = threadIdx.x, ty = tid >> 3, tx = tid & 7;
  const int64_t rs = (int64_t)H * D;
  const int64_t n_work = *n_items * H;
  for (int64_t w = blockIdx.x; w < n_work; w += gridDim.x) {
    const int2 it = items[w / H];
    const int h = (int)(w % H);
    const int64_t b0 = off[it.x], seg = off[it.x + 1] - b0;
    const int64_t nv = valid ? (valid[it.x] < seg ? valid[it.x] : seg) : seg;  // valid keys / rows
    const int q0 = it.y * BQ;                                                  // first query row (local)
    __syncthreads();  // the previous item is done with the staging buffers
    stage_rows<T, D, BQ, false>(q + (int64_t)h * D, b0, q0, seg, rs, Qt, nullptr);
    float m[4], l[4], o[4][DC];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      m[i] = -INFINITY;
      l[i] = 0.f;
#pragma unroll
      for (int j = 0; j < DC; ++j) o[i][j] = 0.f;
    }
    for (int64_t k0 = 0; k0 < nv; k0 += BK) {
      __syncthreads();  // previous block's Kt/V/Pt reads are done (and Q is staged)
      stage_rows<T, D, BK, false>(k + (int64_t)h * D, b0, k0, nv, rs, Kt, nullptr);
      for (int e = tid; e < BK * (D / 4); e += kThreads) {
        const int r = e % BK, d4 = (e / BK) * 4;
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k0 + r < nv) x = ld4(v + (b0 + k0 + r) * rs + (int64_t)h * D + d4);
        *reinterpret_cast<float4*>(Vs + r * (D + 4) + d4) = x;
      }
      __syncthreads();
      // S = Q K^T: rows 4ty..4ty+3, keys 8tx..8tx+7
      float s[4][8];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) s[i][j] = 0.f;
      tile_tn<D, 8, BQ + 4, BK + 4>(Qt, Kt, ty, tx, s);
      // online softmax (log2 units, attention.cpp:205-214); keys past the valid range are -inf
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float mx = -INFINITY;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          s[i][j] = (k0 + 8 * tx + j < nv) ? s[i][j] * scale_log2 : -INFINITY;
          mx = fmaxf(mx, s[i][j]);
        }
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
        const float mn = fmaxf(m[i], mx);
        const float alpha = (m[i] == -INFINITY) ? 0.f : exp2f(m[i] - mn);
        float ps = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float pv = exp2f(s[i][j] - mn);  // -inf -> 0
          ps += pv;
          Pt[(8 * tx + j) * (BQ + 4) + 4 * ty + i] = pv;
        }
        ps += __shfl_xor_sync(0xffffffffu, ps, 1);
        ps += __shfl_xor_sync(0xffffffffu, ps, 2);
        ps += __shfl_xor_sync(0xffffffffu, ps, 4);
        l[i] = l[i] * alpha + ps;
        m[i] = mn;
#pragma unroll
        for (int j = 0; j < DC; ++j) o[i][j] *= alpha;
      }
      __syncthreads();
      tile_pr<D, BQ + 4>(Pt, Vs, nv - k0 < BK ? (int)(nv - k0) : BK, ty, tx, o);  // O += P V
    }
    // epilogue: rows of this tile inside the segment; rows past the valid length are zero with lse = -inf
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t r = q0 + 4 * ty + i;
      if (r >= seg) continue;
      const bool ok = r < nv;
      const float inv = ok ? 1.0f / l[i] : 0.f;
      T* dst = out + (b0 + r) * rs + (int64_t)h * D + tx * DC;
#pragma unroll
      for (int j = 0; j < DC; ++j) st(dst + j, ok ? o[i][j] * inv : 0.f);
      if (tx == 0) lse[(int64_t)h * total_rows + b0 + r] = ok ? (m[i] + log2f(l[i])) * kLn2 : -INFINITY;
    }
  }
}

// Backward without atomics (attention.cpp:227-289): MODE 0 is query-stationary and writes dQ; MODE 1 is
// key-stationary and writes dK, dV. Both recompute P = exp2(S*scale*log2e - lse*log2e) and dS = P (dP - Delta).
template <typename T, int D, int MODE>
__global__ void __launch_bounds__(ft::kThreads, 1) attn_bwd_tiled_kernel(
    const int64_t* __restrict__ off, const int2* __restrict__ items, const int64_t* __restrict__ n_items, int H,
    int64_t total_rows, const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
    const T* __restrict__ go, const float* __restrict__ lse, const float* __restrict__ delta, T* __restrict__ o1,
    T* __restrict__ o2, float scale_log2, float scale, const int64_t* __restrict__ valid) {
  using namespace ft;
  using L = BwdLay<D, MODE>;
  constexpr int DC = D / 8;
  extern __shared__ float4 sm4[];
  float* sm = reinterpret_cast<float*>(sm4);
  float *Xa = sm + L::kXa, *Xb = sm + L::kXb, *Ya = sm + L::kYa, *Yb = sm + L::kYb;
  float *R1 = sm + L::kR1, *R2 = sm + L::kR2, *Ps = sm + L::kPs, *Ls = sm + L::kLs, *Ds = Ls + BN;
  const int tid = threadIdx.x, ty = tid >> 3, tx = tid & 7;
  const int64_t rs = (int64_t)H * D;
  const int64_t n_work = *n_items * H;
  for (int64_t w = blockIdx.x; w < n_work; w += gridDim.x) {
    const int2 it = items[w / H];
    const int h = (int)(w % H);
    const int64_t hd = (int64_t)h * D, hr = (int64_t)h * total_rows;
    const int64_t b0 = off[it.x], seg = off[it.x + 1] - b0;
    const int64_t nv = valid ? (valid[it.x] < seg ? valid[it.x] : seg) : seg;
    const int x0 = it.y * BM;
    __syncthreads();
    stage_rows<T, D, BM, false>((MODE == 0 ? q : k) + hd, b0, x0, nv, rs, Xa, nullptr);
    stage_rows<T, D, BM, false>((MODE == 0 ? go : v) + hd, b0, x0, nv, rs, Xb, nullptr);
    float lr[4] = {0.f, 0.f, 0.f, 0.f}, dr[4] = {0.f, 0.f, 0.f, 0.f};  // MODE 0: this thread's rows
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t r = x0 + 4 * ty + i;
        if (r < nv) {
          lr[i] = lse[hr + b0 + r] * kLog2eA;
          dr[i] = delta[hr + b0 + r];
        }
      }
    }
    float acc1[4][DC], acc2[4][DC];  // acc2 (dV) is dead in MODE 0
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
      for (int j = 0; j < DC; ++j) acc1[i][j] = 0.f;
#pragma unroll
      for (int j = 0; j < DC; ++j) acc2[i][j] = 0.f;
    }
    // stationary rows past the valid length get zero gradients: skip the loop for an all-padding tile
    for (int64_t y0 = 0; x0 < nv && y0 < nv; y0 += BN) {
      __syncthreads();
      if (MODE == 0) {
        stage_rows<T, D, BN, true>(k + hd, b0, y0, nv, rs, Ya, R1);
        stage_rows<T, D, BN, false>(v + hd, b0, y0, nv, rs, Yb, nullptr);
      } else {
        stage_rows<T, D, BN, true>(q + hd, b0, y0, nv, rs, Ya, R1);
        stage_rows<T, D, BN, true>(go + hd, b0, y0, nv, rs, Yb, R2);
        if (tid < BN) {
          const bool in = y0 + tid < nv;
          Ls[tid] = in ? lse[hr + b0 + y0 + tid] * kLog2eA : 0.f;
          Ds[tid] = in ? delta[hr + b0 + y0 + tid] : 0.f;
        }
      }
      __syncthreads();
      float s[4][4], dp[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s[i][j] = dp[i][j] = 0.f;
      tile_tn<D, 4, BM + 4, BN + 4>(Xa, Ya, ty, tx, s);   // MODE 0: S = Q K^T; MODE 1: S^T = K Q^T
      tile_tn<D, 4, BM + 4, BN + 4>(Xb, Yb, ty, tx, dp);  // MODE 0: dP = dO V^T; MODE 1: dP^T = V dO^T
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const bool in = y0 + 4 * tx + j < nv && x0 + 4 * ty + i < nv;  // both rows inside the valid length
          const float l2 = MODE == 0 ? lr[i] : Ls[4 * tx + j];
          const float dl = MODE == 0 ? dr[i] : Ds[4 * tx + j];
          const float p = in ? exp2f(s[i][j] * scale_log2 - l2) : 0.f;
          s[i][j] = p;
          dp[i][j] = p * (dp[i][j] - dl);
        }
      const int kn = nv - y0 < BN ? (int)(nv - y0) : BN;
      if (MODE == 1) {  // dV += P^T dO
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) Ps[(4 * tx + j) * (BM + 4) + 4 * ty + i] = s[i][j];
        __syncthreads();
        tile_pr<D, BM + 4>(Ps, R2, kn, ty, tx, acc2);
        __syncthreads();
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) Ps[(4 * tx + j) * (BM + 4) + 4 * ty + i] = dp[i][j];
      __syncthreads();
      tile_pr<D, BM + 4>(Ps, R1, kn, ty, tx, acc1);  // MODE 0: dQ += dS K; MODE 1: dK += dS^T Q
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t r = x0 + 4 * ty + i;
      if (r >= seg) continue;
      const int64_t base = (b0 + r) * rs + hd + tx * DC;
#pragma unroll
      for (int j = 0; j < DC; ++j) {
        st(o1 + base + j, acc1[i][j] * scale);  // zero for padded rows (never accumulated)
        if (MODE == 1) st(o2 + base + j, acc2[i][j]);
      }
    }
  }
}

// Delta = rowsum(dO * O), accumulated in fp64: the fp32 backward's dS = P (dP - Delta) cancels when P is
// concentrated, so Delta's own rounding must stay well below dP's
template <typename T>
__global__ void attn_delta_kernel(int64_t units, int H, int D, const T* __restrict__ go,
                                  const T* __restrict__ o, int64_t total_rows, float* __restrict__ delta) {
  const int lane = threadIdx.x & 31;
  for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < units;
       u += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t r = u / H;
    const int h = (int)(u - r * H);
    const int64_t base = u * D;  // [r, h, :] is contiguous at (r*H + h)*D
    double acc = 0.0;
    for (int d = lane; d < D; d += 32) acc = fma((double)ld(go + base + d), (double)ld(o + base + d), acc);
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
    if (lane == 0) delta[(int64_t)h * total_rows + r] = (float)acc;
  }
}

// MODE 0: query-stationary dQ; MODE 1: key-stationary dK, dV
template <typename T, int MODE>
__global__ void __launch_bounds__(kAttnWarps * 32) attn_bwd_simt_kernel(
    const int64_t* __restrict__ off, int64_t batch, int64_t total_rows, int H, int D,
    const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v, const T* __restrict__ go,
    const float* __restrict__ lse, const float* __restrict__ delta, T* __restrict__ o1,
    T* __restrict__ o2, float scale_log2, float scale, const int64_t* __restrict__ valid) {
  extern __shared__ float smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* xs = smem + w * 2 * D;  // MODE 0: q row | dO row ; MODE 1: k row | v row
  float* ys = xs + D;
  const int64_t units = total_rows * H;
  const int64_t rs = (int64_t)H * D;
  for (int64_t u = blockIdx.x * (int64_t)kAttnWarps + w; u < units; u += (int64_t)gridDim.x * kAttnWarps) {
    const int64_t r = u / H;
    const int h = (int)(u - r * H);
    const int64_t i = sample_of_row(off, batch, r);
    const int64_t b0 = off[i], seg = off[i + 1] - b0;
    const int64_t hoff = (int64_t)h * D;
    const int64_t n = valid ? (valid[i] < seg ? valid[i] : seg) : seg;  // padded mode: valid rows only
    if (r - b0 >= n) {  // a padded row: no query/key interaction, zero gradient
      for (int d = lane; d < D; d += 32) {
        st(o1 + r * rs + hoff + d, 0.f);
        if (MODE == 1) st(o2 + r * rs + hoff + d, 0.f);
      }
      continue;
    }
    __syncwarp();
    if (MODE == 0) {
      for (int d = lane; d < D; d += 32) { xs[d] = ld(q + r * rs + hoff + d); ys[d] = ld(go + r * rs + hoff + d); }
    } else {
      for (int d = lane; d < D; d += 32) { xs[d] = ld(k + r * rs + hoff + d); ys[d] = ld(v + r * rs + hoff + d); }
    }
    __syncwarp();
    float acc1[kMaxDPL], acc2[kMaxDPL];
#pragma unroll
    for (int j = 0; j < kMaxDPL; ++j) { acc1[j] = 0.f; acc2[j] = 0.f; }
    const float lse_r = MODE == 0 ? lse[(int64_t)h * total_rows + r] * kLog2eA : 0.f;
    const float delta_r = MODE == 0 ? delta[(int64_t)h * total_rows + r] : 0.f;
    for (int64_t c0 = 0; c0 < n; c0 += 32) {
      const int64_t c = c0 + lane;  // the other side's row (key for MODE 0, query for MODE 1)
      float p = 0.f, ds = 0.f;
      if (c < n) {
        const int64_t rr = (b0 + c) * rs + hoff;
        if (MODE == 0) {
          const float s2 = dot_smem_row(xs, k + rr, D) * scale_log2;
          p = exp2f(s2 - lse_r);
          const float dp = dot_smem_row(ys, v + rr, D);
          ds = p * (dp - delta_r);
        } else {
          const int64_t qrow = b0 + c;
          const float s2 = dot_smem_row(xs, q + rr, D) * scale_log2;
          p = exp2f(s2 - lse[(int64_t)h * total_rows + qrow] * kLog2eA);
          const float dp = dot_smem_row(ys, go + rr, D);
          ds = p * (dp - delta[(int64_t)h * total_rows + qrow]);
        }
      }
      const int nj = (int)(n - c0 < 32 ? n - c0 : 32);
      for (int j = 0; j < nj; ++j) {
        const float pj = __shfl_sync(0xffffffffu, p, j);
        const float dsj = __shfl_sync(0xffffffffu, ds, j);
        const int64_t rr = (b0 + c0 + j) * rs + hoff;
#pragma unroll
        for (int jd = 0; jd < kMaxDPL; ++jd) {
          const int d = lane + 32 * jd;
          if (d < D) {
            if (MODE == 0) {
              acc1[jd] = fmaf(dsj, ld(k + rr + d), acc1[jd]);  // dQ
            } else {
              acc1[jd] = fmaf(dsj, ld(q + rr + d), acc1[jd]);  // dK
              acc2[jd] = fmaf(pj, ld(go + rr + d), acc2[jd]);  // dV
            }
          }
        }
      }
    }
#pragma unroll
    for (int jd = 0; jd < kMaxDPL; ++jd) {
      const int d = lane + 32 * jd;
      if (d < D) {
        st(o1 + r * rs + hoff + d, acc1[jd] * scale);
        if (MODE == 1) st(o2 + r * rs + hoff + d, acc2[jd]);
      }
    }
  }
}

template <typename T, int D>
static jg_status fwd_tiled_t(const int64_t* off, int64_t total_rows, int H, const void* q, const void* k,
                             const void* v, void* out, float* lse, const int2* items, const int64_t* n_items,
                             int64_t max_items, const int64_t* valid, cudaStream_t st) {
  const size_t smem = sizeof(float) * ft::FwdLay<D>::kFloats;
  if (jg_status rc = ensure_smem_attr((const void*)attn_fwd_tiled_kernel<T, D>, (int)smem, "attn_fwd_tiled_kernel"))
    return rc;
  int per_sm = 1;
  JG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, attn_fwd_tiled_kernel<T, D>, ft::kThreads, smem));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(max_items * H, (int64_t)std::max(per_sm, 1) *
                                                                                  device_sm_count()));
  const float scale_log2 = kLog2eA / sqrtf((float)D);
  attn_fwd_tiled_kernel<T, D><<<grid, ft::kThreads, smem, st>>>(off, items, n_items, H, total_rows, (const T*)q,
                                                                (const T*)k, (const T*)v, (T*)out, lse, scale_log2,
                                                                valid);
  JG_LAUNCHED("attn_fwd_tiled_kernel");
  return JG_OK;
}

template <typename T>
static jg_status fwd_t(const int64_t* off, int64_t batch, int64_t total_rows, int H, int D, const void* q,
                       const void* k, const void* v, void* out, float* lse, const int2* items,
                       const int64_t* n_items, int64_t max_items, const int64_t* valid, cudaStream_t st) {
  static const bool rowwise = std::getenv("JG_SIMT_ROWWISE") != nullptr;  // A/B knob: the row-per-warp kernel
  if (items && !rowwise) {
    if (D == 32) return fwd_tiled_t<T, 32>(off, total_rows, H, q, k, v, out, lse, items, n_items, max_items, valid, st);
    if (D == 64) return fwd_tiled_t<T, 64>(off, total_rows, H, q, k, v, out, lse, items, n_items, max_items, valid, st);
    if (D == 128)
      return fwd_tiled_t<T, 128>(off, total_rows, H, q, k, v, out, lse, items, n_items, max_items, valid, st);
  }
  const int64_t units = total_rows * H;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((units + kAttnWarps - 1) / kAttnWarps,
                                                               16 * device_sm_count()));
  const float scale_log2 = kLog2eA / sqrtf((float)D);
  attn_fwd_simt_kernel<T><<<grid, kAttnWarps * 32, kAttnWarps * D * sizeof(float), st>>>(
      off, batch, total_rows, H, D, (const T*)q, (const T*)k, (const T*)v, (T*)out, lse, scale_log2, valid);
  JG_LAUNCHED("attn_fwd_simt_kernel");
  return JG_OK;
}

template <typename T, int D, int MODE>
static jg_status bwd_tiled_pass(const int64_t* off, int64_t total_rows, int H, const void* q, const void* k,
                                const void* v, const void* go, const float* lse, const float* delta, void* o1,
                                void* o2, const int2* items, const int64_t* n_items, int64_t max_items,
                                const int64_t* valid, cudaStream_t st) {
  const size_t smem = sizeof(float) * ft::BwdLay<D, MODE>::kFloats;
  if (jg_status rc = ensure_smem_attr((const void*)attn_bwd_tiled_kernel<T, D, MODE>, (int)smem,
                                      "attn_bwd_tiled_kernel"))
    return rc;
  int per_sm = 1;
  JG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, attn_bwd_tiled_kernel<T, D, MODE>, ft::kThreads,
                                                        smem));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(max_items * H, (int64_t)std::max(per_sm, 1) *
                                                                                  device_sm_count()));
  const float scale = 1.0f / sqrtf((float)D), scale_log2 = kLog2eA * scale;
  attn_bwd_tiled_kernel<T, D, MODE><<<grid, ft::kThreads, smem, st>>>(
      off, items, n_items, H, total_rows, (const T*)q, (const T*)k, (const T*)v, (const T*)go, lse, delta, (T*)o1,
      (T*)o2, scale_log2, scale, valid);
  JG_LAUNCHED(MODE == 0 ? "attn_bwd_tiled_kernel<dq>" : "attn_bwd_tiled_kernel<dkdv>");
  return JG_OK;
}

template <typename T, int D>
static jg_status bwd_tiled_t(const int64_t* off, int64_t total_rows, int H, const void* q, const void* k,
                             const void* v, const void* go, const float* lse, const float* delta, void* dq,
                             void* dk, void* dv, const int2* items, const int64_t* n_items, int64_t max_items,
                             const int64_t* valid, cudaStream_t st) {
  if (jg_status rc = bwd_tiled_pass<T, D, 0>(off, total_rows, H, q, k, v, go, lse, delta, dq, nullptr, items,
                                             n_items, max_items, valid, st))
    return rc;
  return bwd_tiled_pass<T, D, 1>(off, total_rows, H, q, k, v, go, lse, delta, dk, dv, items, n_items, max_items,
                                 valid, st);
}

template <typename T>
static jg_status bwd_t(const int64_t* off, int64_t batch, int64_t total_rows, int H, int D, const void* q,
                       const void* k, const void* v, const void* go, const void* o, const float* lse, void* dq,
                       void* dk, void* dv, float* delta, const int2* items, const int64_t* n_items,
                       int64_t max_items, const int64_t* valid, bool x3, cudaStream_t st) {
  const int64_t units = total_rows * H;
  const int sms = device_sm_count();
  if (x3 && items)  // fp32 on tcgen05 (attn_x3_sm100.cu; it computes Delta together with its operand maxima)
    return launch_attn_bwd_x3(off, total_rows, H, D, q, k, v, go, o, lse, delta, dq, dk, dv, items, n_items,
                              max_items, valid, st);
  attn_delta_kernel<T><<<(int)std::min<int64_t>((units + 7) / 8, 16 * sms), 256, 0, st>>>(
      units, H, D, (const T*)go, (const T*)o, total_rows, delta);
  JG_LAUNCHED("attn_delta_kernel");
  static const bool rowwise = std::getenv("JG_SIMT_ROWWISE") != nullptr;  // A/B knob: the row-per-warp kernels
  if (items && !rowwise) {
    if (D == 32)
      return bwd_tiled_t<T, 32>(off, total_rows, H, q, k, v, go, lse, delta, dq, dk, dv, items, n_items, max_items,
                                valid, st);
    if (D == 64)
      return bwd_tiled_t<T, 64>(off, total_rows, H, q, k, v, go, lse, delta, dq, dk, dv, items, n_items, max_items,
                                valid, st);
    if (D == 128)
      return bwd_tiled_t<T, 128>(off, total_rows, H, q, k, v, go, lse, delta, dq, dk, dv, items, n_items,
                                 max_items, valid, st);
  }
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((units + kAttnWarps - 1) / kAttnWarps, 16 * sms));
  const float scale = 1.0f / sqrtf((float)D), scale_log2 = kLog2eA * scale;
  const size_t sm = kAttnWarps * 2 * D * sizeof(float);
  attn_bwd_simt_kernel<T, 0><<<grid, kAttnWarps * 32, sm, st>>>(off, batch, total_rows, H, D, (const T*)q,
                                                               (const T*)k, (const T*)v, (const T*)go, lse,
                                                               delta, (T*)dq, nullptr, scale_log2, scale, valid);
  JG_LAUNCHED("attn_bwd_simt_kernel<dq>");
  attn_bwd_simt_kernel<T, 1><<<grid, kAttnWarps * 32, sm, st>>>(off, batch, total_rows, H, D, (const T*)q,
                                                               (const T*)k, (const T*)v, (const T*)go, lse,
                                                               delta, (T*)dk, (T*)dv, scale_log2, scale, valid);
  JG_LAUNCHED("attn_bwd_simt_kernel<dkdv>");
  return JG_OK;
}

jg_status launch_attn_fwd_simt(const int64_t* off, int64_t batch, int64_t total_rows, int H, int D,
                               const void* q, const void* k, const void* v, void* out, float* lse,
                               jg_dtype dt, const int2* items, const int64_t* n_items, int64_t max_items,
                               const int64_t* valid, cudaStream_t st) {
  if (total_rows == 0) return JG_OK;
  if (D > 32 * kMaxDPL) return fail(JG_UNSUPPORTED, "jagged_flash_attention_forward: head_dim > 256 unsupported");
  if (dt == JG_F32) return fwd_t<float>(off, batch, total_rows, H, D, q, k, v, out, lse, items, n_items, max_items, valid, st);
  if (dt == JG_BF16) return fwd_t<__nv_bfloat16>(off, batch, total_rows, H, D, q, k, v, out, lse, items, n_items, max_items,
                                         valid, st);
  return fail(JG_UNSUPPORTED, "jagged_flash_attention_forward: dtype not supported on device (no CPU fallback)");
}

jg_status launch_attn_bwd_simt(const int64_t* off, int64_t batch, int64_t total_rows, int H, int D,
                               const void* q, const void* k, const void* v, const void* go,
                               const void* o, const float* lse, void* dq, void* dk, void* dv,
                               float* delta, jg_dtype dt, const int2* items, const int64_t* n_items,
                               int64_t max_items, const int64_t* valid, bool x3, cudaStream_t st) {
  if (total_rows == 0) return JG_OK;
  if (D > 32 * kMaxDPL) return fail(JG_UNSUPPORTED, "jagged_flash_attention_backward: head_dim > 256 unsupported");
  if (dt == JG_F32)
    return bwd_t<float>(off, batch, total_rows, H, D, q, k, v, go, o, lse, dq, dk, dv, delta, items, n_items,
                         max_items, valid, x3, st);
  if (dt == JG_BF16)
    return bwd_t<__nv_bfloat16>(off, batch, total_rows, H, D, q, k, v, go, o, lse, dq, dk, dv, delta, items, n_items,
                                  max_items, valid, false, st);
  return fail(JG_UNSUPPORTED, "jagged_flash_attention_backward: dtype not supported on device (no CPU fallback)");
}

}  // namespace jg
