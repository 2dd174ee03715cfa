// softmax.cu — jagged_softmax (per column over a segment's rows) and jagged2_softmax (per row of
// each Bi x Bi block), forward and VJP. HBM-bound: one CTA per (sample, column slab), 128-bit
// vector loads along the contiguous column axis, single-pass online max/sum, warp/CTA reductions.
//
// Semantics (linalg.cpp:98-120, :199-220, :355-388, :474-507): max-subtracted softmax, empty
// segments untouched, p recomputed from x in the VJP. fp32 accumulation; exp via ex2.approx on
// log2(e)-prescaled inputs (relative error ~2^-22, inside the 1e-5 fp32-mode tolerance). The
// prescale is an unfused __fmul_rn so the max pass and the exp pass see the identical value
// (a contracted FMA would leave the product's rounding error in x*log2e - m, and Bi=1 must
// give exactly 1.0).
#include "common.cuh"
#include "internal.h"
#include "tc.cuh"

namespace jg {

constexpr float kLog2e = 1.4426950408889634f;
constexpr int kSmWarps = 8;

template <typename T, int VEC>
struct VecIO {
  static __device__ __forceinline__ void load(const T* p, float (&v)[VEC]) {
    if constexpr (std::is_same_v<T, float> && VEC == 4) {
      float4 x = *reinterpret_cast<const float4*>(p);
      v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    } else if constexpr (std::is_same_v<T, float> && VEC == 2) {
      float2 x = *reinterpret_cast<const float2*>(p);
      v[0] = x.x; v[1] = x.y;
    } else if constexpr (std::is_same_v<T, __nv_bfloat16> && VEC == 8) {
      uint4 x = *reinterpret_cast<const uint4*>(p);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&x);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 f = __bfloat1622float2(h[j]);
        v[2 * j] = f.x; v[2 * j + 1] = f.y;
      }
    } else if constexpr (std::is_same_v<T, __nv_bfloat16> && VEC == 4) {
      uint2 x = *reinterpret_cast<const uint2*>(p);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&x);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        float2 f = __bfloat1622float2(h[j]);
        v[2 * j] = f.x; v[2 * j + 1] = f.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[j] = ld(p + j);
    }
  }
  static __device__ __forceinline__ void store(T* p, const float (&v)[VEC]) {
    if constexpr (std::is_same_v<T, float> && VEC == 4) {
      *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    } else if constexpr (std::is_same_v<T, float> && VEC == 2) {
      *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
    } else if constexpr (std::is_same_v<T, __nv_bfloat16> && VEC == 8) {
      uint4 x;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&x);
#pragma unroll
      for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
      *reinterpret_cast<uint4*>(p) = x;
    } else if constexpr (std::is_same_v<T, __nv_bfloat16> && VEC == 4) {
      uint2 x;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&x);
#pragma unroll
      for (int j = 0; j < 2; ++j) h[j] = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
      *reinterpret_cast<uint2*>(p) = x;
    } else {
#pragma unroll
      for (int j = 0; j < VEC; ++j) st(p + j, v[j]);
    }
  }
};

__device__ __forceinline__ float ex2a(float x) {  // MUFU.EX2 (ex2.approx.ftz; ex2(-inf) = 0)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void online_update(float& m, float& s, float y) {
  // y already in log2 units
  if (y > m) {
    s = s * ex2a(m - y) + 1.0f;
    m = y;
  } else if (m != -INFINITY) {  // y <= m = -inf means y = -inf: weight 0 (ex2(-inf - -inf) would be NaN)
    s += ex2a(y - m);
  }
}

// VJP: the same running update also carries d = sum g 2^(y - m) (rescaled with s), so dot = d / s comes out of
// the statistics pass and x is read twice instead of three times
__device__ __forceinline__ void online_update_d(float& m, float& s, float& d, float y, float g) {
  if (y > m) {
    const float c = ex2a(m - y);
    s = s * c + 1.0f;
    d = d * c + g;
    m = y;
  } else if (m != -INFINITY) {
    const float e = ex2a(y - m);
    s += e;
    d += g * e;
  }
}

// Combine the kSmWarps partial (m, s) of every column held by this thread; result in m, s.
template <int VEC>
__device__ __forceinline__ void combine_ms(float (&m)[VEC], float (&s)[VEC], float* sm_m, float* sm_s,
                                           int col_local) {
  const int w = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    sm_m[w * 32 * VEC + col_local + j] = m[j];
    sm_s[w * 32 * VEC + col_local + j] = s[j];
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    float M = -INFINITY;
    for (int ww = 0; ww < kSmWarps; ++ww) M = fmaxf(M, sm_m[ww * 32 * VEC + col_local + j]);
    float S = 0.f;
    for (int ww = 0; ww < kSmWarps; ++ww) {
      const float mm = sm_m[ww * 32 * VEC + col_local + j];
      if (mm != -INFINITY) S += sm_s[ww * 32 * VEC + col_local + j] * exp2f(mm - M);
    }
    m[j] = M;
    s[j] = S;
  }
}

// grid: x = sample, y = column slab of 32*VEC columns. MODE 0 forward, 1 VJP.
template <typename T, int VEC, int MODE>
__global__ void __launch_bounds__(kSmWarps * 32) jagged_softmax_kernel(
    const int64_t* __restrict__ off, int64_t D, const T* __restrict__ x, const T* __restrict__ g,
    T* __restrict__ out) {
  __shared__ float sm_m[kSmWarps * 32 * VEC];
  __shared__ float sm_s[kSmWarps * 32 * VEC];
  const int64_t i = blockIdx.x;
  const int64_t b0 = off[i], b1 = off[i + 1];
  if (b0 == b1) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int col_local = lane * VEC;
  const int64_t col = (int64_t)blockIdx.y * 32 * VEC + col_local;
  const bool active = col < D;  // D % VEC == 0 is guaranteed by the launcher
  float m[VEC], s[VEC], d[VEC];  // d: VJP only (sum g 2^(y - m))
#pragma unroll
  for (int j = 0; j < VEC; ++j) { m[j] = -INFINITY; s[j] = 0.f; d[j] = 0.f; }
  if (active) {
    // four rows per step: their loads in flight together, one branch-free running-max update per column
    // (s = s * 2^(m - m') + sum_k 2^(y_k - m'), MUFU ex2) instead of a branchy update per element
    int64_t r = b0 + w;
    for (; r + 3 * kSmWarps < b1; r += 4 * kSmWarps) {
      float v[4][VEC], gv[MODE ? 4 : 1][VEC];
#pragma unroll
      for (int u = 0; u < 4; ++u) VecIO<T, VEC>::load(x + (r + u * kSmWarps) * D + col, v[u]);
      if constexpr (MODE == 1) {
#pragma unroll
        for (int u = 0; u < 4; ++u) VecIO<T, VEC>::load(g + (r + u * kSmWarps) * D + col, gv[u]);
      }
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        const float y0 = __fmul_rn(v[0][j], kLog2e), y1 = __fmul_rn(v[1][j], kLog2e);
        const float y2 = __fmul_rn(v[2][j], kLog2e), y3 = __fmul_rn(v[3][j], kLog2e);
        const float mn = fmaxf(m[j], fmaxf(fmaxf(y0, y1), fmaxf(y2, y3)));
        const float ms = mn == -INFINITY ? 0.f : mn;  // safe max: all -inf so far gives weights 0, not NaN
        const float c = ex2a(m[j] - ms);
        const float e0 = ex2a(y0 - ms), e1 = ex2a(y1 - ms), e2 = ex2a(y2 - ms), e3 = ex2a(y3 - ms);
        s[j] = s[j] * c + ((e0 + e1) + (e2 + e3));
        if constexpr (MODE == 1)
          d[j] = d[j] * c + ((gv[0][j] * e0 + gv[1][j] * e1) + (gv[2][j] * e2 + gv[3][j] * e3));
        m[j] = mn;
      }
    }
    for (; r < b1; r += kSmWarps) {
      float v[VEC], gv[VEC];
      VecIO<T, VEC>::load(x + r * D + col, v);
      if constexpr (MODE == 1) VecIO<T, VEC>::load(g + r * D + col, gv);
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        if constexpr (MODE == 1) online_update_d(m[j], s[j], d[j], __fmul_rn(v[j], kLog2e), gv[j]);
        else online_update(m[j], s[j], __fmul_rn(v[j], kLog2e));
      }
    }
  }
  // VJP: fold d into the per-warp partials before combine_ms overwrites m (d_w 2^(m_w - M), summed below)
  float mw[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) mw[j] = m[j];
  combine_ms<VEC>(m, s, sm_m, sm_s, col_local);
  float inv[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) inv[j] = 1.0f / s[j];
  if constexpr (MODE == 0) {
    if (!active) return;
    for (int64_t r = b0 + w; r < b1; r += kSmWarps) {
      float v[VEC];
      VecIO<T, VEC>::load(x + r * D + col, v);
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[j] = ex2a(__fmul_rn(v[j], kLog2e) - m[j]) * inv[j];
      VecIO<T, VEC>::store(out + r * D + col, v);
    }
  } else {
    // dot = sum_rows g p = (sum_w d_w 2^(m_w - M)) / S, then dx = p (g - dot)
    float dot[VEC];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < VEC; ++j)
      sm_s[w * 32 * VEC + col_local + j] = mw[j] == -INFINITY ? 0.f : d[j] * exp2f(mw[j] - m[j]);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      float t = 0.f;
      for (int ww = 0; ww < kSmWarps; ++ww) t += sm_s[ww * 32 * VEC + col_local + j];
      dot[j] = t * inv[j];
    }
    if (!active) return;
    for (int64_t r = b0 + w; r < b1; r += kSmWarps) {
      float v[VEC], gv[VEC];
      VecIO<T, VEC>::load(x + r * D + col, v);
      VecIO<T, VEC>::load(g + r * D + col, gv);
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[j] = ex2a(__fmul_rn(v[j], kLog2e) - m[j]) * inv[j] * (gv[j] - dot[j]);
      VecIO<T, VEC>::store(out + r * D + col, v);
    }
  }
}

// jagged2_softmax: one warp per block row (jagged row index R in [0, total_rows)); MODE 0 forward, 1 VJP.
// A row (n elements at any element alignment) is covered by the aligned 16-byte chunks that overlap it; each lane
// holds up to kCh of them in registers (rows up to 32 kCh chunks: n <= 1017 bf16 / 509 fp32), so the input is
// read from HBM once: max -> sum of 2^(y - M) -> write p (VJP: also g, dot = sum g p, write p (g - dot)).
// Chunks wholly inside the row are stored with one 16-byte store; the (at most two) edge chunks element-wise,
// so neighbouring rows written by other warps are never touched. Longer rows take a two-pass loop.
constexpr int kCh = 4;
template <typename T>
struct Chunk {
  static constexpr int E = 16 / sizeof(T);  // elements per 16-byte chunk
  static __device__ __forceinline__ void unpack(const uint4& c, float (&v)[E]) {
    if constexpr (std::is_same_v<T, float>) {
      v[0] = __uint_as_float(c.x); v[1] = __uint_as_float(c.y); v[2] = __uint_as_float(c.z); v[3] = __uint_as_float(c.w);
    } else {
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&c);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(h[j]);
        v[2 * j] = f.x;
        v[2 * j + 1] = f.y;
      }
    }
  }
  static __device__ __forceinline__ uint4 pack(const float (&v)[E]) {
    uint4 c;
    if constexpr (std::is_same_v<T, float>) {
      c = make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]), __float_as_uint(v[3]));
    } else {
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&c);
#pragma unroll
      for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
    }
    return c;
  }
};

// LPR: lanes per row — 32 (a warp per row) or 16 (two rows per warp, one per half-warp: half the per-row
// reduction and bookkeeping overhead per element for rows that fit)
template <int LPR>
__device__ __forceinline__ float grp_max(float v) {
#pragma unroll
  for (int m = LPR / 2; m > 0; m >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, m));
  return v;
}
template <int LPR>
__device__ __forceinline__ float grp_sum(float v) {
#pragma unroll
  for (int m = LPR / 2; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}
template <typename T, int LPR = 32>
__device__ __forceinline__ bool j2_fits(int64_t base, int64_t n) {
  constexpr int E = Chunk<T>::E;
  return (base + n - (base & ~(int64_t)(E - 1)) + E - 1) / E <= LPR * kCh;
}
// the aligned chunks of row [base, base + n) owned by this lane; elements outside the row read as -inf (inputs:
// weight 0) or 0 (gradients)
template <typename T, bool kZero = false, int LPR = 32>
__device__ __forceinline__ void j2_load(const T* __restrict__ p, int64_t base, int64_t n, int lane, uint4 (&c)[kCh]) {
  constexpr int E = Chunk<T>::E;
  constexpr uint32_t kNegInf2 = kZero ? 0u : std::is_same_v<T, float> ? 0xff800000u : 0xff80ff80u;  // fill, every element
  constexpr uint32_t kFill = kNegInf2 & 0xffffu;  // one bf16 element's fill
  const int64_t a0 = base & ~(int64_t)(E - 1);
  const int lo = (int)(base - a0), hi = lo + (int)n;
#pragma unroll
  for (int k = 0; k < kCh; ++k) {
    const int e0 = (lane + LPR * k) * E;
    c[k] = make_uint4(kNegInf2, kNegInf2, kNegInf2, kNegInf2);
    if (e0 < hi) c[k] = __ldcs(reinterpret_cast<const uint4*>(p + a0) + lane + LPR * k);
    if (e0 < lo || e0 + E > hi) {  // edge chunk (at most two per row): mask the neighbours' elements
      uint32_t* w = reinterpret_cast<uint32_t*>(&c[k]);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if (e0 + e >= lo && e0 + e < hi) continue;
        if constexpr (std::is_same_v<T, float>) w[e] = kNegInf2;
        else w[e >> 1] = (e & 1) ? ((w[e >> 1] & 0xffffu) | (kFill << 16)) : ((w[e >> 1] & 0xffff0000u) | kFill);
      }
    }
  }
}
template <typename T>
__device__ __forceinline__ float2 j2_pair(const uint4& c, int j) {  // elements 2j, 2j+1 of a chunk as floats
  if constexpr (std::is_same_v<T, float>) {
    return j == 0 ? make_float2(__uint_as_float(c.x), __uint_as_float(c.y))
                  : make_float2(__uint_as_float(c.z), __uint_as_float(c.w));
  } else {
    const uint32_t w = j == 0 ? c.x : j == 1 ? c.y : j == 2 ? c.z : c.w;
    return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
  }
}
template <typename T, int MODE, int LPR = 32>
__device__ __forceinline__ void j2_row_regs(const uint4 (&xc)[kCh], const uint4 (&gc)[kCh], T* __restrict__ out,
                                            int64_t base, int64_t n, int lane) {
  using C = Chunk<T>;
  constexpr int E = C::E, P = E / 2;  // element pairs per chunk
  const int64_t a0 = base & ~(int64_t)(E - 1);
  const int lo = (int)(base - a0), hi = lo + (int)n;
  // max over the raw values (masked elements are -inf); y = x log2(e) rounded once (__fmul_rn), so the max
  // element gives 2^(y - M) = 2^0 = 1 exactly
  float m = -INFINITY;
#pragma unroll
  for (int k = 0; k < kCh; ++k) {
    if constexpr (std::is_same_v<T, float>) {
      m = tc::fmax3(m, fmaxf(__uint_as_float(xc[k].x), __uint_as_float(xc[k].y)),
                    fmaxf(__uint_as_float(xc[k].z), __uint_as_float(xc[k].w)));
    } else {
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&xc[k]);
      const __nv_bfloat162 mm = __hmax2(__hmax2(h[0], h[1]), __hmax2(h[2], h[3]));
      m = tc::fmax3(m, __low2float(mm), __high2float(mm));
    }
  }
  const float Ml = __fmul_rn(grp_max<LPR>(m), kLog2e);
  const float2 l2 = make_float2(kLog2e, kLog2e), nM = make_float2(-Ml, -Ml);
  float2 ev[kCh][P];  // 2^(y - M), kept for the output pass (one exponential per element)
  float2 sum2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < kCh; ++k) {
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const float2 y = tc::fadd2(tc::fmul2(j2_pair<T>(xc[k], j), l2), nM);
      ev[k][j] = make_float2(ex2a(y.x), ex2a(y.y));
      sum2 = tc::fadd2(sum2, ev[k][j]);
    }
  }
  const float inv = 1.0f / grp_sum<LPR>(sum2.x + sum2.y);
  const float2 inv2 = make_float2(inv, inv);
  float2 dot2 = make_float2(0.f, 0.f);
  if constexpr (MODE == 1) {
#pragma unroll
    for (int k = 0; k < kCh; ++k)
#pragma unroll
      for (int j = 0; j < P; ++j) {
        dot2 = tc::ffma2(j2_pair<T>(gc[k], j), tc::fmul2(ev[k][j], inv2), dot2);  // masked g elements are 0
      }
  }
  const float dot = MODE == 1 ? grp_sum<LPR>(dot2.x + dot2.y) : 0.f;
  const float2 nd = make_float2(-dot, -dot);
#pragma unroll
  for (int k = 0; k < kCh; ++k) {
    const int e0 = (lane + LPR * k) * E;
    if (e0 >= hi) break;
    float v[E];
#pragma unroll
    for (int j = 0; j < P; ++j) {
      float2 pe = tc::fmul2(ev[k][j], inv2);
      if constexpr (MODE == 1) pe = tc::fmul2(pe, tc::fadd2(j2_pair<T>(gc[k], j), nd));
      v[2 * j] = pe.x;
      v[2 * j + 1] = pe.y;
    }
    if (e0 >= lo && e0 + E <= hi) {
      __stcs(reinterpret_cast<uint4*>(out + a0) + lane + LPR * k, C::pack(v));
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (e0 + e >= lo && e0 + e < hi) st(out + a0 + e0 + e, v[e]);
    }
  }
}
// rows too long for the registers (or unaligned tensors): online max/sum pass, then the output pass
template <typename T, int MODE>
__device__ __noinline__ void j2_row_loop(const T* __restrict__ s, const T* __restrict__ g, T* __restrict__ out,
                                        int64_t base, int64_t n, int lane) {
  float m = -INFINITY, sm = 0.f;
  int64_t c = lane;
  for (; c + 96 < n; c += 128) {  // four elements per step: loads in flight together, one branch-free update
    const float y0 = __fmul_rn(ld(s + base + c), kLog2e), y1 = __fmul_rn(ld(s + base + c + 32), kLog2e);
    const float y2 = __fmul_rn(ld(s + base + c + 64), kLog2e), y3 = __fmul_rn(ld(s + base + c + 96), kLog2e);
    const float mn = fmaxf(m, fmaxf(fmaxf(y0, y1), fmaxf(y2, y3)));
    const float ms = mn == -INFINITY ? 0.f : mn;  // safe max (see online_update)
    sm = sm * ex2a(m - ms) + ((ex2a(y0 - ms) + ex2a(y1 - ms)) + (ex2a(y2 - ms) + ex2a(y3 - ms)));
    m = mn;
  }
  for (; c < n; c += 32) online_update(m, sm, __fmul_rn(ld(s + base + c), kLog2e));
  const float M = warp_max(m);
  const float S = warp_sum(m == -INFINITY ? 0.f : sm * exp2f(m - M));
  const float inv = 1.0f / S;
  if constexpr (MODE == 0) {
    for (int64_t c = lane; c < n; c += 32) st(out + base + c, ex2a(__fmul_rn(ld(s + base + c), kLog2e) - M) * inv);
  } else {
    float dot = 0.f;
    for (int64_t c = lane; c < n; c += 32)
      dot += ld(g + base + c) * (ex2a(__fmul_rn(ld(s + base + c), kLog2e) - M) * inv);
    dot = warp_sum(dot);
    for (int64_t c = lane; c < n; c += 32) {
      const float p = ex2a(__fmul_rn(ld(s + base + c), kLog2e) - M) * inv;
      st(out + base + c, p * (ld(g + base + c) - dot));
    }
  }
}

// Work split: the flat jagged^2 array (sq[batch] elements, rows contiguous across samples) is cut into one
// equal element range per warp; a warp owns the rows that START in its range and walks them in order with a
// (sample, row) cursor — one sample search per warp instead of one per row. In the forward, the next row's
// chunks are loaded before the current row is reduced, so two rows per warp are in flight. (Measured at cfg4:
// 1.26 ms vs 1.44 ms for a lane-strided two-pass warp per row, and 1.53 ms for a CTA variant that stages 32 KB
// spans in shared memory with 1-D bulk copies — the bound is issue/latency per row, not load bandwidth.)
template <typename T, int MODE>
__global__ void __launch_bounds__(256, MODE == 0 ? 3 : 2) jagged2_softmax_kernel(const int64_t* __restrict__ off,
                                                                                 const int64_t* __restrict__ sq,
                                                                                 int64_t batch,
                                                                                 const T* __restrict__ s,
                                                                                 const T* __restrict__ g,
                                                                                 T* __restrict__ out) {
  constexpr int E = Chunk<T>::E;
  const int lane = threadIdx.x & 31;
  __shared__ int64_t coarse_sq[257];
  for (int k = threadIdx.x; k <= 256; k += blockDim.x) coarse_sq[k] = sq[(int64_t)k * batch / 256];
  __syncthreads();
  const int64_t total = coarse_sq[256];  // sq[batch]: total elements
  const int64_t total_al = total & ~(int64_t)(E - 1);  // whole 16-byte chunks inside the tensor
  const int64_t W = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t e_lo = (int64_t)((__int128)total * gw / W), e_hi = (int64_t)((__int128)total * (gw + 1) / W);
  if (e_lo >= e_hi) return;
  // sample holding element e_lo: the largest i with sq[i] <= e_lo (non-empty, since sq[i+1] > e_lo)
  int klo = 0, khi = 255;
  while (klo < khi) {
    const int mid = (klo + khi + 1) >> 1;
    if (coarse_sq[mid] <= e_lo) klo = mid; else khi = mid - 1;
  }
  int64_t lo = (int64_t)klo * batch / 256, hi = (int64_t)(klo + 1) * batch / 256;
  if (hi > batch - 1) hi = batch - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (sq[mid] <= e_lo) lo = mid; else hi = mid - 1;
  }
  int64_t i = lo, sq_i = sq[i], n = off[i + 1] - off[i];
  int64_t r = (e_lo - sq_i + n - 1) / n;  // first row starting at or after e_lo
  const bool aligned = ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(out) |
                         reinterpret_cast<uintptr_t>(MODE ? g : s)) % 16) == 0;
  // register path: the row's aligned chunks fit the lane registers and stay inside the tensor
  // register paths: the row's aligned chunks fit LPR lanes' registers and stay inside the tensor
  auto regs_ok = [&](int64_t b, int64_t len, auto lpr) {
    return aligned && j2_fits<T, decltype(lpr)::value>(b, len) &&
           ((b + len + E - 1) & ~(int64_t)(E - 1)) <= total_al;
  };
  // advance the cursor to the next row start (rolling over empty samples); false past the warp's range
  auto settle = [&]() -> bool {
    while (r >= n) {
      sq_i += n * n;
      if (++i >= batch) return false;
      n = off[i + 1] - off[i];
      r = 0;
    }
    return sq_i + r * n < e_hi;
  };
  using L16 = std::integral_constant<int, 16>;
  using L32 = std::integral_constant<int, 32>;
  // a unit: one row on the whole warp (mode 1), two consecutive short rows on the two half-warps (mode 2), or a
  // long row on the two-pass loop (mode 3); mode 0: the warp's range is done
  struct Unit {
    int64_t b0, n0, b1, n1;
    int mode;
  };
  auto next_unit = [&]() -> Unit {
    Unit u{0, 0, 0, 0, 0};
    if (!settle()) return u;
    u.b0 = sq_i + r * n;
    u.n0 = n;
    ++r;
    if (!regs_ok(u.b0, u.n0, L32{})) {
      u.mode = 3;
      return u;
    }
    u.mode = 1;
    if (regs_ok(u.b0, u.n0, L16{}) && settle()) {
      const int64_t b1 = sq_i + r * n;
      if (regs_ok(b1, n, L16{})) {
        u.b1 = b1;
        u.n1 = n;
        ++r;
        u.mode = 2;
      }
    }
    return u;
  };
  const int half = lane >> 4, sub = lane & 15;
  auto load_unit = [&](const Unit& u, uint4 (&c)[kCh], const T* src, auto zero) {
    constexpr bool Z = decltype(zero)::value;  // grad_out: elements outside the row read as 0
    if (u.mode == 1) j2_load<T, Z, 32>(src, u.b0, u.n0, lane, c);
    if (u.mode == 2) j2_load<T, Z, 16>(src, half ? u.b1 : u.b0, half ? u.n1 : u.n0, sub, c);
  };
  // the VJP also keeps grad_out's chunks (x and g read once)
  uint4 cur[kCh], nxt[kCh], gcur[MODE ? kCh : 1], gnxt[MODE ? kCh : 1];
  Unit uc = next_unit();
  if (uc.mode == 0) return;
  load_unit(uc, cur, s, std::false_type{});
  if constexpr (MODE == 1) load_unit(uc, gcur, g, std::true_type{});
  for (;;) {
    const Unit un = next_unit();
    load_unit(un, nxt, s, std::false_type{});  // in flight while this unit is reduced
    if constexpr (MODE == 1) load_unit(un, gnxt, g, std::true_type{});
    const uint4(&gc)[kCh] = [&]() -> const uint4(&)[kCh] {
      if constexpr (MODE == 1) return gcur;
      else return cur;
    }();
    if (uc.mode == 1) j2_row_regs<T, MODE, 32>(cur, gc, out, uc.b0, uc.n0, lane);
    else if (uc.mode == 2) j2_row_regs<T, MODE, 16>(cur, gc, out, half ? uc.b1 : uc.b0, half ? uc.n1 : uc.n0, sub);
    else j2_row_loop<T, MODE>(s, g, out, uc.b0, uc.n0, lane);
    if (un.mode == 0) break;
    uc = un;
#pragma unroll
    for (int k = 0; k < kCh; ++k) cur[k] = nxt[k];
    if constexpr (MODE == 1) {
#pragma unroll
      for (int k = 0; k < kCh; ++k) gcur[k] = gnxt[k];
    }
  }
}

template <typename T, int MODE>
static jg_status softmax_dispatch(const int64_t* off, int64_t batch, int64_t D, const void* x,
                                  const void* g, void* out, cudaStream_t st) {
  const uintptr_t align = (uintptr_t)x | (uintptr_t)out | (uintptr_t)(g ? g : x);
  auto ok = [&](int vec) {
    return D % vec == 0 && (align % (vec * sizeof(T))) == 0 && vec * sizeof(T) <= 16 && D >= 32 * vec;
  };
  const dim3 block(kSmWarps * 32);
  auto go = [&](auto vec_tag) {
    constexpr int V = decltype(vec_tag)::value;
    dim3 grid((unsigned)batch, (unsigned)((D + 32 * V - 1) / (32 * V)));
    jagged_softmax_kernel<T, V, MODE><<<grid, block, 0, st>>>(off, D, (const T*)x, (const T*)g, (T*)out);
  };
  if (ok(8)) go(std::integral_constant<int, 8>{});
  else if (ok(4)) go(std::integral_constant<int, 4>{});
  else if (ok(2)) go(std::integral_constant<int, 2>{});
  else go(std::integral_constant<int, 1>{});
  JG_LAUNCHED("jagged_softmax_kernel");
  return JG_OK;
}

jg_status launch_jagged_softmax(const int64_t* off, int64_t batch, int64_t D, const void* x,
                                const void* g, void* out, jg_dtype dt, bool vjp, cudaStream_t st) {
  if (batch == 0 || D == 0) return JG_OK;
  if (dt == JG_F32) return vjp ? softmax_dispatch<float, 1>(off, batch, D, x, g, out, st)
                               : softmax_dispatch<float, 0>(off, batch, D, x, g, out, st);
  if (dt == JG_BF16) return vjp ? softmax_dispatch<__nv_bfloat16, 1>(off, batch, D, x, g, out, st)
                                : softmax_dispatch<__nv_bfloat16, 0>(off, batch, D, x, g, out, st);
  return fail(JG_UNSUPPORTED, "jagged_softmax: dtype not supported on device (no CPU fallback)");
}

jg_status launch_jagged2_softmax(const int64_t* off, const int64_t* sq, int64_t batch, int64_t total_rows,
                                 const void* s, const void* g, void* out, jg_dtype dt, bool vjp,
                                 cudaStream_t st) {
  if (total_rows == 0 || batch == 0) return JG_OK;
  auto go = [&](auto tag, auto mode) -> jg_status {
    using T = decltype(tag);
    constexpr int M = decltype(mode)::value;
    // 24 (forward) / 16 (VJP) resident warps per SM, each with its element range; the grid covers 64 ranges per
    // SM so the per-range imbalance (one row) averages out over several waves
    jagged2_softmax_kernel<T, M><<<8 * device_sm_count(), 256, 0, st>>>(off, sq, batch, (const T*)s, (const T*)g,
                                                                       (T*)out);
    JG_LAUNCHED("jagged2_softmax_kernel");
    return JG_OK;
  };
  if (dt == JG_F32) return vjp ? go(float{}, std::integral_constant<int, 1>{}) : go(float{}, std::integral_constant<int, 0>{});
  if (dt == JG_BF16)
    return vjp ? go(__nv_bfloat16{}, std::integral_constant<int, 1>{}) : go(__nv_bfloat16{}, std::integral_constant<int, 0>{});
  return fail(JG_UNSUPPORTED, "jagged2_softmax: dtype not supported on device (no CPU fallback)");
}

}  // namespace jg
