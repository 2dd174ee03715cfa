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
  float m[VEC], s[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) { m[j] = -INFINITY; s[j] = 0.f; }
  if (active) {
    // four rows per step: their loads in flight together, one branch-free running-max update per column
    // (s = s * 2^(m - m') + sum_k 2^(y_k - m'), MUFU ex2) instead of a branchy update per element
    int64_t r = b0 + w;
    for (; r + 3 * kSmWarps < b1; r += 4 * kSmWarps) {
      float v[4][VEC];
#pragma unroll
      for (int u = 0; u < 4; ++u) VecIO<T, VEC>::load(x + (r + u * kSmWarps) * D + col, v[u]);
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        const float y0 = __fmul_rn(v[0][j], kLog2e), y1 = __fmul_rn(v[1][j], kLog2e);
        const float y2 = __fmul_rn(v[2][j], kLog2e), y3 = __fmul_rn(v[3][j], kLog2e);
        const float mn = fmaxf(m[j], fmaxf(fmaxf(y0, y1), fmaxf(y2, y3)));
        const float ms = mn == -INFINITY ? 0.f : mn;  // safe max: all -inf so far gives weights 0, not NaN
        s[j] = s[j] * ex2a(m[j] - ms) + ((ex2a(y0 - ms) + ex2a(y1 - ms)) + (ex2a(y2 - ms) + ex2a(y3 - ms)));
        m[j] = mn;
      }
    }
    for (; r < b1; r += kSmWarps) {
      float v[VEC];
      VecIO<T, VEC>::load(x + r * D + col, v);
#pragma unroll
      for (int j = 0; j < VEC; ++j) online_update(m[j], s[j], __fmul_rn(v[j], kLog2e));
    }
  }
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
    // dot = sum_rows g * p, then dx = p (g - dot)
    float dot[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) dot[j] = 0.f;
    if (active) {
      for (int64_t r = b0 + w; r < b1; r += kSmWarps) {
        float v[VEC], gv[VEC];
        VecIO<T, VEC>::load(x + r * D + col, v);
        VecIO<T, VEC>::load(g + r * D + col, gv);
#pragma unroll
        for (int j = 0; j < VEC; ++j) dot[j] += gv[j] * (ex2a(__fmul_rn(v[j], kLog2e) - m[j]) * inv[j]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < VEC; ++j) sm_s[w * 32 * VEC + col_local + j] = dot[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      float t = 0.f;
      for (int ww = 0; ww < kSmWarps; ++ww) t += sm_s[ww * 32 * VEC + col_local + j];
      dot[j] = t;
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

// one warp per block row (jagged row index R in [0, total_rows)); MODE 0 forward, 1 VJP
template <typename T, int MODE>
__global__ void __launch_bounds__(256) jagged2_softmax_kernel(const int64_t* __restrict__ off,
                                                              const int64_t* __restrict__ sq,
                                                              int64_t batch, int64_t total_rows,
                                                              const T* __restrict__ s,
                                                              const T* __restrict__ g,
                                                              T* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  // row -> sample: a 257-point coarse copy of the offsets in smem narrows each row's search to ~batch/256
  // samples, so only ~log2(batch/256) dependent global loads remain per row
  __shared__ int64_t coarse_off[257];
  for (int k = threadIdx.x; k <= 256; k += blockDim.x) coarse_off[k] = off[(int64_t)k * batch / 256];
  __syncthreads();
  if (total_rows < 0) total_rows = off[batch];  // device-resident row count (no host sync)
  for (int64_t R = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; R < total_rows;
       R += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int klo = 0, khi = 256;  // largest k with coarse_off[k] <= R
    while (klo < khi) {
      const int mid = (klo + khi + 1) >> 1;
      if (coarse_off[mid] <= R) klo = mid; else khi = mid - 1;
    }
    int64_t lo = (int64_t)klo * batch / 256, hi = klo < 256 ? (int64_t)(klo + 1) * batch / 256 : batch;
    if (hi > batch - 1) hi = batch - 1;
    while (lo < hi) {  // sample_of_row restricted to [lo, hi]
      const int64_t mid = (lo + hi) >> 1;
      if (off[mid + 1] <= R) lo = mid + 1; else hi = mid;
    }
    const int64_t i = lo;
    const int64_t n = off[i + 1] - off[i], r = R - off[i];
    const int64_t base = sq[i] + r * n;
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
  if (total_rows == 0) return JG_OK;
  const int grid = total_rows < 0 ? 8 * kNumSMsB200 : (int)std::min<int64_t>((total_rows + 7) / 8, 16 * kNumSMsB200);
  if (dt == JG_F32) {
    if (vjp) jagged2_softmax_kernel<float, 1><<<grid, 256, 0, st>>>(off, sq, batch, total_rows, (const float*)s, (const float*)g, (float*)out);
    else jagged2_softmax_kernel<float, 0><<<grid, 256, 0, st>>>(off, sq, batch, total_rows, (const float*)s, nullptr, (float*)out);
  } else if (dt == JG_BF16) {
    using B = __nv_bfloat16;
    if (vjp) jagged2_softmax_kernel<B, 1><<<grid, 256, 0, st>>>(off, sq, batch, total_rows, (const B*)s, (const B*)g, (B*)out);
    else jagged2_softmax_kernel<B, 0><<<grid, 256, 0, st>>>(off, sq, batch, total_rows, (const B*)s, nullptr, (B*)out);
  } else {
    return fail(JG_UNSUPPORTED, "jagged2_softmax: dtype not supported on device (no CPU fallback)");
  }
  JG_LAUNCHED("jagged2_softmax_kernel");
  return JG_OK;
}

}  // namespace jg
