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

template <typename T>
__global__ void attn_delta_kernel(int64_t units, int H, int D, const T* __restrict__ go,
                                  const T* __restrict__ o, int64_t total_rows, float* __restrict__ delta) {
  const int lane = threadIdx.x & 31;
  for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < units;
       u += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t r = u / H;
    const int h = (int)(u - r * H);
    const int64_t base = u * D;  // [r, h, :] is contiguous at (r*H + h)*D
    float acc = 0.f;
    for (int d = lane; d < D; d += 32) acc = fmaf(ld(go + base + d), ld(o + base + d), acc);
    acc = warp_sum(acc);
    if (lane == 0) delta[(int64_t)h * total_rows + r] = acc;
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

template <typename T>
static jg_status fwd_t(const int64_t* off, int64_t batch, int64_t total_rows, int H, int D, const void* q,
                       const void* k, const void* v, void* out, float* lse, const int64_t* valid, cudaStream_t st) {
  const int64_t units = total_rows * H;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((units + kAttnWarps - 1) / kAttnWarps,
                                                               16 * device_sm_count()));
  const float scale_log2 = kLog2eA / sqrtf((float)D);
  attn_fwd_simt_kernel<T><<<grid, kAttnWarps * 32, kAttnWarps * D * sizeof(float), st>>>(
      off, batch, total_rows, H, D, (const T*)q, (const T*)k, (const T*)v, (T*)out, lse, scale_log2, valid);
  JG_LAUNCHED("attn_fwd_simt_kernel");
  return JG_OK;
}

template <typename T>
static jg_status bwd_t(const int64_t* off, int64_t batch, int64_t total_rows, int H, int D, const void* q,
                       const void* k, const void* v, const void* go, const void* o, const float* lse, void* dq,
                       void* dk, void* dv, float* delta, const int64_t* valid, cudaStream_t st) {
  const int64_t units = total_rows * H;
  const int sms = device_sm_count();
  attn_delta_kernel<T><<<(int)std::min<int64_t>((units + 7) / 8, 16 * sms), 256, 0, st>>>(
      units, H, D, (const T*)go, (const T*)o, total_rows, delta);
  JG_LAUNCHED("attn_delta_kernel");
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
                               jg_dtype dt, const int64_t* valid, cudaStream_t st) {
  if (total_rows == 0) return JG_OK;
  if (D > 32 * kMaxDPL) return fail(JG_UNSUPPORTED, "jagged_flash_attention_forward: head_dim > 256 unsupported");
  if (dt == JG_F32) return fwd_t<float>(off, batch, total_rows, H, D, q, k, v, out, lse, valid, st);
  if (dt == JG_BF16) return fwd_t<__nv_bfloat16>(off, batch, total_rows, H, D, q, k, v, out, lse, valid, st);
  return fail(JG_UNSUPPORTED, "jagged_flash_attention_forward: dtype not supported on device (no CPU fallback)");
}

jg_status launch_attn_bwd_simt(const int64_t* off, int64_t batch, int64_t total_rows, int H, int D,
                               const void* q, const void* k, const void* v, const void* go,
                               const void* o, const float* lse, void* dq, void* dk, void* dv,
                               float* delta, jg_dtype dt, const int64_t* valid, cudaStream_t st) {
  if (total_rows == 0) return JG_OK;
  if (D > 32 * kMaxDPL) return fail(JG_UNSUPPORTED, "jagged_flash_attention_backward: head_dim > 256 unsupported");
  if (dt == JG_F32)
    return bwd_t<float>(off, batch, total_rows, H, D, q, k, v, go, o, lse, dq, dk, dv, delta, valid, st);
  if (dt == JG_BF16)
    return bwd_t<__nv_bfloat16>(off, batch, total_rows, H, D, q, k, v, go, o, lse, dq, dk, dv, delta, valid, st);
  return fail(JG_UNSUPPORTED, "jagged_flash_attention_backward: dtype not supported on device (no CPU fallback)");
}

}  // namespace jg
