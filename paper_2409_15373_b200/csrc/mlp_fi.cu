// mlp_fi.cu — device pieces of the SURVEY §8f "next" rows that are not plain grouped GEMMs:
//   jagged MLP (linalg.cpp:246-277, VJP :509-573): bias + activation epilogue, ReLU mask, deterministic
//   column sums (db), the single-segment offsets {0, rows} the grouped GEMM runs on;
//   feature interaction (attention.cpp:291-309): fp32 -> bf16 cast of the softmax weights.
// The contractions themselves go through the grouped GEMM (gemm_simt.cu / gemm_sm100.cu) from capi.cu.
#include "common.cuh"
#include "internal.h"

namespace jg {

__global__ void two_offsets_kernel(int64_t* o, int64_t rows) {
  o[0] = 0;
  o[1] = rows;
}

// out = act(acc + bias) in T; preact (optional) = acc + bias in T (its sign is all the VJP needs)
template <typename T>
__global__ void bias_act_kernel(const float* __restrict__ acc, const T* __restrict__ bias, int64_t rows, int64_t d,
                                int relu, T* __restrict__ out, T* __restrict__ preact) {
  const int64_t n = rows * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const float v = acc[e] + ld(bias + e % d);
    if (preact) st(preact + e, v);
    st(out + e, relu ? fmaxf(v, 0.f) : v);
  }
}

// delta = relu ? (preact > 0 ? g : 0) : g   (linalg.cpp:531-535: pre-activation <= 0 zeroes the gradient)
template <typename T>
__global__ void relu_mask_kernel(const T* __restrict__ g, const T* __restrict__ preact, int64_t n, int relu,
                                 T* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const float v = ld(g + e);
    st(out + e, (relu && !(ld(preact + e) > 0.f)) ? 0.f : v);
  }
}

// Column sums in a fixed order (deterministic): stage 1, block (column tile of 32, row chunk) -> partial;
// stage 2, one thread per column adds the chunk partials in order.
constexpr int kColChunk = 2048;
template <typename T>
__global__ void __launch_bounds__(256) colsum_partial_kernel(const T* __restrict__ x, int64_t rows, int64_t cols,
                                                             float* __restrict__ partial) {
  __shared__ float red[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t c = blockIdx.x * 32 + tx;
  const int64_t r0 = (int64_t)blockIdx.y * kColChunk, r1 = r0 + kColChunk < rows ? r0 + kColChunk : rows;
  float s = 0.f;
  if (c < cols)
    for (int64_t r = r0 + ty; r < r1; r += 8) s += ld(x + r * cols + c);
  red[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && c < cols) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k][tx];
    partial[(int64_t)blockIdx.y * cols + c] = t;
  }
}
template <typename T>
__global__ void colsum_final_kernel(const float* __restrict__ partial, int64_t chunks, int64_t cols, T* __restrict__ out) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float s = 0.f;
  for (int64_t k = 0; k < chunks; ++k) s += partial[k * cols + c];
  st(out + c, s);
}

template <typename T>
__global__ void cast_f32_kernel(const float* __restrict__ a, int64_t n, T* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    st(out + e, a[e]);
}

static int grid_of(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 8 * (int64_t)device_sm_count()));
}

#define DISPATCH_T2(dtype, ...)                                                \
  do {                                                                         \
    if ((dtype) == JG_F32) { using T = float; __VA_ARGS__; }                   \
    else if ((dtype) == JG_BF16) { using T = __nv_bfloat16; __VA_ARGS__; }     \
    else return fail(JG_UNSUPPORTED, "dtype not supported on device (no CPU fallback)"); \
  } while (0)

__global__ void uniform_offsets_kernel(int64_t* o, int64_t batch, int64_t step) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= batch; i += (int64_t)gridDim.x * blockDim.x)
    o[i] = i * step;
}

jg_status launch_uniform_offsets(int64_t* o, int64_t batch, int64_t step, cudaStream_t st) {
  uniform_offsets_kernel<<<(unsigned)std::min<int64_t>((batch + 256) / 256, 1024), 256, 0, st>>>(o, batch, step);
  JG_LAUNCHED("uniform_offsets_kernel");
  return JG_OK;
}

jg_status launch_two_offsets(int64_t* o, int64_t rows, cudaStream_t st) {
  two_offsets_kernel<<<1, 1, 0, st>>>(o, rows);
  JG_LAUNCHED("two_offsets_kernel");
  return JG_OK;
}

jg_status launch_bias_act(const float* acc, const void* bias, int64_t rows, int64_t d, int relu, void* out,
                          void* preact, jg_dtype dt, cudaStream_t st) {
  if (rows * d == 0) return JG_OK;
  DISPATCH_T2(dt, bias_act_kernel<T><<<grid_of(rows * d), 256, 0, st>>>(acc, (const T*)bias, rows, d, relu, (T*)out,
                                                                         (T*)preact));
  JG_LAUNCHED("bias_act_kernel");
  return JG_OK;
}

jg_status launch_relu_mask(const void* g, const void* preact, int64_t n, int relu, void* out, jg_dtype dt,
                           cudaStream_t st) {
  if (n == 0) return JG_OK;
  DISPATCH_T2(dt, relu_mask_kernel<T><<<grid_of(n), 256, 0, st>>>((const T*)g, (const T*)preact, n, relu, (T*)out));
  JG_LAUNCHED("relu_mask_kernel");
  return JG_OK;
}

int64_t colsum_scratch_floats(int64_t rows, int64_t cols) {
  const int64_t chunks = rows > 0 ? (rows + kColChunk - 1) / kColChunk : 1;
  return chunks * cols;
}

jg_status launch_colsum(const void* x, int64_t rows, int64_t cols, void* out, float* partial, jg_dtype dt,
                        cudaStream_t st) {
  if (cols == 0) return JG_OK;
  const int64_t chunks = rows > 0 ? (rows + kColChunk - 1) / kColChunk : 1;
  if (rows == 0) {
    JG_CUDA(cudaMemsetAsync(partial, 0, sizeof(float) * cols, st));
  } else {
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)chunks);
    DISPATCH_T2(dt, colsum_partial_kernel<T><<<grid, 256, 0, st>>>((const T*)x, rows, cols, partial));
    JG_LAUNCHED("colsum_partial_kernel");
  }
  DISPATCH_T2(dt, colsum_final_kernel<T><<<(unsigned)((cols + 255) / 256), 256, 0, st>>>(partial, chunks, cols, (T*)out));
  JG_LAUNCHED("colsum_final_kernel");
  return JG_OK;
}

jg_status launch_cast_f32(const float* a, int64_t n, void* out, jg_dtype dt, cudaStream_t st) {
  if (n == 0) return JG_OK;
  DISPATCH_T2(dt, cast_f32_kernel<T><<<grid_of(n), 256, 0, st>>>(a, n, (T*)out));
  JG_LAUNCHED("cast_f32_kernel");
  return JG_OK;
}

}  // namespace jg
