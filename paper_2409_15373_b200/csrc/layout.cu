// layout.cu — offsets layer, device tile scheduler, layout conversions, elementwise ops.
//
// Integer work here is bit-exact with the reference (tensor.cpp:72-175): offsets are int64 prefix
// sums, sq_offsets the prefix sum of Bi^2, conversions are pure copies. The scheduler replaces the
// reference's static contiguous chunking of samples over std::threads (parallel.cpp:9-26) with a
// device-built work list of (sample, 128-row tile) items ordered longest-first for persistent CTAs.
#include "common.cuh"
#include "internal.h"

namespace jg {

// ------------------------------------------------------------------ single-CTA exclusive scan
// mode 0: v_i = lengths[i] (negative -> *bad = first i)
// mode 1: v_i = (off[i+1]-off[i])^2
// mode 2: v_i = off[i+1]-off[i]
constexpr int kScanThreads = 1024;

__device__ __forceinline__ int64_t scan_value(int mode, const int64_t* in, int64_t i) {
  if (mode == 0) return in[i];
  const int64_t n = in[i + 1] - in[i];
  return mode == 1 ? n * n : n;
}

__global__ void __launch_bounds__(kScanThreads) scan_kernel(int mode, const int64_t* __restrict__ in,
                                                            int64_t n, int64_t* __restrict__ out,
                                                            int64_t* __restrict__ bad) {
  const int64_t chunk = (n + kScanThreads - 1) / kScanThreads;
  const int64_t b = (int64_t)threadIdx.x * chunk;
  const int64_t e = min(n, b + chunk);
  int64_t local = 0;
  int64_t first_bad = INT64_MAX;
  for (int64_t i = b; i < e; ++i) {
    const int64_t v = scan_value(mode, in, i);
    if (mode == 0 && v < 0 && first_bad == INT64_MAX) first_bad = i;
    local += v;
  }
  int64_t total;
  int64_t run = block_exclusive_scan(local, &total);
  for (int64_t i = b; i < e; ++i) {
    out[i] = run;
    run += scan_value(mode, in, i);
  }
  if (threadIdx.x == 0) out[n] = total;
  if (mode == 0 && bad != nullptr) {
    __shared__ unsigned long long sbad;
    if (threadIdx.x == 0) sbad = (unsigned long long)INT64_MAX;
    __syncthreads();
    if (first_bad != INT64_MAX) atomicMin(&sbad, (unsigned long long)first_bad);
    __syncthreads();
    if (threadIdx.x == 0) *bad = sbad == (unsigned long long)INT64_MAX ? -1 : (int64_t)sbad;
  }
}

__global__ void lengths_kernel(const int64_t* __restrict__ off, int64_t n, int64_t* __restrict__ len) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    len[i] = off[i + 1] - off[i];
}

jg_status launch_scan(int mode, const int64_t* in, int64_t n, int64_t* out, int64_t* bad, cudaStream_t s) {
  scan_kernel<<<1, kScanThreads, 0, s>>>(mode, in, n, out, bad);
  JG_LAUNCHED("scan_kernel");
  return JG_OK;
}

jg_status launch_lengths(const int64_t* off, int64_t n, int64_t* len, cudaStream_t s) {
  if (n == 0) return JG_OK;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 4 * kNumSMsB200);
  lengths_kernel<<<grid, 256, 0, s>>>(off, n, len);
  JG_LAUNCHED("lengths_kernel");
  return JG_OK;
}

// ------------------------------------------------------------------ LPT work list
// Items (sample, tile) for tile in [0, ceil(Bi/kTile)); all tiles of a sample cost the same
// (non-causal attention streams all ceil(Bi/kTile) key blocks), so ordering samples by
// descending tile count is the longest-processing-time-first order. Stable within a bin (sample
// ascending) so the list is deterministic. Bins are clamped at kMaxBins (longer samples share the
// last bin, still stable).
constexpr int kMaxBins = 64;

// Forward sample packing (short samples): a sample is packable when it lies inside one aligned 128-row window of
// the flat row space; the packable samples of window w (and the empty samples between them) become ONE forward
// item (first sample, -count) whose
// query tile and single key block are the window's packed rows, masked block-diagonally per sample by the
// kernel. Zipf-distributed batches (cfg2: median length 14) otherwise spend a whole item latency per sample.
__device__ __forceinline__ bool packable(int64_t a, int64_t b) { return b > a && (a >> 7) == ((b - 1) >> 7); }

__global__ void pack_mark_kernel(const int64_t* __restrict__ off, int64_t batch, int* __restrict__ win_first,
                                 int* __restrict__ win_last) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < batch; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = off[i], b = off[i + 1];
    if (!packable(a, b)) continue;
    atomicMin(win_first + (a >> 7), (int)i);
    atomicMax(win_last + (a >> 7), (int)i);
  }
}

__global__ void __launch_bounds__(kScanThreads) work_list_kernel(const int64_t* __restrict__ off,
                                                                 int64_t batch, int tile,
                                                                 int2* __restrict__ items,
                                                                 int64_t* __restrict__ count,
                                                                 const int* __restrict__ win_first,
                                                                 const int* __restrict__ win_last, int64_t nwin,
                                                                 int64_t split_below) {
  __shared__ int present[kMaxBins + 1];
  for (int b = threadIdx.x; b <= kMaxBins; b += blockDim.x) present[b] = 0;
  __syncthreads();
  const bool pack = win_last != nullptr;
  // packed (forward) list: when the tile-pair items and packs together would not fill the SMs (short batches,
  // cfg2), the unpacked samples are listed as single 128-row query tiles instead (flag bit 30 in the tile field):
  // the longest samples then run on twice the CTAs, and a lone tile's key loop is shorter than a pair's
  if (pack) {
    int64_t t_local = 0;
    for (int64_t i = threadIdx.x; i < batch; i += blockDim.x)
      if (!packable(off[i], off[i + 1])) t_local += (off[i + 1] - off[i] + tile - 1) / tile;
    for (int64_t w = threadIdx.x; w < nwin; w += blockDim.x) t_local += win_last[w] >= 0 ? 1 : 0;
    int64_t total;
    block_exclusive_scan(t_local, &total);
    if (total < split_below) tile = 128;
  }
  const int split = (pack && tile == 128) ? (1 << 30) : 0;
  for (int64_t i = threadIdx.x; i < batch; i += blockDim.x) {
    const int64_t nb = (off[i + 1] - off[i] + tile - 1) / tile;
    if (nb > 0 && !(pack && packable(off[i], off[i + 1]))) present[nb < kMaxBins ? nb : kMaxBins] = 1;
  }
  __syncthreads();
  int64_t base = 0;
  for (int bin = kMaxBins; bin >= 1; --bin) {
    if (!present[bin]) continue;  // uniform across the block
    for (int64_t c0 = 0; c0 < batch; c0 += blockDim.x) {
      const int64_t i = c0 + threadIdx.x;
      int64_t nt = 0;
      if (i < batch) {
        const int64_t nb = (off[i + 1] - off[i] + tile - 1) / tile;
        const int64_t key = nb < kMaxBins ? nb : kMaxBins;
        nt = (key == bin && !(pack && packable(off[i], off[i + 1]))) ? nb : 0;
      }
      int64_t tot;
      const int64_t pos = base + block_exclusive_scan(nt, &tot);
      for (int64_t t = 0; t < nt; ++t) items[pos + t] = make_int2((int)i, (int)t | split);
      base += tot;
    }
  }
  if (pack) {  // one key block each: last in LPT order, windows ascending
    for (int64_t w0 = 0; w0 < nwin; w0 += blockDim.x) {
      const int64_t w = w0 + threadIdx.x;
      const int64_t has = (w < nwin && win_last[w] >= 0) ? 1 : 0;
      int64_t tot;
      const int64_t pos = base + block_exclusive_scan(has, &tot);
      if (has) items[pos] = make_int2(win_first[w], win_first[w] - win_last[w] - 1);
      base += tot;
    }
  }
  if (threadIdx.x == 0) *count = base;
}

jg_status launch_work_list(const int64_t* off, int64_t batch, int tile, int2* items, int64_t* count,
                           cudaStream_t s, int* win_first, int* win_last, int64_t nwin) {
  if (win_last) {
    JG_CUDA(cudaMemsetAsync(win_first, 0x7f, sizeof(int) * nwin, s));
    JG_CUDA(cudaMemsetAsync(win_last, 0xff, sizeof(int) * nwin, s));  // -1: no packable sample
    pack_mark_kernel<<<(int)std::min<int64_t>((batch + 255) / 256, 4 * kNumSMsB200), 256, 0, s>>>(off, batch, win_first,
                                                                                                   win_last);
    JG_LAUNCHED("pack_mark_kernel");
  }
  work_list_kernel<<<1, kScanThreads, 0, s>>>(off, batch, tile, items, count, win_first, win_last, nwin,
                                              2 * (int64_t)device_sm_count());
  JG_LAUNCHED("work_list_kernel");
  return JG_OK;
}

// ------------------------------------------------------------------ conversions
template <typename T>
__global__ void jagged_to_dense_kernel(const int64_t* __restrict__ off, int64_t batch, int64_t dim,
                                       const T* __restrict__ x, int64_t max_len, T pad,
                                       T* __restrict__ out) {
  const int64_t rows = batch * max_len;
  const int lane = threadIdx.x & 31;
  for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; row < rows;
       row += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t i = row / max_len, j = row - i * max_len;
    const int64_t n = off[i + 1] - off[i];
    T* dst = out + row * dim;
    if (j < n) {
      const T* src = x + (off[i] + j) * dim;
      for (int64_t d = lane; d < dim; d += 32) dst[d] = src[d];
    } else {
      for (int64_t d = lane; d < dim; d += 32) dst[d] = pad;
    }
  }
}

template <typename T>
__global__ void dense_to_jagged_kernel(const T* __restrict__ dsrc, int64_t batch, int64_t max_len,
                                       int64_t dim, const int64_t* __restrict__ off,
                                       int64_t total_rows, T* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < total_rows;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t i = sample_of_row(off, batch, r), j = r - off[i];
    const T* src = dsrc + (i * max_len + j) * dim;
    for (int64_t d = lane; d < dim; d += 32) out[r * dim + d] = src[d];
  }
}

// one warp per (sample, padded row); blocks are Bi x Bi at sq[i]
template <typename T>
__global__ void jagged2_to_dense_kernel(const int64_t* __restrict__ off, const int64_t* __restrict__ sq,
                                        int64_t batch, const T* __restrict__ s, int64_t max_len, T pad,
                                        T* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t rows = batch * max_len;
  for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; row < rows;
       row += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t i = row / max_len, r = row - i * max_len;
    const int64_t bi = off[i + 1] - off[i];
    const int64_t n = bi < max_len ? bi : max_len;
    T* dst = out + row * max_len;
    for (int64_t c = lane; c < max_len; c += 32)
      dst[c] = (r < n && c < n) ? s[sq[i] + r * bi + c] : pad;
  }
}

template <typename T>
__global__ void dense_to_jagged2_kernel(const T* __restrict__ dsrc, int64_t batch, int64_t max_len,
                                        const int64_t* __restrict__ off, const int64_t* __restrict__ sq,
                                        T* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t total_rows = off[batch];
  for (int64_t R = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; R < total_rows;
       R += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t i = sample_of_row(off, batch, R), r = R - off[i];
    const int64_t bi = off[i + 1] - off[i];
    const T* src = dsrc + (i * max_len + r) * max_len;
    T* dst = out + sq[i] + r * bi;
    for (int64_t c = lane; c < bi; c += 32) dst[c] = src[c];
  }
}

template <typename T>
__global__ void elementwise_kernel(int op, const T* __restrict__ a, const T* __restrict__ b, int64_t n,
                                   float s, T* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const float x = ld(a + e);
    float r;
    switch (op) {
      case 0: r = x + ld(b + e); break;
      case 1: r = x - ld(b + e); break;
      case 2: r = x * ld(b + e); break;
      default: r = x * s; break;
    }
    st(out + e, r);
  }
}

static int grid_for(int64_t units, int per_block) {
  int64_t g = (units + per_block - 1) / per_block;
  g = std::max<int64_t>(1, std::min<int64_t>(g, 8 * kNumSMsB200));
  return (int)g;
}

template <typename T>
static T pad_as(double p) {
  if constexpr (std::is_same_v<T, float>) return (float)p;
  else return __float2bfloat16_rn((float)p);
}

#define DISPATCH_T(dtype, ...)                                                 \
  do {                                                                         \
    if ((dtype) == JG_F32) { using T = float; __VA_ARGS__; }                   \
    else if ((dtype) == JG_BF16) { using T = __nv_bfloat16; __VA_ARGS__; }     \
    else return fail(JG_UNSUPPORTED, "dtype not supported on device (no CPU fallback)"); \
  } while (0)

jg_status launch_jagged_to_dense(const int64_t* off, int64_t batch, int64_t dim, const void* x,
                                 int64_t max_len, double pad, void* out, jg_dtype dt, cudaStream_t s) {
  if (batch * max_len == 0) return JG_OK;
  DISPATCH_T(dt, jagged_to_dense_kernel<T><<<grid_for(batch * max_len, 8), 256, 0, s>>>(
                     off, batch, dim, (const T*)x, max_len, pad_as<T>(pad), (T*)out));
  JG_LAUNCHED("jagged_to_dense_kernel");
  return JG_OK;
}

jg_status launch_dense_to_jagged(const void* d, int64_t batch, int64_t max_len, int64_t dim,
                                 const int64_t* off, int64_t total_rows, void* out, jg_dtype dt,
                                 cudaStream_t s) {
  if (total_rows == 0) return JG_OK;
  DISPATCH_T(dt, dense_to_jagged_kernel<T><<<grid_for(total_rows, 8), 256, 0, s>>>(
                     (const T*)d, batch, max_len, dim, off, total_rows, (T*)out));
  JG_LAUNCHED("dense_to_jagged_kernel");
  return JG_OK;
}

jg_status launch_jagged2_to_dense(const int64_t* off, const int64_t* sq, int64_t batch, const void* x,
                                  int64_t max_len, double pad, void* out, jg_dtype dt, cudaStream_t s) {
  if (batch * max_len == 0) return JG_OK;
  DISPATCH_T(dt, jagged2_to_dense_kernel<T><<<grid_for(batch * max_len, 8), 256, 0, s>>>(
                     off, sq, batch, (const T*)x, max_len, pad_as<T>(pad), (T*)out));
  JG_LAUNCHED("jagged2_to_dense_kernel");
  return JG_OK;
}

jg_status launch_dense_to_jagged2(const void* d, int64_t batch, int64_t max_len, const int64_t* off,
                                  const int64_t* sq, int64_t total_rows_hint, void* out, jg_dtype dt,
                                  cudaStream_t s) {
  DISPATCH_T(dt, dense_to_jagged2_kernel<T><<<grid_for(std::max<int64_t>(total_rows_hint, 1), 8), 256, 0, s>>>(
                     (const T*)d, batch, max_len, off, sq, (T*)out));
  JG_LAUNCHED("dense_to_jagged2_kernel");
  return JG_OK;
}

jg_status launch_elementwise(int op, const void* a, const void* b, int64_t n, double sc, void* out,
                             jg_dtype dt, cudaStream_t s) {
  if (n == 0) return JG_OK;
  DISPATCH_T(dt, elementwise_kernel<T><<<grid_for(n, 256), 256, 0, s>>>(op, (const T*)a, (const T*)b, n,
                                                                         (float)sc, (T*)out));
  JG_LAUNCHED("elementwise_kernel");
  return JG_OK;
}

}  // namespace jg
