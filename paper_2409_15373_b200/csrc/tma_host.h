// tma_host.h — host-side TMA tensor-map construction (driver entry point fetched through cudart,
// so the library needs no link-time dependency on libcuda).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>
#include <string>

#include "common.cuh"

namespace jg {

inline PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// Encoded maps are cached per host thread by their full key (a tensor map is plain bytes: encoding is pure), so
// repeated calls on the same buffers skip cuTensorMapEncodeTiled (~1 us each; it dominated small launches).
struct MapKey {
  const void* ptr;
  int64_t rows;
  int H, D, box, kind;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && rows == o.rows && H == o.H && D == o.D && box == o.box && kind == o.kind;
  }
};
struct MapCache {
  static constexpr int kSlots = 16;
  MapKey key[kSlots];
  CUtensorMap map[kSlots];
  int used = 0, next = 0;
  bool find(const MapKey& k, CUtensorMap* m) const {
    for (int i = 0; i < used; ++i)
      if (key[i] == k) {
        *m = map[i];
        return true;
      }
    return false;
  }
  void put(const MapKey& k, const CUtensorMap& m) {
    key[next] = k;
    map[next] = m;
    next = (next + 1) % kSlots;
    if (used < kSlots) ++used;
  }
};
inline MapCache& map_cache() {
  static thread_local MapCache c;
  return c;
}

// 3-D map over a [rows, H, D] bf16 tensor: dims (D, H, rows), box (64, 1, box_rows), SWIZZLE_128B.
// Rows past `rows` are zero-filled by the TMA unit; rows of the next sample are masked in-kernel.
inline jg_status make_map(CUtensorMap* m, const void* ptr, int64_t rows, int H, int D, int box_rows) {
  const MapKey key{ptr, rows, H, D, box_rows, 0};
  if (map_cache().find(key, m)) return JG_OK;
  auto enc = tma_encode_fn();
  if (!enc) return fail(JG_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)H, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)H * D * 2};
  cuuint32_t box[3] = {64, 1, (cuuint32_t)box_rows};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(JG_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  map_cache().put(key, *m);
  return JG_OK;
}

// 3-D map over a [rows, H, D] float32 tensor, box (D, 1, box_rows), no swizzle (bulk tensor reductions).
// [rows, H, D] fp32 (the backward's dQ accumulator) or int32, box (D, 1, box_rows)
inline jg_status make_map_f32(CUtensorMap* m, void* ptr, int64_t rows, int H, int D, int box_rows, bool int32 = false) {
  auto enc = tma_encode_fn();
  if (!enc) return fail(JG_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)H, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)D * 4, (cuuint64_t)H * D * 4};
  cuuint32_t box[3] = {(cuuint32_t)D, 1, (cuuint32_t)box_rows};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, int32 ? CU_TENSOR_MAP_DATA_TYPE_INT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ptr, dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(JG_CUDA_ERROR, "cuTensorMapEncodeTiled(f32) failed (" + std::to_string((int)r) + ")");
  return JG_OK;
}

}  // namespace jg

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace jg {
// JG_WAIT_PROF=1: per-role mbarrier wait accounting for the tcgen05 attention kernels (debug only;
// synchronises the stream after the kernel and prints to stderr).
inline unsigned long long* wait_prof_begin(cudaStream_t st) {
  static unsigned long long* buf = nullptr;
  constexpr size_t kWords = 65 + 2 * 5 * 12000;
  const char* e = std::getenv("JG_WAIT_PROF");
  if (!e || (e[0] != '1' && e[0] != '2' && e[0] != '3')) return nullptr;
  if (!buf && cudaMalloc(&buf, kWords * sizeof(unsigned long long)) != cudaSuccess) return nullptr;
  cudaMemsetAsync(buf, 0, kWords * sizeof(unsigned long long), st);
  if (e[0] == '2' || e[0] == '3') {
    static const unsigned long long mode_trace = 1, mode_times = 3;
    cudaMemcpyAsync(buf + 63, e[0] == '2' ? &mode_trace : &mode_times, sizeof(unsigned long long),
                    cudaMemcpyHostToDevice, st);
    static unsigned long long cta = 0;
    if (const char* c = std::getenv("JG_WAIT_PROF_CTA")) cta = std::strtoull(c, nullptr, 10);
    cudaMemcpyAsync(buf + 62, &cta, sizeof(unsigned long long), cudaMemcpyHostToDevice, st);
    cudaStreamSynchronize(st);
  }
  return buf;
}
inline void wait_prof_end(unsigned long long* buf, cudaStream_t st, const char* tag, std::vector<const char*> names) {
  if (!buf) return;
  unsigned long long h[64] = {0};
  cudaStreamSynchronize(st);
  cudaMemcpy(h, buf, sizeof(h), cudaMemcpyDeviceToHost);
  std::fprintf(stderr, "[wait-prof %s]", tag);
  for (size_t r = 0; r + 7 < names.size(); r += 8) {
    const double tot = (double)h[r + 7];
    if (tot <= 0) continue;
    for (size_t i = r; i < r + 7; ++i)
      if (names[i][0]) std::fprintf(stderr, " %s=%.1f%%", names[i], 100.0 * (double)h[i] / tot);
    std::fprintf(stderr, " | %s=%.3g cyc;", names[r + 7], tot);
  }
  std::fprintf(stderr, "\n");
  const char* e = std::getenv("JG_WAIT_PROF");
  if (e && e[0] == '3') {  // per-CTA busy time and the spread of exit times (tail)
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    std::vector<unsigned long long> t(2 * sms);
    cudaMemcpy(t.data(), buf + 65, t.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    unsigned long long s0 = ~0ull, e1 = 0, e0 = ~0ull;
    double busy = 0;
    int n = 0;
    for (int b = 0; b < sms; ++b)
      if (t[2 * b] && t[2 * b + 1]) {
        s0 = std::min(s0, t[2 * b]);
        e1 = std::max(e1, t[2 * b + 1]);
        e0 = std::min(e0, t[2 * b + 1]);
        busy += (double)(t[2 * b + 1] - t[2 * b]);
        ++n;
      }
    if (n)
      std::fprintf(stderr, "[cta-times %s] %d CTAs: makespan %.1f us, mean busy %.1f us, first exit %.1f us\n", tag, n,
                   (e1 - s0) * 1e-3, busy / n * 1e-3, (e0 - s0) * 1e-3);
    if (n && std::getenv("JG_WAIT_PROF_CTAS")) {  // every CTA: start and end relative to the first start
      for (int b = 0; b < sms; ++b)
        if (t[2 * b] && t[2 * b + 1])
          std::fprintf(stderr, "[cta %d] %.2f %.2f\n", b, (t[2 * b] - s0) * 1e-3, (t[2 * b + 1] - s0) * 1e-3);
    }
  }
  if (e && e[0] == '2') {  // dump CTA 0's wait timeline
    const size_t n = 5 * 12000;
    std::vector<unsigned long long> t(2 * n);
    cudaMemcpy(t.data(), buf + 65, t.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    const std::string path = std::string("gpurun_out/trace_") + tag + ".txt";
    if (FILE* f = std::fopen(path.c_str(), "w")) {
      for (size_t i = 0; i < n; ++i)
        if (t[2 * i]) std::fprintf(f, "%llu %llu\n", t[2 * i], t[2 * i + 1]);
      std::fclose(f);
    }
  }
}
}  // namespace jg
