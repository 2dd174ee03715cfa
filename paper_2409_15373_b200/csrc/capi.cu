// capi.cu — the extern "C" boundary (include/jagged_b200.h): argument validation with the
// reference's error texts, per-op GemmDesc construction, stream-ordered scratch, dispatch to the
// SIMT or tcgen05 kernels. No host fallback exists: every op either launches device work or fails.
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace jg {

static thread_local std::string g_last_error;
static thread_local int64_t g_scratch_cur = 0, g_scratch_peak = 0;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }
jg_status fail(jg_status code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
jg_status cuda_status(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? JG_OUT_OF_MEMORY : JG_CUDA_ERROR;
}
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int device_sm_count() {
  static std::mutex mu;
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && cached[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : kNumSMsB200;
    // keep stream-ordered scratch cached in the default pool between calls
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  return dev < 64 ? cached[dev] : kNumSMsB200;
}

jg_status ensure_smem_attr(const void* func, int bytes, const char* name) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;  // (kernel, device) pairs already configured
  int dev = 0;
  JG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  for (const auto& d : done)
    if (d.first == func && d.second == dev) return JG_OK;
  cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return cuda_status(e, name);
  done.emplace_back(func, dev);
  return JG_OK;
}

// RAII stream-ordered scratch
void scratch_note(int64_t bytes) {
  g_scratch_cur += bytes;
  if (g_scratch_cur > g_scratch_peak) g_scratch_peak = g_scratch_cur;
}

struct Scratch {
  void* p = nullptr;
  size_t n = 0;
  cudaStream_t s;
  explicit Scratch(cudaStream_t st) : s(st) {}
  jg_status alloc(size_t bytes) {
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMallocAsync(&p, bytes, s);
    if (e != cudaSuccess) return cuda_status(e, "cudaMallocAsync");
    n = bytes;
    scratch_note((int64_t)n);
    return JG_OK;
  }
  ~Scratch() {
    if (p) {
      cudaFreeAsync(p, s);
      scratch_note(-(int64_t)n);
    }
  }
};

static bool dtype_ok(jg_dtype d) { return d == JG_F32 || d == JG_BF16; }
static size_t dsize(jg_dtype d) { return d == JG_F32 ? 4 : (d == JG_BF16 ? 2 : 8); }

#define REQUIRE(cond, code, msg) \
  do {                           \
    if (!(cond)) return ::jg::fail(code, msg); \
  } while (0)

// device pointers a call dereferences must be non-null whenever there is data (checked before any CUDA call)
#define REQUIRE_PTRS(op, nonempty, ...)                                                                   \
  do {                                                                                                   \
    const void* ptrs_[] = {__VA_ARGS__};                                                                 \
    if (nonempty)                                                                                        \
      for (const void* p_ : ptrs_)                                                                       \
        REQUIRE(p_ != nullptr, JG_INVALID_ARGUMENT, std::string(op) + ": null device pointer");          \
  } while (0)

#define CHECK_DT(op, dt) \
  REQUIRE((dt) != JG_F64, JG_UNSUPPORTED, std::string(op) + ": f64 has no device path (no CPU fallback)"); \
  REQUIRE(dtype_ok(dt), JG_INVALID_ARGUMENT, std::string(op) + ": unknown dtype")

static jg_status gemm(const GemmDesc& g, const int64_t* off, const int64_t* sq, int64_t batch, const void* A,
                      const void* B, void* C, jg_dtype in_dt, jg_dtype out_dt, cudaStream_t st) {
  Scratch prefix(st);
  jg_status rc = prefix.alloc(sizeof(int64_t) * (batch + 1));
  if (rc) return rc;
  return launch_grouped_gemm(g, off, sq, batch, A, B, C, in_dt, out_dt, (int64_t*)prefix.p, st);
}

static GemmDesc desc(Lin M, Lin N, Lin K, Lin a0, Lin sam, Lin sak, Lin b0, Lin sbk, Lin sbn, Lin c0, Lin scm,
                     Lin scn) {
  GemmDesc g;
  g.M = M; g.N = N; g.K = K;
  g.a0 = a0; g.sam = sam; g.sak = sak;
  g.b0 = b0; g.sbk = sbk; g.sbn = sbn;
  g.c0 = c0; g.scm = scm; g.scn = scn;
  return g;
}
static Lin OFF(int64_t k, int64_t c = 0) { Lin l; l.off = k; l.c = c; return l; }
static Lin SQ(int64_t c = 0) { Lin l; l.sq = 1; l.c = c; return l; }
static Lin IDX(int64_t k) { Lin l; l.idx = k; return l; }
static Lin C_(int64_t c) { return L_const(c); }
static Lin BI() { return L_bi(1); }

static jg_status check_out(const char* op, jg_dtype in, jg_dtype out) {
  CHECK_DT(op, in);
  REQUIRE(out == in || (in == JG_BF16 && out == JG_F32), JG_INVALID_ARGUMENT,
          std::string(op) + ": out_dtype must equal in_dtype or be f32 for bf16 inputs");
  return JG_OK;
}

static bool force_simt_gemm() {
  const char* e = std::getenv("JG_GEMM_IMPL");
  return e && std::strcmp(e, "simt") == 0;
}

// tcgen05 path for the bmm family and its VJP contractions (bf16 inputs); op codes as in internal.h
enum TcOp { TC_JJJ = 0, TC_AJ = 1, TC_JJ = 2, TC_JD = 3, TC_JDT = 4, TC_AJT = 5 };
static jg_status tc_gemm(int op, const int64_t* off, const int64_t* sq, int64_t batch, int64_t total_rows, int64_t D,
                         int64_t T, const void* a, const void* b, void* out, jg_dtype out_dt, cudaStream_t st,
                         int64_t sum_sq = -1, const AjBlocks* pre = nullptr) {
  if (batch == 0) return JG_OK;
  Scratch prefix(st);
  if (jg_status rc = prefix.alloc(sizeof(int64_t) * (batch + 1))) return rc;
  return launch_gemm_sm100(op, off, sq, batch, total_rows, D, T, a, b, out, out_dt, (int64_t*)prefix.p, st, nullptr, 0,
                           nullptr, 1, 0, sum_sq, pre);
}
static bool tc_ok(int op, int64_t D, int64_t T, jg_dtype in_dt) {
  return !force_simt_gemm() && gemm_sm100_supported(op, D, T, in_dt);
}

}  // namespace jg

using namespace jg;

// ============================================================================ misc
extern "C" const char* jg_last_error(void) { return g_last_error.c_str(); }

extern "C" void jg_scratch_counters(int64_t* current_bytes, int64_t* peak_bytes) {
  if (current_bytes) *current_bytes = g_scratch_cur;
  if (peak_bytes) *peak_bytes = g_scratch_peak;
}
extern "C" void jg_scratch_reset_peak(void) { g_scratch_peak = g_scratch_cur; }
extern "C" void jg_scratch_raise_peak(int64_t peak_bytes) {
  if (peak_bytes > g_scratch_peak) g_scratch_peak = peak_bytes;
}
extern "C" const char* jg_version(void) { return "jagged_b200 0.1 (sm_100a)"; }
extern "C" int64_t jg_launch_count(void) { return g_launches.load(); }
extern "C" void jg_reset_launch_count(void) { g_launches.store(0); }

// ============================================================================ offsets layer
extern "C" jg_status jg_make_offsets(const int64_t* lengths, int64_t batch, int64_t* offsets,
                                     int64_t* bad_sample, void* stream) {
  REQUIRE(batch >= 0, JG_INVALID_ARGUMENT, "make_jagged: batch must be >= 0");
  return launch_scan(0, lengths, batch, offsets, bad_sample, as_stream(stream));
}

extern "C" jg_status jg_segment_lengths(const int64_t* offsets, int64_t batch, int64_t* lengths, void* stream) {
  REQUIRE(batch >= 0, JG_INVALID_ARGUMENT, "segment_lengths: batch must be >= 0");
  return launch_lengths(offsets, batch, lengths, as_stream(stream));
}

extern "C" jg_status jg_sq_offsets(const int64_t* offsets, int64_t batch, int64_t* sq_offsets, void* stream) {
  REQUIRE(batch >= 0, JG_INVALID_ARGUMENT, "Jagged2Tensor: batch must be >= 0");
  return launch_scan(1, offsets, batch, sq_offsets, nullptr, as_stream(stream));
}

// Three LPT lists over the same offsets: (sample, 128-row tile) items for the key-stationary backward,
// (sample, 256-row tile pair) items for the two-tile forward (padded and cross modes), and the same with the
// short samples packed per 128-row window (first sample, -count) for the jagged self-attention forward.
struct jg_schedule_s {
  const int64_t* offsets;
  int64_t batch, total_rows, max_items, max_items2, max_itemsf, nwin;
  int64_t* lengths;
  int64_t* sq;
  int2* items;
  int64_t* n_items;
  int2* items2;
  int64_t* n_items2;
  int2* itemsf;
  int64_t* n_itemsf;
  int* win;  // [2][nwin]: first and last packable sample per 128-row window
  int64_t bytes;  // device block size (scratch accounting)
  unsigned long long* counters;  // [4]: forward kernel (next item, exited CTAs), backward kernel (same)
  void* block;
};

extern "C" jg_status jg_schedule_create(const int64_t* offsets, int64_t batch, int64_t total_rows, void* stream,
                                        jg_schedule* out) {
  REQUIRE(batch >= 0 && total_rows >= 0 && out, JG_INVALID_ARGUMENT, "schedule: bad arguments");
  cudaStream_t st = as_stream(stream);
  device_sm_count();
  auto* s = new jg_schedule_s();
  s->offsets = offsets;
  s->batch = batch;
  s->total_rows = total_rows;
  s->max_items = total_rows / 128 + batch + 1;
  s->max_items2 = total_rows / 256 + batch + 1;
  s->nwin = total_rows / 128 + 1;
  s->max_itemsf = s->max_items2 + s->nwin;
  const size_t b_len = sizeof(int64_t) * (batch + 1), b_sq = sizeof(int64_t) * (batch + 1),
               b_items = sizeof(int2) * s->max_items, b_items2 = sizeof(int2) * s->max_items2,
               b_itemsf = sizeof(int2) * s->max_itemsf, b_win = sizeof(int) * 2 * s->nwin;
  const size_t bytes = b_len + b_sq + 192 + b_items + b_items2 + b_itemsf + b_win;
  cudaError_t e = cudaMallocAsync(&s->block, bytes, st);
  if (e != cudaSuccess) {
    delete s;
    return cuda_status(e, "schedule alloc");
  }
  s->bytes = (int64_t)bytes;
  scratch_note(s->bytes);
  char* p = (char*)s->block;
  s->lengths = (int64_t*)p; p += b_len;
  s->sq = (int64_t*)p; p += b_sq;
  s->n_items = (int64_t*)p; p += 64;
  s->n_items2 = (int64_t*)p; p += 32;
  s->counters = (unsigned long long*)p; p += 32;
  s->n_itemsf = (int64_t*)p; p += 64;
  s->items = (int2*)p; p += b_items;
  s->items2 = (int2*)p; p += b_items2;
  s->itemsf = (int2*)p; p += b_itemsf;
  s->win = (int*)p;
  jg_status rc = JG_OK;
  JG_CUDA(cudaMemsetAsync(s->counters, 0, 32, st));  // self-resetting afterwards (internal.h)
  if (batch > 0) {
    if ((rc = launch_lengths(offsets, batch, s->lengths, st))) goto err;
    if ((rc = launch_scan(1, offsets, batch, s->sq, nullptr, st))) goto err;
    if ((rc = launch_work_list(offsets, batch, 128, s->items, s->n_items, st))) goto err;
    if ((rc = launch_work_list(offsets, batch, 256, s->items2, s->n_items2, st))) goto err;
    if ((rc = launch_work_list(offsets, batch, 256, s->itemsf, s->n_itemsf, st, s->win, s->win + s->nwin, s->nwin)))
      goto err;
  } else {
    JG_CUDA(cudaMemsetAsync(s->n_items, 0, 64, st));
    JG_CUDA(cudaMemsetAsync(s->n_itemsf, 0, 8, st));
    JG_CUDA(cudaMemsetAsync(s->sq, 0, sizeof(int64_t), st));
  }
  *out = s;
  return JG_OK;
err:
  cudaFreeAsync(s->block, st);
  scratch_note(-s->bytes);
  delete s;
  return rc;
}

extern "C" jg_status jg_schedule_destroy(jg_schedule s) {
  if (!s) return JG_OK;
  cudaError_t e = cudaFree(s->block);
  scratch_note(-s->bytes);
  delete s;
  if (e != cudaSuccess) return cuda_status(e, "schedule free");
  return JG_OK;
}

// A per-call schedule is released stream-ordered (no host synchronisation): its device block is freed after
// the work queued on `st` that reads it.
static void schedule_release(jg_schedule s, cudaStream_t st) {
  if (!s) return;
  cudaFreeAsync(s->block, st);
  scratch_note(-s->bytes);
  delete s;
}

extern "C" const int64_t* jg_schedule_sq_offsets(jg_schedule s) { return s ? s->sq : nullptr; }

extern "C" jg_status jg_schedule_work_list(jg_schedule s, int32_t* host_items, int64_t capacity, int64_t* count) {
  REQUIRE(s && count, JG_INVALID_ARGUMENT, "schedule_work_list: null argument");
  JG_CUDA(cudaDeviceSynchronize());
  int64_t n = 0;
  JG_CUDA(cudaMemcpy(&n, s->n_items, sizeof(int64_t), cudaMemcpyDeviceToHost));
  *count = n;
  if (host_items && capacity > 0) {
    const int64_t m = n < capacity ? n : capacity;
    JG_CUDA(cudaMemcpy(host_items, s->items, sizeof(int2) * m, cudaMemcpyDeviceToHost));
  }
  return JG_OK;
}

// ============================================================================ conversions
extern "C" jg_status jg_jagged_to_dense(const int64_t* offsets, int64_t batch, int64_t dim, const void* x,
                                        int64_t max_len, double pad_value, void* out, jg_dtype dtype, void* stream) {
  CHECK_DT("jagged_to_dense", dtype);
  REQUIRE(max_len >= 0, JG_INVALID_ARGUMENT, "jagged_to_dense: max_len must be >= 0");
  REQUIRE(dim > 0, JG_INVALID_ARGUMENT, "JaggedTensor: dim must be positive");
  return launch_jagged_to_dense(offsets, batch, dim, x, max_len, pad_value, out, dtype, as_stream(stream));
}

extern "C" jg_status jg_dense_to_jagged(const void* d, int64_t batch, int64_t max_len, int64_t dim,
                                        const int64_t* offsets, int64_t total_rows, int64_t max_segment, void* out,
                                        jg_dtype dtype, void* stream) {
  CHECK_DT("dense_to_jagged", dtype);
  REQUIRE(max_segment <= max_len, JG_INVALID_ARGUMENT,
          "dense_to_jagged: a sample length " + std::to_string(max_segment) + " exceeds max_len " +
              std::to_string(max_len));
  return launch_dense_to_jagged(d, batch, max_len, dim, offsets, total_rows, out, dtype, as_stream(stream));
}

extern "C" jg_status jg_jagged2_to_dense(const int64_t* offsets, const int64_t* sq_offsets, int64_t batch,
                                         const void* s, int64_t max_len, double pad_value, void* out, jg_dtype dtype,
                                         void* stream) {
  CHECK_DT("jagged2_to_dense", dtype);
  REQUIRE(max_len >= 0, JG_INVALID_ARGUMENT, "jagged2_to_dense: max_len must be >= 0");
  return launch_jagged2_to_dense(offsets, sq_offsets, batch, s, max_len, pad_value, out, dtype, as_stream(stream));
}

extern "C" jg_status jg_dense_to_jagged2(const void* d, int64_t batch, int64_t max_len, const int64_t* offsets,
                                         const int64_t* sq_offsets, int64_t max_segment, void* out, jg_dtype dtype,
                                         void* stream) {
  CHECK_DT("dense_to_jagged2", dtype);
  REQUIRE(max_segment <= max_len, JG_INVALID_ARGUMENT,
          "dense_to_jagged2: a sample length " + std::to_string(max_segment) + " exceeds max_len " +
              std::to_string(max_len));
  return launch_dense_to_jagged2(d, batch, max_len, offsets, sq_offsets, batch * max_len, out, dtype,
                                 as_stream(stream));
}

extern "C" jg_status jg_elementwise(int32_t op, const void* a, const void* b, int64_t n, void* out, jg_dtype dtype,
                                    void* stream) {
  CHECK_DT("elementwise", dtype);
  REQUIRE(op >= 0 && op <= 2, JG_INVALID_ARGUMENT, "elementwise: op must be 0 (add), 1 (sub) or 2 (mul)");
  return launch_elementwise(op, a, b, n, 0.0, out, dtype, as_stream(stream));
}

extern "C" jg_status jg_scale(const void* a, int64_t n, double s, void* out, jg_dtype dtype, void* stream) {
  CHECK_DT("scale", dtype);
  return launch_elementwise(3, a, nullptr, n, s, out, dtype, as_stream(stream));
}

// ============================================================================ Table-1 operators
extern "C" jg_status jg_jagged_dense_bmm(const int64_t* off, int64_t batch, int64_t total_rows, int64_t D, int64_t T,
                                         const void* x, const void* w, void* out, jg_dtype in_dt, jg_dtype out_dt,
                                         void* stream) {
  if (jg_status rc = check_out("jagged_dense_bmm", in_dt, out_dt)) return rc;
  REQUIRE(D > 0 && T > 0, JG_INVALID_ARGUMENT, "jagged_dense_bmm: w must be [B, D, T]");
  (void)total_rows;
  if (!force_simt_gemm() && gemm_sm100_supported(3, D, T, in_dt))
    return tc_gemm(3, off, nullptr, batch, total_rows, D, T, x, w, out, out_dt, as_stream(stream));
  GemmDesc g = desc(BI(), C_(T), C_(D), OFF(D), C_(D), C_(1), IDX(D * T), C_(T), C_(1), OFF(T), C_(T), C_(1));
  return gemm(g, off, nullptr, batch, x, w, out, in_dt, out_dt, as_stream(stream));
}

extern "C" jg_status jg_jagged_jagged_bmm(const int64_t* off, int64_t batch, int64_t total_rows, int64_t D, int64_t T,
                                          const void* x, const void* y, void* out, jg_dtype in_dt, jg_dtype out_dt,
                                          void* stream) {
  if (jg_status rc = check_out("jagged_jagged_bmm", in_dt, out_dt)) return rc;
  REQUIRE(D > 0 && T > 0, JG_INVALID_ARGUMENT, "jagged_jagged_bmm: dims must be positive");
  (void)total_rows;
  if (!force_simt_gemm() && gemm_sm100_supported(2, D, T, in_dt))
    return tc_gemm(2, off, nullptr, batch, total_rows, D, T, x, y, out, out_dt, as_stream(stream));
  GemmDesc g = desc(C_(D), C_(T), BI(), OFF(D), C_(1), C_(D), OFF(T), C_(T), C_(1), IDX(D * T), C_(T), C_(1));
  return gemm(g, off, nullptr, batch, x, y, out, in_dt, out_dt, as_stream(stream));
}

extern "C" jg_status jg_jagged_softmax(const int64_t* off, int64_t batch, int64_t total_rows, int64_t D,
                                       const void* x, void* out, jg_dtype dtype, void* stream) {
  CHECK_DT("jagged_softmax", dtype);
  (void)total_rows;
  return launch_jagged_softmax(off, batch, D, x, nullptr, out, dtype, false, as_stream(stream));
}

extern "C" jg_status jg_jagged_jagged_bmm_jagged_out(const int64_t* off, const int64_t* sq, int64_t batch,
                                                     int64_t total_rows, int64_t D, const void* q, const void* k,
                                                     void* out, jg_dtype in_dt, jg_dtype out_dt, void* stream) {
  if (jg_status rc = check_out("jagged_jagged_bmm_jagged_out", in_dt, out_dt)) return rc;
  REQUIRE(sq, JG_INVALID_ARGUMENT, "jagged_jagged_bmm_jagged_out: sq_offsets required");
  (void)total_rows;
  if (!force_simt_gemm() && gemm_sm100_supported(0, D, D, in_dt))
    return tc_gemm(0, off, sq, batch, total_rows, D, D, q, k, out, out_dt, as_stream(stream));
  GemmDesc g = desc(BI(), BI(), C_(D), OFF(D), C_(D), C_(1), OFF(D), C_(1), C_(D), SQ(), BI(), C_(1));
  return gemm(g, off, sq, batch, q, k, out, in_dt, out_dt, as_stream(stream));
}

extern "C" jg_status jg_array_jagged_bmm_jagged_out(const int64_t* off, const int64_t* sq, int64_t batch,
                                                    int64_t total_rows, int64_t sum_sq, int64_t D, const void* a,
                                                    const void* v, void* out, jg_dtype in_dt, jg_dtype out_dt,
                                                    void* stream) {
  if (jg_status rc = check_out("array_jagged_bmm_jagged_out", in_dt, out_dt)) return rc;
  REQUIRE(sq, JG_INVALID_ARGUMENT, "array_jagged_bmm_jagged_out: sq_offsets required");
  if (tc_ok(TC_AJ, D, D, in_dt))
    return tc_gemm(TC_AJ, off, sq, batch, total_rows, D, D, a, v, out, out_dt, as_stream(stream), sum_sq);
  GemmDesc g = desc(BI(), C_(D), BI(), SQ(), BI(), C_(1), OFF(D), C_(D), C_(1), OFF(D), C_(D), C_(1));
  return gemm(g, off, sq, batch, a, v, out, in_dt, out_dt, as_stream(stream));
}

extern "C" jg_status jg_jagged2_softmax(const int64_t* off, const int64_t* sq, int64_t batch, const void* s, void* out,
                                        jg_dtype dtype, void* stream) {
  CHECK_DT("jagged2_softmax", dtype);
  REQUIRE(sq, JG_INVALID_ARGUMENT, "jagged2_softmax: sq_offsets required");
  const int64_t total_rows = -1;  // read from offsets[batch] on device
  return launch_jagged2_softmax(off, sq, batch, total_rows, s, nullptr, out, dtype, false, as_stream(stream));
}

// ---------------------------------------------------------------------------- VJPs
// Every contraction of the six VJPs runs on the tcgen05 grouped GEMM for bf16 (the transposed forms JDT / AJT,
// or a forward form); fp32 (and shapes the tensor-core path does not cover) on the SIMT grouped GEMM.
extern "C" jg_status jg_jagged_dense_bmm_vjp(const int64_t* off, int64_t batch, int64_t total_rows, int64_t D,
                                             int64_t T, const void* x, const void* w, const void* go, void* dx,
                                             void* dw, jg_dtype in_dt, jg_dtype out_dt, void* stream) {
  if (jg_status rc = check_out("jagged_dense_bmm_vjp", in_dt, out_dt)) return rc;
  cudaStream_t st = as_stream(stream);
  // dX = dO W^T (linalg.cpp:296-305): [rows, T] x W_i^T -> [rows, D]
  if (tc_ok(TC_JDT, D, T, in_dt)) {
    if (jg_status rc = tc_gemm(TC_JDT, off, nullptr, batch, total_rows, D, T, go, w, dx, out_dt, st)) return rc;
  } else {
    GemmDesc gx = desc(BI(), C_(D), C_(T), OFF(T), C_(T), C_(1), IDX(D * T), C_(1), C_(T), OFF(D), C_(D), C_(1));
    if (jg_status rc = gemm(gx, off, nullptr, batch, go, w, dx, in_dt, out_dt, st)) return rc;
  }
  // dW = X^T dO (linalg.cpp:307-314): a jagged_jagged_bmm
  if (tc_ok(TC_JJ, D, T, in_dt)) return tc_gemm(TC_JJ, off, nullptr, batch, total_rows, D, T, x, go, dw, out_dt, st);
  GemmDesc gw = desc(C_(D), C_(T), BI(), OFF(D), C_(1), C_(D), OFF(T), C_(T), C_(1), IDX(D * T), C_(T), C_(1));
  return gemm(gw, off, nullptr, batch, x, go, dw, in_dt, out_dt, st);
}

extern "C" jg_status jg_jagged_jagged_bmm_vjp(const int64_t* off, int64_t batch, int64_t total_rows, int64_t D,
                                              int64_t T, const void* x, const void* y, const void* go, void* dx,
                                              void* dy, jg_dtype in_dt, jg_dtype out_dt, void* stream) {
  if (jg_status rc = check_out("jagged_jagged_bmm_vjp", in_dt, out_dt)) return rc;
  cudaStream_t st = as_stream(stream);
  // dX = Y dZ^T (linalg.cpp:334-341): [rows, T] x dZ_i^T -> [rows, D]
  if (tc_ok(TC_JDT, D, T, in_dt)) {
    if (jg_status rc = tc_gemm(TC_JDT, off, nullptr, batch, total_rows, D, T, y, go, dx, out_dt, st)) return rc;
  } else {
    GemmDesc gx = desc(BI(), C_(D), C_(T), OFF(T), C_(T), C_(1), IDX(D * T), C_(1), C_(T), OFF(D), C_(D), C_(1));
    if (jg_status rc = gemm(gx, off, nullptr, batch, y, go, dx, in_dt, out_dt, st)) return rc;
  }
  // dY = X dZ (linalg.cpp:342-349): a jagged_dense_bmm
  if (tc_ok(TC_JD, D, T, in_dt)) return tc_gemm(TC_JD, off, nullptr, batch, total_rows, D, T, x, go, dy, out_dt, st);
  GemmDesc gy = desc(BI(), C_(T), C_(D), OFF(D), C_(D), C_(1), IDX(D * T), C_(T), C_(1), OFF(T), C_(T), C_(1));
  return gemm(gy, off, nullptr, batch, x, go, dy, in_dt, out_dt, st);
}

extern "C" jg_status jg_jagged_softmax_vjp(const int64_t* off, int64_t batch, int64_t total_rows, int64_t D,
                                           const void* x, const void* go, void* dx, jg_dtype dtype, void* stream) {
  CHECK_DT("jagged_softmax_vjp", dtype);
  (void)total_rows;
  return launch_jagged_softmax(off, batch, D, x, go, dx, dtype, true, as_stream(stream));
}

extern "C" jg_status jg_jagged_jagged_bmm_jagged_out_vjp(const int64_t* off, const int64_t* sq, int64_t batch,
                                                         int64_t total_rows, int64_t sum_sq, int64_t D, const void* q,
                                                         const void* k, const void* go, void* dq, void* dk,
                                                         jg_dtype in_dt, jg_dtype out_dt, void* stream) {
  if (jg_status rc = check_out("jagged_jagged_bmm_jagged_out_vjp", in_dt, out_dt)) return rc;
  REQUIRE(sq, JG_INVALID_ARGUMENT, "jagged_jagged_bmm_jagged_out_vjp: sq_offsets required");
  cudaStream_t st = as_stream(stream);
  if (tc_ok(TC_AJ, D, D, in_dt) && tc_ok(TC_AJT, D, D, in_dt)) {
    // dQ = dS K (linalg.cpp:405-412): array_jagged_bmm_jagged_out; dK = dS^T Q (:413-420): the transposed form.
    // Both read dS through the same repacked 64 x 64 sub-block images: one repack pass for the two contractions.
    AjBlocks ds;
    if (jg_status rc = aj_repack(off, sq, batch, total_rows, sum_sq, go, &ds, st)) return rc;
    jg_status rc = tc_gemm(TC_AJ, off, sq, batch, total_rows, D, D, go, k, dq, out_dt, st, sum_sq, &ds);
    if (!rc) rc = tc_gemm(TC_AJT, off, sq, batch, total_rows, D, D, go, q, dk, out_dt, st, sum_sq, &ds);
    aj_release(&ds, st);
    return rc;
  }
  GemmDesc gq = desc(BI(), C_(D), BI(), SQ(), BI(), C_(1), OFF(D), C_(D), C_(1), OFF(D), C_(D), C_(1));
  if (jg_status rc = gemm(gq, off, sq, batch, go, k, dq, in_dt, out_dt, st)) return rc;
  GemmDesc gk = desc(BI(), C_(D), BI(), SQ(), C_(1), BI(), OFF(D), C_(D), C_(1), OFF(D), C_(D), C_(1));
  return gemm(gk, off, sq, batch, go, q, dk, in_dt, out_dt, st);
}

extern "C" jg_status jg_array_jagged_bmm_jagged_out_vjp(const int64_t* off, const int64_t* sq, int64_t batch,
                                                        int64_t total_rows, int64_t sum_sq, int64_t D, const void* a,
                                                        const void* v, const void* go, void* da, void* dv,
                                                        jg_dtype in_dt, jg_dtype out_dt, void* stream) {
  if (jg_status rc = check_out("array_jagged_bmm_jagged_out_vjp", in_dt, out_dt)) return rc;
  REQUIRE(sq, JG_INVALID_ARGUMENT, "array_jagged_bmm_jagged_out_vjp: sq_offsets required");
  cudaStream_t st = as_stream(stream);
  if (tc_ok(TC_JJJ, D, D, in_dt) && tc_ok(TC_AJT, D, D, in_dt)) {
    // dA = dO V^T (linalg.cpp:447-455): jagged_jagged_bmm_jagged_out; dV = A^T dO (:456-466): the transposed form
    if (jg_status rc = tc_gemm(TC_JJJ, off, sq, batch, total_rows, D, D, go, v, da, out_dt, st)) return rc;
    return tc_gemm(TC_AJT, off, sq, batch, total_rows, D, D, a, go, dv, out_dt, st, sum_sq);
  }
  GemmDesc ga = desc(BI(), BI(), C_(D), OFF(D), C_(D), C_(1), OFF(D), C_(1), C_(D), SQ(), BI(), C_(1));
  if (jg_status rc = gemm(ga, off, sq, batch, go, v, da, in_dt, out_dt, st)) return rc;
  GemmDesc gv = desc(BI(), C_(D), BI(), SQ(), C_(1), BI(), OFF(D), C_(D), C_(1), OFF(D), C_(D), C_(1));
  return gemm(gv, off, sq, batch, a, go, dv, in_dt, out_dt, st);
}

extern "C" jg_status jg_jagged2_softmax_vjp(const int64_t* off, const int64_t* sq, int64_t batch, const void* s,
                                            const void* go, void* ds, jg_dtype dtype, void* stream) {
  CHECK_DT("jagged2_softmax_vjp", dtype);
  const int64_t total_rows = -1;  // read from offsets[batch] on device
  return launch_jagged2_softmax(off, sq, batch, total_rows, s, go, ds, dtype, true, as_stream(stream));
}

// ============================================================================ attention
static bool force_simt() {
  const char* e = std::getenv("JG_ATTN_IMPL");
  return e && std::strcmp(e, "simt") == 0;
}

static int64_t round256(int64_t x) { return (x + 255) / 256 * 256; }
extern "C" int64_t jg_attention_backward_workspace_size(int64_t total_rows, int64_t batch, int32_t num_heads,
                                                        int32_t head_dim) {
  const int64_t delta = attn_lsd_bytes(total_rows, num_heads);  // >= the SIMT path's [H, total_rows] Delta
  (void)batch;  // (kept in the signature: layouts sized per sample stay possible without an ABI change)
  return delta + round256(total_rows * num_heads * (int64_t)head_dim * 4) + 256;  // fp32 / int32 accumulator
}

// Shared by the jagged entry points (valid == nullptr) and the padded dense_flash_attention mode (valid =
// per-sample lengths on device, offsets i*max_len): same kernels, masks from `valid`.
// A caller-supplied schedule must be the one built for these offsets: the kernels index offsets[] with its
// sample ids, so a schedule of another batch would read out of bounds and write rows of other samples.
static jg_status check_schedule(const char* op, jg_schedule s, const int64_t* off, int64_t batch, int64_t total_rows) {
  if (!s) return JG_OK;
  REQUIRE(s->offsets == off && s->batch == batch && s->total_rows == total_rows, JG_INVALID_ARGUMENT,
          std::string(op) + ": schedule was built for other offsets (batch " + std::to_string(s->batch) + ", rows " +
              std::to_string(s->total_rows) + " vs " + std::to_string(batch) + ", " + std::to_string(total_rows) + ")");
  return JG_OK;
}

// The tensor-core and tiled kernels move 16-byte vectors (TMA boxes, float4 / uint2 loads): tensors whose base is
// not 16-byte aligned (views into a larger buffer) take the row-per-warp kernels, which load scalars.
static bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

static jg_status attn_forward(const int64_t* off, int64_t batch, int64_t total_rows, int32_t H, int32_t D,
                              const void* q, const void* k, const void* v, void* out, float* lse, jg_dtype dtype,
                              jg_schedule sched, const int64_t* valid, cudaStream_t st) {
  if (total_rows == 0) return JG_OK;
  if (jg_status rc = check_schedule("jagged_flash_attention_forward", sched, off, batch, total_rows)) return rc;
  if (!(al16(q) && al16(k) && al16(v) && al16(out)))
    return launch_attn_fwd_simt(off, batch, total_rows, H, D, q, k, v, out, lse, dtype, nullptr, nullptr, 0, valid, st);
  if (!force_simt() && attn_sm100_supported(D, dtype)) {
    jg_schedule own = nullptr;
    if (!sched) {
      if (jg_status rc = jg_schedule_create(off, batch, total_rows, st, &own)) return rc;
      sched = own;
    }
    // jagged mode: the packed list (short samples share a query tile); padded mode: one item per segment
    static const bool no_pack = std::getenv("JG_FWD_NOPACK") != nullptr;  // A/B knob (diagnostic)
    jg_status rc = (valid || no_pack) ? launch_attn_fwd_sm100(off, batch, total_rows, H, D, q, k, v, out, lse, sched->items2,
                                                 sched->n_items2, sched->max_items2, valid, sched->counters, st)
                         : launch_attn_fwd_sm100(off, batch, total_rows, H, D, q, k, v, out, lse, sched->itemsf,
                                                 sched->n_itemsf, sched->max_itemsf, nullptr, sched->counters, st);
    if (own) {
      schedule_release(own, st);
    }
    return rc;
  }
  // fp32 (or forced SIMT): tiled FFMA kernel over the (sample, 128-row tile) list
  jg_schedule own = nullptr;
  if (!sched) {
    if (jg_status rc = jg_schedule_create(off, batch, total_rows, st, &own)) return rc;
    sched = own;
  }
  jg_status rc = (!force_simt() && attn_x3_supported(D, dtype))
                     ? launch_attn_fwd_x3(off, total_rows, H, D, q, k, v, out, lse, sched->items, sched->n_items,
                                          sched->max_items, valid, st)
                     : launch_attn_fwd_simt(off, batch, total_rows, H, D, q, k, v, out, lse, dtype, sched->items,
                                            sched->n_items, sched->max_items, valid, st);
  if (own) schedule_release(own, st);
  return rc;
}

static jg_status attn_backward(const int64_t* off, int64_t batch, int64_t total_rows, int32_t H, int32_t D,
                               const void* q, const void* k, const void* v, const void* go, const void* o,
                               const float* lse, void* dq, void* dk, void* dv, jg_dtype dtype, bool deterministic,
                               jg_schedule sched, void* workspace, const int64_t* valid, cudaStream_t st) {
  if (total_rows == 0) return JG_OK;
  if (jg_status rc = check_schedule("jagged_flash_attention_backward", sched, off, batch, total_rows)) return rc;
  Scratch ws(st);
  if (!workspace) {
    if (jg_status rc = ws.alloc(jg_attention_backward_workspace_size(total_rows, batch, H, D))) return rc;
    workspace = ws.p;
  }
  float* delta = (float*)workspace;
  void* dq_acc = (char*)workspace + attn_lsd_bytes(total_rows, H);
  if (!(al16(q) && al16(k) && al16(v) && al16(go) && al16(o) && al16(dq) && al16(dk) && al16(dv)))
    return launch_attn_bwd_simt(off, batch, total_rows, H, D, q, k, v, go, o, lse, dq, dk, dv, delta, dtype, nullptr,
                                nullptr, 0, valid, false, st);

  if (!force_simt() && attn_sm100_bwd_supported(D, dtype)) {
    jg_schedule own = nullptr;
    if (!sched) {
      if (jg_status rc = jg_schedule_create(off, batch, total_rows, st, &own)) return rc;
      sched = own;
    }
    jg_status rc = launch_attn_bwd_sm100(off, batch, total_rows, H, D, q, k, v, go, o, lse, dq, dk, dv, delta,
                                         dq_acc, deterministic, sched->items, sched->n_items, sched->max_items, valid,
                                         sched->counters + 2, st);
    if (own) {
      schedule_release(own, st);
    }
    return rc;
  }
  jg_schedule own = nullptr;  // fp32 (or forced SIMT): tiled FFMA kernels over the (sample, 128-row tile) list
  if (!sched) {
    if (jg_status rc = jg_schedule_create(off, batch, total_rows, st, &own)) return rc;
    sched = own;
  }
  jg_status rc = launch_attn_bwd_simt(off, batch, total_rows, H, D, q, k, v, go, o, lse, dq, dk, dv, delta, dtype,
                                      sched->items, sched->n_items, sched->max_items, valid,
                                      !force_simt() && attn_x3_supported(D, dtype), st);
  if (own) schedule_release(own, st);
  return rc;
}

extern "C" jg_status jg_jagged_flash_attention_forward(const int64_t* off, int64_t batch, int64_t total_rows,
                                                       int32_t H, int32_t D, const void* q, const void* k,
                                                       const void* v, int64_t block_q, int64_t block_k, void* out,
                                                       float* lse, jg_dtype dtype, jg_schedule sched, void* stream) {
  CHECK_DT("jagged_flash_attention_forward", dtype);
  REQUIRE(block_q >= 1 && block_k >= 1, JG_INVALID_ARGUMENT,
          "jagged_flash_attention_forward: block sizes must be >= 1");
  REQUIRE(H >= 1 && D >= 1, JG_INVALID_ARGUMENT, "jagged_flash_attention_forward: dim mismatch");
  REQUIRE_PTRS("jagged_flash_attention_forward", total_rows > 0, off, q, k, v, out, lse);
  return attn_forward(off, batch, total_rows, H, D, q, k, v, out, lse, dtype, sched, nullptr, as_stream(stream));
}

extern "C" jg_status jg_jagged_flash_attention_backward(const int64_t* off, int64_t batch, int64_t total_rows,
                                                        int32_t H, int32_t D, const void* q, const void* k,
                                                        const void* v, const void* go, const void* o,
                                                        const float* lse, int64_t block_q, int64_t block_k, void* dq,
                                                        void* dk, void* dv, jg_dtype dtype, int32_t deterministic,
                                                        jg_schedule sched, void* workspace, void* stream) {
  CHECK_DT("jagged_flash_attention_backward", dtype);
  REQUIRE(block_q >= 1 && block_k >= 1, JG_INVALID_ARGUMENT,
          "jagged_flash_attention_backward: saved state does not match inputs");
  REQUIRE(H >= 1 && D >= 1, JG_INVALID_ARGUMENT, "jagged_flash_attention_backward: grad_out layout mismatch");
  REQUIRE_PTRS("jagged_flash_attention_backward", total_rows > 0, off, q, k, v, go, o, lse, dq, dk, dv);
  return attn_backward(off, batch, total_rows, H, D, q, k, v, go, o, lse, dq, dk, dv, dtype, deterministic != 0, sched,
                       workspace,
                       nullptr, as_stream(stream));
}

// Padded mode: validate lengths like attention.cpp:19-31 (require_self_attention_inputs), then upload
// offsets i*max_len and the lengths into one stream-ordered scratch block.
static jg_status padded_layout(const char* op, const int64_t* lengths, int64_t batch, int64_t max_len,
                               Scratch& buf, const int64_t** d_off, const int64_t** d_valid) {
  REQUIRE(batch >= 0 && max_len >= 0, JG_INVALID_ARGUMENT, std::string(op) + ": q, k, v must share a [B, L, D] shape");
  REQUIRE(batch == 0 || lengths, JG_INVALID_ARGUMENT, std::string(op) + ": lengths size mismatch");
  for (int64_t i = 0; i < batch; ++i)
    REQUIRE(lengths[i] >= 0 && lengths[i] <= max_len, JG_INVALID_ARGUMENT,
            std::string(op) + ": sample " + std::to_string(i) + " length " + std::to_string(lengths[i]) +
                " out of bounds for L=" + std::to_string(max_len));
  // the staging vector lives until the stream has consumed it (released by a host callback, no host sync)
  auto* h = new std::vector<int64_t>(2 * batch + 1);
  for (int64_t i = 0; i < batch; ++i) {
    (*h)[i] = i * max_len;
    (*h)[batch + 1 + i] = lengths[i];
  }
  (*h)[batch] = batch * max_len;
  if (jg_status rc = buf.alloc(sizeof(int64_t) * h->size())) {
    delete h;
    return rc;
  }
  cudaError_t e = cudaMemcpyAsync(buf.p, h->data(), sizeof(int64_t) * h->size(), cudaMemcpyHostToDevice, buf.s);
  if (e == cudaSuccess)
    e = cudaLaunchHostFunc(buf.s, [](void* v) { delete static_cast<std::vector<int64_t>*>(v); }, h);
  if (e != cudaSuccess) {
    cudaStreamSynchronize(buf.s);
    delete h;
    return cuda_status(e, "padded layout upload");
  }
  *d_off = (const int64_t*)buf.p;
  *d_valid = (const int64_t*)buf.p + batch + 1;
  return JG_OK;
}

extern "C" jg_status jg_dense_flash_attention_forward(const int64_t* lengths, int64_t batch, int64_t max_len,
                                                      int32_t H, int32_t D, const void* q, const void* k,
                                                      const void* v, int64_t block_q, int64_t block_k, void* out,
                                                      float* lse, jg_dtype dtype, void* stream) {
  CHECK_DT("dense_flash_attention", dtype);
  REQUIRE(block_q >= 1 && block_k >= 1, JG_INVALID_ARGUMENT, "dense_flash_attention: block sizes must be >= 1");
  REQUIRE(H >= 1 && D >= 1, JG_INVALID_ARGUMENT, "dense_flash_attention: q, k, v must share a [B, L, D] shape");
  REQUIRE_PTRS("dense_flash_attention", batch * max_len > 0, q, k, v, out, lse);
  cudaStream_t st = as_stream(stream);
  Scratch buf(st);
  const int64_t *d_off = nullptr, *d_valid = nullptr;
  if (jg_status rc = padded_layout("dense_flash_attention", lengths, batch, max_len, buf, &d_off, &d_valid)) return rc;
  return attn_forward(d_off, batch, batch * max_len, H, D, q, k, v, out, lse, dtype, nullptr, d_valid, st);
}

extern "C" jg_status jg_dense_flash_attention_backward(const int64_t* lengths, int64_t batch, int64_t max_len,
                                                       int32_t H, int32_t D, const void* q, const void* k,
                                                       const void* v, const void* go, const void* o,
                                                       const float* lse, int64_t block_q, int64_t block_k, void* dq,
                                                       void* dk, void* dv, jg_dtype dtype, void* workspace,
                                                       void* stream) {
  CHECK_DT("dense_flash_attention_backward", dtype);
  REQUIRE(block_q >= 1 && block_k >= 1, JG_INVALID_ARGUMENT,
          "dense_flash_attention_backward: block sizes must be >= 1");
  REQUIRE(H >= 1 && D >= 1, JG_INVALID_ARGUMENT, "dense_flash_attention_backward: q, k, v must share a [B, L, D] shape");
  REQUIRE_PTRS("dense_flash_attention_backward", batch * max_len > 0, q, k, v, go, o, lse, dq, dk, dv);
  cudaStream_t st = as_stream(stream);
  Scratch buf(st);
  const int64_t *d_off = nullptr, *d_valid = nullptr;
  if (jg_status rc = padded_layout("dense_flash_attention_backward", lengths, batch, max_len, buf, &d_off, &d_valid))
    return rc;
  return attn_backward(d_off, batch, batch * max_len, H, D, q, k, v, go, o, lse, dq, dk, dv, dtype, true, nullptr,
                       workspace, d_valid, st);
}

extern "C" jg_status jg_jagged_attention(const int64_t* off, const int64_t* sq, int64_t batch, int64_t total_rows,
                                         int64_t sum_sq, int32_t H, int32_t D, const void* q, const void* k,
                                         const void* v, void* out, jg_dtype dtype, void* scores_ws, void* stream) {
  CHECK_DT("jagged_attention", dtype);
  REQUIRE(sq, JG_INVALID_ARGUMENT, "jagged_attention: sq_offsets required");
  REQUIRE_PTRS("jagged_attention", total_rows > 0, off, q, k, v, out);
  cudaStream_t st = as_stream(stream);
  if (total_rows == 0) return JG_OK;
  const size_t es = dsize(dtype);
  const size_t s_bytes = ((es * (size_t)sum_sq * H + 255) / 256) * 256;  // P starts 256-byte aligned
  Scratch ws(st);
  if (!scores_ws) {
    if (jg_status rc = ws.alloc(2 * s_bytes)) return rc;
    scores_ws = ws.p;
  }
  char* S = (char*)scores_ws;
  char* P = S + s_bytes;
  const int64_t RS = (int64_t)H * D;
  // bf16: the two contractions run on the tcgen05 grouped GEMM, one head of the [rows, H, D] tensors at a time
  // (TMA head coordinate); otherwise the SIMT grouped GEMM with strided descriptors
  const bool tc = !force_simt_gemm() && gemm_sm100_supported(0, D, D, dtype) && gemm_sm100_supported(1, D, D, dtype);
  Scratch prefix(st);
  if (tc)
    if (jg_status rc = prefix.alloc(sizeof(int64_t) * (batch + 1))) return rc;
  for (int h = 0; h < H; ++h) {
    const int64_t ho = (int64_t)h * D;
    char* Sh = S + es * (size_t)sum_sq * h;
    // jagged_jagged_bmm_jagged_out (attention.cpp:167) on head h
    if (tc) {
      if (jg_status rc = launch_gemm_sm100(0, off, sq, batch, total_rows, D, D, q, k, Sh, dtype, (int64_t*)prefix.p, st,
                                           nullptr, 0, nullptr, H, h))
        return rc;
      continue;
    }
    GemmDesc gs = desc(BI(), BI(), C_(D), OFF(RS, ho), C_(RS), C_(1), OFF(RS, ho), C_(1), C_(RS), SQ(), BI(), C_(1));
    if (jg_status rc = gemm(gs, off, sq, batch, q, k, Sh, dtype, dtype, st)) return rc;
  }
  // scale by 1/sqrt(D), rounded to the element type (attention.cpp:166-167)
  const double inv = dtype == JG_F32 ? (double)(float)(1.0 / std::sqrt((double)D)) : 1.0 / std::sqrt((double)D);
  if (jg_status rc = launch_elementwise(3, S, nullptr, sum_sq * H, inv, S, dtype, st)) return rc;
  for (int h = 0; h < H; ++h) {
    const int64_t ho = (int64_t)h * D;
    char* Sh = S + es * (size_t)sum_sq * h;
    char* Ph = P + es * (size_t)sum_sq * h;
    if (jg_status rc = launch_jagged2_softmax(off, sq, batch, total_rows, Sh, nullptr, Ph, dtype, false, st)) return rc;
    if (tc) {  // array_jagged_bmm_jagged_out (attention.cpp:169) on head h, into out[:, h, :]
      if (jg_status rc = launch_gemm_sm100(1, off, sq, batch, total_rows, D, D, Ph, v, (char*)out + es * ho, dtype,
                                           (int64_t*)prefix.p, st, nullptr, 0, nullptr, H, h, sum_sq))
        return rc;
      continue;
    }
    GemmDesc go = desc(BI(), C_(D), BI(), SQ(), BI(), C_(1), OFF(RS, ho), C_(RS), C_(1), OFF(RS, ho), C_(RS), C_(1));
    if (jg_status rc = gemm(go, off, sq, batch, Ph, v, out, dtype, dtype, st)) return rc;
  }
  return JG_OK;
}

extern "C" jg_status jg_jagged_flash_attention_fwd_bwd_host(const int64_t* host_offsets, int64_t batch, int32_t H,
                                                            int32_t D, const void* q, const void* k, const void* v,
                                                            const void* go, void* out, float* lse, void* dq, void* dk,
                                                            void* dv, jg_dtype dtype, void* stream) {
  CHECK_DT("jagged_flash_attention", dtype);
  REQUIRE(host_offsets && batch >= 0, JG_INVALID_ARGUMENT, "jagged_flash_attention: offsets required");
  REQUIRE(host_offsets[0] == 0, JG_INVALID_ARGUMENT, "JaggedTensor: offsets must start with 0");
  for (int64_t i = 1; i <= batch; ++i)
    REQUIRE(host_offsets[i] >= host_offsets[i - 1], JG_INVALID_ARGUMENT,
            "JaggedTensor: offsets must be non-decreasing at index " + std::to_string(i));
  cudaStream_t user = as_stream(stream);
  const int64_t S = host_offsets[batch];
  if (S == 0) return JG_OK;
  // Samples are independent, so the batch is cut into contiguous sample chunks of ~equal rows and run as a
  // kSlots-stream pipeline: later chunks' host->device copies and earlier chunks' device->host copies
  // (separate copy engines) overlap a chunk's forward + backward. Host buffers should be pinned.
  constexpr int kSlots = 3;
#ifndef JG_HOST_CHUNKS
#define JG_HOST_CHUNKS 32  // e2e on cfg3: 16 chunks 48.9 ms, 32 chunks 46.4-47.8 ms, 48 chunks 47.8 ms
#endif
  const int64_t n_chunks = std::max<int64_t>(1, std::min<int64_t>(JG_HOST_CHUNKS, batch));
  std::vector<int64_t> cut{0};
  for (int64_t c = 1; c < n_chunks; ++c) {
    const int64_t target = S * c / n_chunks;
    int64_t b = cut.back();
    while (b < batch && host_offsets[b] < target) ++b;
    if (b > cut.back() && b < batch) cut.push_back(b);
  }
  cut.push_back(batch);
  const int64_t nc = (int64_t)cut.size() - 1;
  int64_t max_rows = 0, max_b = 0;
  std::vector<std::vector<int64_t>> offs(nc);
  for (int64_t c = 0; c < nc; ++c) {
    const int64_t b0 = cut[c], b1 = cut[c + 1], r0 = host_offsets[b0];
    max_rows = std::max(max_rows, host_offsets[b1] - r0);
    max_b = std::max(max_b, b1 - b0);
    offs[c].resize(b1 - b0 + 1);
    for (int64_t i = b0; i <= b1; ++i) offs[c][i - b0] = host_offsets[i] - r0;
  }
  const size_t es = dsize(dtype);
  const size_t row_b = (size_t)H * D * es;
  const size_t tb = (size_t)max_rows * row_b, lb = (size_t)max_rows * H * sizeof(float);
  const size_t ob = sizeof(int64_t) * (max_b + 1);
  const size_t ws = (size_t)jg_attention_backward_workspace_size(max_rows, max_b, H, D);
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t slot_bytes = al(ob) + 8 * al(tb) + al(lb) + al(ws);
  cudaStream_t sx[kSlots];
  cudaEvent_t ev_start, ev_done[kSlots];
  for (int j = 0; j < kSlots; ++j) {
    JG_CUDA(cudaStreamCreateWithFlags(&sx[j], cudaStreamNonBlocking));
    JG_CUDA(cudaEventCreateWithFlags(&ev_done[j], cudaEventDisableTiming));
  }
  JG_CUDA(cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming));
  JG_CUDA(cudaEventRecord(ev_start, user));  // work already queued on the caller's stream comes first
  Scratch buf(sx[0]);
  jg_status rc = buf.alloc(kSlots * slot_bytes);
  std::vector<jg_schedule> scheds;
  for (int j = 0; j < kSlots && !rc; ++j) JG_CUDA(cudaStreamWaitEvent(sx[j], ev_start, 0));
  {
    cudaEvent_t alloc_done;
    JG_CUDA(cudaEventCreateWithFlags(&alloc_done, cudaEventDisableTiming));
    JG_CUDA(cudaEventRecord(alloc_done, sx[0]));  // the scratch allocation is ordered on sx[0]
    for (int j = 1; j < kSlots; ++j) JG_CUDA(cudaStreamWaitEvent(sx[j], alloc_done, 0));
    cudaEventDestroy(alloc_done);
  }
  for (int64_t c = 0; c < nc && !rc; ++c) {
    const int j = (int)(c % kSlots);
    cudaStream_t st = sx[j];
    char* p = (char*)buf.p + j * slot_bytes;
    int64_t* d_off = (int64_t*)p; p += al(ob);
    char* t[8];
    for (int u = 0; u < 8; ++u) { t[u] = p; p += al(tb); }
    float* d_lse = (float*)p; p += al(lb);
    void* d_ws = p;
    const int64_t b0 = cut[c], bc = cut[c + 1] - b0, r0 = host_offsets[b0], rows = offs[c].back();
    const size_t cb = (size_t)rows * row_b, hoff = (size_t)r0 * row_b;
    JG_CUDA(cudaMemcpyAsync(d_off, offs[c].data(), sizeof(int64_t) * (bc + 1), cudaMemcpyHostToDevice, st));
    JG_CUDA(cudaMemcpyAsync(t[0], (const char*)q + hoff, cb, cudaMemcpyHostToDevice, st));
    JG_CUDA(cudaMemcpyAsync(t[1], (const char*)k + hoff, cb, cudaMemcpyHostToDevice, st));
    JG_CUDA(cudaMemcpyAsync(t[2], (const char*)v + hoff, cb, cudaMemcpyHostToDevice, st));
    JG_CUDA(cudaMemcpyAsync(t[3], (const char*)go + hoff, cb, cudaMemcpyHostToDevice, st));
    if (rows == 0) continue;
    jg_schedule sched = nullptr;
    if ((rc = jg_schedule_create(d_off, bc, rows, st, &sched))) break;
    scheds.push_back(sched);
    rc = jg_jagged_flash_attention_forward(d_off, bc, rows, H, D, t[0], t[1], t[2], 64, 64, t[4], d_lse, dtype, sched, st);
    if (!rc)
      rc = jg_jagged_flash_attention_backward(d_off, bc, rows, H, D, t[0], t[1], t[2], t[3], t[4], d_lse, 64, 64, t[5],
                                              t[6], t[7], dtype, 1, sched, d_ws, st);
    if (rc) break;
    JG_CUDA(cudaMemcpyAsync((char*)out + hoff, t[4], cb, cudaMemcpyDeviceToHost, st));
    JG_CUDA(cudaMemcpy2DAsync(lse + r0, (size_t)S * sizeof(float), d_lse, (size_t)rows * sizeof(float),
                              (size_t)rows * sizeof(float), (size_t)H, cudaMemcpyDeviceToHost, st));
    JG_CUDA(cudaMemcpyAsync((char*)dq + hoff, t[5], cb, cudaMemcpyDeviceToHost, st));
    JG_CUDA(cudaMemcpyAsync((char*)dk + hoff, t[6], cb, cudaMemcpyDeviceToHost, st));
    JG_CUDA(cudaMemcpyAsync((char*)dv + hoff, t[7], cb, cudaMemcpyDeviceToHost, st));
  }
  // the scratch is released on sx[0] after every stream's work
  for (int j = 1; j < kSlots; ++j) {
    JG_CUDA(cudaEventRecord(ev_done[j], sx[j]));
    JG_CUDA(cudaStreamWaitEvent(sx[0], ev_done[j], 0));
  }
  for (int j = 0; j < kSlots; ++j) {
    cudaError_t e = cudaStreamSynchronize(sx[j]);
    if (e != cudaSuccess && !rc) rc = cuda_status(e, "fwd_bwd_host");
  }
  for (jg_schedule s : scheds) jg_schedule_destroy(s);
  if (buf.p) cudaFreeAsync(buf.p, sx[0]);
  buf.p = nullptr;
  cudaStreamSynchronize(sx[0]);
  for (int j = 0; j < kSlots; ++j) {
    cudaStreamDestroy(sx[j]);
    cudaEventDestroy(ev_done[j]);
  }
  cudaEventDestroy(ev_start);
  return rc;
}

// ============================================================================ SURVEY §8f next rows
extern "C" int64_t jg_feature_interaction_workspace_size(int64_t total_rows, int64_t num_targets) {
  const int64_t n = total_rows * num_targets;
  return 2 * ((n * 4 + 255) / 256) * 256 + ((n * 2 + 255) / 256) * 256;
}

// attention.cpp:291-309: s = jdbmm(k, targets^T) (fp32 out), scale, jagged_softmax over rows, jjbmm(p, v)
extern "C" jg_status jg_feature_interaction(const int64_t* off, int64_t batch, int64_t total_rows, int64_t D,
                                            int64_t Tq, const void* k_feat, const void* v_feat, const void* targets,
                                            void* out, jg_dtype dtype, void* workspace, void* stream) {
  CHECK_DT("feature_interaction", dtype);
  REQUIRE(D >= 1 && Tq >= 1, JG_INVALID_ARGUMENT, "feature_interaction: targets must be [B, Tq, D]");
  cudaStream_t st = as_stream(stream);
  if (batch == 0) return JG_OK;
  REQUIRE_PTRS("feature_interaction", true, off, targets, out);
  if (total_rows == 0) {  // every sample empty: the reference returns [B, Tq, D] zeros
    JG_CUDA(cudaMemsetAsync(out, 0, (size_t)batch * Tq * D * dsize(dtype), st));
    return JG_OK;
  }
  if (dtype == JG_BF16 && !force_simt() && attn_sm100_supported((int)D, dtype)) {
    // fused: feature_interaction is attention with the Tq targets of sample i as queries over
    // its k_feat rows (softmax over the segment axis per target) and v_feat as values — the forward JFA
    // kernel in cross mode, one launch; samples without rows give zero outputs
    Scratch qo(st);
    if (jg_status rc = qo.alloc(sizeof(int64_t) * (batch + 1))) return rc;
    if (jg_status rc = launch_uniform_offsets((int64_t*)qo.p, batch, Tq, st)) return rc;
    jg_schedule qs = nullptr;  // (sample, 256-target pair) items over the query segments
    if (jg_status rc = jg_schedule_create((const int64_t*)qo.p, batch, batch * Tq, st, &qs)) return rc;
    jg_status rc = launch_attn_fwd_sm100(off, batch, total_rows, 1, (int)D, targets, k_feat, v_feat, out, nullptr,
                                         qs->items2, qs->n_items2, qs->max_items2, nullptr, qs->counters, st,
                                         (const int64_t*)qo.p, batch * Tq);
    schedule_release(qs, st);
    return rc;
  }
  const int64_t n = total_rows * Tq;
  Scratch ws(st);
  if (!workspace) {
    if (jg_status rc = ws.alloc(std::max<int64_t>(256, jg_feature_interaction_workspace_size(total_rows, Tq)))) return rc;
    workspace = ws.p;
  }
  float* s = (float*)workspace;
  float* pr = (float*)((char*)workspace + ((n * 4 + 255) / 256) * 256);
  void* p16 = (char*)pr + ((n * 4 + 255) / 256) * 256;
  // scores: M = Bi rows, N = Tq, K = D; B(d, t) = targets[i, t, d] (transpose_per_sample folded into strides)
  GemmDesc gs = desc(BI(), C_(Tq), C_(D), OFF(D), C_(D), C_(1), IDX(Tq * D), C_(1), C_(D), OFF(Tq), C_(Tq), C_(1));
  if (jg_status rc = gemm(gs, off, nullptr, batch, k_feat, targets, s, dtype, JG_F32, st)) return rc;
  // scale by 1/sqrt(D) rounded to float (the reference's T(1/sqrt(d)), attention.cpp:300)
  if (jg_status rc = launch_elementwise(3, s, nullptr, n, (double)(float)(1.0 / std::sqrt((double)D)), s, JG_F32, st))
    return rc;
  if (jg_status rc = launch_jagged_softmax(off, batch, Tq, s, nullptr, pr, JG_F32, false, st)) return rc;
  // out_i = P_i^T V_i: M = Tq, N = D, K = Bi
  GemmDesc gz = desc(C_(Tq), C_(D), BI(), OFF(Tq), C_(1), C_(Tq), OFF(D), C_(D), C_(1), IDX(Tq * D), C_(D), C_(1));
  if (dtype == JG_F32) return gemm(gz, off, nullptr, batch, pr, v_feat, out, JG_F32, JG_F32, st);
  if (jg_status rc = launch_cast_f32(pr, n, p16, JG_BF16, st)) return rc;
  if (!force_simt_gemm() && gemm_sm100_supported(2, Tq, D, JG_BF16))
    return tc_gemm(2, off, nullptr, batch, total_rows, Tq, D, p16, v_feat, out, JG_BF16, st);
  return gemm(gz, off, nullptr, batch, p16, v_feat, out, JG_BF16, JG_BF16, st);
}

// linalg.cpp:246-261 one affine layer over all rows: fp32 accumulation, bias + activation epilogue
extern "C" jg_status jg_mlp_layer_forward(int64_t rows, int64_t d_in, int64_t d_out, const void* x, const void* w,
                                          const void* bias, int32_t relu, void* out, void* preact, jg_dtype dtype,
                                          void* stream) {
  CHECK_DT("jagged_mlp", dtype);
  REQUIRE(d_in >= 1 && d_out >= 1, JG_INVALID_ARGUMENT, "jagged_mlp: layer dims must be positive");
  cudaStream_t st = as_stream(stream);
  if (rows == 0) return JG_OK;
  const bool tc = !force_simt_gemm() && gemm_sm100_supported(3, d_in, d_out, dtype);
  Scratch sc(st);
  if (jg_status rc = sc.alloc(512 + (tc ? 0 : rows * d_out * 4))) return rc;
  int64_t* off = (int64_t*)sc.p;
  int64_t* prefix = (int64_t*)((char*)sc.p + 256);
  float* acc = (float*)((char*)sc.p + 512);
  if (jg_status rc = launch_two_offsets(off, rows, st)) return rc;
  if (tc)  // bias + activation fused into the tcgen05 GEMM epilogue: no fp32 round trip through HBM
    return launch_gemm_sm100(3, off, nullptr, 1, rows, d_in, d_out, x, w, out, JG_BF16, prefix, st, bias, relu, preact);
  {
    GemmDesc g = desc(BI(), C_(d_out), C_(d_in), C_(0), C_(d_in), C_(1), C_(0), C_(d_out), C_(1), C_(0), C_(d_out),
                      C_(1));
    if (jg_status rc = gemm(g, off, nullptr, 1, x, w, acc, dtype, JG_F32, st)) return rc;
  }
  return launch_bias_act(acc, bias, rows, d_out, relu, out, preact, dtype, st);
}

// linalg.cpp:526-567 one layer of the VJP
extern "C" jg_status jg_mlp_layer_backward(int64_t rows, int64_t d_in, int64_t d_out, const void* x, const void* w,
                                           const void* preact, int32_t relu, const void* grad_out, void* dw, void* db,
                                           void* dx, jg_dtype dtype, void* stream) {
  CHECK_DT("jagged_mlp_vjp", dtype);
  REQUIRE(d_in >= 1 && d_out >= 1, JG_INVALID_ARGUMENT, "jagged_mlp_vjp: layer dims must be positive");
  REQUIRE(!relu || preact || rows == 0, JG_INVALID_ARGUMENT, "jagged_mlp_vjp: relu layers need their pre-activations");
  cudaStream_t st = as_stream(stream);
  const size_t es = dsize(dtype);
  const int64_t part = colsum_scratch_floats(rows, d_out);
  Scratch sc(st);
  if (jg_status rc = sc.alloc(256 + ((rows * d_out * es + 255) / 256) * 256 + part * 4 + 256)) return rc;
  int64_t* off = (int64_t*)sc.p;
  void* delta = (char*)sc.p + 256;
  float* partial = (float*)((char*)delta + ((rows * d_out * es + 255) / 256) * 256);
  if (jg_status rc = launch_two_offsets(off, rows, st)) return rc;
  if (jg_status rc = launch_relu_mask(grad_out, preact, rows * d_out, relu, delta, dtype, st)) return rc;
  if (db)
    if (jg_status rc = launch_colsum(delta, rows, d_out, db, partial, dtype, st)) return rc;
  if (dw) {  // dW = x^T delta: a one-segment jagged_jagged_bmm
    if (!force_simt_gemm() && gemm_sm100_supported(2, d_in, d_out, dtype)) {
      if (jg_status rc = tc_gemm(2, off, nullptr, 1, rows, d_in, d_out, x, delta, dw, dtype, st)) return rc;
    } else {
      GemmDesc g = desc(C_(d_in), C_(d_out), BI(), C_(0), C_(1), C_(d_in), C_(0), C_(d_out), C_(1), C_(0), C_(d_out),
                        C_(1));
      if (rows == 0) {
        JG_CUDA(cudaMemsetAsync(dw, 0, d_in * d_out * es, st));
      } else if (jg_status rc = gemm(g, off, nullptr, 1, x, delta, dw, dtype, dtype, st)) {
        return rc;
      }
    }
  }
  if (dx && rows > 0 && tc_ok(TC_JDT, d_in, d_out, dtype))  // dx = delta W^T: one segment, W [1, d_in, d_out]
    return tc_gemm(TC_JDT, off, nullptr, 1, rows, d_in, d_out, delta, w, dx, dtype, st);
  if (dx && rows > 0) {  // dx = delta W^T: B(k = o, n = i) = W[i, o]
    GemmDesc g = desc(BI(), C_(d_in), C_(d_out), C_(0), C_(d_out), C_(1), C_(0), C_(1), C_(d_out), C_(0), C_(d_in),
                      C_(1));
    if (jg_status rc = gemm(g, off, nullptr, 1, delta, w, dx, dtype, dtype, st)) return rc;
  }
  return JG_OK;
}
