// jagged_dropin.cpp — link-level drop-in for the reference's operator objects (linalg.o, attention.o).
//
// Compiled against the reference library's PUBLIC headers (proj/core/include/jagged/*.hpp, found on
// the include path like any consumer of jagged::jagged), this translation unit defines the operator
// templates of linalg.hpp and attention.hpp for T = float on the B200: each call copies the operands
// to the device, runs the C-ABI (include/jagged_b200.h, libjagged_b200.so) and copies the results
// back into the reference's owning tensor types. Validation happens on the host with the reference's
// exception texts (linalg.cpp:16-26, :37-44, :165-172, attention.cpp:33-40, :179-180, :234-241).
//
// T = double (the registry/gradcheck substrate) and dense_attention (the materialised padded baseline) have
// no device implementation: they throw std::invalid_argument naming the operator. There is no CPU fallback.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "jagged/attention.hpp"
#include "jagged/linalg.hpp"
#include "jagged/tensor.hpp"
#include "jagged_b200.h"

namespace jagged {
namespace {

[[noreturn]] void device_fail(const char* op, jg_status rc) {
  const std::string msg = std::string(op) + ": " + jg_last_error();
  if (rc == JG_INVALID_ARGUMENT) throw std::invalid_argument(jg_last_error());
  throw std::runtime_error(msg);
}

void ck(const char* op, jg_status rc) {
  if (rc != JG_OK) device_fail(op, rc);
}

void ckc(const char* op, cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(op) + ": " + cudaGetErrorString(e));
}

// Owning device buffer.
struct Dev {
  void* p = nullptr;
  size_t bytes = 0;
  Dev() = default;
  Dev(size_t n, const char* op) : bytes(n) { ckc(op, cudaMalloc(&p, n ? n : 16)); }
  template <typename T>
  static Dev from(const std::vector<T>& v, const char* op) {
    Dev d(v.size() * sizeof(T), op);
    if (!v.empty()) ckc(op, cudaMemcpy(d.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
  }
  template <typename T>
  std::vector<T> to(size_t n, const char* op) const {
    std::vector<T> v(n);
    if (n) ckc(op, cudaMemcpy(v.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost));
    return v;
  }
  ~Dev() {
    if (p) cudaFree(p);
  }
  Dev(Dev&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; }
  Dev& operator=(Dev&& o) noexcept {
    if (this != &o) {
      if (p) cudaFree(p);
      p = o.p;
      bytes = o.bytes;
      o.p = nullptr;
    }
    return *this;
  }
  Dev(const Dev&) = delete;
};

template <typename T>
void require_matching_offsets(const JaggedTensor<T>& a, const JaggedTensor<T>& b, const char* op) {
  if (a.batch() != b.batch())
    throw std::invalid_argument(std::string(op) + ": batch mismatch (" + std::to_string(a.batch()) + " vs " +
                                std::to_string(b.batch()) + ")");
  for (int64_t i = 0; i < a.batch(); ++i)
    if (a.length(i) != b.length(i))
      throw std::invalid_argument(std::string(op) + ": offsets differ first at sample " + std::to_string(i));
}

template <typename T>
[[noreturn]] void no_device_path(const char* op) {
  throw std::invalid_argument(std::string(op) + ": no B200 device path for " +
                              (sizeof(T) == 8 ? "binary64" : "this operator") + " (no CPU fallback)");
}

template <typename T>
constexpr bool is_f32 = std::is_same_v<T, float>;

// KernelOptions.meter (linalg.hpp:19, scratch.hpp:12-55): the device scratch a call allocates for its own
// intermediates, in elements of T, reported as one allocation window per operator (jg_scratch_counters). The
// reference counts its host scratch buffers the same way (e.g. attention.cpp:190-191 per-thread score rows);
// on-chip tiles (TMEM / shared memory) are registers of the kernel, not allocations. Nested windows are safe.
class MeterScope {
 public:
  MeterScope(const KernelOptions& o, size_t elem) : meter_(o.meter), elem_(elem) {
    if (!meter_) return;
    jg_scratch_counters(&cur0_, &peak0_);
    jg_scratch_reset_peak();
  }
  ~MeterScope() {
    if (!meter_) return;
    int64_t cur = 0, peak = 0;
    jg_scratch_counters(&cur, &peak);
    const int64_t elems = (peak - cur0_ + (int64_t)elem_ - 1) / (int64_t)elem_;
    if (elems > 0) {
      meter_->on_alloc(elems);
      meter_->on_release(elems);
    }
    jg_scratch_raise_peak(peak0_);
  }
  MeterScope(const MeterScope&) = delete;
  MeterScope& operator=(const MeterScope&) = delete;

 private:
  ScratchMeter* meter_;
  size_t elem_;
  int64_t cur0_ = 0, peak0_ = 0;
};

std::vector<int64_t> lengths_of(const std::vector<int64_t>& off) {
  std::vector<int64_t> l(off.size() - 1);
  for (size_t i = 0; i + 1 < off.size(); ++i) l[i] = off[i + 1] - off[i];
  return l;
}

}  // namespace

// ============================================================================ Table-1 forward ops
template <typename T>
JaggedTensor<T> jagged_dense_bmm(const JaggedTensor<T>& x, const DenseTensor<T>& w, const KernelOptions& opts) {
  MeterScope meter_scope(opts, sizeof(T));
  const char* op = "jagged_dense_bmm";
  if (w.rank() != 3) throw std::invalid_argument("jagged_dense_bmm: w must be [B, D, T]");
  const int64_t b = x.batch(), d = x.dim(), t = w.shape()[2];
  if (w.shape()[0] != b)
    throw std::invalid_argument("jagged_dense_bmm: batch mismatch (" + std::to_string(b) + " vs " +
                                std::to_string(w.shape()[0]) + ")");
  if (w.shape()[1] != d)
    throw std::invalid_argument("jagged_dense_bmm: dim mismatch (" + std::to_string(d) + " vs " +
                                std::to_string(w.shape()[1]) + ")");
  if constexpr (!is_f32<T>) no_device_path<T>(op);
  Dev off = Dev::from(x.offsets(), op), dx = Dev::from(x.values(), op), dw = Dev::from(w.data(), op);
  Dev out(sizeof(T) * x.total_rows() * t, op);
  ck(op, jg_jagged_dense_bmm((const int64_t*)off.p, b, x.total_rows(), d, t, dx.p, dw.p, out.p, JG_F32, JG_F32, 0));
  return JaggedTensor<T>(x.offsets(), out.to<T>(x.total_rows() * t, op), t);
}

template <typename T>
DenseTensor<T> jagged_jagged_bmm(const JaggedTensor<T>& x, const JaggedTensor<T>& y, const KernelOptions& opts) {
  MeterScope meter_scope(opts, sizeof(T));
  const char* op = "jagged_jagged_bmm";
  require_matching_offsets(x, y, op);
  if constexpr (!is_f32<T>) no_device_path<T>(op);
  const int64_t b = x.batch(), d = x.dim(), t = y.dim();
  Dev off = Dev::from(x.offsets(), op), dx = Dev::from(x.values(), op), dy = Dev::from(y.values(), op);
  Dev out(sizeof(T) * b * d * t, op);
  ck(op, jg_jagged_jagged_bmm((const int64_t*)off.p, b, x.total_rows(), d, t, dx.p, dy.p, out.p, JG_F32, JG_F32, 0));
  return DenseTensor<T>({b, d, t}, out.to<T>(b * d * t, op));
}

template <typename T>
JaggedTensor<T> jagged_softmax(const JaggedTensor<T>& x, const KernelOptions& opts) {
  MeterScope meter_scope(opts, sizeof(T));
  const char* op = "jagged_softmax";
  if constexpr (!is_f32<T>) no_device_path<T>(op);
  Dev off = Dev::from(x.offsets(), op), dx = Dev::from(x.values(), op), out(sizeof(T) * x.values().size(), op);
  ck(op, jg_jagged_softmax((const int64_t*)off.p, x.batch(), x.total_rows(), x.dim(), dx.p, out.p, JG_F32, 0));
  return JaggedTensor<T>(x.offsets(), out.to<T>(x.values().size(), op), x.dim());
}

template <typename T>
Jagged2Tensor<T> jagged_jagged_bmm_jagged_out(const JaggedTensor<T>& q, const JaggedTensor<T>& k,
                                              const KernelOptions& opts) {
  MeterScope meter_scope(opts, sizeof(T));
  const char* op = "jagged_jagged_bmm_jagged_out";
  require_matching_offsets(q, k, op);
  if (q.dim() != k.dim())
    throw std::invalid_argument("jagged_jagged_bmm_jagged_out: dim mismatch (" + std::to_string(q.dim()) + " vs " +
                                std::to_string(k.dim()) + ")");
  if constexpr (!is_f32<T>) no_device_path<T>(op);
  const auto lengths = segment_lengths(q);
  int64_t sq = 0;
  for (int64_t n : lengths) sq += n * n;
  Dev off = Dev::from(q.offsets(), op), sqo(sizeof(int64_t) * (q.batch() + 1), op);
  Dev dq = Dev::from(q.values(), op), dk = Dev::from(k.values(), op), out(sizeof(T) * sq, op);
  ck(op, jg_sq_offsets((const int64_t*)off.p, q.batch(), (int64_t*)sqo.p, 0));
  ck(op, jg_jagged_jagged_bmm_jagged_out((const int64_t*)off.p, (const int64_t*)sqo.p, q.batch(), q.total_rows(),
                                         q.dim(), dq.p, dk.p, out.p, JG_F32, JG_F32, 0));
  return Jagged2Tensor<T>(lengths, out.to<T>(sq, op));
}

template <typename T>
JaggedTensor<T> array_jagged_bmm_jagged_out(const Jagged2Tensor<T>& a, const JaggedTensor<T>& v, const KernelOptions& opts) {
  MeterScope meter_scope(opts, sizeof(T));
  const char* op = "array_jagged_bmm_jagged_out";
  if (a.batch() != v.batch())
    throw std::invalid_argument("array_jagged_bmm_jagged_out: batch mismatch (" + std::to_string(a.batch()) +
                                " vs " + std::to_string(v.batch()) + ")");
  for (int64_t i = 0; i < a.batch(); ++i)
    if (a.length(i) != v.length(i))
      throw std::invalid_argument("array_jagged_bmm_jagged_out: length mismatch at sample " + std::to_string(i));
  if constexpr (!is_f32<T>) no_device_path<T>(op);
  Dev off = Dev::from(v.offsets(), op), sqo = Dev::from(a.sq_offsets(), op);
  Dev da = Dev::from(a.values(), op), dv = Dev::from(v.values(), op), out(sizeof(T) * v.values().size(), op);
  ck(op, jg_array_jagged_bmm_jagged_out((const int64_t*)off.p, (const int64_t*)sqo.p, v.batch(), v.total_rows(),
                                        (int64_t)a.values().size(), v.dim(), da.p, dv.p, out.p, JG_F32, JG_F32, 0));
  return JaggedTensor<T>(v.offsets(), out.to<T>(v.values().size(), op), v.dim());
}

template <typename T>
Jagged2Tensor<T> jagged2_softmax(const Jagged2Tensor<T>& s, const KernelOptions& opts) {
  MeterScope meter_scope(opts, sizeof(T));
  const char* op = "jagged2_softmax";
  if constexpr (!is_f32<T>) no_device_path<T>(op);
  std::vector<int64_t> off(s.batch() + 1, 0);
  for (int64_t i = 0; i < s.batch(); ++i) off[i + 1] = off[i] + s.length(i);
  Dev doff = Dev::from(off, op), sqo = Dev::from(s.sq_offsets(), op), ds = Dev::from(s.values(), op);
  Dev out(sizeof(T) * s.values().size(), op);
  ck(op, jg_jagged2_softmax((const int64_t*)doff.p, (const int64_t*)sqo.p, s.batch(), ds.p, out.p, JG_F32, 0));
  return Jagged2Tensor<T>(s.seq_lengths(), out.to<T>(s.values().size(), op));
}

// linalg.cpp:224-243 validation (same messages)
template <typename T>
void validate_mlp(const JaggedTensor<T>& x, std::span<const MlpLayer<T>> layers) {
  if (layers.empty()) throw std::invalid_argument("jagged_mlp: at least one layer required");
  int64_t cur = x.dim();
  for (size_t l = 0; l < layers.size(); ++l) {
    const auto& w = layers[l].weights;
    if (w.rank() != 2)
      throw std::invalid_argument("jagged_mlp: layer " + std::to_string(l) + " weights must be rank 2");
    if (w.shape()[0] != cur)
      throw std::invalid_argument("jagged_mlp: layer " + std::to_string(l) + " input dim mismatch (" +
                                  std::to_string(cur) + " vs " + std::to_string(w.shape()[0]) + ")");
    if (static_cast<int64_t>(layers[l].bias.size()) != w.shape()[1])
      throw std::invalid_argument("jagged_mlp: layer " + std::to_string(l) + " bias size " +
                                  std::to_string(layers[l].bias.size()) + " != " + std::to_string(w.shape()[1]));
    cur = w.shape()[1];
  }
}

// linalg.cpp:265-277 via jg_mlp_layer_forward per layer (activations stay on the device between layers)
template <typename T>
JaggedTensor<T> jagged_mlp(const JaggedTensor<T>& x, std::span<const MlpLayer<T>> layers, const KernelOptions& opts) {
  MeterScope meter_scope(opts, sizeof(T));
  const char* op = "jagged_mlp";
  validate_mlp(x, layers);
  if constexpr (!is_f32<T>) no_device_path<T>(op);
  const int64_t rows = x.total_rows();
  Dev cur = Dev::from(x.values(), op);
  for (const auto& L : layers) {
    const int64_t di = L.weights.shape()[0], dout = L.weights.shape()[1];
    Dev w = Dev::from(L.weights.data(), op), b = Dev::from(L.bias, op), out(sizeof(T) * rows * dout, op);
    ck(op, jg_mlp_layer_forward(rows, di, dout, cur.p, w.p, b.p, L.activation == Activation::relu ? 1 : 0, out.p,
                                nullptr, JG_F32, 0));
    cur = std::move(out);
  }
  const int64_t dl = layers.back().weights.shape()[1];
  return JaggedTensor<T>(x.offsets(), cur.to<T>(rows * dl, op), dl);
}

// ============================================================================ VJPs
template <typename T>
JaggedDenseBmmGrads<T> jagged_dense_bmm_vjp(const JaggedTensor<T>& x, const DenseTensor<T>& w,
                                            const JaggedTensor<T>& grad_out, const KernelOptions& opts) {
  MeterScope meter_scope(opts, sizeof(T));
  const char* op = "jagged_dense_bmm_vjp";
  if (w.rank() != 3) throw std::invalid_argument("jagged_dense_bmm_vjp: w must be [B, D, T]");
  require_matching_offsets(x, grad_out, op);
  const int64_t b = x.batch(), d = x.dim(), t = w.shape()[2];
  if (grad_out.dim() != t) throw std::invalid_argument("jagged_dense_bmm_vjp: grad_out dim mismatch");
  if constexpr (!is_f32<T>) no_device_path<T>(op);
  Dev off = Dev::from(x.offsets(), op), dx_in = Dev::from(x.values(), op), dw_in = Dev::from(w.data(), op),
      dgo = Dev::from(grad_out.values(), op), dx(sizeof(T) * x.values().size(), op), dw(sizeof(T) * w.data().size(), op);
  ck(op, jg_jagged_dense_bmm_vjp((const int64_t*)off.p, b, x.total_rows(), d, t, dx_in.p, dw_in.p, dgo.p, dx.p, dw.p,
                                 JG_F32, JG_F32, 0));
  return {JaggedTensor<T>(x.offsets(), dx.to<T>(x.values().size(), op), d),
          DenseTensor<T>(w.shape(), dw.to<T>(w.data().size(), op))};
}

template <typename T>
JaggedJaggedBmmGrads<T> jagged_jagged_bmm_vjp(const JaggedTensor<T>& x, const JaggedTensor<T>& y,
                                              const DenseTensor<T>& grad_out, const KernelOptions& opts) {
  MeterScope meter_scope(opts, sizeof(T));
  const char* op = "jagged_jagged_bmm_vjp";
  require_matching_offsets(x, y, op);
  const int64_t b = x.batch(), d = x.dim(), t = y.dim();
  if (grad_out.rank() != 3 || grad_out.shape()[0] != b || grad_out.shape()[1] != d || grad_out.shape()[2] != t)
    throw std::invalid_argument("jagged_jagged_bmm_vjp: grad_out must be [B, D, T]");
  if constexpr (!is_f32<T>) no_device_path<T>(op);
  Dev off = Dev::from(x.offsets(), op), dxi = Dev::from(x.values(), op), dyi = Dev::from(y.values(), op),
      dgo = Dev::from(grad_out.data(), op), dx(sizeof(T) * x.values().size(), op), dy(sizeof(T) * y.values().size(), op);
  ck(op, jg_jagged_jagged_bmm_vjp((const int64_t*)off.p, b, x.total_rows(), d, t, dxi.p, dyi.p, dgo.p, dx.p, dy.p,
                                  JG_F32, JG_F32, 0));
  return {JaggedTensor<T>(x.offsets(), dx.to<T>(x.values().size(), op), d),
          JaggedTensor<T>(y.offsets(), dy.to<T>(y.values().size(), op), t)};
}

template <typename T>
JaggedTensor<T> jagged_softmax_vjp(const JaggedTensor<T>& x, const JaggedTensor<T>& grad_out, const KernelOptions& opts) {
  MeterScope meter_scope(opts, sizeof(T));
  const char* op = "jagged_softmax_vjp";
  require_matching_offsets(x, grad_out, op);
  if (x.dim() != grad_out.dim()) throw std::invalid_argument("jagged_softmax_vjp: dim mismatch");
  if constexpr (!is_f32<T>) no_device_path<T>(op);
  Dev off = Dev::from(x.offsets(), op), dxi = Dev::from(x.values(), op), dgo = Dev::from(grad_out.values(), op),
      dx(sizeof(T) * x.values().size(), op);
  ck(op, jg_jagged_softmax_vjp((const int64_t*)off.p, x.batch(), x.total_rows(), x.dim(), dxi.p, dgo.p, dx.p, JG_F32, 0));
  return JaggedTensor<T>(x.offsets(), dx.to<T>(x.values().size(), op), x.dim());
}

template <typename T>
BmmJaggedOutGrads<T> jagged_jagged_bmm_jagged_out_vjp(const JaggedTensor<T>& q, const JaggedTensor<T>& k,
                                                      const Jagged2Tensor<T>& grad_out, const KernelOptions& opts) {
  MeterScope meter_scope(opts, sizeof(T));
  const char* op = "jagged_jagged_bmm_jagged_out_vjp";
  require_matching_offsets(q, k, op);
  for (int64_t i = 0; i < q.batch(); ++i)
    if (grad_out.length(i) != q.length(i))
      throw std::invalid_argument("jagged_jagged_bmm_jagged_out_vjp: grad_out length mismatch at sample " +
                                  std::to_string(i));
  if constexpr (!is_f32<T>) no_device_path<T>(op);
  Dev off = Dev::from(q.offsets(), op), sqo = Dev::from(grad_out.sq_offsets(), op), dqi = Dev::from(q.values(), op),
      dki = Dev::from(k.values(), op), dgo = Dev::from(grad_out.values(), op), dq(sizeof(T) * q.values().size(), op),
      dk(sizeof(T) * k.values().size(), op);
  ck(op, jg_jagged_jagged_bmm_jagged_out_vjp((const int64_t*)off.p, (const int64_t*)sqo.p, q.batch(), q.total_rows(),
                                             (int64_t)grad_out.values().size(), q.dim(), dqi.p, dki.p, dgo.p, dq.p, dk.p, JG_F32, JG_F32, 0));
  return {JaggedTensor<T>(q.offsets(), dq.to<T>(q.values().size(), op), q.dim()),
          JaggedTensor<T>(k.offsets(), dk.to<T>(k.values().size(), op), k.dim())};
}

template <typename T>
ArrayJaggedBmmGrads<T> array_jagged_bmm_jagged_out_vjp(const Jagged2Tensor<T>& a, const JaggedTensor<T>& v,
                                                       const JaggedTensor<T>& grad_out, const KernelOptions& opts) {
  MeterScope meter_scope(opts, sizeof(T));
  const char* op = "array_jagged_bmm_jagged_out_vjp";
  require_matching_offsets(v, grad_out, op);
  for (int64_t i = 0; i < v.batch(); ++i)
    if (a.length(i) != v.length(i))
      throw std::invalid_argument("array_jagged_bmm_jagged_out_vjp: length mismatch at sample " + std::to_string(i));
  if constexpr (!is_f32<T>) no_device_path<T>(op);
  Dev off = Dev::from(v.offsets(), op), sqo = Dev::from(a.sq_offsets(), op), dai = Dev::from(a.values(), op),
      dvi = Dev::from(v.values(), op), dgo = Dev::from(grad_out.values(), op), da(sizeof(T) * a.values().size(), op),
      dv(sizeof(T) * v.values().size(), op);
  ck(op, jg_array_jagged_bmm_jagged_out_vjp((const int64_t*)off.p, (const int64_t*)sqo.p, v.batch(), v.total_rows(),
                                            (int64_t)a.values().size(), v.dim(), dai.p, dvi.p, dgo.p, da.p, dv.p, JG_F32, JG_F32, 0));
  return {Jagged2Tensor<T>(a.seq_lengths(), da.to<T>(a.values().size(), op)),
          JaggedTensor<T>(v.offsets(), dv.to<T>(v.values().size(), op), v.dim())};
}

template <typename T>
Jagged2Tensor<T> jagged2_softmax_vjp(const Jagged2Tensor<T>& s, const Jagged2Tensor<T>& grad_out, const KernelOptions& opts) {
  MeterScope meter_scope(opts, sizeof(T));
  const char* op = "jagged2_softmax_vjp";
  if (s.batch() != grad_out.batch() || s.seq_lengths() != grad_out.seq_lengths())
    throw std::invalid_argument("jagged2_softmax_vjp: layout mismatch");
  if constexpr (!is_f32<T>) no_device_path<T>(op);
  std::vector<int64_t> off(s.batch() + 1, 0);
  for (int64_t i = 0; i < s.batch(); ++i) off[i + 1] = off[i] + s.length(i);
  Dev doff = Dev::from(off, op), sqo = Dev::from(s.sq_offsets(), op), dsi = Dev::from(s.values(), op),
      dgo = Dev::from(grad_out.values(), op), ds(sizeof(T) * s.values().size(), op);
  ck(op, jg_jagged2_softmax_vjp((const int64_t*)doff.p, (const int64_t*)sqo.p, s.batch(), dsi.p, dgo.p, ds.p, JG_F32, 0));
  return Jagged2Tensor<T>(s.seq_lengths(), ds.to<T>(s.values().size(), op));
}

// linalg.cpp:509-573: device forward keeping activations and pre-activations, then jg_mlp_layer_backward
template <typename T>
JaggedMlpGrads<T> jagged_mlp_vjp(const JaggedTensor<T>& x, std::span<const MlpLayer<T>> layers,
                                 const JaggedTensor<T>& grad_out, const KernelOptions& opts) {
  MeterScope meter_scope(opts, sizeof(T));
  const char* op = "jagged_mlp_vjp";
  validate_mlp(x, layers);
  require_matching_offsets(x, grad_out, op);
  if constexpr (!is_f32<T>) no_device_path<T>(op);
  const int64_t rows = x.total_rows();
  const size_t n = layers.size();
  std::vector<Dev> acts, pres, ws;
  acts.push_back(Dev::from(x.values(), op));
  for (size_t l = 0; l < n; ++l) {
    const auto& L = layers[l];
    const int64_t di = L.weights.shape()[0], dout = L.weights.shape()[1];
    ws.push_back(Dev::from(L.weights.data(), op));
    Dev b = Dev::from(L.bias, op), out(sizeof(T) * rows * dout, op), pre(sizeof(T) * rows * dout, op);
    ck(op, jg_mlp_layer_forward(rows, di, dout, acts.back().p, ws.back().p, b.p,
                                L.activation == Activation::relu ? 1 : 0, out.p, pre.p, JG_F32, 0));
    acts.push_back(std::move(out));
    pres.push_back(std::move(pre));
  }
  JaggedMlpGrads<T> g{JaggedTensor<T>(x.offsets(), std::vector<T>(x.values().size()), x.dim()), {}};
  g.dlayers.resize(n, MlpLayerGrads<T>{DenseTensor<T>::zeros({1, 1}), {}});
  Dev delta = Dev::from(grad_out.values(), op);
  for (size_t li = n; li-- > 0;) {
    const auto& L = layers[li];
    const int64_t di = L.weights.shape()[0], dout = L.weights.shape()[1];
    Dev dw(sizeof(T) * di * dout, op), db(sizeof(T) * dout, op), dx(sizeof(T) * rows * di, op);
    ck(op, jg_mlp_layer_backward(rows, di, dout, acts[li].p, ws[li].p, pres[li].p,
                                 L.activation == Activation::relu ? 1 : 0, delta.p, dw.p, db.p, dx.p, JG_F32, 0));
    g.dlayers[li] = MlpLayerGrads<T>{DenseTensor<T>({di, dout}, dw.to<T>(di * dout, op)), db.to<T>(dout, op)};
    delta = std::move(dx);
  }
  g.dx = JaggedTensor<T>(x.offsets(), delta.to<T>(rows * x.dim(), op), x.dim());
  return g;
}

// ============================================================================ attention
template <typename T>
DenseTensor<T> transpose_per_sample(const DenseTensor<T>& x) {
  if (x.rank() != 3) throw std::invalid_argument("transpose_per_sample: rank-3 input required");
  const int64_t b = x.shape()[0], m = x.shape()[1], n = x.shape()[2];
  std::vector<T> out(static_cast<size_t>(b * m * n));
  for (int64_t i = 0; i < b; ++i)
    for (int64_t r = 0; r < m; ++r)
      for (int64_t c = 0; c < n; ++c) out[(i * n + c) * m + r] = x.at(i, r, c);
  return DenseTensor<T>({b, n, m}, std::move(out));
}

template <typename T>
DenseTensor<T> dense_attention(const DenseTensor<T>&, const DenseTensor<T>&, const DenseTensor<T>&,
                               std::span<const int64_t>, const KernelOptions& opts) {
  MeterScope meter_scope(opts, sizeof(T));
  no_device_path<T>("dense_attention");
}

// attention.cpp:106-160 on the device: the jagged attention kernels in padded mode
// (jg_dense_flash_attention_forward validates the shape/lengths with the reference's messages).
template <typename T>
DenseAttentionSaved<T> dense_flash_attention(const DenseTensor<T>& q, const DenseTensor<T>& k, const DenseTensor<T>& v,
                                             std::span<const int64_t> lengths, int64_t block_q, int64_t block_k,
                                             const KernelOptions& opts) {
  MeterScope meter_scope(opts, sizeof(T));
  const char* op = "dense_flash_attention";
  if (q.rank() != 3 || q.shape() != k.shape() || q.shape() != v.shape())
    throw std::invalid_argument("dense_flash_attention: q, k, v must share a [B, L, D] shape");
  if (static_cast<int64_t>(lengths.size()) != q.shape()[0])
    throw std::invalid_argument("dense_flash_attention: lengths size mismatch");
  if constexpr (!is_f32<T>) no_device_path<T>(op);
  const int64_t B = q.shape()[0], L = q.shape()[1], D = q.shape()[2];
  Dev dq = Dev::from(q.data(), op), dk = Dev::from(k.data(), op), dv = Dev::from(v.data(), op),
      out(sizeof(T) * q.data().size(), op), lse(sizeof(float) * B * L, op);
  ck(op, jg_dense_flash_attention_forward(lengths.data(), B, L, 1, (int32_t)D, dq.p, dk.p, dv.p, block_q, block_k,
                                          out.p, (float*)lse.p, JG_F32, 0));
  const std::vector<float> lse_f = lse.to<float>(B * L, op);
  return {DenseTensor<T>({B, L, D}, out.to<T>(q.data().size(), op)), std::vector<T>(lse_f.begin(), lse_f.end()),
          block_q, block_k};
}

namespace {
template <typename T>
void require_jagged_attention_inputs(const JaggedTensor<T>& q, const JaggedTensor<T>& k, const JaggedTensor<T>& v,
                                     const char* op) {
  if (q.dim() != k.dim() || q.dim() != v.dim()) throw std::invalid_argument(std::string(op) + ": dim mismatch");
  if (!q.same_offsets(k) || !q.same_offsets(v))
    throw std::invalid_argument(std::string(op) + ": q, k, v must share offsets");
}
}  // namespace

template <typename T>
JaggedTensor<T> jagged_attention(const JaggedTensor<T>& q, const JaggedTensor<T>& k, const JaggedTensor<T>& v,
                                 const KernelOptions& opts) {
  MeterScope meter_scope(opts, sizeof(T));
  const char* op = "jagged_attention";
  require_jagged_attention_inputs(q, k, v, op);
  if constexpr (!is_f32<T>) no_device_path<T>(op);
  int64_t sq = 0;
  for (int64_t i = 0; i < q.batch(); ++i) sq += q.length(i) * q.length(i);
  Dev off = Dev::from(q.offsets(), op), sqo(sizeof(int64_t) * (q.batch() + 1), op), dq = Dev::from(q.values(), op),
      dk = Dev::from(k.values(), op), dv = Dev::from(v.values(), op), out(sizeof(T) * q.values().size(), op);
  ck(op, jg_sq_offsets((const int64_t*)off.p, q.batch(), (int64_t*)sqo.p, 0));
  ck(op, jg_jagged_attention((const int64_t*)off.p, (const int64_t*)sqo.p, q.batch(), q.total_rows(), sq, 1,
                             (int32_t)q.dim(), dq.p, dk.p, dv.p, out.p, JG_F32, nullptr, 0));
  return JaggedTensor<T>(q.offsets(), out.to<T>(q.values().size(), op), q.dim());
}

template <typename T>
JaggedAttentionSaved<T> jagged_flash_attention_forward(const JaggedTensor<T>& q, const JaggedTensor<T>& k,
                                                       const JaggedTensor<T>& v, int64_t block_q, int64_t block_k,
                                                       const KernelOptions& opts) {
  MeterScope meter_scope(opts, sizeof(T));
  const char* op = "jagged_flash_attention_forward";
  require_jagged_attention_inputs(q, k, v, op);
  if (block_q < 1 || block_k < 1)
    throw std::invalid_argument("jagged_flash_attention_forward: block sizes must be >= 1");
  if constexpr (!is_f32<T>) no_device_path<T>(op);
  const int64_t S = q.total_rows();
  Dev off = Dev::from(q.offsets(), op), dq = Dev::from(q.values(), op), dk = Dev::from(k.values(), op),
      dv = Dev::from(v.values(), op), out(sizeof(T) * q.values().size(), op), lse(sizeof(float) * S, op);
  ck(op, jg_jagged_flash_attention_forward((const int64_t*)off.p, q.batch(), S, 1, (int32_t)q.dim(), dq.p, dk.p, dv.p,
                                           block_q, block_k, out.p, (float*)lse.p, JG_F32, nullptr, 0));
  const std::vector<float> lse_f = lse.to<float>(S, op);
  return {JaggedTensor<T>(q.offsets(), out.to<T>(q.values().size(), op), q.dim()),
          std::vector<T>(lse_f.begin(), lse_f.end()), block_q, block_k};
}

template <typename T>
AttentionGrads<T> jagged_flash_attention_backward(const JaggedTensor<T>& q, const JaggedTensor<T>& k,
                                                  const JaggedTensor<T>& v, const JaggedTensor<T>& grad_out,
                                                  const JaggedAttentionSaved<T>& saved, const KernelOptions& opts) {
  MeterScope meter_scope(opts, sizeof(T));
  const char* op = "jagged_flash_attention_backward";
  require_jagged_attention_inputs(q, k, v, op);
  if (!grad_out.same_offsets(q) || grad_out.dim() != q.dim())
    throw std::invalid_argument("jagged_flash_attention_backward: grad_out layout mismatch");
  if (!saved.output.same_offsets(q) || saved.output.dim() != q.dim() ||
      static_cast<int64_t>(saved.logsumexp.size()) != q.total_rows() || saved.block_q < 1 || saved.block_k < 1)
    throw std::invalid_argument("jagged_flash_attention_backward: saved state does not match inputs");
  if constexpr (!is_f32<T>) no_device_path<T>(op);
  const int64_t S = q.total_rows();
  std::vector<float> lse(saved.logsumexp.begin(), saved.logsumexp.end());
  Dev off = Dev::from(q.offsets(), op), dq_in = Dev::from(q.values(), op), dk_in = Dev::from(k.values(), op),
      dv_in = Dev::from(v.values(), op), dgo = Dev::from(grad_out.values(), op),
      dout = Dev::from(saved.output.values(), op), dlse = Dev::from(lse, op), dq(sizeof(T) * q.values().size(), op),
      dk(sizeof(T) * k.values().size(), op), dv(sizeof(T) * v.values().size(), op);
  ck(op, jg_jagged_flash_attention_backward((const int64_t*)off.p, q.batch(), S, 1, (int32_t)q.dim(), dq_in.p, dk_in.p,
                                            dv_in.p, dgo.p, dout.p, (const float*)dlse.p, saved.block_q, saved.block_k,
                                            dq.p, dk.p, dv.p, JG_F32, 1, nullptr, nullptr, 0));
  return {JaggedTensor<T>(q.offsets(), dq.to<T>(q.values().size(), op), q.dim()),
          JaggedTensor<T>(k.offsets(), dk.to<T>(k.values().size(), op), k.dim()),
          JaggedTensor<T>(v.offsets(), dv.to<T>(v.values().size(), op), v.dim())};
}

// attention.cpp:291-309 composition, every step on the device
template <typename T>
DenseTensor<T> feature_interaction(const JaggedTensor<T>& k_feat, const JaggedTensor<T>& v_feat,
                                   const DenseTensor<T>& targets, const KernelOptions& opts) {
  MeterScope meter_scope(opts, sizeof(T));
  if (!k_feat.same_offsets(v_feat) || k_feat.dim() != v_feat.dim())
    throw std::invalid_argument("feature_interaction: k_feat/v_feat layout mismatch");
  if (targets.rank() != 3 || targets.shape()[0] != k_feat.batch() || targets.shape()[2] != k_feat.dim())
    throw std::invalid_argument("feature_interaction: targets must be [B, Tq, D]");
  (void)opts;
  const char* op = "feature_interaction";
  if constexpr (!is_f32<T>) no_device_path<T>(op);
  const int64_t b = k_feat.batch(), d = k_feat.dim(), tq = targets.shape()[1];
  Dev off = Dev::from(k_feat.offsets(), op), k = Dev::from(k_feat.values(), op), v = Dev::from(v_feat.values(), op);
  Dev tg = Dev::from(targets.data(), op), out(sizeof(T) * b * tq * d, op);
  ck(op, jg_feature_interaction((const int64_t*)off.p, b, k_feat.total_rows(), d, tq, k.p, v.p, tg.p, out.p, JG_F32,
                                nullptr, 0));
  return DenseTensor<T>({b, tq, d}, out.to<T>(b * tq * d, op));
}

// ---------------------------------------------------------------------------- instantiations
#define JG_DROPIN(T)                                                                                               \
  template JaggedTensor<T> jagged_dense_bmm(const JaggedTensor<T>&, const DenseTensor<T>&, const KernelOptions&);  \
  template DenseTensor<T> jagged_jagged_bmm(const JaggedTensor<T>&, const JaggedTensor<T>&, const KernelOptions&); \
  template JaggedTensor<T> jagged_softmax(const JaggedTensor<T>&, const KernelOptions&);                           \
  template Jagged2Tensor<T> jagged_jagged_bmm_jagged_out(const JaggedTensor<T>&, const JaggedTensor<T>&,           \
                                                         const KernelOptions&);                                    \
  template JaggedTensor<T> array_jagged_bmm_jagged_out(const Jagged2Tensor<T>&, const JaggedTensor<T>&,            \
                                                       const KernelOptions&);                                      \
  template Jagged2Tensor<T> jagged2_softmax(const Jagged2Tensor<T>&, const KernelOptions&);                        \
  template JaggedTensor<T> jagged_mlp(const JaggedTensor<T>&, std::span<const MlpLayer<T>>, const KernelOptions&); \
  template JaggedDenseBmmGrads<T> jagged_dense_bmm_vjp(const JaggedTensor<T>&, const DenseTensor<T>&,              \
                                                       const JaggedTensor<T>&, const KernelOptions&);              \
  template JaggedJaggedBmmGrads<T> jagged_jagged_bmm_vjp(const JaggedTensor<T>&, const JaggedTensor<T>&,           \
                                                         const DenseTensor<T>&, const KernelOptions&);             \
  template JaggedTensor<T> jagged_softmax_vjp(const JaggedTensor<T>&, const JaggedTensor<T>&, const KernelOptions&); \
  template BmmJaggedOutGrads<T> jagged_jagged_bmm_jagged_out_vjp(const JaggedTensor<T>&, const JaggedTensor<T>&,   \
                                                                 const Jagged2Tensor<T>&, const KernelOptions&);   \
  template ArrayJaggedBmmGrads<T> array_jagged_bmm_jagged_out_vjp(const Jagged2Tensor<T>&, const JaggedTensor<T>&, \
                                                                  const JaggedTensor<T>&, const KernelOptions&);   \
  template Jagged2Tensor<T> jagged2_softmax_vjp(const Jagged2Tensor<T>&, const Jagged2Tensor<T>&,                  \
                                                const KernelOptions&);                                             \
  template JaggedMlpGrads<T> jagged_mlp_vjp(const JaggedTensor<T>&, std::span<const MlpLayer<T>>,                  \
                                            const JaggedTensor<T>&, const KernelOptions&);                         \
  template DenseTensor<T> transpose_per_sample(const DenseTensor<T>&);                                             \
  template DenseTensor<T> dense_attention(const DenseTensor<T>&, const DenseTensor<T>&, const DenseTensor<T>&,     \
                                          std::span<const int64_t>, const KernelOptions&);                         \
  template DenseAttentionSaved<T> dense_flash_attention(const DenseTensor<T>&, const DenseTensor<T>&,              \
                                                        const DenseTensor<T>&, std::span<const int64_t>, int64_t,  \
                                                        int64_t, const KernelOptions&);                            \
  template JaggedTensor<T> jagged_attention(const JaggedTensor<T>&, const JaggedTensor<T>&, const JaggedTensor<T>&, \
                                            const KernelOptions&);                                                 \
  template JaggedAttentionSaved<T> jagged_flash_attention_forward(const JaggedTensor<T>&, const JaggedTensor<T>&,  \
                                                                  const JaggedTensor<T>&, int64_t, int64_t,        \
                                                                  const KernelOptions&);                           \
  template AttentionGrads<T> jagged_flash_attention_backward(const JaggedTensor<T>&, const JaggedTensor<T>&,       \
                                                             const JaggedTensor<T>&, const JaggedTensor<T>&,       \
                                                             const JaggedAttentionSaved<T>&, const KernelOptions&); \
  template DenseTensor<T> feature_interaction(const JaggedTensor<T>&, const JaggedTensor<T>&, const DenseTensor<T>&, \
                                              const KernelOptions&);

JG_DROPIN(float)
JG_DROPIN(double)

}  // namespace jagged
