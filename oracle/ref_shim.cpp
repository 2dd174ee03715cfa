// ref_shim.cpp — extern "C" entry points over the COMPILED REFERENCE (test infrastructure).
//
// oracle/Makefile compiles this file together with the reference's own sources, in place under
// /root/reference/proj/core/src (tensor.cpp, rng.cpp, parallel.cpp, linalg.cpp, attention.cpp),
// into oracle/_ref/libjagged_ref.so. Nothing here restates arithmetic: each function builds the
// reference's own JaggedTensor/Jagged2Tensor/DenseTensor and calls the reference operator, so the
// results are the reference's results. Used to (1) pin oracle/jagged_oracle.c, (2) generate
// tests/golden fixtures, (3) time the reference CPU path in bench.py (cpu_baseline, --impl reference).
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "jagged/attention.hpp"
#include "jagged/bench.hpp"
#include "jagged/cost_model.hpp"
#include "jagged/linalg.hpp"
#include "jagged/rng.hpp"
#include "jagged/tensor.hpp"

namespace {
thread_local std::string g_err;

template <typename T>
std::vector<T> vec(const T* p, int64_t n) {
  return std::vector<T>(p, p + n);
}

template <typename T>
jagged::JaggedTensor<T> jt(const int64_t* off, int64_t B, int64_t dim, const T* v) {
  return jagged::JaggedTensor<T>(vec(off, B + 1), vec(v, off[B] * dim), dim);
}

template <typename T>
jagged::Jagged2Tensor<T> j2(const int64_t* off, int64_t B, const T* v) {
  std::vector<int64_t> lens(B);
  int64_t sq = 0;
  for (int64_t i = 0; i < B; ++i) {
    lens[i] = off[i + 1] - off[i];
    sq += lens[i] * lens[i];
  }
  return jagged::Jagged2Tensor<T>(lens, vec(v, sq));
}

template <typename T>
void put(const std::vector<T>& src, T* dst) {
  std::memcpy(dst, src.data(), src.size() * sizeof(T));
}

jagged::KernelOptions kopts(int threads, int64_t block) {
  jagged::KernelOptions o;
  o.block = block > 0 ? block : 64;
  o.threads = threads > 0 ? threads : 1;
  return o;
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}
}  // namespace

#define REF_T(T, SUF)                                                                              \
  extern "C" int ref_jagged_dense_bmm_##SUF(const int64_t* off, int64_t B, int64_t D, int64_t Tt, \
                                            const T* x, const T* w, int threads, T* out) {         \
    return guard([&] {                                                                             \
      auto r = jagged::jagged_dense_bmm(jt(off, B, D, x),                                          \
                                        jagged::DenseTensor<T>({B, D, Tt}, vec(w, B * D * Tt)),   \
                                        kopts(threads, 64));                                       \
      put(r.values(), out);                                                                        \
    });                                                                                            \
  }                                                                                                \
  extern "C" int ref_jagged_jagged_bmm_##SUF(const int64_t* off, int64_t B, int64_t D, int64_t Tt,\
                                             const T* x, const T* y, int threads, T* out) {        \
    return guard([&] {                                                                             \
      auto r = jagged::jagged_jagged_bmm(jt(off, B, D, x), jt(off, B, Tt, y), kopts(threads, 64)); \
      put(r.data(), out);                                                                          \
    });                                                                                            \
  }                                                                                                \
  extern "C" int ref_jagged_softmax_##SUF(const int64_t* off, int64_t B, int64_t D, const T* x,   \
                                          int threads, T* out) {                                   \
    return guard([&] { put(jagged::jagged_softmax(jt(off, B, D, x), kopts(threads, 64)).values(), out); }); \
  }                                                                                                \
  extern "C" int ref_jagged_jagged_bmm_jagged_out_##SUF(const int64_t* off, int64_t B, int64_t D,  \
                                                        const T* q, const T* k, int threads,       \
                                                        T* out) {                                  \
    return guard([&] {                                                                             \
      put(jagged::jagged_jagged_bmm_jagged_out(jt(off, B, D, q), jt(off, B, D, k),                \
                                               kopts(threads, 64)).values(), out);                 \
    });                                                                                            \
  }                                                                                                \
  extern "C" int ref_array_jagged_bmm_jagged_out_##SUF(const int64_t* off, int64_t B, int64_t D,   \
                                                       const T* a, const T* v, int threads,        \
                                                       T* out) {                                   \
    return guard([&] {                                                                             \
      put(jagged::array_jagged_bmm_jagged_out(j2(off, B, a), jt(off, B, D, v),                    \
                                              kopts(threads, 64)).values(), out);                  \
    });                                                                                            \
  }                                                                                                \
  extern "C" int ref_jagged2_softmax_##SUF(const int64_t* off, int64_t B, const T* s, int threads, \
                                           T* out) {                                               \
    return guard([&] { put(jagged::jagged2_softmax(j2(off, B, s), kopts(threads, 64)).values(), out); }); \
  }                                                                                                \
  extern "C" int ref_jagged_attention_##SUF(const int64_t* off, int64_t B, int64_t D, const T* q,  \
                                            const T* k, const T* v, int threads, T* out) {         \
    return guard([&] {                                                                             \
      put(jagged::jagged_attention(jt(off, B, D, q), jt(off, B, D, k), jt(off, B, D, v),          \
                                   kopts(threads, 64)).values(), out);                             \
    });                                                                                            \
  }                                                                                                \
  extern "C" int ref_jfa_forward_##SUF(const int64_t* off, int64_t B, int64_t D, const T* q,       \
                                       const T* k, const T* v, int64_t bq, int64_t bk,             \
                                       int threads, T* out, T* lse) {                              \
    return guard([&] {                                                                             \
      auto s = jagged::jagged_flash_attention_forward(jt(off, B, D, q), jt(off, B, D, k),         \
                                                      jt(off, B, D, v), bq, bk,                    \
                                                      kopts(threads, 64));                         \
      put(s.output.values(), out);                                                                 \
      put(s.logsumexp, lse);                                                                       \
    });                                                                                            \
  }                                                                                                \
  extern "C" int ref_jfa_backward_##SUF(const int64_t* off, int64_t B, int64_t D, const T* q,      \
                                        const T* k, const T* v, const T* go, const T* o,           \
                                        const T* lse, int64_t bq, int64_t bk, int threads, T* dq,  \
                                        T* dk, T* dv) {                                            \
    return guard([&] {                                                                             \
      jagged::JaggedAttentionSaved<T> saved{jt(off, B, D, o), vec(lse, off[B]), bq, bk};           \
      auto g = jagged::jagged_flash_attention_backward(jt(off, B, D, q), jt(off, B, D, k),        \
                                                       jt(off, B, D, v), jt(off, B, D, go), saved, \
                                                       kopts(threads, 64));                        \
      put(g.dq.values(), dq);                                                                      \
      put(g.dk.values(), dk);                                                                      \
      put(g.dv.values(), dv);                                                                      \
    });                                                                                            \
  }

REF_T(float, f32)
REF_T(double, f64)

// the reference's padded dense_flash_attention (attention.cpp:106-160) on [B, L, D] inputs.
#define REF_DENSE(T, SUF)                                                                                  \
  extern "C" int ref_dense_flash_attention_##SUF(const int64_t* lengths, int64_t B, int64_t L, int64_t D,  \
                                                 const T* q, const T* k, const T* v, int64_t bq,           \
                                                 int64_t bk, int threads, T* out, T* lse) {                \
    return guard([&] {                                                                                   \
      auto dt = [&](const T* p) { return jagged::DenseTensor<T>({B, L, D}, vec(p, B * L * D)); };        \
      const std::vector<int64_t> ln = vec(lengths, B);                                                   \
      auto s = jagged::dense_flash_attention(dt(q), dt(k), dt(v), std::span<const int64_t>(ln), bq, bk,  \
                                             kopts(threads, 64));                                        \
      put(s.output.data(), out);                                                                         \
      put(s.logsumexp, lse);                                                                             \
    });                                                                                                  \
  }
REF_DENSE(float, f32)
REF_DENSE(double, f64)

// VJPs: the reference's registry and gradcheck use the double instantiation. KernelOptions.threads for them
// (default 1, as the registry calls them) is set by ref_set_vjp_threads (scale parity tests run them threaded).
namespace {
int g_vjp_threads = 1;
jagged::KernelOptions vjp_opts() { return kopts(g_vjp_threads, 64); }
}  // namespace
extern "C" void ref_set_vjp_threads(int threads) { g_vjp_threads = threads > 0 ? threads : 1; }
extern "C" int ref_jagged_dense_bmm_vjp_f64(const int64_t* off, int64_t B, int64_t D, int64_t T,
                                            const double* x, const double* w, const double* go,
                                            double* dx, double* dw) {
  return guard([&] {
    auto g = jagged::jagged_dense_bmm_vjp(jt(off, B, D, x),
                                          jagged::DenseTensor<double>({B, D, T}, vec(w, B * D * T)),
                                          jt(off, B, T, go), vjp_opts());
    put(g.dx.values(), dx);
    put(g.dw.data(), dw);
  });
}
extern "C" int ref_jagged_jagged_bmm_vjp_f64(const int64_t* off, int64_t B, int64_t D, int64_t T,
                                             const double* x, const double* y, const double* go,
                                             double* dx, double* dy) {
  return guard([&] {
    auto g = jagged::jagged_jagged_bmm_vjp(jt(off, B, D, x), jt(off, B, T, y),
                                           jagged::DenseTensor<double>({B, D, T}, vec(go, B * D * T)), vjp_opts());
    put(g.dx.values(), dx);
    put(g.dy.values(), dy);
  });
}
extern "C" int ref_jagged_softmax_vjp_f64(const int64_t* off, int64_t B, int64_t D,
                                          const double* x, const double* go, double* dx) {
  return guard([&] { put(jagged::jagged_softmax_vjp(jt(off, B, D, x), jt(off, B, D, go), vjp_opts()).values(), dx); });
}
extern "C" int ref_jagged_jagged_bmm_jagged_out_vjp_f64(const int64_t* off, int64_t B, int64_t D,
                                                        const double* q, const double* k,
                                                        const double* go, double* dq, double* dk) {
  return guard([&] {
    auto g = jagged::jagged_jagged_bmm_jagged_out_vjp(jt(off, B, D, q), jt(off, B, D, k), j2(off, B, go),
                                                      vjp_opts());
    put(g.dq.values(), dq);
    put(g.dk.values(), dk);
  });
}
extern "C" int ref_array_jagged_bmm_jagged_out_vjp_f64(const int64_t* off, int64_t B, int64_t D,
                                                       const double* a, const double* v,
                                                       const double* go, double* da, double* dv) {
  return guard([&] {
    auto g = jagged::array_jagged_bmm_jagged_out_vjp(j2(off, B, a), jt(off, B, D, v), jt(off, B, D, go),
                                                     vjp_opts());
    put(g.da.values(), da);
    put(g.dv.values(), dv);
  });
}
extern "C" int ref_jagged2_softmax_vjp_f64(const int64_t* off, int64_t B, const double* s,
                                           const double* go, double* ds) {
  return guard([&] { put(jagged::jagged2_softmax_vjp(j2(off, B, s), j2(off, B, go), vjp_opts()).values(), ds); });
}

// feature_interaction (attention.cpp:291-309) and jagged_mlp (linalg.cpp:265-277,
// VJP :509-573) through the reference's own templates. MLP layers come in as dims[n+1], concatenated
// row-major weights and biases, and relu flags.
namespace {
template <typename T>
std::vector<jagged::MlpLayer<T>> mlp_layers(int n, const int64_t* dims, const T* w, const T* b, const int* relu) {
  std::vector<jagged::MlpLayer<T>> layers;
  int64_t wo = 0, bo = 0;
  for (int l = 0; l < n; ++l) {
    jagged::MlpLayer<T> L{jagged::DenseTensor<T>({dims[l], dims[l + 1]}, vec(w + wo, dims[l] * dims[l + 1])),
                          vec(b + bo, dims[l + 1]), relu[l] ? jagged::Activation::relu : jagged::Activation::none};
    layers.push_back(std::move(L));
    wo += dims[l] * dims[l + 1];
    bo += dims[l + 1];
  }
  return layers;
}
}  // namespace

#define REF_FI_MLP(T, SUF)                                                                              \
  extern "C" int ref_feature_interaction_##SUF(const int64_t* off, int64_t B, int64_t D, int64_t Tq,   \
                                                const T* k, const T* v, const T* tg, T* out) {          \
    return guard([&] {                                                                                  \
      auto r = jagged::feature_interaction(jt(off, B, D, k), jt(off, B, D, v),                          \
                                           jagged::DenseTensor<T>({B, Tq, D}, vec(tg, B * Tq * D)),     \
                                           kopts(1, 64));                                               \
      put(r.data(), out);                                                                               \
    });                                                                                                 \
  }                                                                                                     \
  extern "C" int ref_jagged_mlp_##SUF(int64_t rows, int n, const int64_t* dims, const T* w, const T* b, \
                                      const int* relu, const T* x, T* out) {                            \
    return guard([&] {                                                                                  \
      const int64_t off[2] = {0, rows};                                                                 \
      auto layers = mlp_layers<T>(n, dims, w, b, relu);                                                 \
      auto r = jagged::jagged_mlp(jt(off, 1, dims[0], x), std::span<const jagged::MlpLayer<T>>(layers)); \
      put(r.values(), out);                                                                             \
    });                                                                                                 \
  }
REF_FI_MLP(double, f64)
REF_FI_MLP(float, f32)

extern "C" int ref_jagged_mlp_vjp_f64(int64_t rows, int n, const int64_t* dims, const double* w, const double* b,
                                      const int* relu, const double* x, const double* go, double* dx, double* dw,
                                      double* db) {
  return guard([&] {
    const int64_t off[2] = {0, rows};
    auto layers = mlp_layers<double>(n, dims, w, b, relu);
    auto g = jagged::jagged_mlp_vjp(jt(off, 1, dims[0], x), std::span<const jagged::MlpLayer<double>>(layers),
                                    jt(off, 1, dims[n], go));
    put(g.dx.values(), dx);
    int64_t wo = 0, bo = 0;
    for (int l = 0; l < n; ++l) {
      put(g.dlayers[l].dweights.data(), dw + wo);
      put(g.dlayers[l].dbias, db + bo);
      wo += dims[l] * dims[l + 1];
      bo += dims[l + 1];
    }
  });
}

// Reference generators (rng.cpp) so the oracle's restated RNG can be pinned bit-exactly.
extern "C" int ref_gen_lengths(int kind, int64_t max_len, uint64_t seed, int64_t batch,
                               int64_t* out) {
  return guard([&] {
    jagged::LengthDistribution d;
    d.kind = kind == 0 ? jagged::LengthKind::fixed
                       : (kind == 1 ? jagged::LengthKind::uniform : jagged::LengthKind::half_mean);
    d.max_len = max_len;
    d.seed = seed;
    put(jagged::gen_lengths(d, batch), out);
  });
}
extern "C" int ref_uniform_values_f64(uint64_t seed, int64_t n, double lo, double hi, double* out) {
  return guard([&] {
    jagged::Rng r(seed);
    put(jagged::uniform_values<double>(r, n, lo, hi), out);
  });
}
extern "C" int ref_uniform_values_f32(uint64_t seed, int64_t n, double lo, double hi, float* out) {
  return guard([&] {
    jagged::Rng r(seed);
    put(jagged::uniform_values<float>(r, n, lo, hi), out);
  });
}
// A stateful reference generator: successive draws continue one jagged::Rng stream, as bench.cpp draws q, k, v
// (then grad_out) from Rng(seed + 1) one tensor after another (bench.cpp:323-329). Values are the reference's
// uniform_values<float> (rng.cpp:59-64), produced in bounded chunks.
extern "C" void* ref_rng_new(uint64_t seed) { return new jagged::Rng(seed); }
extern "C" void ref_rng_free(void* r) { delete static_cast<jagged::Rng*>(r); }
extern "C" int ref_rng_uniform_f32(void* r, int64_t n, double lo, double hi, float* out) {
  return guard([&] {
    auto& rng = *static_cast<jagged::Rng*>(r);
    constexpr int64_t kChunk = int64_t(1) << 24;
    for (int64_t i = 0; i < n; i += kChunk) {
      const int64_t m = n - i < kChunk ? n - i : kChunk;
      const auto v = jagged::uniform_values<float>(rng, m, lo, hi);
      std::memcpy(out + i, v.data(), m * sizeof(float));
    }
  });
}
extern "C" int ref_make_offsets(const int64_t* lengths, int64_t B, int64_t* offsets) {
  return guard([&] {
    auto x = jagged::make_jagged<double>(std::span<const int64_t>(lengths, B), std::vector<double>(
        [&] { int64_t s = 0; for (int64_t i = 0; i < B; ++i) s += lengths[i] > 0 ? lengths[i] : 0; return s; }()), 1);
    put(x.offsets(), offsets);
  });
}
extern "C" int ref_jagged_to_dense_f64(const int64_t* off, int64_t B, int64_t D, const double* x,
                                       int64_t L, double pad, double* out) {
  return guard([&] { put(jagged::jagged_to_dense(jt(off, B, D, x), L, pad).data(), out); });
}
extern "C" int ref_hardware_threads(void) {
  return static_cast<int>(std::thread::hardware_concurrency());
}
extern "C" const char* ref_last_error(void) { return g_err.c_str(); }

// the reference's analytic cost model (cost_model.cpp) and CSV header (bench.hpp:79-81), to pin
// paper_2409_15373_b200/report.py. out: flops (jagged, padded), bytes (jagged, padded), intermediate elements
// (jagged, padded), and — when `variant` is non-null — variant_flops, variant_bytes.
extern "C" int ref_cost_model(const char* op, const char* variant, const int64_t* lengths, int64_t B, int64_t D,
                              int64_t T, int64_t eb, int64_t padded_len, int64_t bq, int64_t bk, int64_t* out) {
  return guard([&] {
    jagged::OpConfig c;
    c.op_id = op;
    c.batch = B;
    c.dim = D;
    c.t = T;
    c.lengths = vec(lengths, B);
    c.element_bytes = eb;
    if (padded_len >= 0) c.padded_len = padded_len;
    c.block_q = bq;
    c.block_k = bk;
    const auto [fj, fp] = jagged::flops_of(c);
    const auto [bj, bp] = jagged::bytes_of(c);
    const auto [ij, ip] = jagged::intermediate_elements(c);
    out[0] = fj, out[1] = fp, out[2] = bj, out[3] = bp, out[4] = ij, out[5] = ip;
    if (variant) {
      out[6] = jagged::variant_flops(c, variant);
      out[7] = jagged::variant_bytes(c, variant);
    }
  });
}

extern "C" const char* ref_csv_header() { return jagged::bench::kCsvHeader.data(); }
