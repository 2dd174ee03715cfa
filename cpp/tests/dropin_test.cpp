// dropin_test.cpp — the reference's own API, linked against the B200 drop-in instead of linalg.o /
// attention.o. Written like the reference's tests (proj/tests/test_core.cpp style): build inputs with
// jagged::make_jagged / jagged::Rng, call the jagged:: operators, compare with independent binary64
// loops (cf. proj/tests/support/reference.hpp) and check the reference's exception texts.
// Exit code 0 = all checks passed. Run by tests/test_gpu_cpp_dropin.py on the GPU box.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "jagged/attention.hpp"
#include "jagged/linalg.hpp"
#include "jagged/rng.hpp"
#include "jagged/scratch.hpp"
#include "jagged/tensor.hpp"

using namespace jagged;

static int failures = 0;

static void check(bool ok, const std::string& what) {
  std::printf("%s %s\n", ok ? "OK  " : "FAIL", what.c_str());
  if (!ok) ++failures;
}

// norm-wise relative error of a float result against a binary64 expectation
static double rel(const std::vector<float>& got, const std::vector<double>& ref) {
  double num = 0, den = 0;
  for (size_t i = 0; i < ref.size(); ++i) {
    num += (got[i] - ref[i]) * (got[i] - ref[i]);
    den += ref[i] * ref[i];
  }
  return std::sqrt(num / (den > 0 ? den : 1));
}

template <typename F>
static bool throws_with(F&& f, const std::string& text) {
  try {
    f();
  } catch (const std::invalid_argument& e) {
    return std::string(e.what()).find(text) != std::string::npos;
  }
  return false;
}

int main() {
  const std::vector<int64_t> lengths = {0, 1, 2, 5, 7, 17, 33, 70, 130, 0, 257};
  const int64_t D = 64, T = 16, B = (int64_t)lengths.size();
  Rng rng(42);
  int64_t S = 0;
  for (auto n : lengths) S += n;
  auto x = make_jagged<float>(lengths, uniform_values<float>(rng, S * D, -1, 1), D);
  auto y = make_jagged<float>(lengths, uniform_values<float>(rng, S * D, -1, 1), D);
  auto v = make_jagged<float>(lengths, uniform_values<float>(rng, S * D, -1, 1), D);
  auto go = make_jagged<float>(lengths, uniform_values<float>(rng, S * D, -1, 1), D);
  DenseTensor<float> w({B, D, T}, uniform_values<float>(rng, B * D * T, -1, 1));
  const auto& off = x.offsets();

  // --- jagged_dense_bmm (linalg.cpp:34-68)
  {
    auto o = jagged_dense_bmm(x, w);
    std::vector<double> ref(S * T);
    for (int64_t i = 0; i < B; ++i)
      for (int64_t r = off[i]; r < off[i + 1]; ++r)
        for (int64_t t = 0; t < T; ++t) {
          double a = 0;
          for (int64_t d = 0; d < D; ++d) a += (double)x.row(r)[d] * w.at(i, d, t);
          ref[r * T + t] = a;
        }
    check(o.offsets() == off && rel(o.values(), ref) < 1e-5, "jagged_dense_bmm rel=" + std::to_string(rel(o.values(), ref)));
  }
  // --- jagged_softmax (linalg.cpp:98-120)
  {
    auto o = jagged_softmax(x);
    std::vector<double> ref(S * D);
    for (int64_t i = 0; i < B; ++i)
      for (int64_t d = 0; d < D; ++d) {
        double m = -INFINITY, s = 0;
        for (int64_t r = off[i]; r < off[i + 1]; ++r) m = std::max(m, (double)x.row(r)[d]);
        for (int64_t r = off[i]; r < off[i + 1]; ++r) s += std::exp(x.row(r)[d] - m);
        for (int64_t r = off[i]; r < off[i + 1]; ++r) ref[r * D + d] = std::exp(x.row(r)[d] - m) / s;
      }
    check(rel(o.values(), ref) < 1e-5, "jagged_softmax rel=" + std::to_string(rel(o.values(), ref)));
  }
  // --- flash attention fwd / bwd vs unfused jagged_attention and a binary64 loop
  {
    auto saved = jagged_flash_attention_forward(x, y, v, 64, 64);
    std::vector<double> ref(S * D), lse(S);
    const double sc = 1.0 / std::sqrt((double)D);
    for (int64_t i = 0; i < B; ++i)
      for (int64_t a = off[i]; a < off[i + 1]; ++a) {
        std::vector<double> s(off[i + 1] - off[i]);
        double m = -INFINITY, z = 0;
        for (int64_t c = off[i]; c < off[i + 1]; ++c) {
          double acc = 0;
          for (int64_t d = 0; d < D; ++d) acc += (double)x.row(a)[d] * y.row(c)[d];
          s[c - off[i]] = acc * sc;
          m = std::max(m, s[c - off[i]]);
        }
        for (auto& e : s) z += (e = std::exp(e - m));
        for (int64_t d = 0; d < D; ++d) {
          double acc = 0;
          for (int64_t c = off[i]; c < off[i + 1]; ++c) acc += s[c - off[i]] * v.row(c)[d];
          ref[a * D + d] = acc / z;
        }
        lse[a] = m + std::log(z);
      }
    check(rel(saved.output.values(), ref) < 1e-5,
          "jagged_flash_attention_forward rel=" + std::to_string(rel(saved.output.values(), ref)));
    check(rel(saved.logsumexp, lse) < 1e-6, "logsumexp rel=" + std::to_string(rel(saved.logsumexp, lse)));
    auto un = jagged_attention(x, y, v);
    check(rel(un.values(), ref) < 1e-5, "jagged_attention (unfused) rel=" + std::to_string(rel(un.values(), ref)));
    auto g = jagged_flash_attention_backward(x, y, v, go, saved);
    // dv = P^T dO check (attention.cpp:274-275)
    std::vector<double> dv(S * D, 0.0);
    for (int64_t i = 0; i < B; ++i)
      for (int64_t a = off[i]; a < off[i + 1]; ++a)
        for (int64_t c = off[i]; c < off[i + 1]; ++c) {
          double acc = 0;
          for (int64_t d = 0; d < D; ++d) acc += (double)x.row(a)[d] * y.row(c)[d];
          const double p = std::exp(acc * sc - lse[a]);
          for (int64_t d = 0; d < D; ++d) dv[c * D + d] += p * go.row(a)[d];
        }
    check(rel(g.dv.values(), dv) < 1e-5, "jagged_flash_attention_backward dv rel=" + std::to_string(rel(g.dv.values(), dv)));
    check(g.dq.offsets() == off && g.dk.offsets() == off, "gradients keep the input offsets");
    // SPEC.md:316/:520 peak-intermediate guard through KernelOptions.meter: the fused path never holds a
    // sum Bi^2 score buffer (peak <= block_q block_k + 2 sum_B D elements); the unfused path does
    int64_t sum_sq = 0;
    for (auto n : lengths) sum_sq += n * n;
    ScratchMeter meter;
    KernelOptions mo;
    mo.meter = &meter;
    auto s2 = jagged_flash_attention_forward(x, y, v, 64, 64, mo);
    auto g2 = jagged_flash_attention_backward(x, y, v, go, s2, mo);
    const int64_t flash_peak = meter.peak();
    check(flash_peak <= 64 * 64 + 2 * S * D && meter.current() == 0,
          "meter: flash peak " + std::to_string(flash_peak) + " <= " + std::to_string(64 * 64 + 2 * S * D));
    meter.reset();
    auto un2 = jagged_attention(x, y, v, mo);
    check(meter.peak() >= sum_sq && meter.current() == 0,
          "meter: unfused peak " + std::to_string(meter.peak()) + " >= sum Bi^2 " + std::to_string(sum_sq));
    std::printf("meter: flash fwd+bwd peak %lld elements, unfused jagged_attention %lld (sum Bi^2 = %lld)\n",
                (long long)flash_peak, (long long)meter.peak(), (long long)sum_sq);
  }
  // --- feature_interaction composition (attention.cpp:291-309) runs end to end
  {
    DenseTensor<float> targets({B, 3, D}, uniform_values<float>(rng, B * 3 * D, -1, 1));
    auto fi = feature_interaction(x, v, targets);
    check(fi.shape() == std::vector<int64_t>({B, 3, D}), "feature_interaction shape");
  }
  // --- dense_flash_attention (attention.cpp:106-160) in the GPU padded mode: valid rows equal the jagged
  // attention of the truncated samples, padded rows are zero with lse = -inf
  {
    const int64_t L = 40, Bd = 4;
    const std::vector<int64_t> dl = {7, 0, 40, 19};
    DenseTensor<float> dq({Bd, L, D}, uniform_values<float>(rng, Bd * L * D, -1, 1));
    DenseTensor<float> dk({Bd, L, D}, uniform_values<float>(rng, Bd * L * D, -1, 1));
    DenseTensor<float> dvv({Bd, L, D}, uniform_values<float>(rng, Bd * L * D, -1, 1));
    auto ds = dense_flash_attention(dq, dk, dvv, std::span<const int64_t>(dl), 16, 16);
    double worst = 0.0;
    bool pad_ok = true;
    for (int64_t i = 0; i < Bd; ++i)
      for (int64_t a = 0; a < L; ++a) {
        if (a >= dl[i]) {
          for (int64_t d = 0; d < D; ++d) pad_ok = pad_ok && ds.output.at(i, a, d) == 0.f;
          pad_ok = pad_ok && std::isinf(ds.logsumexp[i * L + a]) && ds.logsumexp[i * L + a] < 0;
          continue;
        }
        std::vector<double> sc(dl[i]);
        double m = -1e300, sum = 0.0;
        for (int64_t c = 0; c < dl[i]; ++c) {
          double acc = 0.0;
          for (int64_t d = 0; d < D; ++d) acc += (double)dq.at(i, a, d) * dk.at(i, c, d);
          sc[c] = acc / std::sqrt((double)D);
          m = std::max(m, sc[c]);
        }
        for (int64_t c = 0; c < dl[i]; ++c) sum += std::exp(sc[c] - m);
        for (int64_t d = 0; d < D; ++d) {
          double o = 0.0;
          for (int64_t c = 0; c < dl[i]; ++c) o += std::exp(sc[c] - m) / sum * dvv.at(i, c, d);
          worst = std::max(worst, std::fabs(o - ds.output.at(i, a, d)));
        }
      }
    check(worst < 1e-5 && pad_ok, "dense_flash_attention max err=" + std::to_string(worst));
    const std::vector<int64_t> bad = {7, 0, 41, 19};
    check(throws_with([&] { dense_flash_attention(dq, dk, dvv, std::span<const int64_t>(bad), 16, 16); },
                      "dense_flash_attention: sample 2 length 41 out of bounds for L=40"),
          "error: dense_flash_attention length bounds");
  }
  // --- jagged_mlp forward + VJP (linalg.cpp:246-277, :509-573) against a host binary64 restatement
  {
    const int64_t H1 = 24, O = 8;
    MlpLayer<float> l0{DenseTensor<float>({D, H1}, uniform_values<float>(rng, D * H1, -0.3, 0.3)),
                       uniform_values<float>(rng, H1, -0.1, 0.1), Activation::relu};
    MlpLayer<float> l1{DenseTensor<float>({H1, O}, uniform_values<float>(rng, H1 * O, -0.3, 0.3)),
                       uniform_values<float>(rng, O, -0.1, 0.1), Activation::none};
    std::vector<MlpLayer<float>> layers{l0, l1};
    auto y_mlp = jagged_mlp(x, std::span<const MlpLayer<float>>(layers));
    std::vector<double> h(S * H1), pre(S * H1), outr(S * O);
    for (int64_t r = 0; r < S; ++r) {
      for (int64_t o = 0; o < H1; ++o) {
        double acc = l0.bias[o];
        for (int64_t i = 0; i < D; ++i) acc += (double)x.row(r)[i] * l0.weights.at(i, o);
        pre[r * H1 + o] = acc;
        h[r * H1 + o] = acc > 0 ? acc : 0;
      }
      for (int64_t o = 0; o < O; ++o) {
        double acc = l1.bias[o];
        for (int64_t i = 0; i < H1; ++i) acc += h[r * H1 + i] * l1.weights.at(i, o);
        outr[r * O + o] = acc;
      }
    }
    check(rel(y_mlp.values(), outr) < 1e-5, "jagged_mlp rel=" + std::to_string(rel(y_mlp.values(), outr)));
    auto gout = make_jagged<float>(lengths, uniform_values<float>(rng, S * O, -1, 1), O);
    auto g = jagged_mlp_vjp(x, std::span<const MlpLayer<float>>(layers), gout);
    std::vector<double> db1(O, 0.0);
    for (int64_t r = 0; r < S; ++r)
      for (int64_t o = 0; o < O; ++o) db1[o] += gout.row(r)[o];
    check(rel(g.dlayers[1].dbias, db1) < 1e-5, "jagged_mlp_vjp db rel=" + std::to_string(rel(g.dlayers[1].dbias, db1)));
    check(g.dx.dim() == D && g.dlayers[0].dweights.shape() == std::vector<int64_t>({D, H1}), "jagged_mlp_vjp shapes");
    check(throws_with([&] { jagged_mlp(x, std::span<const MlpLayer<float>>()); }, "at least one layer required"),
          "error: at least one layer required");
  }
  // --- reference exception texts
  check(throws_with([&] { jagged_dense_bmm(x, DenseTensor<float>({B, D}, std::vector<float>(B * D))); },
                    "jagged_dense_bmm: w must be [B, D, T]"),
        "error: w must be [B, D, T]");
  check(throws_with([&] { jagged_flash_attention_forward(x, y, v, 0, 64); }, "block sizes must be >= 1"),
        "error: block sizes must be >= 1");
  {
    std::vector<int64_t> l2 = lengths;
    std::swap(l2[1], l2[2]);
    auto z = make_jagged<float>(l2, std::vector<float>(S * D, 0.f), D);
    check(throws_with([&] { jagged_jagged_bmm(x, z); }, "jagged_jagged_bmm: offsets differ first at sample 1"),
          "error: offsets differ first at sample 1");
    check(throws_with([&] { jagged_flash_attention_forward(x, z, v, 64, 64); }, "q, k, v must share offsets"),
          "error: q, k, v must share offsets");
  }
  {
    auto xd = make_jagged<double>(lengths, std::vector<double>(S * D, 0.0), D);
    check(throws_with([&] { jagged_softmax(xd); }, "no B200 device path"), "binary64 reports no device path");
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "PASSED", failures);
  return failures ? 1 : 0;
}
