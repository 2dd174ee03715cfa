/*
 * jagged_oracle.c — CPU restatement of the reference jagged operators (TEST INFRASTRUCTURE ONLY).
 *
 * Not product code: the product path (paper_2409_15373_b200/) never links or calls this file;
 * it is the checker used by tests/, __graft_entry__.smoke() and bench.py's CPU legs.
 * Each function cites the /root/reference/proj/core file:line whose loop nest it restates.
 * Arithmetic follows the reference: products and sums in binary64, reduction order ascending
 * over the contracted index, exp/log from libm.
 */
#include "jagged_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];
const char* or_last_error(void) { return g_err; }
static int fail(const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return 1;
}

#define LEN(off, i) ((off)[(i) + 1] - (off)[(i)])

/* ------------------------------------------------------------------------------------------ */
/* RNG: std::mt19937_64 (the standard pins its output), modulo-method bounded ints and a      */
/* 53-bit real (rng.hpp:10-28, rng.cpp:7-17).                                                  */
/* ------------------------------------------------------------------------------------------ */
void or_rng_seed(or_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

uint64_t or_rng_next(or_rng* r) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* rng.cpp:7-12 */
int64_t or_rng_uniform_int(or_rng* r, int64_t lo, int64_t hi) {
  const uint64_t span = (uint64_t)(hi - lo) + 1;
  if (span == 0) return (int64_t)or_rng_next(r);
  return lo + (int64_t)(or_rng_next(r) % span);
}

/* rng.cpp:14-17 */
double or_rng_uniform_real(or_rng* r, double lo, double hi) {
  const double unit = (double)(or_rng_next(r) >> 11) * 0x1.0p-53;
  return lo + unit * (hi - lo);
}

/* rng.cpp:35-57 (kinds 0..2). Kind 3 is the Zipf generator SURVEY.md §8(d) defines for
 * configs 2 and 5: P(k) ∝ k^-alpha on {1..max_len}, u = Rng(seed).uniform_real(0,1) per
 * sample, length = 1 + lower_bound(cdf, u). Not part of the reference. */
int or_gen_lengths(int kind, int64_t max_len, uint64_t seed, int64_t batch, double zipf_alpha,
                   int64_t* out) {
  if (batch < 1) return fail("gen_lengths: batch must be >= 1");
  if (max_len < 1) return fail("gen_lengths: max_len must be >= 1");
  or_rng r;
  or_rng_seed(&r, seed);
  if (kind == 0) {
    for (int64_t i = 0; i < batch; ++i) out[i] = max_len;
  } else if (kind == 1) {
    for (int64_t i = 0; i < batch; ++i) out[i] = or_rng_uniform_int(&r, 1, max_len);
  } else if (kind == 2) {
    for (int64_t i = 0; i + 1 < batch; i += 2) {
      const int64_t u = or_rng_uniform_int(&r, 0, max_len);
      out[i] = u;
      out[i + 1] = max_len - u;
    }
    if (batch % 2 == 1) out[batch - 1] = or_rng_uniform_int(&r, 0, max_len);
  } else if (kind == 3) {
    double* cdf = (double*)malloc(sizeof(double) * (size_t)max_len);
    double tot = 0.0;
    for (int64_t k = 1; k <= max_len; ++k) {
      tot += pow((double)k, -zipf_alpha);
      cdf[k - 1] = tot;
    }
    for (int64_t k = 0; k < max_len; ++k) cdf[k] /= tot;
    cdf[max_len - 1] = 1.0;
    for (int64_t i = 0; i < batch; ++i) {
      const double u = or_rng_uniform_real(&r, 0.0, 1.0);
      int64_t lo = 0, hi = max_len; /* lower_bound: first index with cdf >= u */
      while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (cdf[mid] < u) lo = mid + 1; else hi = mid;
      }
      out[i] = lo + 1;
    }
    free(cdf);
  } else {
    return fail("unknown length distribution");
  }
  return 0;
}

/* rng.cpp:59-64; as_float rounds each draw to binary32 like uniform_values<float>. */
void or_uniform_values(or_rng* r, int64_t n, double lo, double hi, int as_float, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    const double v = or_rng_uniform_real(r, lo, hi);
    out[i] = as_float ? (double)(float)v : v;
  }
}

/* ------------------------------------------------------------------------------------------ */
/* Offsets and layout conversions (tensor.cpp:72-175)                                          */
/* ------------------------------------------------------------------------------------------ */
/* tensor.cpp:72-87 */
int or_make_offsets(const int64_t* lengths, int64_t batch, int64_t* offsets) {
  offsets[0] = 0;
  for (int64_t i = 0; i < batch; ++i) {
    if (lengths[i] < 0) {
      snprintf(g_err, sizeof g_err, "make_jagged: negative length at sample %lld", (long long)i);
      return 1;
    }
    offsets[i + 1] = offsets[i] + lengths[i];
  }
  return 0;
}

/* tensor.cpp:40-48 (Jagged2Tensor ctor) */
int or_sq_offsets(const int64_t* off, int64_t batch, int64_t* sq) {
  sq[0] = 0;
  for (int64_t i = 0; i < batch; ++i) sq[i + 1] = sq[i] + LEN(off, i) * LEN(off, i);
  return 0;
}

int64_t or_sum_sq(const int64_t* off, int64_t B) {
  int64_t s = 0;
  for (int64_t i = 0; i < B; ++i) s += LEN(off, i) * LEN(off, i);
  return s;
}

/* tensor.cpp:102-116: pad to [B,L,D], truncating segments longer than L */
int or_jagged_to_dense(const int64_t* off, int64_t batch, int64_t dim, const double* x,
                       int64_t max_len, double pad, double* out) {
  if (max_len < 0) return fail("jagged_to_dense: max_len must be >= 0");
  for (int64_t e = 0; e < batch * max_len * dim; ++e) out[e] = pad;
  for (int64_t i = 0; i < batch; ++i) {
    int64_t n = LEN(off, i);
    if (n > max_len) n = max_len;
    memcpy(out + i * max_len * dim, x + off[i] * dim, sizeof(double) * (size_t)(n * dim));
  }
  return 0;
}

/* tensor.cpp:118-139 */
int or_dense_to_jagged(const double* d, int64_t batch, int64_t max_len, int64_t dim,
                       const int64_t* lengths, double* out) {
  int64_t r = 0;
  for (int64_t i = 0; i < batch; ++i) {
    if (lengths[i] > max_len) {
      snprintf(g_err, sizeof g_err, "dense_to_jagged: sample %lld length %lld exceeds max_len %lld",
               (long long)i, (long long)lengths[i], (long long)max_len);
      return 1;
    }
  }
  for (int64_t i = 0; i < batch; ++i) {
    memcpy(out + r * dim, d + i * max_len * dim, sizeof(double) * (size_t)(lengths[i] * dim));
    r += lengths[i];
  }
  return 0;
}

/* tensor.cpp:141-155 */
int or_jagged2_to_dense(const int64_t* off, int64_t batch, const double* s, int64_t max_len,
                        double pad, double* out) {
  if (max_len < 0) return fail("jagged2_to_dense: max_len must be >= 0");
  for (int64_t e = 0; e < batch * max_len * max_len; ++e) out[e] = pad;
  int64_t sq = 0;
  for (int64_t i = 0; i < batch; ++i) {
    const int64_t bi = LEN(off, i);
    const int64_t n = bi < max_len ? bi : max_len;
    for (int64_t r = 0; r < n; ++r)
      for (int64_t c = 0; c < n; ++c) out[(i * max_len + r) * max_len + c] = s[sq + r * bi + c];
    sq += bi * bi;
  }
  return 0;
}

/* tensor.cpp:157-175 */
int or_dense_to_jagged2(const double* d, int64_t batch, int64_t max_len, const int64_t* lengths,
                        double* out) {
  int64_t e = 0;
  for (int64_t i = 0; i < batch; ++i) {
    const int64_t n = lengths[i];
    if (n > max_len) {
      snprintf(g_err, sizeof g_err, "dense_to_jagged2: sample %lld length %lld exceeds max_len %lld",
               (long long)i, (long long)n, (long long)max_len);
      return 1;
    }
    for (int64_t r = 0; r < n; ++r)
      for (int64_t c = 0; c < n; ++c) out[e++] = d[(i * max_len + r) * max_len + c];
  }
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* Table-1 forward operators                                                                   */
/* ------------------------------------------------------------------------------------------ */
/* linalg.cpp:34-68: O_i = X_i W_i, w is [B,D,T] */
int or_jagged_dense_bmm(const int64_t* off, int64_t B, int64_t D, int64_t T, const double* x,
                        const double* w, double* out) {
  for (int64_t i = 0; i < B; ++i)
    for (int64_t r = off[i]; r < off[i + 1]; ++r)
      for (int64_t t = 0; t < T; ++t) {
        double acc = 0.0;
        for (int64_t d = 0; d < D; ++d) acc += x[r * D + d] * w[(i * D + d) * T + t];
        out[r * T + t] = acc;
      }
  return 0;
}

/* linalg.cpp:70-96: Z_i = X_i^T Y_i, zero for empty samples */
int or_jagged_jagged_bmm(const int64_t* off, int64_t B, int64_t D, int64_t T, const double* x,
                         const double* y, double* out) {
  for (int64_t i = 0; i < B; ++i)
    for (int64_t d = 0; d < D; ++d)
      for (int64_t t = 0; t < T; ++t) {
        double acc = 0.0;
        for (int64_t r = off[i]; r < off[i + 1]; ++r) acc += x[r * D + d] * y[r * T + t];
        out[(i * D + d) * T + t] = acc;
      }
  return 0;
}

/* linalg.cpp:98-120: softmax over each segment's rows, per column (three passes) */
int or_jagged_softmax(const int64_t* off, int64_t B, int64_t D, const double* x, double* out) {
  for (int64_t i = 0; i < B; ++i) {
    const int64_t b0 = off[i], b1 = off[i + 1];
    if (b0 == b1) continue;
    for (int64_t d = 0; d < D; ++d) {
      double m = -INFINITY, sum = 0.0;
      for (int64_t r = b0; r < b1; ++r) m = fmax(m, x[r * D + d]);
      for (int64_t r = b0; r < b1; ++r) sum += exp(x[r * D + d] - m);
      for (int64_t r = b0; r < b1; ++r) out[r * D + d] = exp(x[r * D + d] - m) / sum;
    }
  }
  return 0;
}

/* linalg.cpp:122-159: S_i = Q_i K_i^T stored as row-major Bi x Bi blocks at sq_offsets[i] */
int or_jagged_jagged_bmm_jagged_out(const int64_t* off, int64_t B, int64_t D, const double* q,
                                    const double* k, double* out) {
  int64_t sq = 0;
  for (int64_t i = 0; i < B; ++i) {
    const int64_t n = LEN(off, i), b0 = off[i];
    for (int64_t r = 0; r < n; ++r)
      for (int64_t c = 0; c < n; ++c) {
        double acc = 0.0;
        for (int64_t d = 0; d < D; ++d) acc += q[(b0 + r) * D + d] * k[(b0 + c) * D + d];
        out[sq + r * n + c] = acc;
      }
    sq += n * n;
  }
  return 0;
}

/* linalg.cpp:161-197: O_i = A_i V_i */
int or_array_jagged_bmm_jagged_out(const int64_t* off, int64_t B, int64_t D, const double* a,
                                   const double* v, double* out) {
  int64_t sq = 0;
  for (int64_t i = 0; i < B; ++i) {
    const int64_t n = LEN(off, i), b0 = off[i];
    for (int64_t r = 0; r < n; ++r)
      for (int64_t d = 0; d < D; ++d) {
        double acc = 0.0;
        for (int64_t c = 0; c < n; ++c) acc += a[sq + r * n + c] * v[(b0 + c) * D + d];
        out[(b0 + r) * D + d] = acc;
      }
    sq += n * n;
  }
  return 0;
}

/* linalg.cpp:199-220: row softmax inside each block */
int or_jagged2_softmax(const int64_t* off, int64_t B, const double* s, double* out) {
  int64_t sq = 0;
  for (int64_t i = 0; i < B; ++i) {
    const int64_t n = LEN(off, i);
    for (int64_t r = 0; r < n; ++r) {
      const double* row = s + sq + r * n;
      double m = -INFINITY, sum = 0.0;
      for (int64_t c = 0; c < n; ++c) m = fmax(m, row[c]);
      for (int64_t c = 0; c < n; ++c) sum += exp(row[c] - m);
      for (int64_t c = 0; c < n; ++c) out[sq + r * n + c] = exp(row[c] - m) / sum;
    }
    sq += n * n;
  }
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* VJPs                                                                                        */
/* ------------------------------------------------------------------------------------------ */
/* linalg.cpp:283-318: dX = dO W^T, dW = X^T dO */
int or_jagged_dense_bmm_vjp(const int64_t* off, int64_t B, int64_t D, int64_t T, const double* x,
                            const double* w, const double* go, double* dx, double* dw) {
  for (int64_t i = 0; i < B; ++i) {
    for (int64_t r = off[i]; r < off[i + 1]; ++r)
      for (int64_t d = 0; d < D; ++d) {
        double acc = 0.0;
        for (int64_t t = 0; t < T; ++t) acc += go[r * T + t] * w[(i * D + d) * T + t];
        dx[r * D + d] = acc;
      }
    for (int64_t d = 0; d < D; ++d)
      for (int64_t t = 0; t < T; ++t) {
        double acc = 0.0;
        for (int64_t r = off[i]; r < off[i + 1]; ++r) acc += x[r * D + d] * go[r * T + t];
        dw[(i * D + d) * T + t] = acc;
      }
  }
  return 0;
}

/* linalg.cpp:320-353: dX = Y dZ^T, dY = X dZ */
int or_jagged_jagged_bmm_vjp(const int64_t* off, int64_t B, int64_t D, int64_t T, const double* x,
                             const double* y, const double* go, double* dx, double* dy) {
  for (int64_t i = 0; i < B; ++i)
    for (int64_t r = off[i]; r < off[i + 1]; ++r) {
      for (int64_t d = 0; d < D; ++d) {
        double acc = 0.0;
        for (int64_t t = 0; t < T; ++t) acc += y[r * T + t] * go[(i * D + d) * T + t];
        dx[r * D + d] = acc;
      }
      for (int64_t t = 0; t < T; ++t) {
        double acc = 0.0;
        for (int64_t d = 0; d < D; ++d) acc += x[r * D + d] * go[(i * D + d) * T + t];
        dy[r * T + t] = acc;
      }
    }
  return 0;
}

/* linalg.cpp:355-388: dx = p (dp - sum_rows(dp p)), p recomputed from x */
int or_jagged_softmax_vjp(const int64_t* off, int64_t B, int64_t D, const double* x,
                          const double* go, double* dx) {
  for (int64_t i = 0; i < B; ++i) {
    const int64_t b0 = off[i], b1 = off[i + 1];
    if (b0 == b1) continue;
    for (int64_t d = 0; d < D; ++d) {
      double m = -INFINITY, sum = 0.0, dot = 0.0;
      for (int64_t r = b0; r < b1; ++r) m = fmax(m, x[r * D + d]);
      for (int64_t r = b0; r < b1; ++r) sum += exp(x[r * D + d] - m);
      for (int64_t r = b0; r < b1; ++r) dot += go[r * D + d] * (exp(x[r * D + d] - m) / sum);
      for (int64_t r = b0; r < b1; ++r) {
        const double p = exp(x[r * D + d] - m) / sum;
        dx[r * D + d] = p * (go[r * D + d] - dot);
      }
    }
  }
  return 0;
}

/* linalg.cpp:390-430: dQ = dS K, dK = dS^T Q */
int or_jagged_jagged_bmm_jagged_out_vjp(const int64_t* off, int64_t B, int64_t D, const double* q,
                                        const double* k, const double* go, double* dq,
                                        double* dk) {
  int64_t sq = 0;
  for (int64_t i = 0; i < B; ++i) {
    const int64_t n = LEN(off, i), b0 = off[i];
    const double* ds = go + sq;
    for (int64_t r = 0; r < n; ++r)
      for (int64_t d = 0; d < D; ++d) {
        double acc = 0.0;
        for (int64_t c = 0; c < n; ++c) acc += ds[r * n + c] * k[(b0 + c) * D + d];
        dq[(b0 + r) * D + d] = acc;
      }
    for (int64_t c = 0; c < n; ++c)
      for (int64_t d = 0; d < D; ++d) {
        double acc = 0.0;
        for (int64_t r = 0; r < n; ++r) acc += ds[r * n + c] * q[(b0 + r) * D + d];
        dk[(b0 + c) * D + d] = acc;
      }
    sq += n * n;
  }
  return 0;
}

/* linalg.cpp:432-472: dA = dO V^T, dV = A^T dO */
int or_array_jagged_bmm_jagged_out_vjp(const int64_t* off, int64_t B, int64_t D, const double* a,
                                       const double* v, const double* go, double* da,
                                       double* dv) {
  int64_t sq = 0;
  for (int64_t i = 0; i < B; ++i) {
    const int64_t n = LEN(off, i), b0 = off[i];
    for (int64_t r = 0; r < n; ++r)
      for (int64_t c = 0; c < n; ++c) {
        double acc = 0.0;
        for (int64_t d = 0; d < D; ++d) acc += go[(b0 + r) * D + d] * v[(b0 + c) * D + d];
        da[sq + r * n + c] = acc;
      }
    for (int64_t c = 0; c < n; ++c)
      for (int64_t d = 0; d < D; ++d) {
        double acc = 0.0;
        for (int64_t r = 0; r < n; ++r) acc += a[sq + r * n + c] * go[(b0 + r) * D + d];
        dv[(b0 + c) * D + d] = acc;
      }
    sq += n * n;
  }
  return 0;
}

/* linalg.cpp:474-507 */
int or_jagged2_softmax_vjp(const int64_t* off, int64_t B, const double* s, const double* go,
                           double* ds) {
  int64_t sq = 0;
  for (int64_t i = 0; i < B; ++i) {
    const int64_t n = LEN(off, i);
    for (int64_t r = 0; r < n; ++r) {
      const double* row = s + sq + r * n;
      const double* g = go + sq + r * n;
      double m = -INFINITY, sum = 0.0, dot = 0.0;
      for (int64_t c = 0; c < n; ++c) m = fmax(m, row[c]);
      for (int64_t c = 0; c < n; ++c) sum += exp(row[c] - m);
      for (int64_t c = 0; c < n; ++c) dot += g[c] * (exp(row[c] - m) / sum);
      for (int64_t c = 0; c < n; ++c) ds[sq + r * n + c] = (exp(row[c] - m) / sum) * (g[c] - dot);
    }
    sq += n * n;
  }
  return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* Attention                                                                                   */
/* ------------------------------------------------------------------------------------------ */
static double dot_rows(const double* a, const double* b, int64_t d) {
  double acc = 0.0;
  for (int64_t i = 0; i < d; ++i) acc += a[i] * b[i];
  return acc;
}

/* attention.cpp:162-170: jjbmm_jout -> scale(1/sqrt D) -> jagged2_softmax -> ajbmm_jout */
int or_jagged_attention(const int64_t* off, int64_t B, int64_t D, const double* q, const double* k,
                        const double* v, double* out) {
  const int64_t n2 = or_sum_sq(off, B);
  double* s = (double*)malloc(sizeof(double) * (size_t)(n2 > 0 ? n2 : 1));
  double* p = (double*)malloc(sizeof(double) * (size_t)(n2 > 0 ? n2 : 1));
  const double inv = 1.0 / sqrt((double)D);
  or_jagged_jagged_bmm_jagged_out(off, B, D, q, k, s);
  for (int64_t e = 0; e < n2; ++e) s[e] *= inv;
  or_jagged2_softmax(off, B, s, p);
  or_array_jagged_bmm_jagged_out(off, B, D, p, v, out);
  free(s);
  free(p);
  return 0;
}

/* attention.cpp:172-225: per-segment streaming online softmax. Empty segments write nothing
 * (callers pre-fill out with 0 and lse with -inf, attention.cpp:183-184). */
int or_jfa_forward(const int64_t* off, int64_t B, int64_t D, const double* q, const double* k,
                   const double* v, int64_t block_q, int64_t block_k, double* out, double* lse) {
  if (block_q < 1 || block_k < 1)
    return fail("jagged_flash_attention_forward: block sizes must be >= 1");
  const double inv = 1.0 / sqrt((double)D);
  double* acc = (double*)malloc(sizeof(double) * (size_t)D);
  double* srow = (double*)malloc(sizeof(double) * (size_t)block_k);
  for (int64_t e = 0; e < off[B]; ++e) lse[e] = -INFINITY;
  for (int64_t e = 0; e < off[B] * D; ++e) out[e] = 0.0;
  for (int64_t i = 0; i < B; ++i) {
    const int64_t b0 = off[i], n = LEN(off, i);
    for (int64_t a = 0; a < n; ++a) {
      const double* qr = q + (b0 + a) * D;
      double m = -INFINITY, sum = 0.0;
      for (int64_t d = 0; d < D; ++d) acc[d] = 0.0;
      for (int64_t c0 = 0; c0 < n; c0 += block_k) {
        const int64_t c1 = c0 + block_k < n ? c0 + block_k : n;
        double bmax = -INFINITY;
        for (int64_t c = c0; c < c1; ++c) {
          srow[c - c0] = dot_rows(qr, k + (b0 + c) * D, D) * inv;
          bmax = fmax(bmax, srow[c - c0]);
        }
        const double m_new = fmax(m, bmax);
        const double rescale = (m == -INFINITY) ? 0.0 : exp(m - m_new);
        sum *= rescale;
        for (int64_t d = 0; d < D; ++d) acc[d] *= rescale;
        for (int64_t c = c0; c < c1; ++c) {
          const double p = exp(srow[c - c0] - m_new);
          sum += p;
          const double* vr = v + (b0 + c) * D;
          for (int64_t d = 0; d < D; ++d) acc[d] += p * vr[d];
        }
        m = m_new;
      }
      for (int64_t d = 0; d < D; ++d) out[(b0 + a) * D + d] = acc[d] / sum;
      lse[b0 + a] = m + log(sum);
    }
  }
  free(acc);
  free(srow);
  return 0;
}

/* attention.cpp:227-289: recompute P from (q, k, lse); queries processed sequentially per
 * segment so the dK/dV accumulation order is fixed. */
int or_jfa_backward(const int64_t* off, int64_t B, int64_t D, const double* q, const double* k,
                    const double* v, const double* go, const double* out, const double* lse,
                    int64_t block_k, double* dq, double* dk, double* dv) {
  if (block_k < 1) return fail("jagged_flash_attention_backward: saved state does not match inputs");
  const double inv = 1.0 / sqrt((double)D);
  double* dqr = (double*)malloc(sizeof(double) * (size_t)D);
  for (int64_t e = 0; e < off[B] * D; ++e) dq[e] = dk[e] = dv[e] = 0.0;
  for (int64_t i = 0; i < B; ++i) {
    const int64_t b0 = off[i], n = LEN(off, i);
    for (int64_t a = 0; a < n; ++a) {
      const double* qr = q + (b0 + a) * D;
      const double* gr = go + (b0 + a) * D;
      const double l = lse[b0 + a];
      const double delta = dot_rows(gr, out + (b0 + a) * D, D);
      for (int64_t d = 0; d < D; ++d) dqr[d] = 0.0;
      for (int64_t c = 0; c < n; ++c) {
        const double* kr = k + (b0 + c) * D;
        const double* vr = v + (b0 + c) * D;
        const double s = dot_rows(qr, kr, D) * inv;
        const double p = exp(s - l);
        const double dp = dot_rows(gr, vr, D);
        const double dsv = p * (dp - delta);
        for (int64_t d = 0; d < D; ++d) {
          dv[(b0 + c) * D + d] += p * gr[d];
          dqr[d] += dsv * kr[d] * inv;
          dk[(b0 + c) * D + d] += dsv * qr[d] * inv;
        }
      }
      for (int64_t d = 0; d < D; ++d) dq[(b0 + a) * D + d] = dqr[d];
    }
  }
  free(dqr);
  return 0;
}

/* attention.cpp:62-104: padded dense attention with the full L x L masked score matrix. */
int or_dense_attention(const int64_t* lengths, int64_t B, int64_t L, int64_t D, const double* q,
                       const double* k, const double* v, double* out) {
  const double inv = 1.0 / sqrt((double)D);
  double* sc = (double*)malloc(sizeof(double) * (size_t)(L > 0 ? L : 1));
  for (int64_t e = 0; e < B * L * D; ++e) out[e] = 0.0;
  for (int64_t i = 0; i < B; ++i) {
    const int64_t n = lengths[i];
    for (int64_t a = 0; a < n; ++a) {
      double m = -INFINITY, sum = 0.0;
      for (int64_t c = 0; c < L; ++c) {
        sc[c] = c < n ? dot_rows(q + (i * L + a) * D, k + (i * L + c) * D, D) * inv : -INFINITY;
        m = fmax(m, sc[c]);
      }
      for (int64_t c = 0; c < L; ++c) {
        sc[c] = exp(sc[c] - m);
        sum += sc[c];
      }
      for (int64_t c = 0; c < L; ++c) sc[c] /= sum;
      for (int64_t d = 0; d < D; ++d) {
        double acc = 0.0;
        for (int64_t c = 0; c < L; ++c) acc += sc[c] * v[(i * L + c) * D + d];
        out[(i * L + a) * D + d] = acc;
      }
    }
  }
  free(sc);
  return 0;
}

/* attention.cpp:106-160: padded dense flash attention. Streams each padded row over key blocks of
 * block_k with an online softmax; scores with a >= n or c >= n are -inf (:130), a block with no valid score
 * yet is skipped (:134), rows with no valid key keep out = 0 and lse = -inf (:151-154). lse: B*L entries. */
int or_dense_flash_attention(const int64_t* lengths, int64_t B, int64_t L, int64_t D, int64_t block_q,
                             int64_t block_k, const double* q, const double* k, const double* v, double* out,
                             double* lse) {
  if (block_q < 1 || block_k < 1) return -1;
  const double inv = 1.0 / sqrt((double)D);
  const int64_t bk = block_k < L ? block_k : L;
  double* row = (double*)malloc(sizeof(double) * (size_t)(bk > 0 ? bk : 1));
  double* acc = (double*)malloc(sizeof(double) * (size_t)(D > 0 ? D : 1));
  for (int64_t e = 0; e < B * L * D; ++e) out[e] = 0.0;
  for (int64_t e = 0; e < B * L; ++e) lse[e] = -INFINITY;
  for (int64_t i = 0; i < B; ++i) {
    const int64_t n = lengths[i];
    for (int64_t a = 0; a < L; ++a) {  /* the block_q loop of :124-125 visits every row once */
      double m = -INFINITY, sum = 0.0;
      for (int64_t d = 0; d < D; ++d) acc[d] = 0.0;
      for (int64_t c0 = 0; c0 < L; c0 += block_k) {
        const int64_t c1 = c0 + block_k < L ? c0 + block_k : L;
        double bmax = -INFINITY;
        for (int64_t c = c0; c < c1; ++c) {
          const double sc = (a < n && c < n) ? dot_rows(q + (i * L + a) * D, k + (i * L + c) * D, D) * inv : -INFINITY;
          row[c - c0] = sc;
          bmax = fmax(bmax, sc);
        }
        const double m_new = fmax(m, bmax);
        if (m_new == -INFINITY) continue;
        const double rescale = m == -INFINITY ? 0.0 : exp(m - m_new);
        sum *= rescale;
        for (int64_t d = 0; d < D; ++d) acc[d] *= rescale;
        for (int64_t c = c0; c < c1; ++c) {
          if (row[c - c0] == -INFINITY) continue;
          const double pr = exp(row[c - c0] - m_new);
          sum += pr;
          for (int64_t d = 0; d < D; ++d) acc[d] += pr * v[(i * L + c) * D + d];
        }
        m = m_new;
      }
      if (sum > 0.0) {
        for (int64_t d = 0; d < D; ++d) out[(i * L + a) * D + d] = acc[d] / sum;
        lse[i * L + a] = m + log(sum);
      }
    }
  }
  free(row);
  free(acc);
  return 0;
}

/* ---- feature interaction, attention.cpp:291-309 ----
 * s = scale(jagged_dense_bmm(k_feat, transpose_per_sample(targets)), 1/sqrt(D))  (:302-303)
 * p = jagged_softmax(s)  (softmax over each segment's rows, per target column)  (:305)
 * out = jagged_jagged_bmm(p, v_feat)  (P_i^T V_i, zero for empty samples)  (:307) */
int or_feature_interaction(const int64_t* off, int64_t B, int64_t D, int64_t Tq, const double* k_feat,
                           const double* v_feat, const double* targets, int as_float, double* out) {
  const int64_t S = off[B];
  const double inv = as_float ? (double)(float)(1.0 / sqrt((double)D)) : 1.0 / sqrt((double)D);
  double* s = (double*)malloc(sizeof(double) * (size_t)(S * Tq > 0 ? S * Tq : 1));
  double* pr = (double*)malloc(sizeof(double) * (size_t)(S * Tq > 0 ? S * Tq : 1));
  for (int64_t i = 0; i < B; ++i)
    for (int64_t r = off[i]; r < off[i + 1]; ++r)
      for (int64_t t = 0; t < Tq; ++t) {
        double acc = 0.0;  /* jagged_dense_bmm against targets_i^T: w(d, t) = targets[i, t, d] */
        for (int64_t d = 0; d < D; ++d) acc += k_feat[r * D + d] * targets[(i * Tq + t) * D + d];
        if (as_float) acc = (double)(float)acc;
        double sc = acc * inv;
        s[r * Tq + t] = as_float ? (double)(float)sc : sc;
      }
  or_jagged_softmax(off, B, Tq, s, pr);
  if (as_float)
    for (int64_t e = 0; e < S * Tq; ++e) pr[e] = (double)(float)pr[e];
  or_jagged_jagged_bmm(off, B, Tq, D, pr, v_feat, out);
  free(s);
  free(pr);
  return 0;
}

/* ---- jagged MLP ---- */
/* linalg.cpp:246-261: one affine layer in binary64, optional pre-activation capture */
static void mlp_layer(int64_t rows, int64_t din, int64_t dout, const double* w, const double* b, int relu,
                      const double* in, double* out, double* pre) {
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t o = 0; o < dout; ++o) {
      double acc = b[o];
      for (int64_t i = 0; i < din; ++i) acc += in[r * din + i] * w[i * dout + o];
      if (pre) pre[r * dout + o] = acc;
      out[r * dout + o] = relu ? fmax(acc, 0.0) : acc;
    }
}

/* linalg.cpp:265-277 */
int or_jagged_mlp(int64_t rows, int n_layers, const int64_t* dims, const double* w, const double* b,
                  const int* relu, const double* x, double* out) {
  if (n_layers < 1) return fail("jagged_mlp: at least one layer required");
  int64_t maxd = 0;
  for (int l = 0; l <= n_layers; ++l) maxd = dims[l] > maxd ? dims[l] : maxd;
  double* a = (double*)malloc(sizeof(double) * (size_t)(rows * maxd > 0 ? rows * maxd : 1));
  double* c = (double*)malloc(sizeof(double) * (size_t)(rows * maxd > 0 ? rows * maxd : 1));
  memcpy(a, x, sizeof(double) * (size_t)(rows * dims[0]));
  int64_t wo = 0, bo = 0;
  for (int l = 0; l < n_layers; ++l) {
    mlp_layer(rows, dims[l], dims[l + 1], w + wo, b + bo, relu[l], a, c, NULL);
    wo += dims[l] * dims[l + 1];
    bo += dims[l + 1];
    double* tmp = a;
    a = c;
    c = tmp;
  }
  memcpy(out, a, sizeof(double) * (size_t)(rows * dims[n_layers]));
  free(a);
  free(c);
  return 0;
}

/* linalg.cpp:509-573: forward with retained activations / pre-activations, then per layer (last first):
 * ReLU mask (pre <= 0 -> 0), db = column sums, dW = act^T delta, delta <- delta W^T */
int or_jagged_mlp_vjp(int64_t rows, int n_layers, const int64_t* dims, const double* w, const double* b,
                      const int* relu, const double* x, const double* grad_out, double* dx, double* dw,
                      double* db) {
  if (n_layers < 1) return fail("jagged_mlp: at least one layer required");
  double** acts = (double**)malloc(sizeof(double*) * (size_t)(n_layers + 1));
  double** pres = (double**)malloc(sizeof(double*) * (size_t)n_layers);
  int64_t* wo = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_layers + 1));
  int64_t* bo = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_layers + 1));
  wo[0] = bo[0] = 0;
  for (int l = 0; l < n_layers; ++l) {
    wo[l + 1] = wo[l] + dims[l] * dims[l + 1];
    bo[l + 1] = bo[l] + dims[l + 1];
  }
  for (int l = 0; l <= n_layers; ++l)
    acts[l] = (double*)malloc(sizeof(double) * (size_t)(rows * dims[l] > 0 ? rows * dims[l] : 1));
  memcpy(acts[0], x, sizeof(double) * (size_t)(rows * dims[0]));
  for (int l = 0; l < n_layers; ++l) {
    pres[l] = (double*)malloc(sizeof(double) * (size_t)(rows * dims[l + 1] > 0 ? rows * dims[l + 1] : 1));
    mlp_layer(rows, dims[l], dims[l + 1], w + wo[l], b + bo[l], relu[l], acts[l], acts[l + 1], pres[l]);
  }
  int64_t maxd = 0;
  for (int l = 0; l <= n_layers; ++l) maxd = dims[l] > maxd ? dims[l] : maxd;
  double* delta = (double*)malloc(sizeof(double) * (size_t)(rows * maxd > 0 ? rows * maxd : 1));
  double* prev = (double*)malloc(sizeof(double) * (size_t)(rows * maxd > 0 ? rows * maxd : 1));
  memcpy(delta, grad_out, sizeof(double) * (size_t)(rows * dims[n_layers]));
  for (int l = n_layers - 1; l >= 0; --l) {
    const int64_t din = dims[l], dout = dims[l + 1];
    if (relu[l])
      for (int64_t e = 0; e < rows * dout; ++e)
        if (pres[l][e] <= 0.0) delta[e] = 0.0;
    for (int64_t o = 0; o < dout; ++o) {
      double acc = 0.0;
      for (int64_t r = 0; r < rows; ++r) acc += delta[r * dout + o];
      db[bo[l] + o] = acc;
    }
    for (int64_t i = 0; i < din; ++i)
      for (int64_t o = 0; o < dout; ++o) {
        double acc = 0.0;
        for (int64_t r = 0; r < rows; ++r) acc += acts[l][r * din + i] * delta[r * dout + o];
        dw[wo[l] + i * dout + o] = acc;
      }
    for (int64_t r = 0; r < rows; ++r)
      for (int64_t i = 0; i < din; ++i) {
        double acc = 0.0;
        for (int64_t o = 0; o < dout; ++o) acc += delta[r * dout + o] * w[wo[l] + i * dout + o];
        prev[r * din + i] = acc;
      }
    double* tmp = delta;
    delta = prev;
    prev = tmp;
  }
  memcpy(dx, delta, sizeof(double) * (size_t)(rows * dims[0]));
  for (int l = 0; l <= n_layers; ++l) free(acts[l]);
  for (int l = 0; l < n_layers; ++l) free(pres[l]);
  free(acts);
  free(pres);
  free(wo);
  free(bo);
  free(delta);
  free(prev);
  return 0;
}
