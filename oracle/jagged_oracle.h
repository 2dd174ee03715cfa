/*
 * jagged_oracle.h — CPU restatement of the reference jagged operators (TEST INFRASTRUCTURE).
 *
 * This is the parity checker, not product code. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it. Every function restates one
 * reference loop nest in plain C with binary64 accumulation, exactly as the reference does
 * ("Accumulation in binary64 internally"); the comment above each definition in
 * jagged_oracle.c names the /root/reference file:line it follows.
 *
 * Pinning: tests/test_oracle.py checks this restatement against (a) the SPEC.md known-answer
 * vectors, (b) tests/golden/*.npz fixtures produced by the compiled reference itself
 * (oracle/_ref/libjagged_ref.so, built from /root/reference sources by oracle/Makefile), and
 * (c) live comparison with oracle/_ref when it is present.
 *
 * Conventions: all values are double; offsets are int64 with offsets[0]=0; Bi = offsets[i+1]-offsets[i].
 * Return codes: 0 ok, 1 invalid argument (message via or_last_error()).
 */
#ifndef JAGGED_ORACLE_H
#define JAGGED_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* or_last_error(void);

/* ---- pinned RNG (std::mt19937_64 restated; reference rng.hpp:10-28, rng.cpp:7-17) ---- */
typedef struct {
  uint64_t mt[312];
  int idx;
} or_rng;
void or_rng_seed(or_rng* r, uint64_t seed);
uint64_t or_rng_next(or_rng* r);
int64_t or_rng_uniform_int(or_rng* r, int64_t lo, int64_t hi);
double or_rng_uniform_real(or_rng* r, double lo, double hi);
/* kind: 0 fixed, 1 uniform, 2 half-mean (rng.cpp:35-57); 3 zipf (not in reference) */
int or_gen_lengths(int kind, int64_t max_len, uint64_t seed, int64_t batch, double zipf_alpha,
                   int64_t* out);
/* n values U[lo,hi) rounded to float (as_float=1) or kept double (rng.cpp:59-64) */
void or_uniform_values(or_rng* r, int64_t n, double lo, double hi, int as_float, double* out);

/* ---- offsets / layout (tensor.cpp:72-175) ---- */
int or_make_offsets(const int64_t* lengths, int64_t batch, int64_t* offsets);
int or_sq_offsets(const int64_t* offsets, int64_t batch, int64_t* sq_offsets);
int or_jagged_to_dense(const int64_t* offsets, int64_t batch, int64_t dim, const double* x,
                       int64_t max_len, double pad, double* out);
int or_dense_to_jagged(const double* d, int64_t batch, int64_t max_len, int64_t dim,
                       const int64_t* lengths, double* out);
int or_jagged2_to_dense(const int64_t* offsets, int64_t batch, const double* s, int64_t max_len,
                        double pad, double* out);
int or_dense_to_jagged2(const double* d, int64_t batch, int64_t max_len, const int64_t* lengths,
                        double* out);

/* ---- Table-1 forward operators (linalg.cpp:34-220) ---- */
int or_jagged_dense_bmm(const int64_t* off, int64_t B, int64_t D, int64_t T, const double* x,
                        const double* w, double* out);
int or_jagged_jagged_bmm(const int64_t* off, int64_t B, int64_t D, int64_t T, const double* x,
                         const double* y, double* out);
int or_jagged_softmax(const int64_t* off, int64_t B, int64_t D, const double* x, double* out);
int or_jagged_jagged_bmm_jagged_out(const int64_t* off, int64_t B, int64_t D, const double* q,
                                    const double* k, double* out);
int or_array_jagged_bmm_jagged_out(const int64_t* off, int64_t B, int64_t D, const double* a,
                                   const double* v, double* out);
int or_jagged2_softmax(const int64_t* off, int64_t B, const double* s, double* out);

/* ---- VJPs (linalg.cpp:283-507) ---- */
int or_jagged_dense_bmm_vjp(const int64_t* off, int64_t B, int64_t D, int64_t T, const double* x,
                            const double* w, const double* go, double* dx, double* dw);
int or_jagged_jagged_bmm_vjp(const int64_t* off, int64_t B, int64_t D, int64_t T, const double* x,
                             const double* y, const double* go, double* dx, double* dy);
int or_jagged_softmax_vjp(const int64_t* off, int64_t B, int64_t D, const double* x,
                          const double* go, double* dx);
int or_jagged_jagged_bmm_jagged_out_vjp(const int64_t* off, int64_t B, int64_t D, const double* q,
                                        const double* k, const double* go, double* dq, double* dk);
int or_array_jagged_bmm_jagged_out_vjp(const int64_t* off, int64_t B, int64_t D, const double* a,
                                       const double* v, const double* go, double* da, double* dv);
int or_jagged2_softmax_vjp(const int64_t* off, int64_t B, const double* s, const double* go,
                           double* ds);

/* ---- attention (attention.cpp:162-289) ---- */
int or_jagged_attention(const int64_t* off, int64_t B, int64_t D, const double* q, const double* k,
                        const double* v, double* out);
int or_jfa_forward(const int64_t* off, int64_t B, int64_t D, const double* q, const double* k,
                   const double* v, int64_t block_q, int64_t block_k, double* out, double* lse);
int or_jfa_backward(const int64_t* off, int64_t B, int64_t D, const double* q, const double* k,
                    const double* v, const double* go, const double* out, const double* lse,
                    int64_t block_k, double* dq, double* dk, double* dv);
/* padded-dense baseline semantics (attention.cpp:62-104) on [B,L,D] with lengths */
int or_dense_attention(const int64_t* lengths, int64_t B, int64_t L, int64_t D, const double* q,
                       const double* k, const double* v, double* out);
int or_dense_flash_attention(const int64_t* lengths, int64_t B, int64_t L, int64_t D, int64_t block_q,
                             int64_t block_k, const double* q, const double* k, const double* v, double* out,
                             double* lse);

/* ---- feature interaction (attention.cpp:291-309). targets [B, Tq, D] -> out [B, Tq, D].
 * as_float != 0 rounds the scores to float after the 1/sqrt(D) scale and the softmax output to float, as
 * the reference's float instantiation does between its composed operators (binary64 otherwise). */
int or_feature_interaction(const int64_t* off, int64_t B, int64_t D, int64_t Tq, const double* k_feat,
                           const double* v_feat, const double* targets, int as_float, double* out);

/* ---- jagged MLP (linalg.cpp:224-277, VJP :509-573). Layer l maps dims[l] -> dims[l+1]
 * with weights w + woff[l] ([dims[l], dims[l+1]] row-major), bias b + boff[l], relu[l] != 0 for ReLU.
 * Activations stay binary64 between layers, as in the reference. */
int or_jagged_mlp(int64_t rows, int n_layers, const int64_t* dims, const double* w, const double* b,
                  const int* relu, const double* x, double* out);
/* grads: dx [rows, dims[0]]; dw, db concatenated like w, b */
int or_jagged_mlp_vjp(int64_t rows, int n_layers, const int64_t* dims, const double* w, const double* b,
                      const int* relu, const double* x, const double* grad_out, double* dx, double* dw,
                      double* db);

/* ---- cost model (cost_model.cpp:94-189), used by bench/tests for algorithmic FLOPs/bytes ---- */
int64_t or_sum_sq(const int64_t* off, int64_t B);

#ifdef __cplusplus
}
#endif
#endif
