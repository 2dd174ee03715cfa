/*
 * jagged_b200.h — C-ABI of the B200-native jagged hot path (libjagged_b200.so).
 *
 * Drop-in boundary for the reference library's operator layer (proj/core, namespace jagged).
 * Every entry point replaces one reference operator; the comment above it cites the reference
 * declaration (include/jagged/<file>.hpp:line) whose semantics it keeps: same operator name,
 * same argument order (inputs, then options), same per-sample math, same empty-segment behaviour.
 *
 * Differences forced by the device boundary:
 *   - tensors are device pointers + sizes (no STL types); the caller owns all memory;
 *   - a JaggedTensor<T> is (offsets[batch+1] int64 on device, values[total_rows*dim] on device);
 *     total_rows = offsets[batch] must also be passed by value (sizes are host-known);
 *   - a Jagged2Tensor<T> is (offsets of the governing jagged tensor, values[sum Bi^2]) with block i
 *     at sq_offsets[i] = sum_{j<i} Bj^2 (tensor.hpp:42-62); jg_sq_offsets computes it on device;
 *   - errors return a jg_status; the reference's exception text is available from jg_last_error()
 *     (thread-local), e.g. "jagged_dense_bmm: dim mismatch (64 vs 32)" (linalg.cpp:42-44);
 *   - every call is stream-ordered on the caller's cudaStream_t (passed as void*) without host
 *     synchronisation (the host `lengths` of jg_dense_flash_attention_* are staged through a buffer
 *     released by a stream callback), except jg_schedule_work_list (a host-side inspection helper);
 *     ops with a jagged^2 operand take its element count sum_sq (= sum Bi^2, what a Jagged2Tensor
 *     holds) so their scratch is sized on the host (-1: unknown -> one 8-byte device read);
 *   - KernelOptions{block, threads, meter} (linalg.hpp:16-20) have no device meaning and are not
 *     taken; block_q/block_k of the flash forward are validated (>= 1) exactly as the reference does
 *     and otherwise ignored (device tiles are fixed at 128x128).
 *
 * dtypes: JG_F32 ("fp32 mode": attention on tcgen05 via an fp16 two-piece split at head_dim 64/128, FFMA
 * otherwise and for the bmm family), JG_BF16 (tcgen05 tensor cores where shapes allow,
 * fp32 accumulation). JG_F64 returns JG_UNSUPPORTED: there is no CPU fallback.
 * Attention tensors carry heads: [total_rows, num_heads, head_dim] row-major (token-major, the
 * reference's single-head layout when num_heads == 1); lse is float32 [num_heads, total_rows].
 * Attention runs on tcgen05 for bf16 with head_dim 64 or 128 (forward and backward); fp32 and other
 * head dims run SIMT kernels with the same semantics.
 */
#ifndef JAGGED_B200_H
#define JAGGED_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  JG_OK = 0,
  JG_INVALID_ARGUMENT = 1, /* reference throws std::invalid_argument */
  JG_CUDA_ERROR = 2,
  JG_OUT_OF_MEMORY = 3,
  JG_UNSUPPORTED = 4 /* e.g. f64: no device path and no CPU fallback */
} jg_status;

typedef enum { JG_F32 = 0, JG_BF16 = 1, JG_F64 = 2 } jg_dtype;

/* Thread-local text of the last failure (the reference's exception message). */
const char* jg_last_error(void);

/* Device scratch accounting, per host thread: bytes of device memory the library allocates for a call's own
 * intermediates (backward workspace, unfused score/probability tensors, repacked jagged^2 operands, per-call
 * schedules); the caller's operands and outputs are not counted. This is what KernelOptions.meter
 * (linalg.hpp:19, scratch.hpp:12-55) observes through the C++ drop-in: a peak window opened with
 * jg_scratch_reset_peak() (peak := current) and read back with jg_scratch_counters(); jg_scratch_raise_peak()
 * restores an enclosing window's peak (nested windows). */
void jg_scratch_counters(int64_t* current_bytes, int64_t* peak_bytes);
void jg_scratch_reset_peak(void);
void jg_scratch_raise_peak(int64_t peak_bytes);
/* Library version string; also forces the CUDA module load. */
const char* jg_version(void);

/* ---------------------------------------------------------------------------------------------
 * Offsets layer and device tile scheduler (replaces parallel.cpp:9-26 work splitting)
 * ------------------------------------------------------------------------------------------- */

/* lengths[batch] -> offsets[batch+1] (exclusive prefix sum). tensor.hpp:96-98 make_jagged;
 * negative lengths are an error ("make_jagged: negative length at sample i", tensor.cpp:78-79).
 * The check is done on device; *bad_sample (device int64, may be NULL) receives the first bad
 * index or -1. Bit-exact integer work. */
jg_status jg_make_offsets(const int64_t* lengths, int64_t batch, int64_t* offsets,
                          int64_t* bad_sample, void* stream);
/* offsets -> lengths (tensor.hpp:104 segment_lengths). */
jg_status jg_segment_lengths(const int64_t* offsets, int64_t batch, int64_t* lengths, void* stream);
/* offsets -> sq_offsets[batch+1], sq_offsets[i+1] = sq_offsets[i] + Bi^2 (tensor.cpp:40-48). */
jg_status jg_sq_offsets(const int64_t* offsets, int64_t batch, int64_t* sq_offsets, void* stream);

/* Opaque device schedule for one offsets array: lengths, sq_offsets and the attention work list
 * of (sample, 128-row tile) items ordered longest-first (LPT) for the persistent kernels. */
typedef struct jg_schedule_s* jg_schedule;
jg_status jg_schedule_create(const int64_t* offsets, int64_t batch, int64_t total_rows,
                             void* stream, jg_schedule* out);
jg_status jg_schedule_destroy(jg_schedule sched);
/* Device pointers owned by the schedule (valid until destroy). */
const int64_t* jg_schedule_sq_offsets(jg_schedule sched);
/* Copies the LPT work list (int32 pairs sample,tile) and its length to host (test hook). */
jg_status jg_schedule_work_list(jg_schedule sched, int32_t* host_items, int64_t capacity,
                                int64_t* count);

/* ---------------------------------------------------------------------------------------------
 * Layout conversions (tensor.hpp:100-118) and elementwise ops (tensor.hpp:122-141); bit-exact.
 * ------------------------------------------------------------------------------------------- */
/* [total_rows, dim] -> [batch, max_len, dim]; pad past Bi, truncate Bi > max_len (tensor.cpp:102). */
jg_status jg_jagged_to_dense(const int64_t* offsets, int64_t batch, int64_t dim, const void* x,
                             int64_t max_len, double pad_value, void* out, jg_dtype dtype,
                             void* stream);
/* [batch, max_len, dim] -> jagged rows given offsets (lengths must be <= max_len; tensor.cpp:118).
 * Host-side validation needs the lengths; pass max_segment = max Bi (host-known) for the check. */
jg_status jg_dense_to_jagged(const void* d, int64_t batch, int64_t max_len, int64_t dim,
                             const int64_t* offsets, int64_t total_rows, int64_t max_segment,
                             void* out, jg_dtype dtype, void* stream);
jg_status jg_jagged2_to_dense(const int64_t* offsets, const int64_t* sq_offsets, int64_t batch,
                              const void* s, int64_t max_len, double pad_value, void* out,
                              jg_dtype dtype, void* stream);
jg_status jg_dense_to_jagged2(const void* d, int64_t batch, int64_t max_len,
                              const int64_t* offsets, const int64_t* sq_offsets,
                              int64_t max_segment, void* out, jg_dtype dtype, void* stream);
/* op: 0 add, 1 sub, 2 mul (tensor.cpp:206-219); scale: out = a * s (tensor.cpp:221-233). */
jg_status jg_elementwise(int32_t op, const void* a, const void* b, int64_t n, void* out,
                         jg_dtype dtype, void* stream);
jg_status jg_scale(const void* a, int64_t n, double s, void* out, jg_dtype dtype, void* stream);

/* ---------------------------------------------------------------------------------------------
 * Table-1 operators (linalg.hpp:27-54). in_dtype is the values dtype; out_dtype may be JG_F32 for
 * bf16 inputs (fp32 output of the fp32 accumulator) or equal to in_dtype.
 * ------------------------------------------------------------------------------------------- */
/* linalg.hpp:27-29: x [total_rows, D], w [batch, D, T] -> out [total_rows, T]. */
jg_status jg_jagged_dense_bmm(const int64_t* offsets, int64_t batch, int64_t total_rows, int64_t D,
                              int64_t T, const void* x, const void* w, void* out,
                              jg_dtype in_dtype, jg_dtype out_dtype, void* stream);
/* linalg.hpp:32-34: x [total_rows, D], y [total_rows, T] -> out [batch, D, T] (zero for Bi=0). */
jg_status jg_jagged_jagged_bmm(const int64_t* offsets, int64_t batch, int64_t total_rows,
                               int64_t D, int64_t T, const void* x, const void* y, void* out,
                               jg_dtype in_dtype, jg_dtype out_dtype, void* stream);
/* linalg.hpp:37-38: softmax over each segment's rows, per column. */
jg_status jg_jagged_softmax(const int64_t* offsets, int64_t batch, int64_t total_rows, int64_t D,
                            const void* x, void* out, jg_dtype dtype, void* stream);
/* linalg.hpp:41-44: q,k [total_rows, D] -> jagged2 [sum Bi^2]. */
jg_status jg_jagged_jagged_bmm_jagged_out(const int64_t* offsets, const int64_t* sq_offsets,
                                          int64_t batch, int64_t total_rows, int64_t D,
                                          const void* q, const void* k, void* out,
                                          jg_dtype in_dtype, jg_dtype out_dtype, void* stream);
/* linalg.hpp:47-50: a jagged2 [sum_sq], v [total_rows, D] -> [total_rows, D]. */
jg_status jg_array_jagged_bmm_jagged_out(const int64_t* offsets, const int64_t* sq_offsets,
                                         int64_t batch, int64_t total_rows, int64_t sum_sq, int64_t D,
                                         const void* a, const void* v, void* out,
                                         jg_dtype in_dtype, jg_dtype out_dtype, void* stream);
/* linalg.hpp:53-54: row softmax inside each Bi x Bi block. */
jg_status jg_jagged2_softmax(const int64_t* offsets, const int64_t* sq_offsets, int64_t batch,
                             const void* s, void* out, jg_dtype dtype, void* stream);

/* VJPs (linalg.hpp:112-146). Gradients have the layout of the matching input. bf16: all eight
 * contractions on the tcgen05 grouped GEMM (incl. the transposed forms dO W^T, Y dZ^T, dS^T Q, A^T dO). */
jg_status jg_jagged_dense_bmm_vjp(const int64_t* offsets, int64_t batch, int64_t total_rows,
                                  int64_t D, int64_t T, const void* x, const void* w,
                                  const void* grad_out, void* dx, void* dw, jg_dtype in_dtype,
                                  jg_dtype out_dtype, void* stream);
jg_status jg_jagged_jagged_bmm_vjp(const int64_t* offsets, int64_t batch, int64_t total_rows,
                                   int64_t D, int64_t T, const void* x, const void* y,
                                   const void* grad_out, void* dx, void* dy, jg_dtype in_dtype,
                                   jg_dtype out_dtype, void* stream);
jg_status jg_jagged_softmax_vjp(const int64_t* offsets, int64_t batch, int64_t total_rows,
                                int64_t D, const void* x, const void* grad_out, void* dx,
                                jg_dtype dtype, void* stream);
jg_status jg_jagged_jagged_bmm_jagged_out_vjp(const int64_t* offsets, const int64_t* sq_offsets,
                                              int64_t batch, int64_t total_rows, int64_t sum_sq, int64_t D,
                                              const void* q, const void* k, const void* grad_out,
                                              void* dq, void* dk, jg_dtype in_dtype,
                                              jg_dtype out_dtype, void* stream);
jg_status jg_array_jagged_bmm_jagged_out_vjp(const int64_t* offsets, const int64_t* sq_offsets,
                                             int64_t batch, int64_t total_rows, int64_t sum_sq, int64_t D,
                                             const void* a, const void* v, const void* grad_out,
                                             void* da, void* dv, jg_dtype in_dtype,
                                             jg_dtype out_dtype, void* stream);
jg_status jg_jagged2_softmax_vjp(const int64_t* offsets, const int64_t* sq_offsets, int64_t batch,
                                 const void* s, const void* grad_out, void* ds, jg_dtype dtype,
                                 void* stream);

/* ---------------------------------------------------------------------------------------------
 * Attention (attention.hpp:63-88). q/k/v/out/grads are [total_rows, num_heads, head_dim].
 * ------------------------------------------------------------------------------------------- */
/* attention.hpp:70-75 jagged_flash_attention_forward: writes out and lse (float32,
 * [num_heads, total_rows]; -inf for rows of empty segments is never needed since such rows do not
 * exist). Scores are scaled by 1/sqrt(head_dim). sched may be NULL (built per call). */
jg_status jg_jagged_flash_attention_forward(const int64_t* offsets, int64_t batch,
                                            int64_t total_rows, int32_t num_heads,
                                            int32_t head_dim, const void* q, const void* k,
                                            const void* v, int64_t block_q, int64_t block_k,
                                            void* out, float* lse, jg_dtype dtype,
                                            jg_schedule sched, void* stream);
/* attention.hpp:82-88 jagged_flash_attention_backward: recompute from (q, k, lse).
 * deterministic != 0 (the default of every wrapper): bit-identical gradients across runs, grid sizes and
 * schedules (the reference's fixed summation order, attention.cpp:252-254). The
 * tcgen05 kernel then rounds each key tile's partial dQ to a per-head power-of-two grid bounded from the
 * inputs (max|K|, max||V||, max||dO||), so every fp32 reduce-add of the partials is exact and the sum is
 * independent of the order in which key tiles finish; 0 selects plain fp32 accumulation (last bits
 * order-dependent). The SIMT path is sequential per key and deterministic either way.
 * workspace: NULL or >= jg_attention_backward_workspace_size(total_rows, batch, ...) bytes of device
 * memory. A schedule (and a workspace) must not be shared by two concurrently running calls. */
jg_status jg_jagged_flash_attention_backward(const int64_t* offsets, int64_t batch,
                                             int64_t total_rows, int32_t num_heads,
                                             int32_t head_dim, const void* q, const void* k,
                                             const void* v, const void* grad_out, const void* out,
                                             const float* lse, int64_t block_q, int64_t block_k,
                                             void* dq, void* dk, void* dv, jg_dtype dtype,
                                             int32_t deterministic, jg_schedule sched,
                                             void* workspace, void* stream);
int64_t jg_attention_backward_workspace_size(int64_t total_rows, int64_t batch, int32_t num_heads,
                                             int32_t head_dim);
/* attention.hpp:55-58 dense_flash_attention (attention.cpp:106-160), GPU padded mode of the same tcgen05 /
 * SIMT kernels: q/k/v/out are padded [batch, max_len, num_heads, head_dim]; `lengths` is a
 * HOST array of batch entries, each in [0, max_len] (validated with the reference's messages). Keys past a
 * sample's length are masked and its rows past the length are zero with lse = -inf (lse: float32
 * [num_heads, batch * max_len]). The kernels run the full padded max_len^2 work per sample (segments at
 * offsets i * max_len), which is what makes this the padded baseline of the jagged kernels. */
jg_status jg_dense_flash_attention_forward(const int64_t* lengths, int64_t batch, int64_t max_len,
                                           int32_t num_heads, int32_t head_dim, const void* q,
                                           const void* k, const void* v, int64_t block_q,
                                           int64_t block_k, void* out, float* lse, jg_dtype dtype,
                                           void* stream);
/* Backward of the padded mode (no reference counterpart; used for the padded-vs-jagged training-step
 * comparison): rows past a sample's length get zero dq/dk/dv. workspace: NULL or
 * >= jg_attention_backward_workspace_size(batch * max_len, batch, num_heads, head_dim) bytes. */
jg_status jg_dense_flash_attention_backward(const int64_t* lengths, int64_t batch, int64_t max_len,
                                            int32_t num_heads, int32_t head_dim, const void* q,
                                            const void* k, const void* v, const void* grad_out,
                                            const void* out, const float* lse, int64_t block_q,
                                            int64_t block_k, void* dq, void* dk, void* dv,
                                            jg_dtype dtype, void* workspace, void* stream);
/* attention.hpp:63-65 jagged_attention (unfused baseline): materializes sum Bi^2 scores per head
 * in `scores_workspace` (scores and probabilities: >= 2 * round_up(num_heads * sum Bi^2 * sizeof(dtype), 256)
 * bytes, or NULL to allocate). */
jg_status jg_jagged_attention(const int64_t* offsets, const int64_t* sq_offsets, int64_t batch,
                              int64_t total_rows, int64_t sum_sq, int32_t num_heads,
                              int32_t head_dim, const void* q, const void* k, const void* v,
                              void* out, jg_dtype dtype, void* scores_workspace, void* stream);

/* ---------------------------------------------------------------- SURVEY §8f "next" rows */
/* attention.hpp:97 / attention.cpp:291-309 feature_interaction: targets [B, Tq, D] attend over each
 * sample's jagged rows: out[i] = softmax_rows(K_i targets_i^T / sqrt(D))^T V_i, [B, Tq, D] (zeros for
 * empty samples). Scores and weights are kept in fp32 for both dtypes (the reference's float
 * instantiation rounds them to float). workspace: NULL or >= jg_feature_interaction_workspace_size()
 * bytes. Errors as the reference: "feature_interaction: targets must be [B, Tq, D]". */
int64_t jg_feature_interaction_workspace_size(int64_t total_rows, int64_t num_targets);
jg_status jg_feature_interaction(const int64_t* offsets, int64_t batch, int64_t total_rows, int64_t dim,
                                 int64_t num_targets, const void* k_feat, const void* v_feat,
                                 const void* targets, void* out, jg_dtype dtype, void* workspace,
                                 void* stream);
/* linalg.hpp:59-68 / linalg.cpp:246-277 jagged_mlp, one layer: out[r] = act(x[r] W + bias) over all
 * rows (weights shared across samples, no padding rows). W [d_in, d_out], bias [d_out]; relu != 0 for
 * Activation::relu. preact: NULL or [rows, d_out] pre-activations (kept for the VJP). */
jg_status jg_mlp_layer_forward(int64_t rows, int64_t d_in, int64_t d_out, const void* x, const void* w,
                               const void* bias, int32_t relu, void* out, void* preact, jg_dtype dtype,
                               void* stream);
/* linalg.cpp:526-567 one layer of jagged_mlp_vjp: delta = grad_out masked by preact <= 0 (relu),
 * db = column sums of delta, dW = x^T delta, dx = delta W^T. Any of dw/db/dx may be NULL.
 * Under sample sharding dW/db are partial sums: all-reduce them across ranks. */
jg_status jg_mlp_layer_backward(int64_t rows, int64_t d_in, int64_t d_out, const void* x, const void* w,
                                const void* preact, int32_t relu, const void* grad_out, void* dw,
                                void* db, void* dx, jg_dtype dtype, void* stream);

/* Host-buffer convenience (what the reference API's by-value std::vector contract implies):
 * copies host q/k/v/grad_out in, runs forward + backward, copies out/lse/dq/dk/dv back.
 * Host pointers should be pinned for full PCIe bandwidth. offsets is a HOST array here. */
jg_status jg_jagged_flash_attention_fwd_bwd_host(const int64_t* host_offsets, int64_t batch,
                                                 int32_t num_heads, int32_t head_dim,
                                                 const void* q, const void* k, const void* v,
                                                 const void* grad_out, void* out, float* lse,
                                                 void* dq, void* dk, void* dv, jg_dtype dtype,
                                                 void* stream);

/* Number of device kernels this library launched on the calling thread since the last reset
 * (instrumentation for bench.py's gpu_launches). */
int64_t jg_launch_count(void);
void jg_reset_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif
