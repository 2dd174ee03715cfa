// internal.h — launcher declarations shared between the kernel files and the C-ABI layer.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "jagged_b200.h"

namespace jg {

// ------------------------------------------------------------------ per-sample affine descriptors
// Every jagged contraction of the bmm family (and its VJPs) is, per sample i, a strided GEMM
// C_i[M x N] = sum_k A_i[m,k] B_i[k,n]. Each size/offset/stride is an affine function of the
// sample's length Bi, row offset off_i, square offset sq_i and index i; one kernel covers all
// eight contractions of linalg.cpp:34-197 and :283-472.
struct Lin {
  int64_t bi = 0, off = 0, sq = 0, idx = 0, c = 0;
  __host__ __device__ int64_t at(int64_t Bi, int64_t o, int64_t s, int64_t i) const {
    return bi * Bi + off * o + sq * s + idx * i + c;
  }
};
inline Lin L_const(int64_t c) { Lin l; l.c = c; return l; }
inline Lin L_bi(int64_t k = 1) { Lin l; l.bi = k; return l; }

struct GemmDesc {
  Lin M, N, K;
  Lin a0, sam, sak;  // A(m,k) = A[a0 + m*sam + k*sak]
  Lin b0, sbk, sbn;  // B(k,n) = B[b0 + k*sbk + n*sbn]
  Lin c0, scm, scn;  // C(m,n) = C[c0 + m*scm + n*scn]
};

// Per-device, mutex-guarded, lazily-set kernel attribute: the opt-in dynamic shared memory size of `func`
// (cudaFuncSetAttribute is per device; a process driving several devices sets it once on each).
jg_status ensure_smem_attr(const void* func, int bytes, const char* name);

// Self-resetting work counters for the persistent kernels: counters[0] = next dynamic item, counters[1] = CTAs
// exited. Zeroed once when allocated (schedule creation); the last CTA of a launch to exit zeroes both, so
// consecutive launches on one stream need no memset. A schedule's counters serialise the launches that use
// it: one schedule must not drive two concurrently running kernels.
#ifdef __CUDACC__
__device__ __forceinline__ void work_counters_exit(unsigned long long* counters) {
  if (counters == nullptr) return;
  __threadfence();
  if (atomicAdd(counters + 1, 1ull) == gridDim.x - 1) {
    counters[0] = 0;
    counters[1] = 0;
    __threadfence();
  }
}
#endif

jg_status launch_scan(int mode, const int64_t* in, int64_t n, int64_t* out, int64_t* bad, cudaStream_t s);
jg_status launch_lengths(const int64_t* off, int64_t n, int64_t* len, cudaStream_t s);
// device scratch accounting (jg_scratch_counters): every library-internal device allocation reports here
void scratch_note(int64_t bytes);  // + on allocation, - on release

jg_status launch_work_list(const int64_t* off, int64_t batch, int tile, int2* items, int64_t* count,
                           cudaStream_t s, int* win_first = nullptr, int* win_last = nullptr, int64_t nwin = 0);

jg_status launch_jagged_to_dense(const int64_t* off, int64_t batch, int64_t dim, const void* x,
                                 int64_t max_len, double pad, void* out, jg_dtype dt, cudaStream_t s);
jg_status launch_dense_to_jagged(const void* d, int64_t batch, int64_t max_len, int64_t dim,
                                 const int64_t* off, int64_t total_rows, void* out, jg_dtype dt,
                                 cudaStream_t s);
jg_status launch_jagged2_to_dense(const int64_t* off, const int64_t* sq, int64_t batch, const void* x,
                                  int64_t max_len, double pad, void* out, jg_dtype dt, cudaStream_t s);
jg_status launch_dense_to_jagged2(const void* d, int64_t batch, int64_t max_len, const int64_t* off,
                                  const int64_t* sq, int64_t total_rows_hint, void* out, jg_dtype dt,
                                  cudaStream_t s);
jg_status launch_elementwise(int op, const void* a, const void* b, int64_t n, double sc, void* out,
                             jg_dtype dt, cudaStream_t s);

jg_status launch_jagged_softmax(const int64_t* off, int64_t batch, int64_t D, const void* x,
                                const void* g, void* out, jg_dtype dt, bool vjp, cudaStream_t st);
jg_status launch_jagged2_softmax(const int64_t* off, const int64_t* sq, int64_t batch, int64_t total_rows,
                                 const void* s, const void* g, void* out, jg_dtype dt, bool vjp,
                                 cudaStream_t st);

// Grouped strided GEMM over samples. tile_prefix: device scratch of batch+1 int64.
jg_status launch_grouped_gemm(const GemmDesc& g, const int64_t* off, const int64_t* sq, int64_t batch,
                              const void* A, const void* B, void* C, jg_dtype in_dt, jg_dtype out_dt,
                              int64_t* tile_prefix, cudaStream_t st);

jg_status launch_gemm_prefix(const GemmDesc& g, const int64_t* off, const int64_t* sq, int64_t batch, int bm, int bn,
                             int64_t* tile_prefix, cudaStream_t st);

// tcgen05 bmm family (bf16 inputs): op 0 jjbmm_jout (q,k), 1 ajbmm_jout (a_j2,v), 2 jjbmm (x,y), 3 jdbmm (x,w),
// 4 x [rows, T] . w^T (w [B, D, T]) -> [rows, D], 5 a_j2^T . v -> [rows, D] (the transposed VJP forms)
struct AjBlocks {  // a jagged^2 operand repacked into 64 x 64 SW128 sub-block images (gemm_sm100.cu)
  uint8_t* blocks = nullptr;
  int64_t* prefix = nullptr;  // 128 x 128 tiles per sample, exclusive prefix
  int64_t n_blocks = 0, blocks_bytes = 0, prefix_bytes = 0;
};
jg_status aj_repack(const int64_t* off, const int64_t* sq, int64_t batch, int64_t total_rows, int64_t sum_sq,
                    const void* a, AjBlocks* out, cudaStream_t st);
void aj_release(AjBlocks* b, cudaStream_t st);
bool gemm_sm100_supported(int op, int64_t D, int64_t T, jg_dtype in_dt);
// JD only: optional fused epilogue out = act(acc + bias[col]) with preact = acc + bias (jagged_mlp layers)
jg_status launch_gemm_sm100(int op, const int64_t* off, const int64_t* sq, int64_t batch, int64_t total_rows, int64_t D,
                            int64_t T, const void* a, const void* b, void* out, jg_dtype out_dt, int64_t* tile_prefix,
                            cudaStream_t st,
                            const void* bias = nullptr, int relu = 0, void* preact = nullptr,
                            // JJJ / AJ on head `head` of [rows, heads, D] q/k (JJJ) or v (AJ); the AJ output
                            // pointer is the head's column block of a [rows, heads, D] tensor
                            int heads = 1, int head = 0,
                            // AJ / AJT: sum Bi^2 (the jagged^2 operand's size) sizes the repack buffer without a
                            // device->host read; -1: unknown (one stream-synchronising read)
                            int64_t sum_sq = -1,
                            // AJ / AJT: already repacked sub-block images of `a` (aj_repack), shared by several GEMMs
                            const struct AjBlocks* pre = nullptr);

// SURVEY §8f next rows (mlp_fi.cu)
jg_status launch_two_offsets(int64_t* o, int64_t rows, cudaStream_t st);
jg_status launch_uniform_offsets(int64_t* o, int64_t batch, int64_t step, cudaStream_t st);  // o[i] = i * step
jg_status launch_bias_act(const float* acc, const void* bias, int64_t rows, int64_t d, int relu, void* out,
                          void* preact, jg_dtype dt, cudaStream_t st);
jg_status launch_relu_mask(const void* g, const void* preact, int64_t n, int relu, void* out, jg_dtype dt,
                           cudaStream_t st);
int64_t colsum_scratch_floats(int64_t rows, int64_t cols);
jg_status launch_colsum(const void* x, int64_t rows, int64_t cols, void* out, float* partial, jg_dtype dt,
                        cudaStream_t st);
jg_status launch_cast_f32(const float* a, int64_t n, void* out, jg_dtype dt, cudaStream_t st);

// SIMT attention (fp32 mode, and any head_dim the tensor-core path does not cover).
// valid: nullptr (jagged), or per-sample valid lengths <= segment lengths (padded dense_flash_attention mode:
// keys past the valid length are masked, rows past it produce zeros / lse = -inf / zero gradients).
jg_status launch_attn_fwd_simt(const int64_t* off, int64_t batch, int64_t total_rows, int H, int D,
                               const void* q, const void* k, const void* v, void* out, float* lse,
                               jg_dtype dt, const int2* items, const int64_t* n_items, int64_t max_items,
                               const int64_t* valid, cudaStream_t st);
// fp32 attention on tcgen05 through a split-bf16 emulation (attn_x3_sm100.cu), head_dim 64 / 128
bool attn_x3_supported(int head_dim, jg_dtype dt);
jg_status launch_attn_fwd_x3(const int64_t* off, int64_t total_rows, int H, int D, const void* q, const void* k,
                             const void* v, void* out, float* lse, const int2* items, const int64_t* n_items,
                             int64_t max_items, const int64_t* valid, cudaStream_t st);
jg_status launch_attn_bwd_x3(const int64_t* off, int64_t total_rows, int H, int D, const void* q, const void* k,
                             const void* v, const void* go, const void* o, const float* lse, float* delta, void* dq, void* dk,
                             void* dv, const int2* items, const int64_t* n_items, int64_t max_items,
                             const int64_t* valid, cudaStream_t st);
jg_status launch_attn_bwd_simt(const int64_t* off, int64_t batch, int64_t total_rows, int H, int D,
                               const void* q, const void* k, const void* v, const void* go,
                               const void* o, const float* lse, void* dq, void* dk, void* dv,
                               float* delta, jg_dtype dt, const int2* items, const int64_t* n_items,
                               int64_t max_items, const int64_t* valid, bool x3, cudaStream_t st);

// The backward workspace starts with lsd fp32
// ([2][H][total_rows]: -lse log2(e), -Delta; then [3][H] per-head max|K|, max||V||^2, max||dO||^2)
inline int64_t attn_lsd_bytes(int64_t total_rows, int H) {
  return ((2 * (int64_t)H * total_rows * 4 + 3 * (int64_t)H * 4 + 255) / 256) * 256;
}

// tcgen05 attention (bf16, head_dim 64/128)
bool attn_sm100_supported(int head_dim, jg_dtype dt);
bool attn_sm100_bwd_supported(int head_dim, jg_dtype dt);
jg_status launch_attn_fwd_sm100(const int64_t* off, int64_t batch, int64_t total_rows, int H, int D,
                                const void* q, const void* k, const void* v, void* out, float* lse,
                                const int2* items, const int64_t* n_items, int64_t max_items,
                                const int64_t* valid, unsigned long long* counters, cudaStream_t st,
                                // cross mode (fused feature_interaction): query segments over the key segments
                                const int64_t* q_off = nullptr, int64_t q_rows = 0);
// dq_accum: fp32, or int64 fixed point when deterministic ([total_rows, H, D], zeroed by the launcher's prologue)
jg_status launch_attn_bwd_sm100(const int64_t* off, int64_t batch, int64_t total_rows, int H, int D,
                                const void* q, const void* k, const void* v, const void* go,
                                const void* o, const float* lse, void* dq, void* dk, void* dv,
                                float* delta, void* dq_accum, bool deterministic, const int2* items,
                                const int64_t* n_items, int64_t max_items, const int64_t* valid,
                                unsigned long long* counters, cudaStream_t st);

}  // namespace jg
