// attn_sm100.cu — placeholder until the tcgen05 kernels land.
#include "common.cuh"
#include "internal.h"
namespace jg {
bool attn_sm100_supported(int, jg_dtype) { return false; }
jg_status launch_attn_fwd_sm100(const int64_t*, int64_t, int64_t, int, int, const void*, const void*, const void*,
                                void*, float*, const int2*, const int64_t*, int64_t, cudaStream_t) {
  return fail(JG_UNSUPPORTED, "tcgen05 attention not built");
}
jg_status launch_attn_bwd_sm100(const int64_t*, int64_t, int64_t, int, int, const void*, const void*, const void*,
                                const void*, const void*, const float*, void*, void*, void*, float*, float*,
                                const int2*, const int64_t*, int64_t, cudaStream_t) {
  return fail(JG_UNSUPPORTED, "tcgen05 attention not built");
}
}  // namespace jg
