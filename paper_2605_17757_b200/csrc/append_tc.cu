// Tensor-core quantize_append (variant 0) — see DESIGN.md §7.
#include "common.cuh"

namespace oscar {

bool append_tc_supported(const oscar_ctx& c) { (void)c; return false; }

cudaError_t launch_append_tc(const oscar_ctx& c, const void* K, const void* V,
                             const int64_t* slots, int64_t T, const float* RK, const float* RV,
                             void* pool, cudaStream_t s) {
  (void)c; (void)K; (void)V; (void)slots; (void)T; (void)RK; (void)RV; (void)pool; (void)s;
  return cudaErrorNotSupported;
}

}  // namespace oscar
