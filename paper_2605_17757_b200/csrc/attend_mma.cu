// Tensor-core split-K decode attention (variant 0) — see DESIGN.md §7.
#include "attend_common.cuh"

namespace oscar {

bool attend_mma_supported(const oscar_ctx& c) { (void)c; return false; }

cudaError_t launch_attend_mma(const AttnParams& p, cudaStream_t s) {
  (void)p; (void)s;
  return cudaErrorNotSupported;
}

}  // namespace oscar
