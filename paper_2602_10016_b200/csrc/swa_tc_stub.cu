// tcgen05 sliding-window attention entry points (placeholder until swa_tc.cu
// lands: returning KL_EUNSUPPORTED routes bf16 to the SIMT flash kernels).
#include "swa.h"
namespace kl {
int swa_fwd_tc(const SwaP&, cudaStream_t) { return KL_EUNSUPPORTED; }
int swa_bwd_tc(const SwaP&, cudaStream_t) { return KL_EUNSUPPORTED; }
}  // namespace kl
