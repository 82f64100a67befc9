// Placeholder tcgen05 entry points (replaced by gemm_tc.cu / swa_tc.cu).
#include "gemm.h"
#include "swa.h"
namespace kl {
int gemm_tc(const GemmDesc&, const Epi&, cudaStream_t) { return KL_EUNSUPPORTED; }
int swa_fwd_tc(const SwaP&, cudaStream_t) { return KL_EUNSUPPORTED; }
int swa_bwd_tc(const SwaP&, cudaStream_t) { return KL_EUNSUPPORTED; }
}  // namespace kl
