// tc_fused.cu -- placeholder: routed to the SIMT kernel until the tcgen05 kernel lands.
#include "kernels.h"
namespace splat {
cudaError_t launch_mhsa_tc(const DevAcsr &A, const void *Q, const void *K, const void *V, int BH, int d,
                           float scale, void *O, cudaStream_t st, int *n_launch)
{
    *n_launch = 1;
    return launch_mhsa_simt(A, Q, K, V, true, BH, d, scale, O, st);
}
}  // namespace splat
