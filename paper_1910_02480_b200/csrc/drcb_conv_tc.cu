// drcb_conv_tc.cu — tensor-core (tcgen05 / TMEM / TMA) implicit-GEMM engine
// for the autoencoder. Placeholder until the kernel lands.
#include "drcb_net.h"

namespace drcb {
int forward_tc(NetImpl& net, const float* x, float* y, int64_t n, int mode, cudaStream_t st) {
  (void)net; (void)x; (void)y; (void)n; (void)mode; (void)st;
  return fail(DRCB_ECONFIG, "tensor-core network mode not built yet");
}
}  // namespace drcb
