// tcgen05 (5th-gen tensor core) implicit-GEMM conv -- placeholder until the
// kernel lands; every conv runs on the SIMT path meanwhile.
#include "kernels.cuh"
#include "tc_layout.cuh"

namespace pcnn {

bool conv_tc_supported(const ConvArgs&) { return false; }
void launch_conv_tc(const ConvArgs&, cudaStream_t) {}

}  // namespace pcnn
