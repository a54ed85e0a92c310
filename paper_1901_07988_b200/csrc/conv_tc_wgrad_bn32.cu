// Weight-gradient kernel instantiations for output-channel tiles of 32.
#include "conv_tc_wgrad.cuh"

namespace qt {
int wg_launch_bn32(const CUtensorMap &m, const CUtensorMap &mc, const WgParams &p, const WgPlan &pl,
                    cudaStream_t st) {
    return launch_wg<32>(m, mc, p, pl, st);
}
}  // namespace qt
