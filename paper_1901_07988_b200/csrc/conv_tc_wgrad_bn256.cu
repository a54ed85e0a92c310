// Weight-gradient kernel instantiations for output-channel tiles of 256.
#include "conv_tc_wgrad.cuh"

namespace qt {
int wg_launch_bn256(const CUtensorMap &m, const CUtensorMap &mc, const WgParams &p, const WgPlan &pl,
                    cudaStream_t st) {
    return launch_wg<256>(m, mc, p, pl, st);
}
}  // namespace qt
