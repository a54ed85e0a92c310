// Weight-gradient kernel instantiations for output-channel tiles of 128.
#include "conv_tc_wgrad.cuh"

namespace qt {
int wg_launch_bn128(const CUtensorMap &m, const CUtensorMap &mc, const WgParams &p, const WgPlan &pl,
                    cudaStream_t st) {
    return launch_wg<128>(m, mc, p, pl, st);
}
}  // namespace qt
