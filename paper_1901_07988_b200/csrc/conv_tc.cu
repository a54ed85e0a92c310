// tcgen05 (5th-gen tensor core) implicit-GEMM convolutions -- placeholder
// until the UMMA path lands; every shape is routed to the SIMT kernels.
#include "common.cuh"

int qt_tc_conv_forward(const float *, const float *, float *, const qt::ConvGeo &, const float *,
                       int64_t, int64_t, cudaStream_t) {
    return QT_EUNSUPPORTED;
}
