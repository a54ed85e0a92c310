// TMA issue rate: one thread issues N tile loads back-to-back (different smem
// destinations, one mbarrier), cycles per issue; box rows x 128 B.
#include <cstdio>
#include <cudaTypedefs.h>
#include "../../paper_1901_07988_b200/csrc/tc_common.cuh"
using namespace qt::tc;

__global__ void k(const __grid_constant__ CUtensorMap m, long long *out, int n, int rows) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); tma_prefetch(&m); }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int bytes = rows * 128;
    mbar_expect_tx(&bar, bytes * n);
    long long t0 = clock64();
    for (int i = 0; i < n; ++i)
      tma_load_2d(sm + (i % 8) * bytes, &m, &bar, 0, (i * rows) % 4096);
    long long t1 = clock64();
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[0] = t1 - t0; out[1] = t2 - t0;
  }
}
int main() {
  float *d; cudaMalloc(&d, 4096 * 32 * 4);
  long long *o; cudaMalloc(&o, 16);
  void *fnp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  for (int rows : {4, 16, 64}) {
    CUtensorMap m;
    cuuint64_t dims[2] = {32, 4096}; cuuint64_t str[1] = {128};
    cuuint32_t box[2] = {32, (cuuint32_t)rows}; cuuint32_t es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int n : {1, 8, 32}) {
      k<<<1, 32, 200000>>>(m, o, n, rows);
      cudaDeviceSynchronize();
      long long h[2]; cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
      printf("rows %2d n %2d: issue %lld cyc (%.0f/op), complete %lld cyc (%.0f B/cyc) %s\n", rows, n, h[0],
             (double)h[0] / n, h[1], (double)n * rows * 128 / h[1], cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
