// TMA 4D tiled load with (possibly negative) start coordinates.
#include <cstdio>
#include <cstdlib>
#include <cudaTypedefs.h>
#include "../paper_1901_07988_b200/csrc/tc_common.cuh"
using namespace qt::tc;
__global__ void k(const __grid_constant__ CUtensorMap m, int c0, int c2, float *out, int nbytes) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t *sm = (uint8_t *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x == 0) { mbar_expect_tx(&bar, nbytes); tma_load_4d(sm, &m, &bar, c0, 0, c2, 0); }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < nbytes / 4; i += blockDim.x) out[i] = ((float *)sm)[i];
}
int main(int argc, char **argv) {
  int c0 = atoi(argv[1]), c2 = atoi(argv[2]), W = 32, C = 16, H = 32, N = 2;
  float *x; cudaMalloc(&x, W * C * H * N * 4);
  float *hx = (float *)malloc(W * C * H * N * 4);
  for (int i = 0; i < W * C * H * N; ++i) hx[i] = i;
  cudaMemcpy(x, hx, W * C * H * N * 4, cudaMemcpyHostToDevice);
  void *p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  CUtensorMap m;
  cuuint64_t dims[4] = {(cuuint64_t)W, (cuuint64_t)C, (cuuint64_t)H, (cuuint64_t)N};
  cuuint64_t st[3] = {(cuuint64_t)H * W * 4, (cuuint64_t)W * 4, (cuuint64_t)C * H * W * 4};
  cuuint32_t box[4] = {32, 16, 4, 1}, es[4] = {1, 1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  float *out; cudaMalloc(&out, 32 * 16 * 4 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  k<<<1, 128, 16384>>>(m, c0, c2, out, 32 * 16 * 4 * 4);
  cudaError_t e = cudaDeviceSynchronize();
  float ho[8]; cudaMemcpy(ho, out, 32, cudaMemcpyDeviceToHost);
  printf("c0=%d c2=%d encode=%d err=%s first=%g %g %g %g\n", c0, c2, (int)r, cudaGetErrorString(e), ho[0], ho[1], ho[2], ho[3]);
  return 0;
}
