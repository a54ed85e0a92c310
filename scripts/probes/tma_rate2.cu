// TMA issue rate for the conv kernel's box shapes: A 4D (w=32, c=16, h=4, n=1)
// and B 3D (ci=16, co=16, taps=3), interleaved as in the producer loop.
#include <cstdio>
#include <cudaTypedefs.h>
#include "../../paper_1901_07988_b200/csrc/tc_common.cuh"
using namespace qt::tc;

__global__ void k(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                  long long *out, int n, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); tma_prefetch(&ma); tma_prefetch(&mb); }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int abytes = 32 * 16 * 4 * 4, bbytes = 16 * 16 * 3 * 4;
    int per = (mode == 0 ? abytes : mode == 1 ? bbytes : abytes + 2 * bbytes);
    mbar_expect_tx(&bar, per * n);
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
      uint8_t *dst = sm + (i % 4) * 32768;
      if (mode == 0 || mode == 2) tma_load_4d(dst, &ma, &bar, 0, 0, (i * 4) % 32 - 1, i % 128);
      if (mode == 1 || mode == 2) {
        tma_load_3d(dst + 8192, &mb, &bar, 0, 0, (i % 3) * 3);
        if (mode == 2) tma_load_3d(dst + 8192 + 3072, &mb, &bar, 0, 0, (i % 3) * 3);
      }
    }
    long long t1 = clock64();
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[0] = t1 - t0; out[1] = t2 - t0;
  }
}
int main() {
  float *x, *w; cudaMalloc(&x, 128ull * 16 * 32 * 32 * 4); cudaMalloc(&w, 9 * 16 * 16 * 4);
  long long *o; cudaMalloc(&o, 16);
  void *fnp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
  CUtensorMap ma, mb;
  { cuuint64_t dims[4] = {32, 16, 32, 128}; cuuint64_t str[3] = {32 * 32 * 4, 32 * 4, 16 * 32 * 32 * 4};
    cuuint32_t box[4] = {32, 16, 4, 1}; cuuint32_t es[4] = {1, 1, 1, 1};
    printf("enc a %d\n", (int)enc(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)); }
  { cuuint64_t dims[3] = {16, 16, 9}; cuuint64_t str[2] = {16 * 4, 16 * 16 * 4};
    cuuint32_t box[3] = {16, 16, 3}; cuuint32_t es[3] = {1, 1, 1};
    printf("enc b %d\n", (int)enc(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)); }
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  const char *nm[3] = {"A 4D", "B 3D", "A+2B"};
  for (int mode = 0; mode < 3; ++mode)
    for (int n : {1, 8, 32}) {
      k<<<1, 32, 200000>>>(ma, mb, o, n, mode);
      cudaDeviceSynchronize();
      long long h[2]; cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
      printf("%s n %2d: issue %lld cyc (%.0f/iter), complete %lld cyc (%.0f /iter) %s\n", nm[mode], n, h[0],
             (double)h[0] / n, h[1], (double)h[1] / n, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
