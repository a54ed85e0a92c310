// Cost of the MMA-issuer loop pieces: tcgen05.mma (ts, bf16, N=48) x2 per
// iteration, with/without per-iteration commit and fence.
#include <cstdio>
#include "../paper_1901_07988_b200/csrc/tc_common.cuh"
using namespace qt::tc;

template <int MODE>
__global__ void k(long long *out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t *sb = (uint8_t *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar[4];
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) ((uint32_t *)sb)[i] = 0x3f803f80u;
  fence_async_smem();
  if (threadIdx.x == 0) { for (int j = 0; j < 4; ++j) mbar_init(&bar[j], 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tmem = slot;
  if (threadIdx.x < 32) {
    const uint32_t idesc = instr_desc(128, 48, 1, 0, 0);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (MODE >= 2) tc_fence_after();
      if (elect_one()) {
        const uint32_t gb = smem_u32(sb) + (i & 3) * 8192;
        const uint32_t a = tmem + 256 + (i & 3) * 16;
        for (int j = 0; j < 2; ++j)
          mma_bf16_ts(tmem, a + j * 8, smem_desc(gb + j * 32, 16, 512, 4), idesc, 1u);
        if (MODE >= 1) mma_commit(&bar[i & 3]);
      }
      __syncwarp();
    }
    long long t1 = clock64();
    if (elect_one()) mma_commit(&bar[0]);
    __syncwarp();
    out[0] = t1 - t0;
  }
  __syncthreads();
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}
template <int MODE> void run() {
  long long *d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  k<MODE><<<1, 128, 70000>>>(d, 256); cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("mode %d: %.1f cycles/iter (2 MMAs)  %s\n", MODE, h / 256.0, cudaGetErrorString(cudaGetLastError()));
}
int main() { run<0>(); run<1>(); run<2>(); return 0; }
