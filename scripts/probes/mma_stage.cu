// Per-"stage" cost of the conv MMA issue loop: wait a completed mbarrier,
// fence, 6 x tcgen05.mma kind::tf32 (A in TMEM, N = 48 / 96), 2 commits.
#include <cstdio>
#include "../../paper_1901_07988_b200/csrc/tc_common.cuh"
using namespace qt::tc;
template <int N, int NMMA, int NCOMMIT>
__global__ void k(long long *out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t *sb = (uint8_t *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar[4]; __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 32 * 1024 / 4; i += blockDim.x) ((float *)sb)[i] = 1.0f;
  fence_async_smem();
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tmem = slot;
  if (threadIdx.x < 32) {
    uint32_t idesc = instr_desc(128, N, 2, 0, 0);
    uint64_t db = smem_desc(smem_u32(sb), 16, 512, 4);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      tc_fence_after();
      if (elect_one()) {
        for (int j = 0; j < NMMA; ++j) mma_tf32_ts(tmem, tmem + 256 + (j & 1) * 8, db + (j & 1) * 2, idesc, 1);
        for (int c = 0; c < NCOMMIT; ++c) mma_commit(&bar[c]);
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(&bar[3]);
    __syncwarp();
    mbar_wait(&bar[3], 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}
template <int N, int NMMA, int NCOMMIT> void run() {
  long long *d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k<N, NMMA, NCOMMIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  k<N, NMMA, NCOMMIT><<<1, 128, 40000>>>(d, 256); cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("tf32 N=%3d mma/stage=%d commits/stage=%d: %.1f cyc per stage (%.1f per mma)\n", N, NMMA, NCOMMIT, (double)h / 256, (double)h / 256 / NMMA);
}
int main() {
  run<48, 6, 0>(); run<48, 6, 1>(); run<48, 6, 2>(); run<48, 6, 3>();
  run<96, 6, 2>(); run<48, 4, 2>(); run<16, 6, 2>(); run<64, 6, 2>(); run<128, 6, 2>();
  return 0;
}
