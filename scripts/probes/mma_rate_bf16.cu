// Throughput of back-to-back tcgen05.mma kind::f16 (bf16), M=128, K=16, A in TMEM or SMEM.
#include <cstdio>
#include "../../paper_1901_07988_b200/csrc/tc_common.cuh"
using namespace qt::tc;
template <int N, bool TS>
__global__ void k(long long *out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t *sb = (uint8_t *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar; __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t *)sb)[i] = 0x3f803f80u;
  fence_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    uint32_t idesc = instr_desc(128, N, 1, 0, 0);
    uint64_t db = smem_desc(smem_u32(sb), 16, 512, 4);
    uint64_t da = smem_desc(smem_u32(sb) + 32768, 16, 512, 4);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (TS) mma_bf16_ts(tmem, tmem + 256 + (i & 1) * 8, db + (i & 1) * 2, idesc, 1);
      else mma_bf16(tmem, da + (i & 1) * 2, db + (i & 1) * 2, idesc, 1);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[0] = t1 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}
template <int N, bool TS> void run() {
  long long *d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  for (int it : {64, 512}) {
    k<N, TS><<<1, 128, 70000>>>(d, it); cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("bf16 N=%3d %s iters=%4d per-mma=%.1f cyc  (128xNx16 MAC / 4096 = %d)\n", N, TS ? "A=TMEM" : "A=SMEM", it, (double)h / it, 128 * N * 16 / 4096);
  }
}
int main() { run<64, true>(); run<64, false>(); run<128, true>(); run<128, false>(); run<192, true>(); run<192, false>(); run<256, true>(); run<256, false>(); return 0; }
