// The conv kernel's MMA-warp loop in isolation (completed barriers): which
// part of a stage costs.  VARIANT bits: 1 mbar_wait per stage, 2 clock64
// trace stores, 4 per-stage descriptor build, 8 (i|j) accumulate predicate.
#include <cstdio>
#include "../../paper_1901_07988_b200/csrc/tc_common.cuh"
using namespace qt::tc;
template <int VARIANT>
__global__ void k(long long *out, long long *tr, int iters) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t *sb = (uint8_t *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar[8]; __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 32 * 1024 / 4; i += blockDim.x) ((float *)sb)[i] = 1.0f;
  fence_async_smem();
  if (threadIdx.x == 0) { for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x == 0) { mbar_arrive(&bar[4]); }   // bar[4]: completed phase 0
  __syncthreads();
  uint32_t tmem = slot;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    constexpr uint32_t idesc = instr_desc(128, 48, 2, 0, 0);
    uint64_t db0 = smem_desc(smem_u32(sb), 16, 512, 4);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if ((VARIANT & 2) && lane == 0) tr[(i & 63) * 8 + 6] = clock64();
      if (VARIANT & 1) mbar_wait(&bar[4], 0);
      if ((VARIANT & 2) && lane == 0) tr[(i & 63) * 8 + 4] = clock64();
      tc_fence_after();
      if (elect_one()) {
        const uint32_t ah = tmem + 256 + (i & 7) * 32, al = ah + 16;
        uint64_t dbh = db0, dbl = db0 + 64;
        if (VARIANT & 4) {
          dbh = smem_desc(smem_u32(sb + (i % 3) * 3072), 16, 512, 4);
          dbl = smem_desc(smem_u32(sb + 16384 + (i % 3) * 3072), 16, 512, 4);
        }
        const int ii = (VARIANT & 8) ? (i % 3) : 1;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          mma_tf32_ts(tmem, ah + j * 8, dbh + j * 2, idesc, (ii | j) ? 1u : 0u);
          mma_tf32_ts(tmem, ah + j * 8, dbl + j * 2, idesc, 1u);
          mma_tf32_ts(tmem, al + j * 8, dbh + j * 2, idesc, 1u);
        }
        mma_commit(&bar[0]); mma_commit(&bar[1]);
      }
      __syncwarp();
      if ((VARIANT & 2) && lane == 0) tr[(i & 63) * 8 + 5] = clock64();
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
template <int V> void run() {
  long long *d, *tr; cudaMalloc(&d, 8); cudaMalloc(&tr, 8 * 1024);
  cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  k<V><<<1, 576, 40000>>>(d, tr, 512); cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("variant %2d (wait=%d trace=%d desc=%d pred=%d): %.1f cyc per stage\n", V, V & 1, (V >> 1) & 1, (V >> 2) & 1, (V >> 3) & 1, (double)h / 512);
}
int main() { run<0>(); run<1>(); run<2>(); run<4>(); run<8>(); run<15>(); return 0; }
