// MMA issue rate (tf32, A in TMEM, N=48, 6 MMAs + 2 commits per stage) while
// other warps hammer TMEM with tcgen05.st (split-warp pattern) and/or
// tcgen05.ld (epilogue pattern), or spin on mbarrier try_wait.
#include <cstdio>
#include "../../paper_1901_07988_b200/csrc/tc_common.cuh"
using namespace qt::tc;
template <int MODE>   // 0 none, 1 st, 2 ld, 3 st+ld, 4 spin, 5 st+ld+spin
__global__ void k(long long *out, int iters, volatile int *stop) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t *sb = (uint8_t *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar[4]; __shared__ uint32_t slot; __shared__ int done;
  for (int i = threadIdx.x; i < 32 * 1024 / 4; i += blockDim.x) ((float *)sb)[i] = 1.0f;
  fence_async_smem();
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1); fence_barrier_init(); done = 0; }
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tmem = slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    uint32_t idesc = instr_desc(128, 48, 2, 0, 0);
    uint64_t db = smem_desc(smem_u32(sb), 16, 512, 4);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      tc_fence_after();
      if (elect_one()) {
        for (int j = 0; j < 6; ++j) mma_tf32_ts(tmem, tmem + 256 + (j & 1) * 8, db + (j & 1) * 2, idesc, 1);
        mma_commit(&bar[0]); mma_commit(&bar[1]);
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(&bar[3]);
    __syncwarp();
    mbar_wait(&bar[3], 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; done = 1; }
  } else {
    const int q = warp & 3;
    const uint32_t lb = tmem + ((uint32_t)(32 * q) << 16);
    uint32_t r[16];
    for (int j = 0; j < 16; ++j) r[j] = threadIdx.x + j;
    int it = 0;
    while (!*(volatile int *)&done && it < 200000) {
      ++it;
      if ((MODE == 1 || MODE == 3 || MODE == 5) && warp < 5) {   // 4 warps: st 2x16 cols
        tmem_st16(lb + 320, r); tmem_st16(lb + 336, r); tmem_wait_st();
      }
      if ((MODE == 2 || MODE == 3 || MODE == 5) && warp >= 5 && warp < 9) {   // 4 warps: ld 3x16 cols
        uint32_t a[16], b[16], c[16];
        tmem_ld16(lb + 0, a); tmem_ld16(lb + 48, b); tmem_ld16(lb + 96, c); tmem_wait_ld();
        for (int j = 0; j < 16; ++j) r[j] += a[j] ^ b[j] ^ c[j];
      }
      if ((MODE == 4 || MODE == 5) && warp >= 9) {   // spinners on an incomplete barrier
        uint32_t ok;
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar[2])), "r"(0u) : "memory");
      }
    }
    if (r[0] == 12345 && stop) *stop = r[1];
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}
template <int MODE> void run(const char *name) {
  long long *d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  k<MODE><<<1, 576, 40000>>>(d, 512, nullptr); cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-24s %.1f cyc per stage (6 tf32 MMAs N=48 + 2 commits)\n", name, (double)h / 512);
}
int main() {
  run<0>("alone"); run<1>("+ tcgen05.st warps"); run<2>("+ tcgen05.ld warps"); run<3>("+ st + ld");
  run<4>("+ mbarrier spinners"); run<5>("+ st + ld + spinners");
  return 0;
}
