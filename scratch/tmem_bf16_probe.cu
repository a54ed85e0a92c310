// Probe: tcgen05.mma kind::f16 (bf16) with A in TMEM (lane = row m, column j
// holds k = 2j (low half) and 2j+1 (high half)), B K-major SW64 in smem
// (row = 32 bf16 = 64 B).  Also: back-to-back rate, and the bf16x2
// magic-number decode (0x4300 + t, fma.rn.relu(x, 1, -128)).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_bf16.h>
#include "../paper_1901_07988_b200/csrc/tc_common.cuh"
using namespace qt::tc;

__device__ __forceinline__ void mma_bf16_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               :: "r"(d), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
static __host__ __device__ uint16_t bf(float x) { uint32_t u; memcpy(&u, &x, 4); return (uint16_t)(u >> 16); }

template <int N>
__global__ void probe(const float *A, const float *B, float *D, int K, long long *cyc, int iters) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t *sb = (uint8_t *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {   // K = 32 exactly: one 64-B row
    int n = i / K, k = i % K;
    uint32_t off = (n / 8) * 512 + (n % 8) * 64 + k * 2;
    off = swz_off<64>(off);
    *(uint16_t *)(sb + off) = bf(B[i]);
  }
  fence_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc<256>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem = slot;
  const uint32_t acol = 128;
  {
    int w = threadIdx.x / 32;
    uint32_t r[16];
    for (int j = 0; j < 16; ++j)
      r[j] = (uint32_t)bf(A[threadIdx.x * K + 2 * j]) | ((uint32_t)bf(A[threadIdx.x * K + 2 * j + 1]) << 16);
    tmem_st16(tmem + ((32 * w) << 16) + acol, r);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    uint32_t idesc = instr_desc(128, N, 1, 0, 0);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
      for (int j = 0; j < 2; ++j) {
        uint64_t db = smem_desc(smem_u32(sb) + j * 32, 16, 512, 4);
        mma_bf16_ts(tmem, tmem + acol + j * 8, db, idesc, (it | j) > 0);
      }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    cyc[0] = clock64() - t0;
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  {
    int w = threadIdx.x / 32;
    for (int c = 0; c < N; c += 16) {
      uint32_t r[16];
      tmem_ld16(tmem + ((32 * w) << 16) + c, r);
      tmem_wait_ld();
      for (int j = 0; j < 16; ++j) D[threadIdx.x * N + c + j] = __uint_as_float(r[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<256>(tmem); }
}

__global__ void magic(int *out) {
  // t in [-200, 140): lane = 0x4300 + t; relu(x - 128) should equal max(t, 0) for t < 128
  int t = threadIdx.x - 200;
  uint32_t lane = (uint32_t)(0x4300 + t);
  uint32_t x = lane | (lane << 16);
  uint32_t one = 0x3F803F80u, m128 = 0xC300C300u, y;
  asm("fma.rn.relu.bf16x2 %0, %1, %2, %3;" : "=r"(y) : "r"(x), "r"(one), "r"(m128));
  float lo = __uint_as_float((y & 0xFFFFu) << 16), hi = __uint_as_float(y & 0xFFFF0000u);
  out[threadIdx.x] = (lo == (float)(t > 0 ? t : 0) && hi == lo && !signbit(lo)) ? 1 : 0;
}

template <int N> void run(int iters) {
  const int K = 32;
  std::vector<float> A(128 * K), B(N * K), D(128 * N), R(128 * N);
  srand(1);
  for (auto &v : A) v = (rand() % 31) - 15;
  for (auto &v : B) v = ((rand() % 255) - 127) / 64.0f;
  for (int m = 0; m < 128; ++m) for (int n = 0; n < N; ++n) {
    double s = 0; for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[n * K + k];
    R[m * N + n] = (float)(s * iters);
  }
  float *dA, *dB, *dD; long long *dc;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4); cudaMalloc(&dc, 8);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  int smem = 64 * 1024;
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<N><<<1, 128, smem>>>(dA, dB, dD, K, dc, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long cyc; cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double err = 0, ref = 0;
  for (size_t i = 0; i < D.size(); ++i) { err = fmax(err, fabs(D[i] - R[i])); ref = fmax(ref, fabs(R[i])); }
  printf("bf16 ts N=%3d iters=%4d err=%g ref=%g %s  cycles/mma=%.1f\n", N, iters, err, ref, cudaGetErrorString(e),
         (double)cyc / (2 * iters));
}
int main() {
  run<16>(1); run<16>(256); run<32>(256); run<64>(256); run<128>(256); run<256>(256);
  int *d; cudaMalloc(&d, 340 * 4); magic<<<1, 340>>>(d); int h[340]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  int bad = 0; for (int i = 0; i < 328; ++i) bad += !h[i];   // t < 128
  int hi_ok = 0; for (int i = 328; i < 340; ++i) hi_ok += h[i];
  printf("magic relu: bad(t<128)=%d  ok(t>=128, expected inexact)=%d\n", bad, hi_ok);
  return 0;
}
