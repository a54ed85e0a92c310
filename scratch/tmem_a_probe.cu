// Probe: tcgen05.mma kind::tf32 with the A operand in TMEM (lane = row m,
// column = k), B K-major SW128 in smem.  M=128, N=16/64, K=8..32.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include "../paper_1901_07988_b200/csrc/tc_common.cuh"
using namespace qt::tc;

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
               :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                  "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
}
__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
               :: "r"(d), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}

template <int N>
__global__ void probe(const float *A, const float *B, float *D, int K) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t *sb = (uint8_t *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  // B K-major SW128: row n = 128 B (32 tf32), 8-row atoms
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    int n = i / K, k = i % K;
    uint32_t off = (n / 8) * 1024 + (n % 8) * 128 + k * 4;
    off ^= ((off >> 7) & 7) << 4;
    *(float *)(sb + off) = B[i];
  }
  fence_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc<256>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem = slot;
  const uint32_t acol = 128;   // A at columns [128, 128+K)
  {  // thread t writes row t of A into TMEM lane t
    int w = threadIdx.x / 32;
    for (int c = 0; c < K; c += 16) {
      uint32_t r[16];
      for (int j = 0; j < 16; ++j) r[j] = __float_as_uint(A[threadIdx.x * K + c + j]);
      tmem_st16(tmem + ((32 * w) << 16) + acol + c, r);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    uint32_t idesc = instr_desc(128, N, 2, 0, 0);
    for (int j = 0; j < K / 8; ++j) {
      uint64_t db = smem_desc(smem_u32(sb) + j * 32, 16, 1024, 2);
      mma_tf32_ts(tmem, tmem + acol + j * 8, db, idesc, j > 0);
    }
    mma_commit(&bar);
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
static float tf32(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return y; }
template <int N> void run(int K) {
  std::vector<float> A(128 * K), B(N * K), D(128 * N), R(128 * N);
  srand(3);
  for (auto &v : A) v = (rand() % 17) - 8;
  for (auto &v : B) v = (rand() % 13) - 6;
  for (int m = 0; m < 128; ++m) for (int n = 0; n < N; ++n) { double s = 0; for (int k = 0; k < K; ++k) s += (double)tf32(A[m*K+k]) * tf32(B[n*K+k]); R[m*N+n] = s; }
  float *dA, *dB, *dD; cudaMalloc(&dA, A.size()*4); cudaMalloc(&dB, B.size()*4); cudaMalloc(&dD, D.size()*4);
  cudaMemcpy(dA, A.data(), A.size()*4, cudaMemcpyHostToDevice); cudaMemcpy(dB, B.data(), B.size()*4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, D.size()*4);
  int smem = N * 128 + 2048;
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<N><<<1, 128, smem>>>(dA, dB, dD, K);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D.data(), dD, D.size()*4, cudaMemcpyDeviceToHost);
  double err = 0; for (size_t i = 0; i < D.size(); ++i) err = fmax(err, fabs(D[i] - R[i]));
  printf("TMEM-A tf32 N=%d K=%d err=%g %s D=%g %g R=%g %g\n", N, K, err, cudaGetErrorString(e), D[0], D[1], R[0], R[1]);
  if (e) exit(1);
}
int main() { run<16>(8); run<16>(32); run<64>(32); run<128>(16); return 0; }
