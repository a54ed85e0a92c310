// Probe of tcgen05.mma kind::tf32 descriptor encodings (M=128).
// For each (A layout, B layout) case: fill smem from row-major fp32 A[M][K],
// B[N][K] with the layout formula, run K/8 MMAs, read TMEM, compare.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_1901_07988_b200/csrc/tc_common.cuh"
using namespace qt::tc;

// layout codes: 0 = K-major none, 1 = K-major SW(kbytes), 2 = MN-major SW(sw)
struct Lay { int kind; int sw; };

__device__ uint32_t swz(uint32_t off, int sw) {
  if (sw == 128) return off ^ (((off >> 7) & 7) << 4);
  if (sw == 64) return off ^ (((off >> 7) & 3) << 4);
  if (sw == 32) return off ^ (((off >> 7) & 1) << 4);
  return off;
}

// byte offset of element (r, k) for a tile with R rows and K cols
__device__ uint32_t lay_off(Lay L, int r, int k, int R, int K, uint32_t &lbo, uint32_t &sbo) {
  if (L.kind == 0) {  // K-major interleave: core 8 rows x 16B; LBO = K chunk stride, SBO = 8-row stride
    lbo = 128; sbo = (K / 4) * 128;
    return (r / 8) * sbo + (k / 4) * lbo + (r % 8) * 16 + (k % 4) * 4;
  }
  if (L.kind == 1) {  // K-major swizzled, row = K*4 bytes = sw
    sbo = 8 * L.sw; lbo = 16;
    uint32_t lo = (r / 8) * sbo + (r % 8) * L.sw + k * 4;
    return swz(lo, L.sw);
  }
  // MN-major swizzled: M atom = sw bytes of rows (sw/4 elements), 8 k-rows
  int me = L.sw / 4;
  lbo = K * L.sw;            // stride between M atoms
  sbo = 8 * L.sw;            // stride between 8-k groups
  uint32_t lo = (r / me) * lbo + (k / 8) * sbo + (k % 8) * L.sw + (r % me) * 4;
  return swz(lo, L.sw);
}

template <int N>
__global__ void probe(const float *A, const float *B, float *D, Lay la, Lay lb, int K) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t *sm = (uint8_t *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *sa = sm, *sb = sm + 128 * K * 4;
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint32_t alb, asb, blb, bsb;
  for (int i = threadIdx.x; i < 128 * K; i += blockDim.x) {
    int r = i / K, k = i % K;
    *(float *)(sa + lay_off(la, r, k, 128, K, alb, asb)) = A[i];
  }
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    int r = i / K, k = i % K;
    *(float *)(sb + lay_off(lb, r, k, N, K, blb, bsb)) = B[i];
  }
  lay_off(la, 0, 0, 128, K, alb, asb);
  lay_off(lb, 0, 0, N, K, blb, bsb);
  fence_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc<N < 32 ? 32 : N>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    uint32_t idesc = instr_desc(128, N, 2, la.kind == 2, lb.kind == 2);
    for (int j = 0; j < K / 8; ++j) {
      uint32_t aoff, boff;
      // k-step advance: K-major: 32 bytes within the row (none: 2 chunks = 2*LBO); MN-major: SBO
      if (la.kind == 0) aoff = j * 2 * alb; else if (la.kind == 1) aoff = j * 32; else aoff = j * asb;
      if (lb.kind == 0) boff = j * 2 * blb; else if (lb.kind == 1) boff = j * 32; else boff = j * bsb;
      uint64_t da = smem_desc(smem_u32(sa) + aoff, alb, asb, la.kind == 0 ? 0 : swizzle_layout(la.sw));
      uint64_t db = smem_desc(smem_u32(sb) + boff, blb, bsb, lb.kind == 0 ? 0 : swizzle_layout(lb.sw));
      mma_tf32(tmem, da, db, idesc, j > 0);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (threadIdx.x < 128) {
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
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<N < 32 ? 32 : N>(tmem); }
}

static float tf32(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return y; }

template <int N>
void run(Lay la, Lay lb, int K, const char *name) {
  std::vector<float> A(128 * K), B(N * K), D(128 * N), R(128 * N);
  srand(1);
  for (auto &v : A) v = (rand() % 17) - 8;
  for (auto &v : B) v = (rand() % 13) - 6;
  for (int m = 0; m < 128; ++m) for (int n = 0; n < N; ++n) {
    double s = 0; for (int k = 0; k < K; ++k) s += (double)tf32(A[m * K + k]) * tf32(B[n * K + k]);
    R[m * N + n] = s;
  }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, D.size() * 4);
  int smem = 128 * K * 4 + N * K * 4 + 2048;
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<N><<<1, 128, smem>>>(dA, dB, dD, la, lb, K);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double err = 0, ref = 0;
  for (size_t i = 0; i < D.size(); ++i) { err = fmax(err, fabs(D[i] - R[i])); ref = fmax(ref, fabs(R[i])); }
  printf("%-40s N=%3d K=%3d  err=%g ref=%g %s  D[0..3]=%g %g %g %g R=%g %g %g %g\n", name, N, K, err, ref,
         cudaGetErrorString(e), D[0], D[1], D[2], D[3], R[0], R[1], R[2], R[3]);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  if (e != cudaSuccess) exit(1);
}

int main() {
  run<16>({0, 0}, {0, 0}, 8, "Kmaj-none x Kmaj-none");
  run<16>({0, 0}, {0, 0}, 32, "Kmaj-none x Kmaj-none");
  run<64>({1, 128}, {1, 128}, 32, "Kmaj-SW128 x Kmaj-SW128");
  run<16>({1, 64}, {1, 64}, 16, "Kmaj-SW64 x Kmaj-SW64");
  run<16>({1, 32}, {1, 32}, 8, "Kmaj-SW32 x Kmaj-SW32");
  run<16>({2, 128}, {1, 128}, 32, "MN-SW128 x Kmaj-SW128");
  run<16>({2, 64}, {1, 64}, 16, "MN-SW64 x Kmaj-SW64");
  run<16>({2, 32}, {1, 32}, 8, "MN-SW32 x Kmaj-SW32");
  run<64>({2, 128}, {1, 64}, 16, "MN-SW128 x Kmaj-SW64");
  run<32>({2, 32}, {1, 128}, 32, "MN-SW32 x Kmaj-SW128");
  return 0;
}
