// tf32_tmem_a_test.cu -- tcgen05.mma kind::tf32 with the A operand in TMEM (written by tcgen05.st,
// lane m = row m, column k = element k) and a K-major B in shared memory: D vs a CPU product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2006_13714_b200/csrc -o tools/tf32_tmem_a_test tools/tf32_tmem_a_test.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace scbm::sm100;

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

// D[128][N] = A[128][16] (TMEM, two K=8 steps) x B[N][16]^T (smem K-major)
__global__ void k_test(const float* A, const float* B, float* D, int N) {
  __shared__ __align__(1024) uint8_t sb[256 * 16 * 4];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  for (int e = tid; e < N * 16; e += blockDim.x) {
    const int n = e / 16, k = e % 16;
    // K-major canonical: [n/8 group][k/4 chunk (4 chunks)][n%8][k%4]: LBO 128, SBO 512
    *reinterpret_cast<float*>(sb + (n / 8) * 512 + (k / 4) * 128 + (n % 8) * 16 + (k % 4) * 4) = B[n * 16 + k];
  }
  const uint32_t sbar = uint32_t(__cvta_generic_to_shared(&bar));
  if (warp == 0) tmem_alloc(uint32_t(__cvta_generic_to_shared(&tslot)), 256);
  if (tid == 0) { mbar_init(sbar, 1); fence_barrier_init(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = tslot;
  // A at columns [0, 16), D at [128, 128 + N)
  {
    const int m = 32 * warp + lane;
    uint32_t v[8];
    for (int c = 0; c < 2; ++c) {
      for (int i = 0; i < 8; ++i) v[i] = __float_as_uint(A[m * 16 + 8 * c + i]);
      tmem_st8(base + (uint32_t(32 * warp) << 16) + 8 * c, v);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t b0 = uint32_t(__cvta_generic_to_shared(sb));
    const uint32_t idesc = idesc_tf32(128, N, false, false);
    for (int s = 0; s < 2; ++s) {
      const uint64_t db = smem_desc(b0 + 256u * s, 128, 512);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(base + 128),
                   "r"(base + 8 * s), "l"(db), "r"(idesc), "r"(s) : "memory");
    }
    mma_commit(sbar);
  }
  __syncwarp();
  mbar_wait(sbar, 0);
  tc_fence_after();
  for (int c = 0; c < N; c += 16) {
    uint32_t v[16];
    tmem_ld16(base + (uint32_t(32 * warp) << 16) + 128 + c, v);
    tmem_wait_ld();
    for (int i = 0; i < 16; ++i) D[(32 * warp + lane) * N + c + i] = __uint_as_float(v[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(base, 256); }
}

int main() {
  const int N = 64;
  float hA[128 * 16], hB[N * 16], hD[128 * N];
  unsigned s = 777;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return float((s >> 8) & 0xffff) / 65536.0f - 0.5f; };
  for (auto& x : hA) x = rnd();
  for (auto& x : hB) x = rnd();
  float *A, *B, *D;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  k_test<<<1, 128>>>(A, B, D, N);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
  auto trunc = [](float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xffffe000u; float r; memcpy(&r, &u, 4); return r; };
  double et = 0, ex = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double a = 0, b = 0;
      for (int k = 0; k < 16; ++k) { a += double(trunc(hA[m * 16 + k])) * trunc(hB[n * 16 + k]); b += double(hA[m * 16 + k]) * hB[n * 16 + k]; }
      et = fmax(et, fabs(hD[m * N + n] - a));
      ex = fmax(ex, fabs(hD[m * N + n] - b));
    }
  printf("A in TMEM, kind::tf32, N=%d: max|D-trunc| %.3g  max|D-exact| %.3g\n", N, et, ex);
  return 0;
}
