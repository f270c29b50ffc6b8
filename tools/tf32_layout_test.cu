// tf32_layout_test.cu -- which descriptor field carries which stride for an MN-major kind::tf32 B
// operand (no swizzle), and whether tf32 inputs are truncated or rounded.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2006_13714_b200/csrc -o tools/tf32_layout_test tools/tf32_layout_test.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace scbm::sm100;

// A: 128 x 8 K-major canonical (groups of 8 rows x 16 B, 2 K-chunks): off = (m/8)*256 + kc*128 + (m%8)*16
// B: N = 128 MN-major, one K-group of 8: chunk j (4 n) x 8 k rows: off = j*CH + k*16 + (n%4)*4
__global__ void k_test(const float* A, const float* B, float* D, int variant, int bmode) {
  __shared__ __align__(1024) uint8_t sa[128 * 8 * 4];
  __shared__ __align__(1024) uint8_t sb[128 * 8 * 4 * 4];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  for (int e = tid; e < 128 * 8; e += blockDim.x) {
    const int m = e / 8, k = e % 8;
    *reinterpret_cast<float*>(sa + (m / 8) * 256 + (k / 4) * 128 + (m % 8) * 16 + (k % 4) * 4) = A[m * 8 + k];
  }
  const int CH = 128;
  for (int e = tid; e < 128 * 8; e += blockDim.x) {
    const int n = e / 8, k = e % 8;
    const float v = B[n * 8 + k];
    if (bmode == 0) *reinterpret_cast<float*>(sb + (n / 4) * CH + k * 16 + (n % 4) * 4) = v;  // MN-major
    else *reinterpret_cast<float*>(sb + (n / 8) * 256 + (k / 4) * 128 + (n % 8) * 16 + (k % 4) * 4) = v;  // K-major
  }
  const uint32_t sbar = uint32_t(__cvta_generic_to_shared(&bar));
  if (warp == 0) tmem_alloc(uint32_t(__cvta_generic_to_shared(&tslot)), 128);
  if (tid == 0) { mbar_init(sbar, 1); fence_barrier_init(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = tslot;
  if (tid == 0) {
    const uint32_t a0 = uint32_t(__cvta_generic_to_shared(sa)), b0 = uint32_t(__cvta_generic_to_shared(sb));
    const uint64_t da = smem_desc(a0, 128, 256);
    uint64_t db;
    if (bmode == 1) db = smem_desc(b0, 128, 256);
    else db = variant == 0 ? smem_desc(b0, 512, CH) : smem_desc(b0, CH, 512);
    const uint32_t idesc = idesc_tf32(128, 128, false, bmode == 0);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(da), "l"(db),
                 "r"(idesc), "r"(0u) : "memory");
    mma_commit(sbar);
  }
  __syncwarp();
  mbar_wait(sbar, 0);
  tc_fence_after();
  for (int c = 0; c < 128; c += 16) {
    uint32_t v[16];
    tmem_ld16(d + (uint32_t(32 * warp) << 16) + c, v);
    tmem_wait_ld();
    for (int i = 0; i < 16; ++i) D[(32 * warp + lane) * 128 + c + i] = __uint_as_float(v[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(d, 128); }
}

int main() {
  float hA[128 * 8], hB[128 * 8], hD[128 * 128];
  unsigned s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return float((s >> 8) & 0xffff) / 65536.0f - 0.5f; };
  for (auto& x : hA) x = rnd();
  for (auto& x : hB) x = rnd();
  float *A, *B, *D;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  auto trunc = [](float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xffffe000u; float r; memcpy(&r, &u, 4); return r; };
  for (int bmode = 0; bmode < 2; ++bmode)
    for (int variant = 0; variant < (bmode == 0 ? 2 : 1); ++variant) {
      k_test<<<1, 128>>>(A, B, D, variant, bmode);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
      double e_exact = 0, e_trunc = 0, e_round = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 128; ++n) {
          double ex = 0, et = 0;
          for (int k = 0; k < 8; ++k) {
            ex += double(hA[m * 8 + k]) * hB[n * 8 + k];
            et += double(trunc(hA[m * 8 + k])) * trunc(hB[n * 8 + k]);
          }
          e_exact = fmax(e_exact, fabs(hD[m * 128 + n] - ex));
          e_trunc = fmax(e_trunc, fabs(hD[m * 128 + n] - et));
        }
      printf("bmode %s variant %d (LBO,SBO)=%s: max|D-exact| %.3g  max|D-trunc| %.3g\n", bmode ? "K-major" : "MN-major",
             variant, bmode ? "(128,256)" : (variant == 0 ? "(512,128)" : "(128,512)"), e_exact, e_trunc);
    }
  return 0;
}
