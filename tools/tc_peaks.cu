// tc_peaks.cu -- measured tcgen05 peaks on this B200: the tensor-core roofline
// denominators the bench line quotes, instead of assuming int8 = 2x and tf32 = 1/2x bf16.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2006_13714_b200/csrc \
//        -o tools/tc_peaks tools/tc_peaks.cu && tools/tc_peaks
//
// * MMA rate: one CTA per SM, one elected thread issues back-to-back tcgen05.mma.cta_group::1
//   (M = 128, N = 256, A and B from shared memory, no-swizzle K-major canonical layouts) into
//   one TMEM accumulator, for kind::i8 (K = 32 per instruction), kind::f16 with bf16 operands
//   (K = 16) and kind::tf32 (K = 8); MACs = 148 * iters * 128 * 256 * K.
// * TMEM read rate: W warps per CTA (one CTA per SM) stream tcgen05.ld.32x32b.x32 over the
//   512 allocated columns; bytes = 128 B per warp-column.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace scbm::sm100;

// kind::f16 / kind::tf32 instruction descriptor: D f32, A/B format fmt (1 = bf16, 2 = tf32), both K-major.
__host__ __device__ constexpr uint32_t idesc_f(int M, int N, uint32_t fmt) {
  return (1u << 4) | (fmt << 7) | (fmt << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc),
               "r"(acc)
               : "memory");
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b),
               "r"(idesc), "r"(acc)
               : "memory");
}

// kind: 0 = i8, 1 = bf16, 2 = tf32
template <int KIND>
__global__ void __launch_bounds__(128, 1) k_mma(int iters, int n, unsigned long long* sink) {
  __shared__ __align__(1024) uint8_t sm[128 * 32 + 256 * 32];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < int(sizeof(sm)) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  const int warp = threadIdx.x / 32;
  const uint32_t sbar = uint32_t(__cvta_generic_to_shared(&bar));
  if (warp == 0) tmem_alloc(uint32_t(__cvta_generic_to_shared(&tbase)), 256);
  if (threadIdx.x == 32) { mbar_init(sbar, 1); fence_barrier_init(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = tbase;
  if (threadIdx.x == 0) {
    const uint32_t a0 = uint32_t(__cvta_generic_to_shared(sm));
    // 32 bytes of K per row: core matrices [row group][k chunk][8 rows][16 B]: LBO = 128, SBO = 256
    const uint64_t da = smem_desc(a0, 128, 256), db = smem_desc(a0 + 128 * 32, 128, 256);
    for (int it = 0; it < iters; ++it) {
      if (KIND == 0) mma_i8(d, da, db, idesc_i8(128, n, false, false), it > 0);
      if (KIND == 1) mma_f16(d, da, db, idesc_f(128, n, 1), it > 0);
      if (KIND == 2) mma_tf32(d, da, db, idesc_f(128, n, 2), it > 0);
    }
    mma_commit(sbar);
  }
  __syncwarp();
  if (warp == 0) mbar_wait(sbar, 0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    uint32_t v[16];
    tmem_ld16(d, v);
    tmem_wait_ld();
    if (v[0] == 0x12345678u) sink[0] = v[1];
    tmem_dealloc(d, 256);
  }
}

// TMEM -> register streaming: every warp reads its lane quarter, columns [c0, c0+256) x reps.
template <int X>
__global__ void __launch_bounds__(512, 1) k_ldtm(int reps, unsigned long long* sink) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(uint32_t(__cvta_generic_to_shared(&tbase)), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
  const uint32_t col0 = (warp >> 2) * 64;  // warps sharing a quarter read different columns
  uint32_t acc = 0;
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int c = 0; c < 256; c += X) {
      uint32_t v[32];
      const uint32_t ta = tbase + lane_base + ((col0 + c) & 511);
      if (X == 32) {
        tmem_ld32(ta, v);
      } else {
        uint32_t (&w)[16] = *reinterpret_cast<uint32_t(*)[16]>(v);
        tmem_ld16(ta, w);
      }
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < X; ++i) acc ^= v[i];
    }
  }
  if (acc == 0x9abcdef1u) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

template <typename F>
static float best_ms(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 7; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  const int iters = 20000;
  const double per = double(sms) * clk * 1e3;
  printf("{\"sms\": %d, \"clock_mhz\": %.0f", sms, clk / 1e3);
  const int kk[3] = {32, 16, 8};
  const char* names[3] = {"i8", "bf16", "tf32"};
  for (int kind = 0; kind < 3; ++kind) {
    for (int n : {128, 256}) {
      float ms;
      if (kind == 0) ms = best_ms([&] { k_mma<0><<<sms, 128>>>(iters, n, sink); });
      else if (kind == 1) ms = best_ms([&] { k_mma<1><<<sms, 128>>>(iters, n, sink); });
      else ms = best_ms([&] { k_mma<2><<<sms, 128>>>(iters, n, sink); });
      const double macs = double(sms) * iters * 128.0 * n * kk[kind];
      printf(", \"%s_m128n%d_tops\": %.1f, \"%s_m128n%d_mac_per_sm_clk\": %.0f", names[kind], n,
             2 * macs / (ms * 1e-3) / 1e12, names[kind], n, macs / (ms * 1e-3) / per);
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf(", \"mma_error\": \"%s\"", cudaGetErrorString(e));
  const int reps = 2000;
  for (int w : {4, 8, 16}) {
    for (int x : {16, 32}) {
      float ms = x == 32 ? best_ms([&] { k_ldtm<32><<<sms, 32 * w>>>(reps, sink); })
                         : best_ms([&] { k_ldtm<16><<<sms, 32 * w>>>(reps, sink); });
      const double bytes = double(sms) * w * reps * 256.0 * 128.0;  // 256 columns x 32 lanes x 4 B per warp
      printf(", \"ldtm_x%d_w%d_bytes_per_sm_clk\": %.1f", x, w, bytes / (ms * 1e-3) / per);
    }
  }
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf(", \"error\": \"%s\"", cudaGetErrorString(e));
  printf("}\n");
  return 0;
}
