// peaks.cu -- measured CUDA-core issue rates on this B200 (the ALU roofline denominators).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks tools/peaks.cu && tools/peaks
// Each kernel runs 8 independent dependency chains per thread, 148*8 CTAs x 256 threads, and
// reports thread-ops/s (FFMA / IMAD / IDP4A each count as one op; MACs = ops, or 4x for dp4a).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void k_ffma(float* out, float a, float b) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1234.5f) out[0] = s;
}

__global__ void k_ffma3(float* out, float a) {  // 3-register form: c varies
  float x[8], y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x * 0.001f + i; y[i] = i * 0.5f; }
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(y[i], a, x[i]);
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1234.5f) out[0] = s;
}

// packed fp32x2 FMA (sm_100: FFMA2): two FMAs per lane per instruction
__device__ __forceinline__ void ffma2(float2& x, float2 y, float2 a) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;"
      : "+l"(*reinterpret_cast<unsigned long long*>(&x))
      : "l"(*reinterpret_cast<unsigned long long*>(&y)), "l"(*reinterpret_cast<unsigned long long*>(&a)));
}
__global__ void k_ffma2(float* out, float a) {
  float2 x[8], y[8];
  const float2 a2 = make_float2(a, a);
#pragma unroll
  for (int i = 0; i < 8; ++i) { x[i] = make_float2(threadIdx.x * 0.001f + i, i); y[i] = make_float2(i * 0.5f, i * 0.25f); }
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) ffma2(x[i], y[i], a2);
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
  if (s == 1234.5f) out[0] = s;
}

__global__ void k_imad(int* out, int a) {
  int x[8], y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x + i; y[i] = i * 3 + 1; }
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = x[i] * a + y[i];
  int s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1234567) out[0] = s;
}

__global__ void k_dp4a(int* out, int a) {
  int x[8], y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x + i; y[i] = 0x01020304 * (i + 1); }
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __dp4a(y[i], a, x[i]);
  int s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1234567) out[0] = s;
}

template <typename F>
double rate(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double ops = double(sms) * 8 * 256 * kIters * 8;
  return ops / (best * 1e-3);
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* fo;
  int* io;
  cudaMalloc(&fo, 4);
  cudaMalloc(&io, 4);
  dim3 g(sms * 8), b(256);
  const double ffma = rate([&] { k_ffma<<<g, b>>>(fo, 1.0001f, 0.5f); });
  const double ffma3 = rate([&] { k_ffma3<<<g, b>>>(fo, 1.0001f); });
  const double ffma2 = 2.0 * rate([&] { k_ffma2<<<g, b>>>(fo, 1.0001f); });  // FMAs
  const double imad = rate([&] { k_imad<<<g, b>>>(io, 3); });
  const double dp4a = rate([&] { k_dp4a<<<g, b>>>(io, 0x01010101); });
  const double per = double(sms) * clk * 1e3;  // SM-cycles per second at the reported max clock
  printf("{\"sms\": %d, \"clock_mhz\": %.0f, \"ffma_imm_ops\": %.4g, \"ffma_3reg_ops\": %.4g, "
         "\"imad_ops\": %.4g, \"dp4a_ops\": %.4g, \"ffma_lanes_per_sm_clk\": %.1f, "
         "\"ffma3_lanes_per_sm_clk\": %.1f, \"imad_lanes_per_sm_clk\": %.1f, \"dp4a_lanes_per_sm_clk\": %.1f, "
         "\"ffma2_fma_per_sm_clk\": %.1f}\n",
         sms, clk / 1e3, ffma, ffma3, imad, dp4a, ffma / per, ffma3 / per, imad / per, dp4a / per, ffma2 / per);
  return 0;
}
