// nlm.cuh -- one reference row of NLM weights (Eq. 2), normalised in place by
// one warp: clipped slots hold -1 (weight 0), d_min is subtracted before the exponential (the
// ratio is unchanged: numerator and Theta_i share exp(d_min / h^2)), then Theta_i normalises.
// Shared by the stand-alone nlm_normalize kernel and the dense matcher's fused epilogue.
#pragma once
#include <math.h>

namespace scbm {

template <typename T>
__device__ __forceinline__ void nlm_normalize_row(void* row, int slots, float inv_h2, int lane) {
  T* d = static_cast<T*>(row);
  float* w = static_cast<float*>(row);
  float dmin = __int_as_float(0x7f800000);
  for (int k = lane; k < slots; k += 32) {
    const float v = float(d[k]);
    // clipped slots hold -1; a float identity distance may round slightly below 0 (clamped)
    if (v > -0.5f) dmin = fminf(dmin, fmaxf(v, 0.f));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmin = fminf(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
  float theta = 0.f;
  for (int k = lane; k < slots; k += 32) {
    const float v = float(d[k]);
    const float e = v > -0.5f ? expf(-(fmaxf(v, 0.f) - dmin) * inv_h2) : 0.f;
    w[k] = e;  // in place: the same slot, read before it is written by this lane
    theta += e;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) theta += __shfl_xor_sync(0xffffffffu, theta, o);
  const float inv = 1.f / theta;
  for (int k = lane; k < slots; k += 32) w[k] *= inv;
}

}  // namespace scbm
