// nlm.cuh -- one reference row of NLM weights (Eq. 2), normalised in place by
// one warp: clipped slots (decided from the window geometry) get weight 0, d_min is subtracted before the exponential (the
// ratio is unchanged: numerator and Theta_i share exp(d_min / h^2)), then Theta_i normalises.
// Shared by the stand-alone nlm_normalize kernel and the dense matcher's fused epilogue.
#pragma once
#include <math.h>

namespace scbm {

// A slot is a real candidate iff its window position lies inside the image (footnote 2,
// PAPER.md:280): decided from the geometry (slot k = (dy, dx) = (k / Wn + lo, k % Wn + lo) of the
// reference at (ry, rx), valid iff 0 <= ry + dy <= cy_max and 0 <= rx + dx <= cx_max), never from
// the stored value, so a real distance that rounds below 0 (fp32 identity cancellation on inputs
// of any scale) keeps its weight; real distances are clamped at 0.
struct NlmRowGeom {
  int ry, rx, cy_max, cx_max, Wn, lo;
};

template <typename T>
__device__ __forceinline__ void nlm_normalize_row(void* row, const NlmRowGeom& gm, float inv_h2, int lane) {
  T* d = static_cast<T*>(row);
  float* w = static_cast<float*>(row);
  const int slots = gm.Wn * gm.Wn;
  auto valid = [&](int k) {
    const int cy = gm.ry + k / gm.Wn + gm.lo, cx = gm.rx + k % gm.Wn + gm.lo;
    return cy >= 0 && cy <= gm.cy_max && cx >= 0 && cx <= gm.cx_max;
  };
  float dmin = __int_as_float(0x7f800000);
  for (int k = lane; k < slots; k += 32)
    if (valid(k)) dmin = fminf(dmin, fmaxf(float(d[k]), 0.f));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmin = fminf(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
  float theta = 0.f;
  for (int k = lane; k < slots; k += 32) {
    const float e = valid(k) ? expf(-(fmaxf(float(d[k]), 0.f) - dmin) * inv_h2) : 0.f;
    w[k] = e;  // in place: the same slot, read before it is written by this lane
    theta += e;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) theta += __shfl_xor_sync(0xffffffffu, theta, o);
  const float inv = 1.f / theta;
  for (int k = lane; k < slots; k += 32) w[k] *= inv;
}

}  // namespace scbm
