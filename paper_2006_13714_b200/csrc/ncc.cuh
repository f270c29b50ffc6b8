// ncc.cuh -- the exact NCC re-rank shared by the box kernels (SC_METRIC_NCC, Eq. 4,
// PAPER.md:264-269): the K+8 candidates a kernel kept by its float filter are re-scored exactly
// and sorted by (NCC descending, idx ascending) with one warp bitonic sort (one item per lane).
// uint8: the double NCC values decide unless they are within rounding of each other, then an
// exact 128-bit comparison of sign(C) C^2 n_other (n_r is common to the reference) does.
#pragma once
#include <stdint.h>

namespace scbm {

// One candidate of the NCC re-rank (a5 for the NCC metric): exact integer cross term / squared
// norm for uint8 input (compared by cross-multiplication in 128 bits), double NCC for float.
struct NccItem {
  int c, n;  // uint8: C, ||X_c||^2 (<= 8 * 64 * 255^2 < 2^31; NCC := 0 for zero norms: c = 0, n = 1)
  double f;  // NCC value (float input: the comparison key)
  int idx;   // -1: empty slot (sorts last)
};
template <bool EXACT>
__device__ __forceinline__ bool ncc_better(const NccItem& x, const NccItem& y) {
  if (x.idx < 0 || y.idx < 0) return y.idx < 0 && x.idx >= 0;
  if constexpr (EXACT) {
    // the double NCC values decide unless they are within rounding of each other; then the
    // exact 128-bit comparison of sign(C) C^2 n_other (n_r is common) does
    const double df = x.f - y.f;
    if (fabs(df) > 1e-12 * fmax(fabs(x.f), fabs(y.f))) return df > 0.0;
    const __int128 lx = (__int128)((long long)(x.c < 0 ? -x.c : x.c) * x.c) * y.n;
    const __int128 ly = (__int128)((long long)(y.c < 0 ? -y.c : y.c) * y.c) * x.n;
    if (lx != ly) return lx > ly;
  } else {
    if (x.f != y.f) return x.f > y.f;
  }
  return x.idx < y.idx;
}
__device__ __forceinline__ NccItem shfl_item(const NccItem& v, int src_lane_xor) {
  NccItem o;
  o.c = __shfl_xor_sync(0xffffffffu, v.c, src_lane_xor);
  o.n = __shfl_xor_sync(0xffffffffu, v.n, src_lane_xor);
  o.f = __shfl_xor_sync(0xffffffffu, v.f, src_lane_xor);
  o.idx = __shfl_xor_sync(0xffffffffu, v.idx, src_lane_xor);
  return o;
}
// warp bitonic sort, best first, one item per lane
template <bool EXACT>
__device__ __noinline__ NccItem warp_sort_ncc(NccItem x, int lane) {
#pragma unroll 1
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll 1
    for (int j = k >> 1; j > 0; j >>= 1) {
      const NccItem p = shfl_item(x, j);
      const bool lower = (lane & j) == 0, up = (lane & k) == 0;
      const bool p_better = ncc_better<EXACT>(p, x);
      // ascending (best first) when up: the lower lane keeps the better item
      if ((lower == up) ? p_better : !p_better && ncc_better<EXACT>(x, p)) x = p;
    }
  }
  return x;
}


}  // namespace scbm
