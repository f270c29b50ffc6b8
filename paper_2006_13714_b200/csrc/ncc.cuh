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

// The same order at a fraction of the cost: a warp bitonic sort of 64-bit keys (order-preserving
// bits of float(-f), then idx) that carries only the source lane, the items fetched once at the
// end; float(-f) is monotone in f, so the key order can disagree with ncc_better only between
// neighbours whose float keys are equal or whose f are within the exact path's rounding band --
// those are repaired by odd-even transposition passes with the full comparator (rarely entered).
template <bool EXACT>
__device__ __forceinline__ NccItem warp_rank_ncc(const NccItem x, int lane) {
  uint32_t hi = 0xffffffffu, lo = 0xffffffffu;  // empty slots sort last
  if (x.idx >= 0) {
    const uint32_t u = __float_as_uint(float(-x.f) + 0.0f);  // -0 -> +0 (ncc_better: equal)
    hi = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    lo = uint32_t(x.idx);
  }
  int src = lane;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint32_t phi = __shfl_xor_sync(0xffffffffu, hi, j), plo = __shfl_xor_sync(0xffffffffu, lo, j);
      const int psrc = __shfl_xor_sync(0xffffffffu, src, j);
      const bool p_less = phi < hi || (phi == hi && plo < lo);
      const bool take_min = ((lane & j) == 0) == ((lane & k) == 0);
      if (take_min == p_less) hi = phi, lo = plo, src = psrc;
    }
  }
  NccItem y;
  y.c = __shfl_sync(0xffffffffu, x.c, src);
  y.n = __shfl_sync(0xffffffffu, x.n, src);
  y.f = __shfl_sync(0xffffffffu, x.f, src);
  y.idx = __shfl_sync(0xffffffffu, x.idx, src);
  // neighbours the keys may have mis-ordered
  const uint32_t nhi = __shfl_down_sync(0xffffffffu, hi, 1);
  const double nf = __shfl_down_sync(0xffffffffu, y.f, 1);
  const int nidx = __shfl_down_sync(0xffffffffu, y.idx, 1);
  bool amb = lane < 31 && y.idx >= 0 && nidx >= 0 && nhi == hi;
  if constexpr (EXACT) amb |= lane < 31 && y.idx >= 0 && nidx >= 0 && fabs(y.f - nf) <= 1e-12 * fmax(fabs(y.f), fabs(nf));
  if (__any_sync(0xffffffffu, amb)) {
    for (int pass = 0, quiet = 0; quiet < 2; ++pass) {
      const int ph = pass & 1;
      const int partner = ((lane & 1) == ph) ? min(lane + 1, 31) : max(lane - 1, 0);
      NccItem p;
      p.c = __shfl_sync(0xffffffffu, y.c, partner);
      p.n = __shfl_sync(0xffffffffu, y.n, partner);
      p.f = __shfl_sync(0xffffffffu, y.f, partner);
      p.idx = __shfl_sync(0xffffffffu, y.idx, partner);
      const bool swap = partner != lane && (partner > lane ? ncc_better<EXACT>(p, y) : ncc_better<EXACT>(y, p));
      if (swap) y = p;
      quiet = __any_sync(0xffffffffu, swap) ? 0 : quiet + 1;
    }
  }
  return y;
}

// Items that arrive already ordered by a monotone approximation of the key (the kept quantised
// filter keys, empty slots last): one check of every neighbour pair with the full comparator, and
// odd-even transposition passes only when some pair is out of order -- the passes are a complete
// sort, so the result is exact however far the approximation was off.
template <bool EXACT>
__device__ __forceinline__ NccItem warp_repair_ncc(NccItem y, int lane) {
  auto fetch = [&](int src) {
    NccItem p;
    p.c = __shfl_sync(0xffffffffu, y.c, src);
    p.n = __shfl_sync(0xffffffffu, y.n, src);
    p.f = __shfl_sync(0xffffffffu, y.f, src);
    p.idx = __shfl_sync(0xffffffffu, y.idx, src);
    return p;
  };
  const NccItem nx = fetch(min(lane + 1, 31));
  const bool bad = lane < 31 && ncc_better<EXACT>(nx, y);
  if (!__any_sync(0xffffffffu, bad)) return y;
  for (int pass = 0, quiet = 0; quiet < 2; ++pass) {
    const int ph = pass & 1;
    const int partner = ((lane & 1) == ph) ? min(lane + 1, 31) : max(lane - 1, 0);
    const NccItem p = fetch(partner);
    const bool swap = partner != lane && (partner > lane ? ncc_better<EXACT>(p, y) : ncc_better<EXACT>(y, p));
    if (swap) y = p;
    quiet = __any_sync(0xffffffffu, swap) ? 0 : quiet + 1;
  }
  return y;
}

}  // namespace scbm
