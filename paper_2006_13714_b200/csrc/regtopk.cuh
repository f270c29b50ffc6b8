// regtopk.cuh -- per-lane register top-K on 32-bit keys (u8 kernels whose lanes own references).
//
// key32 = (min(d, DSAT) << RB) | rel, where d = d' + ||X_i||^2 is the exact integer distance
// (Lemma 2) and rel = (dy - lo) * Wn + (dx - lo) is the candidate's index
// inside the reference's window. For a fixed reference rel is monotone in idx = cy*W + cx, so
// ascending key32 order is exactly the (distance, idx) order of DESIGN.md reading R7 -- as long
// as no key of the final top-K is saturated (d >= DSAT). A lane whose K-th key is saturated or
// still +inf (fewer than K unsaturated candidates) is flagged and its reference is recomputed
// by the exact fix-up kernel (fixup.cu), so the output is always exact.
//
// Insertion is the branch-free network r[k] = max(r[k-1], min(r[k], x)) (k = KR-1..1),
// r[0] = min(r[0], x): 2 IMNMX per slot, no memory traffic, no divergence; x = 0xffffffff is
// a no-op, so lanes without a survivor simply insert +inf.
#pragma once
#include <stdint.h>

namespace scbm {

template <int KR>
struct RegTopK32 {
  uint32_t r[KR];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int i = 0; i < KR; ++i) r[i] = 0xffffffffu;
  }
  __device__ __forceinline__ void insert(uint32_t x) {
#pragma unroll
    for (int k = KR - 1; k > 0; --k) r[k] = max(r[k - 1], min(r[k], x));
    r[0] = min(r[0], x);
  }
  // r[kp1] for a warp-uniform runtime index (select chain over the registers)
  __device__ __forceinline__ uint32_t at(int kp1) const {
    uint32_t v = r[KR - 1];
#pragma unroll
    for (int i = 0; i < KR - 1; ++i)
      if (i == kp1) v = r[i];
    return v;
  }
};

struct Key32 {
  int rb;        // bits of the window-relative index
  uint32_t dsat; // saturation value of the distance field
  __device__ __forceinline__ uint32_t make(int d, int rel) const {
    const uint32_t dd = d < 0 ? 0u : (uint32_t(d) > dsat ? dsat : uint32_t(d));
    return (dd << rb) | uint32_t(rel);
  }
  __device__ __forceinline__ int dist(uint32_t k) const { return int(k >> rb); }
  __device__ __forceinline__ int rel(uint32_t k) const { return int(k & ((1u << rb) - 1u)); }
  // largest distance that may still pass the filter given the K-th key
  __device__ __forceinline__ int thr(uint32_t kth) const { return int(kth >> rb); }
  __device__ __forceinline__ bool exact(uint32_t kth) const { return (kth >> rb) < dsat; }
};

__host__ __device__ inline int key32_rel_bits(int Wn) {
  int rb = 0;
  while ((1 << rb) < Wn * Wn) ++rb;
  return rb < 1 ? 1 : rb;
}

}  // namespace scbm
