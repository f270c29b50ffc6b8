// topk.cuh -- step a4: per-reference top-K on packed 64-bit keys (Theorem 1's l0-ball
// projection keeps the K largest b_i = the K smallest distances).
//
// key = (ord(d') << 32) | idx, ord order-preserving to uint32, idx = cy*W + cx. Keys are
// unique per reference (idx is unique), so ascending key order is the (distance, idx)
// lexicographic order of DESIGN.md reading R7 and every tie breaks deterministically.
//
// Warp-cooperative: the warp owns a shared-memory array of MS keys:
//   arr[0, KP)        the current best KP keys, sorted ascending
//   arr[KP, KP+64)    a buffer of survivors of the threshold filter (key < arr[KP-1])
//   arr[KP+64, MS)    +inf padding
// When >= 32 survivors are buffered the warp runs a bitonic sort over arr[0, MS) and the
// buffer is reset; the filter threshold only ever decreases, so filtering against a
// stale threshold is conservative (never drops a true top-K key).
#pragma once
#include <stdint.h>

namespace scbm {

constexpr uint64_t kKeyInf = ~0ull;

__device__ __forceinline__ uint32_t ord_i32(int32_t v) { return uint32_t(v) ^ 0x80000000u; }
__device__ __forceinline__ int32_t unord_i32(uint32_t u) { return int32_t(u ^ 0x80000000u); }
__device__ __forceinline__ uint32_t ord_f32(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unord_f32(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// Ascending bitonic sort of arr[0, n) (n a power of two) by one warp.
__device__ __forceinline__ void warp_bitonic_sort(uint64_t* arr, int n, int lane) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int p = lane; p < (n >> 1); p += 32) {
        const int i = ((p & ~(j - 1)) << 1) | (p & (j - 1));
        const int q = i | j;
        const uint64_t a = arr[i], b = arr[q];
        const bool up = (i & k) == 0;
        if ((a > b) == up) {
          arr[i] = b;
          arr[q] = a;
        }
      }
      __syncwarp();
    }
  }
}

// Merge the survivor buffer into the sorted list; returns the new threshold arr[KP-1].
__device__ __forceinline__ uint64_t warp_topk_merge(uint64_t* arr, int KP, int MS, int lane) {
  warp_bitonic_sort(arr, MS, lane);
  for (int i = KP + lane; i < MS; i += 32) arr[i] = kKeyInf;
  __syncwarp();
  return arr[KP - 1];
}

}  // namespace scbm
