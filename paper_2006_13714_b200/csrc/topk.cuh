// topk.cuh -- step a4: per-reference top-K on packed 64-bit keys (Theorem 1's l0-ball
// projection keeps the K largest b_i = the K smallest distances).
//
// key = (ord(d') << 32) | idx, ord order-preserving to uint32, idx = cy*W + cx. Keys are
// unique per reference (idx is unique), so ascending key order is the (distance, idx)
// lexicographic order of DESIGN.md reading R7 and every tie breaks deterministically.
//
// WarpTopK<NJ>: the sorted list of the best 32*NJ keys lives in REGISTERS, distributed over
// the warp: lane i holds list[i + 32 j] in v[j]. Survivors of the threshold filter are
// buffered (one per lane, <= 32) and merged in one shot:
//   1. bitonic sort of the 32 buffered keys across lanes (15 shuffle stages);
//   2. for each slot j: the 32 smallest of (v[j] U carry) stay in v[j] and the 32 largest
//      become the carry for slot j+1 (reverse + min/max + two 5-stage bitonic merges).
// The filter threshold (the KP-th key) only ever decreases, so filtering against a stale
// threshold is conservative (never drops a true top-K key).
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

__device__ __forceinline__ uint64_t shfl_xor64(uint64_t x, int m) {
  return __shfl_xor_sync(0xffffffffu, x, m);
}
__device__ __forceinline__ uint64_t kmin(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint64_t kmax(uint64_t a, uint64_t b) { return a < b ? b : a; }

// Ascending bitonic sort of one key per lane. The stage loops are deliberately NOT unrolled:
// the merge runs rarely, and unrolled copies blow the instruction cache.
__device__ __forceinline__ uint64_t warp_sort32(uint64_t x, int lane) {
#pragma unroll 1
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll 1
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint64_t p = shfl_xor64(x, j);
      const bool keep_min = ((lane & j) == 0) == ((lane & k) == 0);
      x = keep_min ? kmin(x, p) : kmax(x, p);
    }
  }
  return x;
}

// A bitonic sequence (one key per lane) -> ascending.
__device__ __forceinline__ uint64_t warp_bitonic_merge32(uint64_t x, int lane) {
#pragma unroll 1
  for (int j = 16; j > 0; j >>= 1) {
    const uint64_t p = shfl_xor64(x, j);
    x = (lane & j) ? kmax(x, p) : kmin(x, p);
  }
  return x;
}

// Ascending bitonic sort of 128 keys held 4 per lane: element e = 4 lane + i sits in v[i]. Stages
// with j < 4 exchange inside a lane (no shuffle), the others with lane ^ (j / 4). One sort of the
// whole kept set instead of one WarpTopK merge per 32-key batch (a5 with K + m > 64: ~4x fewer
// instructions). Unrolled: the stage pattern is static.
__device__ __forceinline__ void warp_sort128(uint64_t (&v)[4], int lane) {
#pragma unroll
  for (int k = 2; k <= 128; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j < 4) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int p = i ^ j;
          if (p > i) {
            const bool up = (((lane << 2) + i) & k) == 0;
            const uint64_t a = v[i], b = v[p];
            const uint64_t lo = kmin(a, b), hi = kmax(a, b);
            v[i] = up ? lo : hi;
            v[p] = up ? hi : lo;
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint64_t o = shfl_xor64(v[i], j >> 2);
          const int e = (lane << 2) + i;
          const bool keep_min = ((e & j) == 0) == ((e & k) == 0);
          v[i] = keep_min ? kmin(v[i], o) : kmax(v[i], o);
        }
      }
    }
  }
}

template <int NJ>
struct WarpTopK {
  uint64_t v[NJ];

  __device__ __forceinline__ void init() {
#pragma unroll
    for (int j = 0; j < NJ; ++j) v[j] = kKeyInf;
  }

  // Merge one unsorted key per lane (kKeyInf = none) into the list.
  __device__ __forceinline__ void merge(uint64_t b, int lane) {
    b = warp_sort32(b, lane);
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const uint64_t br = __shfl_sync(0xffffffffu, b, 31 - lane);
      const uint64_t lo = kmin(v[j], br), hi = kmax(v[j], br);
      v[j] = warp_bitonic_merge32(lo, lane);
      if (j + 1 < NJ) b = warp_bitonic_merge32(hi, lane);
    }
  }

  // list[k] (warp-uniform k), broadcast to all lanes.
  __device__ __forceinline__ uint64_t at(int k) const {
    const int js = k >> 5;
    uint64_t x = v[0];
#pragma unroll
    for (int j = 1; j < NJ; ++j)
      if (j == js) x = v[j];
    return __shfl_sync(0xffffffffu, x, k & 31);
  }

  // Sort the (possibly unsorted after re-scoring) 32*NJ keys ascending.
  __device__ __forceinline__ void resort(int lane) {
    uint64_t w[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) w[j] = v[j];
    init();
#pragma unroll
    for (int j = 0; j < NJ; ++j) merge(w[j], lane);
  }
};

// Shared-memory-resident list of 32*NJ sorted keys (list[i + 32 j] at lst[i + 32 j]); one
// non-inlined merge routine per NJ keeps a single copy of the merge code in the kernel.
template <int NJ>
__device__ __noinline__ uint32_t smem_list_merge(uint64_t* lst, const uint64_t* buf, int cnt, int KP,
                                                int lane) {
  WarpTopK<NJ> t;
#pragma unroll
  for (int j = 0; j < NJ; ++j) t.v[j] = lst[lane + 32 * j];
  t.merge(lane < cnt ? buf[lane] : kKeyInf, lane);
#pragma unroll
  for (int j = 0; j < NJ; ++j) lst[lane + 32 * j] = t.v[j];
  const uint64_t kth = t.at(KP - 1);
  __syncwarp();
  return uint32_t(kth >> 32);
}

// Sort an unsorted shared list of 32*NJ keys ascending (after f32 re-scoring).
template <int NJ>
__device__ __noinline__ void smem_list_sort(uint64_t* lst, int lane) {
  WarpTopK<NJ> t;
#pragma unroll
  for (int j = 0; j < NJ; ++j) t.v[j] = lst[lane + 32 * j];
  t.resort(lane);
#pragma unroll
  for (int j = 0; j < NJ; ++j) lst[lane + 32 * j] = t.v[j];
  __syncwarp();
}

}  // namespace scbm
