// refq.cuh -- step a4 for kernels whose lanes own REFERENCES (bm_lanes.cu, bm_tc.cu).
//
// Each reference r of a CTA owns a MAX-HEAP of KP 64-bit keys in shared memory
// (key = (ord(d') << 32) | idx; ascending key order = (distance, idx) order, R7),
// initialised to +inf. The root is the current KP-th best key, i.e. the filter threshold:
// a candidate survives when ord(d') <= hi32(root) (a superset; exact ties are resolved by the
// heap's full 64-bit compare). Inserting x < root replaces the root and sifts it down through
// a FIXED number of levels (ceil(log2(KP+1))) with predicated moves: no data-dependent loop,
// so 32 lanes inserting into 32 different heaps stay converged. After the scan every heap is
// sorted once (heapsort by its owning lane).
//
// Survivors of a warp are compacted into a per-warp queue (ballot + popc) so that insertion
// runs with all 32 lanes busy (lane j inserts queue entry j into its reference's heap);
// entries of the same reference inside one batch are serialised with __match_any_sync rounds.
#pragma once
#include <stdint.h>

#include "topk.cuh"

namespace scbm {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t lds64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts64(uint32_t a, uint64_t v) {
  asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v));
}
__device__ __forceinline__ int32_t lds32(uint32_t a) {
  int32_t v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, int32_t v) {
  asm volatile("st.shared.s32 [%0], %1;" ::"r"(a), "r"(v));
}

struct RefHeaps {
  uint32_t base;  // shared address of heap 0
  int pitch;      // entries per heap (>= KP, odd to spread banks)
  int KP;
  int depth;      // ceil(log2(KP + 1))
  __device__ __forceinline__ uint32_t heap(int r) const { return base + uint32_t(r) * uint32_t(pitch) * 8u; }
  __device__ __forceinline__ uint64_t root(int r) const { return lds64(heap(r)); }
  __device__ __forceinline__ uint32_t thr_hi(int r) const { return uint32_t(root(r) >> 32); }
};

// Replace the root of heap h (KP keys) by x if x < root, restoring the max-heap property.
__device__ __forceinline__ void heap_push(uint32_t h, int KP, int depth, uint64_t x) {
  if (x >= lds64(h)) return;
  int pos = 0;
#pragma unroll 1
  for (int lvl = 0; lvl < depth; ++lvl) {
    int c = 2 * pos + 1;
    if (c >= KP) break;
    const uint64_t l = lds64(h + 8u * c);
    const uint64_t r = (c + 1 < KP) ? lds64(h + 8u * (c + 1)) : 0ull;
    const bool right = r > l;
    const uint64_t big = right ? r : l;
    if (big <= x) break;
    sts64(h + 8u * pos, big);
    pos = c + (right ? 1 : 0);
  }
  sts64(h + 8u * pos, x);
}

// Heapsort in place: afterwards h[0..KP) is ascending.
__device__ __forceinline__ void heap_sort(uint32_t h, int KP, int depth) {
  for (int n = KP - 1; n > 0; --n) {
    const uint64_t top = lds64(h);
    const uint64_t x = lds64(h + 8u * n);
    sts64(h + 8u * n, top);
    // sift x down within the first n entries
    int pos = 0;
    bool done = false;
    for (int lvl = 0; lvl < depth; ++lvl) {
      const int c = 2 * pos + 1;
      const uint64_t a = (!done && c < n) ? lds64(h + 8u * c) : 0ull;
      const uint64_t b = (!done && c + 1 < n) ? lds64(h + 8u * (c + 1)) : 0ull;
      const bool right = b > a;
      const uint64_t big = right ? b : a;
      const bool move = !done && big > x;
      if (move) sts64(h + 8u * pos, big);
      pos = move ? c + (right ? 1 : 0) : pos;
      done = done || !move;
    }
    sts64(h + 8u * pos, x);
  }
}

// Per-warp survivor queue: up to 64 entries (drained 32 at a time).
struct WarpQueue {
  uint32_t key;  // shared address of uint64_t[64]
  uint32_t ref;  // shared address of int32_t[64]
};

// Insert the first min(cnt, 32) queued entries; returns the new count (the undrained tail is
// moved to the front).
static __device__ __noinline__ int queue_drain(WarpQueue q, RefHeaps hp, int cnt, int lane) {
  const int n = cnt < 32 ? cnt : 32;
  const bool has = lane < n;
  const uint64_t k = has ? lds64(q.key + 8u * lane) : 0ull;
  const int r = has ? lds32(q.ref + 4u * lane) : -1 - lane;  // unique dummies for empty lanes
  const unsigned grp = __match_any_sync(0xffffffffu, r);
  const int rank = __popc(grp & ((1u << lane) - 1u));
  const int rounds = __reduce_max_sync(0xffffffffu, __popc(grp));
  for (int rd = 0; rd < rounds; ++rd) {
    if (has && rank == rd) heap_push(hp.heap(r), hp.KP, hp.depth, k);
    __syncwarp();
  }
  const int rest = cnt - n;
  uint64_t tk = 0;
  int tr = 0;
  if (lane < rest) {
    tk = lds64(q.key + 8u * (32 + lane));
    tr = lds32(q.ref + 4u * (32 + lane));
  }
  __syncwarp();
  if (lane < rest) {
    sts64(q.key + 8u * lane, tk);
    sts32(q.ref + 4u * lane, tr);
  }
  __syncwarp();
  return rest;
}

// Append this lane's survivor (if pass) to the queue; drains when >= 32 are queued.
// Returns true if a drain happened (callers refresh their cached thresholds).
__device__ __forceinline__ bool queue_push(WarpQueue q, RefHeaps hp, int& cnt, bool pass, uint64_t key,
                                           int ref, int lane) {
  const unsigned m = __ballot_sync(0xffffffffu, pass);
  if (m == 0) return false;
  if (pass) {
    const int pos = cnt + __popc(m & ((1u << lane) - 1u));
    sts64(q.key + 8u * pos, key);
    sts32(q.ref + 4u * pos, ref);
  }
  cnt += __popc(m);
  __syncwarp();
  if (cnt >= 32) {
    cnt = queue_drain(q, hp, cnt, lane);
    return true;
  }
  return false;
}

__host__ __device__ inline int heap_depth(int KP) {
  int d = 0;
  while ((1 << d) < KP + 1) ++d;
  return d;
}

}  // namespace scbm

namespace scbm {
// Out-of-line heap push for rarely taken paths (keeps one copy of the sift code per kernel).
static __device__ __noinline__ void heap_push_cold(uint32_t h, int KP, int depth, uint64_t x) {
  heap_push(h, KP, depth, x);
}
}  // namespace scbm
