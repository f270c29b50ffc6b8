// group.cu -- patch grouping Y_i (the "next" row after block matching).
//
// For every reference i and each of its K matches S_i(k) (the idx_out table of a run), copy the
// matched b x b x C patch of the input into the group matrix
//     Y_i = [ y_{S_i(1)}, y_{S_i(2)}, ..., y_{S_i(K)} ]          (footnote P:548)
// column k = vecT of the full-depth patch, stored channel-major ([C][b][b], reading R13),
// in the input dtype and uncentred. idx = -1 (fewer than K candidates) -> a zero column.
//
// Pure gather: HBM-bound on the writes (c5: 8.4 GB of groups per 64 frames), so threads write
// consecutive patch rows (8-byte stores for u8 b = 8, 16-byte stores for f32 b % 4 = 0) and read
// the image through L1/L2 (each image row segment is reused by the many groups that contain it).
#include <algorithm>

#include "sc_internal.h"

namespace scbm {
namespace {

// Exact unsigned division of n < 2^32 by a runtime d >= 1 with one 64-bit multiply-high:
// q = umulhi64(n, ceil(2^64 / d)) (d = 1 handled by the all-ones multiplier + 1 fix-up).
struct FastDiv {
  unsigned long long m;
  uint32_t d;
  __host__ FastDiv() : m(0), d(1) {}
  __host__ explicit FastDiv(uint32_t dd) : d(dd) {
    m = dd == 1 ? 0ull : (~0ull / dd) + 1ull;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return d == 1 ? n : uint32_t(__umul64hi(n, m)); }
};

struct GroupArgs {
  const void* imgs;    // [n][C][H][W]
  const int32_t* idx;  // [n][refs][K]
  void* out;           // [n][refs][K][C][b][b]
  int H, W, C, b, K;
  long long n_patches;  // n * refs * K (< 2^31)
  size_t img_elems;     // n * C * H * W (bound for the aligned word loads)
  FastDiv fdW, fdImg;   // divide by W (pixel index -> row), by refs * K (patch -> image)
};

#ifndef SCBM_GROUP_UNROLL
#define SCBM_GROUP_UNROLL 4
#endif
constexpr int kGroupUnroll = SCBM_GROUP_UNROLL;  // patches in flight per thread (memory-level parallelism)

// Thread = one fixed row r (of the R = C b rows of a patch) of a fixed patch slot of its CTA;
// the CTA walks patch blocks grid-stride, so consecutive threads write consecutive rows of
// consecutive patches (contiguous stores) with no per-row integer divisions. Every thread keeps
// kGroupUnroll patches in flight: all index and image loads are issued before the stores.
template <typename T>
__global__ void __launch_bounds__(256) group_kernel(GroupArgs a) {
  const int R = a.C * a.b;                  // rows per patch
  const int ppb = 256 / R;                  // patches per CTA step
  if (int(threadIdx.x) >= ppb * R) return;  // idle tail threads (R does not divide 256)
  const int slot = threadIdx.x / R, r = threadIdx.x - slot * R;
  const int c = r / a.b, l = r - c * a.b;
  const size_t plane = size_t(a.H) * a.W;
  const long long step = (long long)gridDim.x * ppb;
  // software pipeline: the match indices of the next batch are loaded while this batch's image
  // rows are fetched (two dependent memory latencies per batch otherwise)
  int jn[kGroupUnroll];
  auto load_idx = [&](long long q0) {
#pragma unroll
    for (int u = 0; u < kGroupUnroll; ++u) {
      const long long p = q0 + u * step;
      jn[u] = p < a.n_patches ? __ldg(a.idx + p) : -2;
    }
  };
  load_idx((long long)blockIdx.x * ppb + slot);
  for (long long p0 = (long long)blockIdx.x * ppb + slot; p0 < a.n_patches; p0 += step * kGroupUnroll) {
    size_t off[kGroupUnroll];
    int jv[kGroupUnroll];
#pragma unroll
    for (int u = 0; u < kGroupUnroll; ++u) jv[u] = jn[u];
    load_idx(p0 + step * kGroupUnroll);
#pragma unroll
    for (int u = 0; u < kGroupUnroll; ++u) {
      const long long p = p0 + u * step;
      off[u] = 0;
      const int j = jv[u];
      {
        if (j >= 0) {
          const uint32_t cy = a.fdW.div(uint32_t(j)), cx = uint32_t(j) - cy * uint32_t(a.W);
          const uint32_t img = a.fdImg.div(uint32_t(p));
          off[u] = (size_t(img) * a.C + c) * plane + size_t(cy + l) * a.W + cx;
        }
      }
    }
    if constexpr (sizeof(T) == 1) {
      if (a.b == 8) {  // u8, 8-byte rows: one (or two) aligned 16-byte loads + funnel shifts
        uint32_t w[kGroupUnroll][3];
#pragma unroll
        for (int u = 0; u < kGroupUnroll; ++u) {
          const size_t base = off[u] & ~size_t(15);
          const int sh = int(off[u] & 15);
          const bool fast = jv[u] >= 0 && base + 32 <= a.img_elems;
          const uint4* src = reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(a.imgs) + (fast ? base : 0));
          const uint4 A = fast ? __ldg(src) : make_uint4(0u, 0u, 0u, 0u);
          const uint4 B = (fast && sh > 8) ? __ldg(src + 1) : A;  // the 8 bytes cross into the next 16
          const int q = sh >> 2;
          w[u][0] = q == 0 ? A.x : q == 1 ? A.y : q == 2 ? A.z : A.w;
          w[u][1] = q == 0 ? A.y : q == 1 ? A.z : q == 2 ? A.w : B.x;
          w[u][2] = q == 0 ? A.z : q == 1 ? A.w : q == 2 ? B.x : B.y;
        }
#pragma unroll
        for (int u = 0; u < kGroupUnroll; ++u) {
          if (jv[u] == -2) continue;
          const long long p = p0 + u * step;
          uint2* dst = reinterpret_cast<uint2*>(static_cast<uint8_t*>(a.out) + (size_t(p) * R + r) * 8);
          const size_t base = off[u] & ~size_t(15);
          // streaming (evict-first) stores: the groups must not push the image out of L2
          if (jv[u] < 0) {
            __stcs(dst, make_uint2(0u, 0u));
          } else if (base + 32 <= a.img_elems) {
            const int sh = 8 * int(off[u] & 3);
            __stcs(dst, make_uint2(__funnelshift_r(w[u][0], w[u][1], sh), __funnelshift_r(w[u][1], w[u][2], sh)));
          } else {
            const uint8_t* src = static_cast<const uint8_t*>(a.imgs) + off[u];
            uint8_t* d8 = reinterpret_cast<uint8_t*>(dst);
            for (int m = 0; m < 8; ++m) d8[m] = src[m];
          }
        }
        continue;
      }
    }
#pragma unroll
    for (int u = 0; u < kGroupUnroll; ++u) {
      if (jv[u] == -2) continue;
      const long long p = p0 + u * step;
      T* dst = static_cast<T*>(a.out) + (size_t(p) * R + r) * a.b;
      const T* src = static_cast<const T*>(a.imgs) + off[u];
      if (jv[u] < 0) {
        for (int m = 0; m < a.b; ++m) dst[m] = T(0);
      } else if (sizeof(T) == 4 && (a.b & 3) == 0) {
        for (int m = 0; m < a.b; m += 4)
          __stcs(reinterpret_cast<float4*>(dst + m),
                 make_float4(__ldg(src + m), __ldg(src + m + 1), __ldg(src + m + 2), __ldg(src + m + 3)));
      } else {
        for (int m = 0; m < a.b; ++m) dst[m] = __ldg(src + m);
      }
    }
  }
}

template <typename T>
cudaError_t launch_group_t(const GroupArgs& a, int sm_count, cudaStream_t st) {
  const int ppb = 256 / (a.C * a.b);
  const long long blocks = std::min<long long>((a.n_patches + ppb - 1) / ppb, (long long)sm_count * 8);
  group_kernel<T><<<unsigned(std::max<long long>(blocks, 1)), 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_group(const sc_bm_plan_s& p, const void* imgs, int64_t n_images, const int32_t* idx,
                         void* out, cudaStream_t st, int64_t* launches) {
  const Geometry& g = p.g;
  GroupArgs a{};
  a.imgs = imgs;
  a.idx = idx;
  a.out = out;
  a.H = g.H; a.W = g.W; a.C = g.C; a.b = g.b; a.K = g.K;
  const long long n_refs = (long long)g.ny * g.nx;
  a.n_patches = n_images * n_refs * g.K;
  a.img_elems = size_t(n_images) * g.C * g.H * g.W;
  if (a.n_patches >= (1ll << 31)) return cudaErrorInvalidValue;  // 32-bit patch / pixel indices
  a.fdW = FastDiv(uint32_t(g.W));
  a.fdImg = FastDiv(uint32_t(n_refs * g.K));
  if (launches) *launches += 1;
  if (g.dtype == SC_DTYPE_U8) return launch_group_t<uint8_t>(a, p.sm_count, st);
  return launch_group_t<float>(a, p.sm_count, st);
}

}  // namespace scbm
