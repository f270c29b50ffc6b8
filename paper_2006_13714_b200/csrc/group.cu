// group.cu -- patch grouping Y_i (the "next" row after block matching).
//
// For every reference i and each of its K matches S_i(k) (the idx_out table of a run), copy the
// matched b x b x C patch of the input into the group matrix
//     Y_i = [ y_{S_i(1)}, y_{S_i(2)}, ..., y_{S_i(K)} ]          (footnote P:548)
// column k = vecT of the full-depth patch, stored channel-major ([C][b][b], reading R13),
// in the input dtype and uncentred. idx = -1 (fewer than K candidates) -> a zero column.
//
// Pure gather, HBM-bound on the writes (c5: 8.4 GB of groups per 64 frames). Two kernels:
// group_staged_kernel (default, per-image idx) stages each reference tile's windows in shared
// memory and writes every group segment with 16-byte streaming stores; group_kernel (batch-global
// temporal idx, tiles that do not fit) reads the image through L1/L2, one thread per patch row.
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
  FastDiv fdHW;         // divide by H * W: batch-global idx (3D / temporal runs) -> frame
  int global_idx;       // idx entries are frame * H * W + pixel (sc_bm_set_temporal), not per image
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
          uint32_t img, pix = uint32_t(j);
          if (a.global_idx) {
            img = a.fdHW.div(pix);
            pix -= img * uint32_t(a.H * a.W);
          } else {
            img = a.fdImg.div(uint32_t(p));
          }
          const uint32_t cy = a.fdW.div(pix), cx = pix - cy * uint32_t(a.W);
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

// Region-staged gather (the default for per-image idx tables): a CTA owns a TRY x TRX tile of
// references of one image, stages the union of their search windows (+ patch extent) in shared
// memory with coalesced loads -- every matched patch lies inside it -- converts the tile's idx
// rows into region offsets (a shared match table), then writes the tile's groups: one warp per
// reference, whose K C b b elements are one contiguous output segment; lanes take 16-byte items
// (two 8-byte u8 rows via aligned words + funnel shifts, or four floats) or single elements,
// consecutive lanes consecutive bytes. The image is read once per tile instead of once per match.
struct StagedArgs {
  int s, lo, hi, nx, ny, TRY, TRX, tiles_x, RH, RWp;  // RWp: region row pitch in elements
  int tab_off, tab_len;                              // item table: byte offset in shared memory, entries
};

// BT: match-table entry type (int16_t when every region offset fits); BFIX: compile-time patch
// size (0: a.b at run time).
template <typename T, typename BT, int BFIX>
__global__ void __launch_bounds__(256) group_staged_kernel(GroupArgs a, StagedArgs sa) {
  const int bb = BFIX ? BFIX : a.b;
  extern __shared__ __align__(16) uint8_t gsm[];
  T* reg = reinterpret_cast<T*>(gsm);
  const int f = blockIdx.y;
  const int ty = blockIdx.x / sa.tiles_x, tx = blockIdx.x - ty * sa.tiles_x;
  const int iy_first = ty * sa.TRY, ix_first = tx * sa.TRX;
  const int iy_n = min(sa.TRY, sa.ny - iy_first), ix_n = min(sa.TRX, sa.nx - ix_first);
  const int Ybase = iy_first * sa.s + sa.lo, Xbase = ix_first * sa.s + sa.lo;
  const size_t plane = size_t(a.H) * a.W;
  const T* img = static_cast<const T*>(a.imgs) + size_t(f) * a.C * plane;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int per_plane = sa.RH * sa.RWp;
  const long long n_refs = (long long)sa.ny * sa.nx;
  const int n_tile = iy_n * ix_n;
  const long long ref00 = (long long)f * n_refs + (long long)iy_first * sa.nx + ix_first;  // tile's first ref
  // Match table of the tile: bases[t K + k] = region offset of match k of tile reference t
  // (t row-major over the tile), -1 for no match, -2 for a match outside the staged region
  // (an idx not from this plan). The idx rows of a tile row are contiguous: coalesced loads,
  // kMatchBatch in flight per thread.
  BT* bases = reinterpret_cast<BT*>(reinterpret_cast<int*>(gsm + sa.tab_off) + sa.tab_len);
  {
    constexpr int kMatchBatch = 8;
    const int rowK = ix_n * a.K, nq = iy_n * rowK;
    const float inv_rowK = 1.0f / float(rowK);
    for (int q0 = threadIdx.x; q0 < nq; q0 += kMatchBatch * blockDim.x) {
      int jv[kMatchBatch];
#pragma unroll
      for (int u = 0; u < kMatchBatch; ++u) {
        const int q = q0 + u * blockDim.x;
        int r = __float2int_rz(float(q) * inv_rowK), e = q - r * rowK;  // q / rowK, corrected below
        if (e < 0) --r, e += rowK;
        if (e >= rowK) ++r, e -= rowK;
        jv[u] = q < nq ? __ldg(a.idx + (ref00 + (long long)r * sa.nx) * a.K + e) : -1;
      }
#pragma unroll
      for (int u = 0; u < kMatchBatch; ++u) {
        const int q = q0 + u * blockDim.x, j = jv[u];
        int v = -1;
        if (j >= 0) {
          const uint32_t cy = a.fdW.div(uint32_t(j)), cx = uint32_t(j) - cy * uint32_t(a.W);
          const int ry = int(cy) - Ybase, rx = int(cx) - Xbase;
          const bool in = ry >= 0 && ry + bb <= sa.RH && rx >= 0 && rx + bb + 4 <= sa.RWp;
          v = in ? ry * sa.RWp + rx : -2;
        }
        if (q < nq) bases[q] = BT(v);
      }
    }
  }
  const size_t img_end = a.img_elems - size_t(f) * a.C * plane;  // elements of img[] from this image on
  for (int row = warp; row < a.C * sa.RH; row += nwarps) {  // warp per region row, lanes along it
    const int c = row / sa.RH, r = row - c * sa.RH, y = Ybase + r;
    const bool yin = y >= 0 && y < a.H;
    const T* src = img + c * plane + size_t(yin ? y : 0) * a.W;
    T* d = reg + c * per_plane + r * sa.RWp;
    if constexpr (sizeof(T) == 1) {  // interior rows: aligned 4-byte loads + funnel shifts
      const size_t g0 = c * plane + size_t(y) * a.W + Xbase;
      if (yin && Xbase >= 0 && Xbase + sa.RWp <= a.W && g0 + sa.RWp + 4 <= img_end) {
        const uint8_t* rp = reinterpret_cast<const uint8_t*>(img) + g0;
        const int mis = int(reinterpret_cast<uintptr_t>(rp) & 3);
        const uint32_t* wp = reinterpret_cast<const uint32_t*>(rp - mis);
        uint32_t* d32 = reinterpret_cast<uint32_t*>(d);
        for (int x4 = lane; x4 < sa.RWp / 4; x4 += 32)
          d32[x4] = __funnelshift_r(__ldg(wp + x4), __ldg(wp + x4 + 1), 8 * mis);
        continue;
      }
    }
    for (int x = lane; x < sa.RWp; x += 32) {
      const int xx = Xbase + x;
      d[x] = (yin && xx >= 0 && xx < a.W) ? __ldg(src + xx) : T(0);
    }
  }
  __syncthreads();
  const int R = a.C * bb;  // patch rows
  // Items of a reference's contiguous output segment (K patches of R b elements): a 16-byte vector
  // (two 8-byte rows for uint8 b = 8, four floats for float32 b % 4 == 0), one element otherwise;
  // lane i writes items i, i + 32, ... so consecutive lanes write consecutive bytes. tab[e] is the
  // region offset of item e of a patch; wb[k] the region offset of match k of the current reference.
  const int vec = sizeof(T) == 1 ? (bb == 8 ? 16 : 1) : (bb % 4 == 0 ? 4 : 1);
  const int ppv = R * bb / vec, items = a.K * ppv;
  int* tab = reinterpret_cast<int*>(gsm + sa.tab_off);
  for (int e = threadIdx.x; e < ppv; e += blockDim.x) {
    const int el = e * vec, rr = el / bb, m = el - rr * bb, c = rr / bb, l = rr - c * bb;
    tab[e] = c * per_plane + l * sa.RWp + m;
  }
  __syncthreads();
  const int kstep = 32 / ppv, estep = 32 - kstep * ppv;
  const int k_lane = lane / ppv, e_lane = lane - k_lane * ppv;
  const uint32_t* reg32 = reinterpret_cast<const uint32_t*>(gsm);
  // one item: region offset ro (base < 0: no match / outside the region), destination dst
  auto put = [&](int base, int te, int e, T* dst, long long ref, int k) {
    if (base < 0) {
      const int el = e * vec, rr = el / bb, m0 = el - rr * bb, c = rr / bb, l = rr - c * bb;
      const int j = base == -1 ? 0 : __ldg(a.idx + ref * a.K + k);  // (an idx not from this plan)
      const uint32_t cy = a.fdW.div(uint32_t(max(j, 0))), cx = uint32_t(max(j, 0)) - cy * uint32_t(a.W);
      const T* src = img + c * plane + size_t(cy + l) * a.W + cx + m0;
      const int nrow = (vec == 16 && sizeof(T) == 1) ? 2 : 1, per_row = vec / nrow;
      for (int q = 0; q < nrow; ++q)
        for (int m = 0; m < per_row; ++m) dst[q * bb + m] = base == -1 ? T(0) : src[size_t(q) * a.W + m];
      return;
    }
    const int ro = base + te;
    if constexpr (sizeof(T) == 1) {
      if (vec == 16) {  // two 8-byte patch rows: aligned words + funnel shifts
        uint32_t o[4];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int rq = ro + q * sa.RWp;
          const uint32_t* w = reg32 + (rq >> 2);
          const int sh = 8 * (rq & 3);
          const uint32_t w0 = w[0], w1 = w[1], w2 = w[2];
          o[2 * q] = __funnelshift_r(w0, w1, sh);
          o[2 * q + 1] = __funnelshift_r(w1, w2, sh);
        }
        __stcs(reinterpret_cast<uint4*>(dst), make_uint4(o[0], o[1], o[2], o[3]));
      } else {
        *dst = reg[ro];
      }
    } else {
      if (vec == 4) __stcs(reinterpret_cast<float4*>(dst), make_float4(reg[ro], reg[ro + 1], reg[ro + 2], reg[ro + 3]));
      else __stcs(dst, reg[ro]);
    }
  };
  const int ref_elems = a.K * R * bb;                      // group elements per reference
  T* out_tile = static_cast<T*>(a.out) + size_t(ref00) * ref_elems;
  // float patches with an odd row length (c3: b = 7) are written as element pairs when every
  // reference's segment starts 8-byte aligned (K C b^2 even)
  const bool pair = sizeof(T) == 4 && vec == 1 && (ref_elems & 1) == 0;
  const int pkstep = 64 / ppv, pestep = 64 - pkstep * ppv;  // 64 elements per warp iteration
  const int k_pair = (2 * lane) / ppv, e_pair = 2 * lane - k_pair * ppv;
  int ty_w = warp / ix_n, tx_w = warp - ty_w * ix_n;  // this warp's current tile reference
  for (int t = warp; t < n_tile; t += nwarps) {
    const int rofs = ty_w * sa.nx + tx_w;  // reference - ref00
    const long long ref = ref00 + rofs;
    const BT* wb = bases + t * a.K;
    tx_w += nwarps;
    while (tx_w >= ix_n) tx_w -= ix_n, ++ty_w;
    T* out_ref = out_tile + (long long)rofs * ref_elems;
    if (estep == 0) {  // ppv divides 32: every lane keeps its item e and strides over the matches
      const int te = tab[e_lane];
      T* dst = out_ref + lane * vec;
      for (int k = k_lane; k < a.K; k += kstep, dst += 32 * vec) put(int(wb[k]), te, e_lane, dst, ref, k);
    } else if (pair) {  // float, odd row length: element pairs -> one 8-byte store (segment is 8-B aligned)
      int k0 = k_pair, e0 = e_pair;
      for (int it = lane; 2 * it < ref_elems; it += 32) {
        int k1 = k0, e1 = e0 + 1;
        if (e1 == ppv) e1 = 0, ++k1;
        T v[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int k = u ? k1 : k0, e = u ? e1 : e0;
          const int base = int(wb[k]);
          if (base >= 0) {
            v[u] = reg[base + tab[e]];
          } else {  // no match (0) / outside the staged region (global read)
            const int j = base == -1 ? -1 : __ldg(a.idx + ref * a.K + k);
            const int rr = e / bb, c = rr / bb, l = rr - c * bb, m = e - rr * bb;
            const uint32_t cy = a.fdW.div(uint32_t(max(j, 0))), cx = uint32_t(max(j, 0)) - cy * uint32_t(a.W);
            v[u] = j < 0 ? T(0) : img[c * plane + size_t(cy + l) * a.W + cx + m];
          }
        }
        if constexpr (sizeof(T) == 4)
          __stcs(reinterpret_cast<float2*>(out_ref + 2 * it), make_float2(float(v[0]), float(v[1])));
        e0 += pestep;
        k0 += pkstep;
        if (e0 >= ppv) e0 -= ppv, ++k0;
      }
    } else {
      int k = k_lane, e = e_lane;
      for (int it = lane; it < items; it += 32) {
        put(int(wb[k]), tab[e], e, out_ref + it * vec, ref, k);
        e += estep;
        k += kstep;
        if (e >= ppv) e -= ppv, ++k;
      }
    }
  }
}

#ifndef SCBM_GROUP_SMEM
#define SCBM_GROUP_SMEM 96
#endif
constexpr size_t kGroupSmem = size_t(SCBM_GROUP_SMEM) * 1024;  // shared-memory budget of a tile

template <typename T>
cudaError_t launch_group_staged_t(const GroupArgs& a, const sc_bm_plan_s& p, int64_t n_images, cudaStream_t st) {
  const Geometry& g = p.g;
  StagedArgs sa{};
  sa.s = g.s; sa.lo = g.lo; sa.hi = g.hi; sa.nx = g.nx; sa.ny = g.ny;
  const int vec = sizeof(T) == 1 ? (g.b == 8 ? 16 : 1) : (g.b % 4 == 0 ? 4 : 1);
  sa.tab_len = (g.C * g.b * g.b / vec + 3) & ~3;
  size_t bytes = 0;
  bool short_bases = false;
  // 16 x 32 reference tiles, halved while region + tables exceed kGroupSmem, the tile writes more
  // than max(1 MB, 8 x its shared memory) of groups (measured: c3's 70 float patches per reference
  // prefer 8 x 8 tiles) or the grid is under 4 waves of CTAs on the SMs (small images)
  for (int t = 0;; ++t) {
    sa.TRY = std::max(1, 16 >> (t / 2)), sa.TRX = std::max(1, 32 >> ((t + 1) / 2));
    sa.RH = (sa.TRY - 1) * g.s + g.Wn + g.b - 1;
    sa.RWp = ((sa.TRX - 1) * g.s + g.Wn + g.b - 1 + 4 + 3) & ~3;  // + 1 word of slack for the funnel
    sa.tab_off = int((size_t(g.C) * sa.RH * sa.RWp * sizeof(T) + 16 + 15) & ~size_t(15));
    short_bases = size_t(sa.RH) * sa.RWp <= 32767;  // match offsets (within one channel plane) fit int16
    bytes = size_t(sa.tab_off) + size_t(sa.tab_len) * sizeof(int) +
            size_t(sa.TRY) * sa.TRX * g.K * (short_bases ? 2 : 4);
    const long long ctas = (long long)((g.nx + sa.TRX - 1) / sa.TRX) * ((g.ny + sa.TRY - 1) / sa.TRY) * n_images;
    const size_t out_bytes = size_t(sa.TRY) * sa.TRX * g.K * g.C * g.b * g.b * sizeof(T);  // groups per CTA
    const bool small_out = out_bytes <= std::max(size_t(1) << 20, 8 * bytes);  // else: staging amortised enough
    if ((bytes <= kGroupSmem && ctas >= 4LL * p.sm_count && small_out) || sa.TRY * sa.TRX <= 4) break;
  }
  if (bytes > 96 * 1024) return cudaErrorInvalidValue;
  sa.tiles_x = (g.nx + sa.TRX - 1) / sa.TRX;
  const int tiles_y = (g.ny + sa.TRY - 1) / sa.TRY;
  const dim3 grid(sa.tiles_x * tiles_y, unsigned(n_images));
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
    kern<<<grid, 256, bytes, st>>>(a, sa);
  };
  if (g.b == 8) {
    if (short_bases) go(group_staged_kernel<T, int16_t, 8>);
    else go(group_staged_kernel<T, int, 8>);
  } else {
    if (short_bases) go(group_staged_kernel<T, int16_t, 0>);
    else go(group_staged_kernel<T, int, 0>);
  }
  return cudaGetLastError();
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
  a.fdHW = FastDiv(uint32_t(g.H * g.W));
  a.global_idx = p.T > 0;
  if (launches) *launches += 1;
  if (p.T == 0 && n_images <= 65535) {  // per-image idx: the region-staged gather
    cudaError_t e = g.dtype == SC_DTYPE_U8 ? launch_group_staged_t<uint8_t>(a, p, n_images, st)
                                           : launch_group_staged_t<float>(a, p, n_images, st);
    if (e != cudaErrorInvalidValue) return e;
    cudaGetLastError();
  }
  if (g.dtype == SC_DTYPE_U8) return launch_group_t<uint8_t>(a, p.sm_count, st);
  return launch_group_t<float>(a, p.sm_count, st);
}

}  // namespace scbm
