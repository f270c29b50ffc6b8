// bm_boxf.cu -- the float box-sum Self-Convolution matcher (SC_KERNEL_BOXF): f32 images, any
// channel count (channels summed, Eq. 12), reference stride s <= patch side b (instantiated for
// (s, b) = (3, 8), (1, 7), (4, 8), (2, 8)): steps a0-a6 fused in one kernel.
//
// The same regrouping as the u8 box kernel (bm_box.cu): for one window offset delta the cross
// term of every reference (Eq. 5) is a box sum of the product image
// P_delta(y, x) = x'(y, x) x'(y + dy, x + dx), so references that overlap share work:
//   * lane l holds reference column ix0 + l and correlates only its own s-column strip of the
//     patch rows; a reference's patch is NS = ceil(b / s) consecutive strips (the last one
//     WL = b - (NS-1) s columns wide), i.e. lanes l .. l+NS-1: NS-1 shuffles per pair (a
//     doubling tree for s = 1). Lanes 33-NS .. 31 are helper strips.
//   * the candidate norm (a1) uses the same strips: running sums of the squared
//     candidate rows, so d' = n_c - 2 C (Lemma 2) is assembled per strip,
//     E = strip norm - 2 strip cross term, and summed over the NS strips.
//   * a lane slides over VY vertically adjacent offsets, loading each candidate row once.
// For c2 (s = 3, b = 8) that is 24 FMAs + 24 square FMAs per (reference, candidate row) group
// of 8 offsets, i.e. ~27 FMAs per pair instead of 64; for c3 (s = 1, b = 7) ~8 instead of 49.
//
// a4: per-lane register top-KP of 32-bit keys (regtopk.cuh): key = (float bits of d >> (rb-1))
// << rb | (rel + 1); d >= 0 so the float bits are monotone, and the 21 (20) kept bits give
// a relative resolution of 2^-13 (2^-12). The first KR - KP slots hold a 0 sentinel (real keys
// are >= 1), so the KP-th key always sits in the last register. The filter is a superset
// (threshold = the largest distance of the KP-th key's quantum), and a5 re-scores the KP keys
// of every reference exactly by direct differences in fp32 from the input and keeps the best
// K (BASELINE.json north_star tolerance): a true top-K candidate can only
// be lost if more than KP - K = 8 others lie within one quantum (~1e-4 relative) of it.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "ncc.cuh"
#include "regtopk.cuh"
#include "sc_internal.h"
#include "topk.cuh"

namespace scbm {
namespace {

constexpr int kFWarps = 8;

#ifndef SCBM_BOXF_HEAP4
#define SCBM_BOXF_HEAP4 1  // K + m > 48: a 4-ary heap with the root in a register (0: the binary heap)
#endif
#ifndef SCBM_BOXF_A5HALVES
#define SCBM_BOXF_A5HALVES 1  // WS = 2: both warps of a reference row share a5 (half the references each)
#endif
#ifndef SCBM_BOXF_A5SPLIT
#define SCBM_BOXF_A5SPLIT 1  // a5: the short last key slot re-scored by several lanes per key
#endif
#ifndef SCBM_BOXF_F2
#define SCBM_BOXF_F2 0  // 1: packed FFMA2 cross terms (measured: FFMA2 runs at the FFMA FMA rate, 121 /SM/clk, and its pair accumulators spill on c4: c4 2.66 -> 2.74 ms, c2 unchanged)
#endif

struct BoxfArgs {
  const void* imgs;   // [F][C][H][W] float (or uint8 for the NCC metric)
  int32_t* idx_out;   // [F][band refs][K]
  float* dist_out;    // L2: d; NCC: d_NCC = -NCC
  int H, W, C, Wn, K, KP, lo, hi, nx, iy_begin, iy_end, tiles_x;
  int rows;          // reference rows per CTA (1 .. kFWarps; warps wr >= rows sit idle): the tile height
                     // that fills the last wave (boxf_rows)
  int RH, RWp, PL;  // staged region rows, row pitch (floats), floats per channel plane
  int nblk;         // dy blocks of VY offsets
  int scr;          // per-warp scratch words (survivor staging [+ output staging | + heaps])
  int hp;           // heap pitch (words per reference) when the top-KP lives in shared heaps
  int lofs;         // WS = 2: word offset of the per-row list area (0: the staged region, reused)
  // Z3 (3D search over the planes of a volume, PAPER.md:548 / 697): the launch's reference plane
  // positions z0 .. z0 + gridDim.y - 1 (first plane (z0 + f) * sz), volume planes P, plane offsets
  // [zlo, zhi] of the candidates; C = the patch depth d
  int z0, sz, P, zlo, zhi, zwin;
  int rb;           // window-relative index bits of the 32-bit keys
  int* fix_count;   // references the key quantisation leaves open -> exact fix-up (fixup.cu)
  int* fix_list;
};

__device__ __forceinline__ int centre_out_f(int k) { return (k & 1) ? ((k + 1) >> 1) : -(k >> 1); }

// sum over the reference's strips: full strips of lanes l .. l+NS-2, partial strip of lane l+NS-1
template <int NS, int WL, int S>
__device__ __forceinline__ float hcombine(float ef, float ep) {
  if constexpr (NS == 1) {
    return ep;
  } else if constexpr (NS == 7 && WL == S) {  // s = 1, b = 7: doubling tree, 4 shuffles
    const float s2 = ef + __shfl_down_sync(0xffffffffu, ef, 1);
    const float s4 = s2 + __shfl_down_sync(0xffffffffu, s2, 2);
    const float s6 = s4 + __shfl_down_sync(0xffffffffu, s2, 4);
    return s6 + __shfl_down_sync(0xffffffffu, ef, 6);
  } else {
    float acc = ef;
#pragma unroll
    for (int j = 1; j < NS - 1; ++j) acc += __shfl_down_sync(0xffffffffu, ef, j);
    return acc + __shfl_down_sync(0xffffffffu, ep, NS - 1);
  }
}

// WS = 2 (window split): two warps per reference row, each visiting half of the window's dx pairs
// (alternating, so both start near the reference), with their own top-KP lists and a shared filter
// threshold (the smaller of the two published KP-th keys: each list holds KP real candidates of the
// reference, so the KP-th best of their union can only be smaller -- a valid superset bound); the
// second half's list is merged into the first's before a5. Doubles the warps per staged region
// where the grid or the shared memory leaves the SMs half empty (c2: 132 CTAs; c4: 216 KB, 1 CTA/SM).
// Z3 (3D search): the reference planes are staged once, the candidate planes of every plane offset
// (centre-out) are restaged into a second region; keys carry (offset index) Wn^2 + slot; idx is the
// volume raster (z H + y) W + x of the candidate's first voxel.
template <int S, int BK, int VY, int KR, bool C1, bool NCC, typename TIN, int WS = 1, bool Z3 = false>
__global__ void __launch_bounds__(kFWarps * 32 * WS, WS == 1 ? 2 : 1) bm_boxf_kernel(BoxfArgs a) {
  constexpr int NS = (BK + S - 1) / S;   // strips per patch
  constexpr int WL = BK - (NS - 1) * S;  // width of the last strip
  constexpr int RX = 33 - NS;            // references per warp (lanes RX..31: helper strips)
  constexpr int NT = BK + VY - 1;        // candidate rows per (dy block, dx)
  constexpr int kPairs = SCBM_BOXF_F2 ? WL / 2 : 0;  // FFMA2 column pairs of the partial strip
  // a5: list entries in the last 32-key slot, and lanes per key there (register lists only)
  constexpr int kN1 = KR - 32 * (((KR + 31) / 32) - 1);
  constexpr int kSplitG = (SCBM_BOXF_A5SPLIT && KR > 32 && KR <= 48 && !NCC && !Z3) ? (kN1 <= 8 ? 4 : 2) : 1;
  extern __shared__ __align__(16) float smf[];
  const int f = blockIdx.y;
  const int ty = blockIdx.x / a.tiles_x, tx = blockIdx.x - ty * a.tiles_x;
  const int iy_first = a.iy_begin + ty * a.rows;
  const int ix_first = tx * RX;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = warp % kFWarps, hh = warp / kFWarps;  // reference row of the warp, window half (WS = 2)
  const int Ybase = iy_first * S + a.lo, Xbase = ix_first * S + a.lo;

  // ---- a0: the staged region of every channel (0 outside the image): L2 centres x' = x - 0.5
  // (halves the identity's cancellation); NCC keeps the raw values (not shift-invariant, Eq. 4)
  const int nch = C1 ? 1 : a.C;
  const size_t plane = size_t(a.H) * a.W;
  const int zr = Z3 ? (a.z0 + f) * a.sz : 0;  // Z3: the reference patch's first plane
  const TIN* const vol = static_cast<const TIN*>(a.imgs);
  const TIN* img = Z3 ? vol + size_t(zr) * plane : vol + size_t(f) * nch * plane;
  const int regw = (Z3 ? 2 : 1) * nch * a.PL;  // staged floats: reference (+ candidate) planes
  const float shift = NCC ? 0.f : 0.5f;
  for (int e = threadIdx.x; e < nch * a.PL; e += blockDim.x) {
    const int c = e / a.PL, e2 = e - c * a.PL;
    const int r = e2 / a.RWp, x = e2 - r * a.RWp;
    const int yy = Ybase + r, xx = Xbase + x;
    smf[e] = (yy >= 0 && yy < a.H && xx >= 0 && xx < a.W)
                 ? float(__ldg(img + c * plane + size_t(yy) * a.W + xx)) - shift : 0.f;
  }
  // published KP-th keys of the two window halves (WS = 2), +inf until a list fills
  uint32_t* pub = reinterpret_cast<uint32_t*>(smf + ((regw + 3) & ~3)) + kFWarps * WS * a.scr;
  if (WS == 2) pub[warp * 32 + lane] = 0xffffffffu;
  __syncthreads();

  const int iy0 = iy_first + wr;
  const bool wact = wr < a.rows && iy0 < a.iy_end;  // warp-uniform
  if (WS == 1 && !Z3 && !wact) return;  // (Z3: every warp joins the restaging barriers)
  const int ix = ix_first + lane;
  const bool lane_ok = lane < RX && ix < a.nx;
  const int rx = ix * S, ry = iy0 * S;
  const int rr0 = (iy0 - iy_first) * S - a.lo;  // region row of image row ry
  const int rc0 = lane * S - a.lo;              // region column of the lane's strip
  float R[BK][S];  // the lane's strip of the reference patch (one channel at a time if C > 1)
  auto load_ref = [&](int c) {
#pragma unroll
    for (int r = 0; r < BK; ++r)
#pragma unroll
      for (int m = 0; m < S; ++m) R[r][m] = smf[c * a.PL + (rr0 + r) * a.RWp + rc0 + m];
  };
  float nr;  // ||X_i||^2 of the centred reference, channels summed (Eq. 12)
  {
    float nf = 0.f, np = 0.f;
    for (int c = 0; c < nch; ++c) {
      load_ref(c);
#pragma unroll
      for (int r = 0; r < BK; ++r)
#pragma unroll
        for (int m = 0; m < S; ++m) {
          if (m < WL) np = fmaf(R[r][m], R[r][m], np);
          nf = fmaf(R[r][m], R[r][m], nf);
        }
    }
    nr = hcombine<NS, WL, S>(nf, np);
    if (C1) load_ref(0);
  }
  // NCC: the filter score of a candidate is sqrt(n_r) - C / sqrt(n_c) >= 0 (Cauchy-Schwarz; smaller
  // = larger NCC, NCC := 0 for zero norms); keys quantise it like a distance (no n_r offset)
  const float nrs = NCC ? sqrtf(nr) : 0.f;
  const float nadd = NCC ? 0.f : nr;
  // a4 state. KR <= 48: a sorted register list (0 sentinels in the first KR - KP slots, so the
  // KP-th key is r[KR-1]). KR = 80: a per-reference binary max-heap of KP keys in shared memory
  // (1-indexed, root = the KP-th key): an insertion is a ~7-level sift-down instead of a
  // 160-instruction register network.
  constexpr bool HEAP = KR > 48;
  RegTopK32<HEAP ? 1 : KR> rt;
  if constexpr (!HEAP) {
#pragma unroll
    for (int k = 0; k < KR; ++k) rt.r[k] = k < KR - a.KP ? 0u : 0xffffffffu;
  }
  // (helper lanes RX..31 never insert; they alias lane RX-1's heap for the root reads)
  uint32_t* const scr0 = reinterpret_cast<uint32_t*>(smf + ((regw + 3) & ~3));  // 16-byte aligned
  uint32_t* heap = scr0 + warp * a.scr + 64 * VY + min(lane, RX - 1) * a.hp;
  uint32_t* const pub_own = pub + warp * 32 + lane;
  const uint32_t* const pub_other = pub + ((1 - hh) * kFWarps + wr) * 32 + lane;
  // HEAP4: a 4-ary max-heap, node n at position n + 3 (the children of n, 4n+1 .. 4n+4, are one
  // aligned 16-byte load at 4n+4), root kept in a register, fixed-depth sift-downs with the children
  // of the four children loaded one level ahead (as the 3xTF32 matcher's); zeros past the last node
  constexpr bool HEAP4 = HEAP && SCBM_BOXF_HEAP4;
  constexpr int kHB = HEAP4 ? 3 : 1;       // heap position of the root
  constexpr int kSift4 = KR > 85 ? 4 : 3;  // levels below the root
  uint32_t root_r = 0xffffffffu;           // HEAP4: the root (the KP-th key)
  if constexpr (HEAP4) {
    if (lane < RX) {
      for (int k = kHB; k < kHB + a.KP; ++k) heap[k] = 0xffffffffu;
      for (int k = kHB + a.KP; k < a.hp; ++k) heap[k] = 0u;
    }
  } else if constexpr (HEAP) {
    if (lane < RX)
      for (int k = 1; k <= a.KP; ++k) heap[k] = 0xffffffffu;
    if (lane < RX) heap[a.KP + 1] = 0u;  // padding child: never the larger one
  }
  const int rb = a.rb;
  float thr = __int_as_float(0x7f800000);  // +inf: largest d' that may still enter the top-KP
  uint32_t* scratch = scr0 + warp * a.scr;

  const int b0 = (0 - a.lo) / VY;
  const int span = max(-a.lo, a.hi);
  unsigned pend = 0u;  // survivor bits of the staged group(s)
  int rel1p = 0;
  auto set_thr = [&](uint32_t kth) {
    if (kth != 0xffffffffu) {
      // largest distance whose key can still tie the KP-th key, plus a rounding margin
      const float dmax = __uint_as_float(((kth >> rb) << (rb - 1)) | ((1u << (rb - 1)) - 1u));
      thr = fmaf(dmax, 1.0f + (NCC ? 1e-5f : 1e-6f), -nadd) + 1e-30f;
    }
  };
  auto flush = [&](int rel1c) {
    unsigned bits = pend;
    pend = 0u;
    if (!__any_sync(0xffffffffu, bits != 0u)) {
      if constexpr (WS == 2) {  // the partner half may have tightened the shared threshold
        const uint32_t own = HEAP4 ? root_r : HEAP ? heap[1] : rt.r[KR - 1];
        set_thr(min(own, *pub_other));
      }
      return;
    }
    const uint32_t* sc = scratch + lane;
    while (__any_sync(0xffffffffu, bits != 0u)) {
      const int i = 31 - __clz(bits | 1u);
      const uint32_t q = sc[32 * i] >> (rb - 1);
      const int rel1 = i < VY ? rel1p + i * a.Wn : rel1c + (i - VY) * a.Wn;
      const uint32_t key = bits ? (q << rb) | uint32_t(rel1) : 0xffffffffu;
      bits &= ~(1u << i);
      if constexpr (HEAP4) {
        if (key < root_r) {  // replace the root, sift down
          int n = 0;
          bool alive = true;
          uint32_t nroot = key;
          uint4 vv = *reinterpret_cast<const uint4*>(heap + 4);
          uint4 g0 = *reinterpret_cast<const uint4*>(heap + 8), g1 = *reinterpret_cast<const uint4*>(heap + 12);
          uint4 g2 = *reinterpret_cast<const uint4*>(heap + 16), g3 = *reinterpret_cast<const uint4*>(heap + 20);
#pragma unroll
          for (int lvl = 0; lvl < kSift4; ++lvl) {
            const bool r01 = vv.y > vv.x, r23 = vv.w > vv.z;
            const uint32_t m01 = max(vv.x, vv.y), m23 = max(vv.z, vv.w);
            const bool up = m23 > m01;
            const uint32_t big = max(m01, m23);
            const int cb = 4 * n + 1 + (up ? (r23 ? 3 : 2) : (r01 ? 1 : 0));
            const bool mv = alive && big > key;
            const uint4 nv = up ? (r23 ? g3 : g2) : (r01 ? g1 : g0);
            if (lvl + 1 < kSift4) {
              g0 = g1 = g2 = g3 = make_uint4(0u, 0u, 0u, 0u);
              // (each 16-byte block loaded only if it lies inside the row: blocks past the row hold no node)
              if (mv && 16 * cb + 12 <= a.hp) g0 = *reinterpret_cast<const uint4*>(heap + 16 * cb + 8);
              if (mv && 16 * cb + 16 <= a.hp) g1 = *reinterpret_cast<const uint4*>(heap + 16 * cb + 12);
              if (mv && 16 * cb + 20 <= a.hp) g2 = *reinterpret_cast<const uint4*>(heap + 16 * cb + 16);
              if (mv && 16 * cb + 24 <= a.hp) g3 = *reinterpret_cast<const uint4*>(heap + 16 * cb + 20);
            }
            if (mv) heap[3 + n] = big;
            if (lvl == 0) nroot = mv ? big : key;
            n = mv ? cb : n;
            alive = mv && 4 * cb + 1 < a.KP;
            vv = nv;
          }
          heap[3 + n] = key;
          root_r = nroot;
        }
      } else if constexpr (HEAP) {
        if (key < heap[1]) {  // replace the root, sift down (children of i: 2i, 2i+1)
          int h = 1;
          for (int c = 2; c <= a.KP; c = 2 * h) {
            // both children in one 8-byte load: rows are 8-byte aligned, c is even
            const uint2 vv = *reinterpret_cast<const uint2*>(heap + c);
            const uint32_t v0 = vv.x, v1 = vv.y;
            const int cb = v1 > v0 ? c + 1 : c;
            const uint32_t big = max(v0, v1);
            if (big <= key) break;
            heap[h] = big;
            h = cb;
          }
          heap[h] = key;
        }
      } else {
        rt.insert(key);
      }
    }
    const uint32_t kth = HEAP4 ? root_r : HEAP ? heap[1] : rt.r[KR - 1];
    if constexpr (WS == 2) {
      *pub_own = kth;
      set_thr(min(kth, *pub_other));
    } else {
      set_thr(kth);
    }
    __syncwarp();
  };
  // two phases over the dy blocks: the near offsets (dx pairs j < 5) of every block first (as in
  // the uint8 box kernel: thresholds tighten sooner; measured on c2 / c4). Heap lists (c3, K = 70)
  // measured slower with the split: one phase.
  const int kNearPairs = HEAP ? span + 1 : 5;
  // Z3: candidate plane offsets centre-out (0, +1, -1, ...), each restaged into the second region
  float* const creg = smf + (Z3 ? nch * a.PL : 0);
  for (int kz = 0; kz < (Z3 ? 2 * a.zwin : 1); ++kz) {
  int relz = 0;
  if constexpr (Z3) {
    const int dz = centre_out_f(kz);
    const int zc = zr + dz;
    if (dz < a.zlo || dz > a.zhi || zc < 0 || zc > a.P - nch) continue;  // CTA-uniform
    relz = (dz - a.zlo) * a.Wn * a.Wn;
    __syncthreads();  // every warp is done with the previous candidate planes
    const TIN* cimg = vol + size_t(zc) * plane;
    for (int e = threadIdx.x; e < nch * a.PL; e += blockDim.x) {
      const int c = e / a.PL, e2 = e - c * a.PL;
      const int r = e2 / a.RWp, x = e2 - r * a.RWp;
      const int yy = Ybase + r, xx = Xbase + x;
      creg[e] = (yy >= 0 && yy < a.H && xx >= 0 && xx < a.W)
                    ? float(__ldg(cimg + c * plane + size_t(yy) * a.W + xx)) - shift : 0.f;
    }
    __syncthreads();
  }
  if (wact) {  // (WS = 2: an inactive warp still joins the merge barrier below)
  for (int ph = 0; ph < 2; ++ph) {
  const int j_begin = ph == 0 ? 0 : kNearPairs, j_end = ph == 0 ? min(kNearPairs, span + 1) : span + 1;
  for (int kb = 0; kb < 2 * a.nblk; ++kb) {
    const int bb = b0 + centre_out_f(kb);
    if (bb < 0 || bb >= a.nblk) continue;
    const int dy0 = a.lo + bb * VY;
    const int cy0 = ry + dy0;  // candidate row of offset i = 0
    const int ilo = max(0, -cy0), ihi = min(min(VY - 1, a.hi - dy0), a.H - BK - cy0);
    if (ihi < ilo) continue;  // warp-uniform
    const unsigned rows = ((2u << ihi) - 1u) & ~((1u << ilo) - 1u);
    const float* cbase = creg + (rr0 + dy0) * a.RWp + rc0;
    const unsigned rmask = lane_ok ? rows : 0u;
    // one offset group (fixed dx, offsets dy0 .. dy0+VY-1) into staging half H (compile time)
    auto group = [&](int dx, auto hc) -> int {
      constexpr int H = decltype(hc)::value;
      const float* col = cbase + dx;
      // cross terms of the full / partial strip, and running squared-row sums for the norms;
      // the partial strip's column pairs (2p, 2p+1) go through packed FFMA2 (two FMAs per
      // instruction, __ffma2_rn) into pair accumulators summed at the end
      float Tp[VY], Tr[VY];
      float2 Tp2[VY];
#pragma unroll
      for (int i = 0; i < VY; ++i) {
        Tp[i] = Tr[i] = 0.f;
        Tp2[i] = make_float2(0.f, 0.f);
      }
      float Qp[NT + 1], Qr[NT + 1];
#pragma unroll
      for (int t = 0; t <= NT; ++t) Qp[t] = Qr[t] = 0.f;
      for (int c = 0; c < nch; ++c) {
        if (!C1) load_ref(c);
        const float* colc = col + c * a.PL;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          float cv[S];
#pragma unroll
          for (int m = 0; m < S; ++m) cv[m] = colc[t * a.RWp + m];
          float qp = Qp[t + 1], qr = Qr[t + 1];  // squared row sums (prefix taken below)
#pragma unroll
          for (int m = 0; m < S; ++m) {
            if (m < WL) qp = fmaf(cv[m], cv[m], qp);
            else qr = fmaf(cv[m], cv[m], qr);
          }
          Qp[t + 1] = qp;
          Qr[t + 1] = qr;
#pragma unroll
          for (int i = 0; i < VY; ++i) {
            const int r = t - i;
            if (r >= 0 && r < BK) {
#pragma unroll
              for (int p = 0; p < kPairs; ++p)
                Tp2[i] = __ffma2_rn(make_float2(R[r][2 * p], R[r][2 * p + 1]),
                                    make_float2(cv[2 * p], cv[2 * p + 1]), Tp2[i]);
#pragma unroll
              for (int m = 2 * kPairs; m < S; ++m) {
                if (m < WL) Tp[i] = fmaf(R[r][m], cv[m], Tp[i]);
                else Tr[i] = fmaf(R[r][m], cv[m], Tr[i]);
              }
            }
          }
        }
      }
#pragma unroll
      for (int i = 0; i < VY; ++i) Tp[i] += Tp2[i].x + Tp2[i].y;
#pragma unroll
      for (int t = 1; t <= NT; ++t) {  // prefix sums over the candidate rows
        Qp[t] += Qp[t - 1];
        Qr[t] += Qr[t - 1];
      }
      const bool colok = unsigned(rx + dx) <= unsigned(a.W - BK);
      float dpv[VY];
      unsigned fails = 0u;
#pragma unroll
      for (int i = VY - 1; i >= 0; --i) {
        const float np = Qp[i + BK] - Qp[i], nrest = Qr[i + BK] - Qr[i];
        if constexpr (NCC) {
          const float cc = hcombine<NS, WL, S>(Tp[i] + Tr[i], Tp[i]);  // C (Eq. 5)
          const float nc = hcombine<NS, WL, S>(np + nrest, np);       // ||X_c||^2
          dpv[i] = nrs - (nc > 0.f ? cc * rsqrtf(nc) : 0.f);
        } else {
          const float ep = fmaf(-2.f, Tp[i], np);
          const float ef = ep + fmaf(-2.f, Tr[i], nrest);
          dpv[i] = hcombine<NS, WL, S>(ef, ep);  // d' = n_c - 2 C
        }
        // slack thr - d' >= 0 (or +inf): the candidate may enter the top-KP
        fails = __funnelshift_l(__float_as_uint(thr - dpv[i]), fails, 1);  // (fails << 1) | sign
      }
      const unsigned bits = ~fails & (colok ? rmask : 0u);
      // survivors of two consecutive offset groups are inserted together (fewer, fuller rounds:
      // a round lasts as long as the busiest lane); group h's distances sit in scratch rows
      // h*VY .. h*VY+VY-1 and its bits at the same positions of pend
      if (__any_sync(0xffffffffu, bits != 0u)) {
        uint32_t* sc = scratch + H * (32 * VY) + lane;
#pragma unroll
        for (int i = 0; i < VY; ++i) sc[32 * i] = __float_as_uint(fmaxf(dpv[i] + nadd, 0.f));
        pend |= bits << (H * VY);
      }
      return relz + (dy0 - a.lo) * a.Wn + (dx - a.lo) + 1;  // rel + 1 >= 1 (0 = sentinel)
    };
    // dx centre-out (0, 1, -1, 2, -2, ...): pairs (-j, j+1) staged in the two halves and
    // flushed together (a round lasts as long as the busiest lane); a lone group flushes alone
    for (int j = j_begin; j < j_end; ++j) {
      if (WS == 2 && (j & 1) != hh) continue;  // the other half's dx pair
      const bool va = -j >= a.lo, vb = j + 1 <= a.hi;
      if (!va && !vb) continue;  // warp-uniform
      rel1p = group(va ? -j : j + 1, std::integral_constant<int, 0>{});
      flush(va && vb ? group(j + 1, std::integral_constant<int, 1>{}) : 0);
    }
  }
  }  // phases
  }  // wact
  }  // plane offsets (Z3)
  if (WS == 1 && !wact) return;  // (Z3: reference rows past the band joined the restaging only)

  if constexpr (WS == 2) {
    // merge the second half's list into the first's (0 sentinels skipped), then only the first
    // half's warps go on to a5
    // (in rounds of 16 keys through the second warp's own scratch, [k][lane]: the staged region
    // stays intact for the a5 re-score)
    uint32_t* ml = scr0 + (kFWarps + wr) * a.scr;
#pragma unroll
    for (int k0 = 0; k0 < KR; k0 += 16) {
      __syncthreads();
      if (hh == 1 && wact) {
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (k0 + k < KR) ml[k * 32 + lane] = rt.r[k0 + k < KR ? k0 + k : 0];
      }
      __syncthreads();
      if (hh == 0 && wact && lane < RX) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          if (k0 + k < KR) {
            const uint32_t x = ml[k * 32 + lane];
            rt.insert(x == 0u ? 0xffffffffu : x);
          }
        }
      }
    }
    if constexpr (!SCBM_BOXF_A5HALVES) {
      if (hh == 1 || !wact) return;
    }
  }
  // WS = 2, A5HALVES: both warps of a reference row run a5, the first on references [0, nsplit),
  // the second on [nsplit, nref); the first hands the merged lists of the second half over through
  // the two warps' scratch (keys < kTS: the second warp's, [j'][25]; the rest: the first warp's,
  // [j'][KR - kTS + 1]; odd pitches: conflict-free row reads)
  constexpr int kTS = 24;
  constexpr int kP1 = KR > kTS ? KR - kTS + 1 : 1;
  const int nref_all = min(RX, a.nx - ix_first);
  const int nsplit = (WS == 2 && SCBM_BOXF_A5HALVES) ? (nref_all + 1) / 2 : nref_all;
  uint32_t* const tb0 = scr0 + (kFWarps + wr) * a.scr;
  uint32_t* const tb1 = scr0 + wr * a.scr;
  if constexpr (WS == 2 && SCBM_BOXF_A5HALVES) {
    __syncwarp();
    if (hh == 0 && wact && lane >= nsplit && lane < nref_all) {
      const int jq = lane - nsplit;
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        if (k < kTS) tb0[jq * (kTS + 1) + k] = rt.r[k];
        else tb1[jq * kP1 + (k - kTS)] = rt.r[k];
      }
    }
    __syncthreads();
    if (!wact) return;
  }
  // key k of reference j taken from the hand-over buffers (second warp, WS = 2)
  auto handed = [&](int j, int k) -> uint32_t {
    const int jq = j - nsplit;
    return k < kTS ? tb0[jq * (kTS + 1) + k] : tb1[jq * kP1 + (k - kTS)];
  };
  (void)handed;

  // ---- a5 + a6: stage each reference's KP keys (register lists; the heaps already are in shared
  // memory), then per reference (warp-cooperative) re-score them by direct differences from the
  // input, sort the (distance, idx) keys and write K.
  if constexpr (!HEAP && WS == 1) {
    if (lane_ok) {
#pragma unroll
      for (int k = 0; k < KR; ++k) scratch[lane * (KR + 1) + k] = rt.r[k];
    }
  }
  __syncwarp();
  const int nref = min(RX, a.nx - ix_first);
  const size_t band_refs = size_t(a.iy_end - a.iy_begin) * a.nx;
  const size_t row0 = size_t(f) * band_refs + size_t(iy0 - a.iy_begin) * a.nx + ix_first;
  constexpr int NJ = (KR + 31) / 32;
  if constexpr (NCC && KR > 32) {
    // a5 (NCC, float input, K + m > 32: lists of 40 / 48 keys or the shared-memory heaps): per
    // reference the kept candidates' NCC recomputed in double from the input (Eq. 4), ranked by
    // (float32 d_NCC = -NCC, idx) -- the reported value, as the f32 rule compares -- with the warp's
    // 64-bit key lists (topk.cuh), K written; a reference whose worst kept key's quantum could still
    // hold a score as good as the exact K-th one goes to the exact fix-up
    static_assert(sizeof(TIN) == 4, "wide NCC lists serve float input (uint8 NCC keeps K + m <= 32)");
    constexpr int NJ = (KR + 31) / 32;
    for (int j = 0; j < nref; ++j) {
      const int rxj = (ix_first + j) * S;
      const size_t rowj = row0 + j;
      double nrq = 0.0;
      // kept slot k -> its exact (float32 d_NCC, idx) key (double-precision NCC)
      auto ncc_key = [&](int k) -> uint64_t {
        uint32_t kk;
        if constexpr (HEAP) kk = k < a.KP ? heap[(j - min(lane, RX - 1)) * a.hp + kHB + k] : 0xffffffffu;
        else kk = k < a.KP ? scratch[j * (KR + 1) + (KR - a.KP) + k] : 0xffffffffu;  // skip 0 sentinels
        const bool have = kk != 0u && kk != 0xffffffffu;
        double nrd = 0.0, cd = 0.0, ncd = 0.0;
        int cy = ry, cx = rxj;
        if (have) {
          const int rel = int(kk & ((1u << rb) - 1u)) - 1;
          const int dyy = rel / a.Wn, dxx = rel - dyy * a.Wn;
          cy = ry + dyy + a.lo;
          cx = rxj + dxx + a.lo;
        }
        for (int c = 0; c < nch; ++c) {
          const TIN* pr = img + c * plane + size_t(ry) * a.W + rxj;
          const TIN* pc = img + c * plane + size_t(cy) * a.W + cx;
          for (int l = 0; l < BK; ++l)
#pragma unroll
            for (int m = 0; m < BK; ++m) {
              const double vr = double(__ldg(pr + l * a.W + m)), vc = double(__ldg(pc + l * a.W + m));
              nrd = fma(vr, vr, nrd);
              cd = fma(vr, vc, cd);
              ncd = fma(vc, vc, ncd);
            }
        }
        nrq = nrd;  // the same for every slot (the reference's own norm)
        if (!have) return kKeyInf;
        const double den = sqrt(nrd * ncd);
        const float dn = -float(den > 0.0 ? cd / den : 0.0);  // the reported d_NCC
        return (uint64_t(ord_f32(dn)) << 32) | uint32_t(cy * a.W + cx);
      };
      // > 64 kept keys: one warp bitonic sort of 128 (4 per lane, element e = 4 lane + i); fewer:
      // the warp lists. out(k) -> the k-th smallest key
      uint64_t sv[4];
      WarpTopK<NJ> top;
      if constexpr (NJ >= 3) {
#pragma unroll
        for (int i = 0; i < 4; ++i) sv[i] = ncc_key(4 * lane + i);
        warp_sort128(sv, lane);
      } else {
        top.init();
#pragma unroll
        for (int sl = 0; sl < NJ; ++sl) top.merge(ncc_key(sl * 32 + lane), lane);
      }
      uint64_t kv;
      if constexpr (NJ >= 3) {
        uint64_t kq = sv[0];
#pragma unroll
        for (int i = 1; i < 4; ++i)
          if (i == (a.K - 1) % 4) kq = sv[i];
        kv = __shfl_sync(0xffffffffu, kq, (a.K - 1) / 4);
      } else {
        kv = kKeyInf;
#pragma unroll
        for (int sl = 0; sl < NJ; ++sl)
          if (sl == (a.K - 1) / 32) kv = top.v[sl];
        kv = __shfl_sync(0xffffffffu, kv, (a.K - 1) % 32);
      }
      const uint32_t klast = HEAP ? heap[(j - min(lane, RX - 1)) * a.hp + kHB] : scratch[j * (KR + 1) + KR - 1];
      nrq = __shfl_sync(0xffffffffu, nrq, 0);
      if (lane == 0 && klast != 0u && klast != 0xffffffffu && kv != kKeyInf && nrq > 0.0) {
        const double fK = -double(unord_f32(uint32_t(kv >> 32)));  // exact K-th NCC (float32)
        const float smin = __uint_as_float((klast >> rb) << (rb - 1));  // quantum minimum
        const double nrs_d = sqrt(nrq), scK = nrs_d * (1.0 - fK);    // exact K-th filter score
        if (double(smin) <= scK * (1.0 + 1e-5) + 1e-6 * nrs_d) {
          const int pos = atomicAdd(a.fix_count, 1);
          a.fix_list[pos] = int(rowj);
        }
      }
#pragma unroll
      for (int sl = 0; sl < (NJ >= 3 ? 4 : NJ); ++sl) {
        const int k = NJ >= 3 ? 4 * lane + sl : sl * 32 + lane;
        if (k < a.K) {
          const uint64_t key = NJ >= 3 ? sv[sl] : top.v[sl < NJ ? sl : 0];
          const bool none = key == kKeyInf;
          a.idx_out[rowj * a.K + k] = none ? -1 : int32_t(uint32_t(key));
          a.dist_out[rowj * a.K + k] = none ? __int_as_float(0x7f800000) : unord_f32(uint32_t(key >> 32));
        }
      }
    }
    return;
  } else if constexpr (NCC) {
    // a5 (NCC): exact cross terms / norms of the KP (<= 32) kept candidates, which arrive in key
    // order; exact neighbour checks + odd-even repair (128-bit comparisons for uint8, ncc.cuh),
    // write K (idx, d_NCC = -NCC)
    constexpr bool EXACT = sizeof(TIN) == 1;
    for (int j = 0; j < nref; ++j) {
      const int rxj = (ix_first + j) * S;
      const uint32_t kk = lane < a.KP ? scratch[j * (KR + 1) + (KR - a.KP) + lane] : 0xffffffffu;  // skip 0 sentinels
      NccItem it;
      it.c = 0; it.n = 1; it.f = 0.0; it.idx = -1;
      double nrd = 0.0, cd = 0.0, ncd = 0.0;
      int nri = 0, ci = 0, nci = 0;
      int cy = 0, cx = 0;
      const bool have = kk != 0u && kk != 0xffffffffu;
      if (have) {
        const int rel = int(kk & ((1u << rb) - 1u)) - 1;
        const int dyy = rel / a.Wn, dxx = rel - dyy * a.Wn;
        cy = ry + dyy + a.lo;
        cx = rxj + dxx + a.lo;
      }
      for (int c = 0; c < nch; ++c) {
        const TIN* pr = img + c * plane + size_t(ry) * a.W + rxj;
        const TIN* pc = img + c * plane + size_t(cy) * a.W + cx;
        for (int l = 0; l < BK; ++l)
#pragma unroll
          for (int m = 0; m < BK; ++m) {
            const TIN vr = __ldg(pr + l * a.W + m), vc = have ? __ldg(pc + l * a.W + m) : TIN(0);
            if constexpr (EXACT) {
              nri += int(vr) * int(vr);
              ci += int(vr) * int(vc);
              nci += int(vc) * int(vc);
            } else {
              nrd = fma(double(vr), double(vr), nrd);
              cd = fma(double(vr), double(vc), cd);
              ncd = fma(double(vc), double(vc), ncd);
            }
          }
      }
      if (have) {
        it.idx = cy * a.W + cx;
        if constexpr (EXACT) {
          const bool zero = nri == 0 || nci == 0;
          it.c = zero ? 0 : ci;
          it.n = zero ? 1 : nci;
          it.f = zero ? 0.0 : double(ci) / sqrt(double(nri) * double(nci));
        } else {
          const double den = sqrt(nrd * ncd);
          // ordered by the reported float32 value, ties by idx (rows sorted by (dist, idx))
          it.f = double(float(den > 0.0 ? cd / den : 0.0));
        }
      }
      // the worst kept key's quantum could still hold a score as good as the exact K-th one:
      // a dropped candidate might belong to the top-K -> exact re-rank of the window (fixup.cu)
      const uint32_t klast = __shfl_sync(0xffffffffu, kk, a.KP - 1);
      it = warp_repair_ncc<EXACT>(it, lane);  // kept keys arrive in (quantised score, idx) order
      const double fK = __shfl_sync(0xffffffffu, it.f, a.K - 1);
      const double nrq = EXACT ? double(nri) : nrd;
      if (lane == 0 && klast != 0u && klast != 0xffffffffu && nrq > 0.0) {
        const float smin = __uint_as_float((klast >> rb) << (rb - 1));  // quantum minimum
        const double nrs_d = sqrt(nrq), scK = nrs_d * (1.0 - fK);     // exact K-th filter score
        if (double(smin) <= scK * (1.0 + 1e-5) + 1e-6 * nrs_d) {
          const int pos = atomicAdd(a.fix_count, 1);
          a.fix_list[pos] = int(row0 + j);
        }
      }
      if (lane < a.K) {
        a.idx_out[(row0 + j) * a.K + lane] = it.idx;
        a.dist_out[(row0 + j) * a.K + lane] = it.idx < 0 ? __int_as_float(0x7f800000) : float(-it.f);
      }
    }
    return;
  } else {
  const int j_lo = (WS == 2 && hh == 1) ? nsplit : 0, j_hi = (WS == 2 && hh == 0) ? nsplit : nref;
  for (int j = j_lo; j < j_hi; ++j) {
    const int rxj = (ix_first + j) * S;
    const float nrj_a5 = __shfl_sync(0xffffffffu, nr, j);  // ||X_i||^2 (centred) of reference j
    WarpTopK<NJ> top;
    top.init();
#pragma unroll
    for (int sl = 0; sl < NJ; ++sl) {
      if constexpr (kSplitG > 1) {
        if (sl == NJ - 1) {
          // the last slot holds only kN1 (<= 16) list entries: kSplitG lanes per key, each a strided
          // share of the patch columns, summed by xor shuffles (instead of a full-length pass with
          // kN1 of 32 lanes busy)
          const int kq = lane / kSplitG, part = lane % kSplitG;
          uint32_t kk = 0xffffffffu;
          if constexpr (WS == 2) {
            if (hh == 0 || !SCBM_BOXF_A5HALVES) {
#pragma unroll
              for (int q = 0; q < kN1; ++q) {
                const uint32_t v = __shfl_sync(0xffffffffu, rt.r[sl * 32 + q], j);
                if (kq == q) kk = v;
              }
            } else if (kq < kN1) {
              kk = handed(j, sl * 32 + kq);
            }
          } else {
            if (kq < kN1) kk = scratch[j * (KR + 1) + sl * 32 + kq];
          }
          const bool have = kq < kN1 && kk != 0u && kk != 0xffffffffu;
          int cy = ry, cx = rxj;
          if (have) {
            const int rel = int(kk & ((1u << rb) - 1u)) - 1;
            const int dyy = rel / a.Wn, dxx = rel - dyy * a.Wn;
            cy = ry + dyy + a.lo;
            cx = rxj + dxx + a.lo;
          }
          const float* prs = smf + (ry - Ybase) * a.RWp + (rxj - Xbase);
          const float* pcs = smf + (cy - Ybase) * a.RWp + (cx - Xbase);
          float acc[4] = {0.f, 0.f, 0.f, 0.f};
          for (int c = 0; c < nch; ++c) {
#pragma unroll 4
            for (int l = 0; l < BK; ++l) {
              float t = 0.f;
#pragma unroll
              for (int m = 0; m < BK; m += kSplitG) {
                if (m + part < BK) {
                  const float df = prs[c * a.PL + l * a.RWp + m + part] - pcs[c * a.PL + l * a.RWp + m + part];
                  t = fmaf(df, df, t);
                }
              }
              acc[l & 3] += t;
            }
          }
          float d = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
          for (int o = 1; o < kSplitG; o <<= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
          if (have && part == 0 && d * 180.f < nrj_a5 && (cy != ry || cx != rxj)) {
            // near-duplicate pair: re-scored from the input in global memory (as the full-length path)
            float g[4] = {0.f, 0.f, 0.f, 0.f};
            for (int c = 0; c < nch; ++c) {
#pragma unroll 4
              for (int l = 0; l < BK; ++l) {
                float t = 0.f;
#pragma unroll
                for (int m = 0; m < BK; ++m) {
                  const float df = __ldg(img + c * plane + size_t(ry + l) * a.W + rxj + m) -
                                   __ldg(img + c * plane + size_t(cy + l) * a.W + cx + m);
                  t = fmaf(df, df, t);
                }
                g[l & 3] += t;
              }
            }
            d = (g[0] + g[1]) + (g[2] + g[3]);
          }
          uint64_t key = (have && part == 0) ? (uint64_t(__float_as_uint(d)) << 32) | uint32_t(cy * a.W + cx) : kKeyInf;
          key = __shfl_sync(0xffffffffu, key, min(lane * kSplitG, 31));
          top.merge(lane < kN1 ? key : kKeyInf, lane);
          continue;
        }
      }
      const int k = sl * 32 + lane;
      uint64_t key = kKeyInf;
      uint32_t kk;
      if constexpr (HEAP) {
        kk = k < a.KP ? heap[(j - min(lane, RX - 1)) * a.hp + kHB + k] : 0xffffffffu;
      } else if constexpr (WS == 2) {  // lane j's register list, one key per lane by shuffles
        kk = 0xffffffffu;
        if (hh == 0 || !SCBM_BOXF_A5HALVES) {
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            if (sl * 32 + q < KR) {
              const uint32_t v = __shfl_sync(0xffffffffu, rt.r[sl * 32 + q < KR ? sl * 32 + q : 0], j);
              if (lane == q) kk = v;
            }
          }
        } else if (k < KR) {  // (the second warp: from the hand-over buffers)
          kk = handed(j, k);
        }
      } else {
        kk = k < KR ? scratch[j * (KR + 1) + k] : 0xffffffffu;
      }
      if (kk != 0u && kk != 0xffffffffu) {
        int rel = int(kk & ((1u << rb) - 1u)) - 1;
        int zc = 0;
        if constexpr (Z3) {  // plane offset index, then the window slot
          const int zi = rel / (a.Wn * a.Wn);
          rel -= zi * a.Wn * a.Wn;
          zc = zr + a.zlo + zi;
        }
        const int dyy = rel / a.Wn, dxx = rel - dyy * a.Wn;
        const int cy = ry + dyy + a.lo, cx = rxj + dxx + a.lo;
        const float* cimg = Z3 ? reinterpret_cast<const float*>(vol) + size_t(zc) * plane : img;
        // (rows in independent partial sums, 4 in flight: the loads of a row do not wait for the
        // previous row's FMA chain)
        auto rescore = [&](auto ld_r, auto ld_c) -> float {
          float acc[4] = {0.f, 0.f, 0.f, 0.f};
          for (int c = 0; c < nch; ++c) {
#pragma unroll 4
            for (int l = 0; l < BK; ++l) {
              float t = 0.f;
#pragma unroll
              for (int m = 0; m < BK; ++m) {
                const float df = ld_r(c, l, m) - ld_c(c, l, m);
                t = fmaf(df, df, t);
              }
              acc[l & 3] += t;
            }
          }
          return (acc[0] + acc[1]) + (acc[2] + acc[3]);
        };
        auto from_global = [&]() {
          return rescore([&](int c, int l, int m) { return __ldg(img + c * plane + size_t(ry + l) * a.W + rxj + m); },
                         [&](int c, int l, int m) { return __ldg(cimg + c * plane + size_t(cy + l) * a.W + cx + m); });
        };
        float d;
        if constexpr (Z3) {
          d = from_global();
        } else {
          // from the staged region (x' = fl(x - 0.5), shared memory): x' differs from x - 0.5 by at
          // most 2^-24 |x'|, which moves d by at most 2^-23 sqrt(2 d) (2 sqrt(n_r) + sqrt(d))
          // (Cauchy-Schwarz) -- below 5e-6 d whenever d >= n_r / 205. Closer pairs (near-duplicate
          // patches) are re-scored from the input in global memory.
          const float* prs = smf + (ry - Ybase) * a.RWp + (rxj - Xbase);
          const float* pcs = smf + (cy - Ybase) * a.RWp + (cx - Xbase);
          d = rescore([&](int c, int l, int m) { return prs[c * a.PL + l * a.RWp + m]; },
                      [&](int c, int l, int m) { return pcs[c * a.PL + l * a.RWp + m]; });
          // (the reference itself, d = 0 exactly, needs no second look)
          if (d * 180.f < nrj_a5 && (cy != ry || cx != rxj)) d = from_global();
        }
        key = (uint64_t(__float_as_uint(d)) << 32) | uint32_t((Z3 ? zc * a.H : 0) * a.W + cy * a.W + cx);
      }
      top.merge(key, lane);
    }
    {  // worst kept key vs the exact K-th distance (see the NCC branch; fp32 filter error margin)
      uint64_t kv = kKeyInf;
#pragma unroll
      for (int sl = 0; sl < NJ; ++sl)
        if (sl == (a.K - 1) / 32) kv = top.v[sl];
      kv = __shfl_sync(0xffffffffu, kv, (a.K - 1) % 32);
      const float nrj = __shfl_sync(0xffffffffu, nr, j);
      uint32_t klast;
      if constexpr (HEAP) klast = heap[(j - min(lane, RX - 1)) * a.hp + kHB];  // max-heap root
      else if constexpr (WS == 2) klast = (hh == 0 || !SCBM_BOXF_A5HALVES) ? __shfl_sync(0xffffffffu, rt.r[KR - 1], j)
                                                                           : handed(j, KR - 1);
      else klast = scratch[j * (KR + 1) + KR - 1];
      if (lane == 0 && klast != 0u && klast != 0xffffffffu && kv != kKeyInf) {
        const float dK = __uint_as_float(uint32_t(kv >> 32));
        const float smin = __uint_as_float((klast >> rb) << (rb - 1));
        // (1.5e-5: the exact K-th distance comes from the staged region, within 5e-6 of the input's)
        if (smin <= fmaf(dK, 1.0f + 1.5e-5f, 4e-6f * (nrj + dK))) {
          const int pos = atomicAdd(a.fix_count, 1);
          a.fix_list[pos] = int(row0 + j);
        }
      }
    }
#pragma unroll
    for (int sl = 0; sl < NJ; ++sl) {
      const int k = sl * 32 + lane;
      if (k < a.K) {
        const uint64_t key = top.v[sl];
        const bool none = key == kKeyInf;
        a.idx_out[(row0 + j) * a.K + k] = none ? -1 : int32_t(uint32_t(key));
        a.dist_out[(row0 + j) * a.K + k] = none ? __int_as_float(0x7f800000) : __uint_as_float(uint32_t(key >> 32));
      }
    }
  }
  }
}

constexpr int kFVY = 8;

// window split (WS = 2) where one 8-warp CTA per SM would be all the SM gets: several channel
// planes (the staged region takes the SM's shared memory) or fewer CTAs than 2 per SM; register
// lists only (the c3-style shared heaps keep WS = 1)
size_t boxf_bytes(const Geometry& g, int KR, int ws, BoxfArgs* a);

int boxf_ws(const Geometry& g, int KR) {
  if (KR > 48 || g.metric != SC_METRIC_L2 || g.z3) return 1;
  const int ns = (g.b + g.s - 1) / g.s, rx = 33 - ns;
  const long long ctas = (long long)((g.nx + rx - 1) / rx) * ((g.ny + kFWarps - 1) / kFWarps);
  if (!(g.C > 1 || ctas < 2 * 148)) return 1;
  BoxfArgs t{};
  return boxf_bytes(g, KR, 2, &t) <= 227 * 1024 ? 2 : 1;  // (else the plain layout)
}

size_t boxf_layout(const Geometry& g, int KR, BoxfArgs* a) { return boxf_bytes(g, KR, boxf_ws(g, KR), a); }

size_t boxf_bytes(const Geometry& g, int KR, int ws, BoxfArgs* a) {
  const int ns = (g.b + g.s - 1) / g.s, rx = 33 - ns;
  a->nblk = (g.Wn + kFVY - 1) / kFVY;
  a->RH = (kFWarps - 1) * g.s + a->nblk * kFVY + g.b;
  a->RWp = 32 * g.s + g.Wn - 1 + 1;
  a->PL = a->RH * a->RWp;
  // heap pitch: 1-indexed heap + a padding child, = 2 (mod 4) words: 8-byte aligned rows whose
  // 64-bit child loads hit distinct bank pairs across a half-warp
  a->hp = ((g.KP + 2 + 1) & ~3) + 2;
  if (SCBM_BOXF_HEAP4 && KR > 48) {  // 4-ary: nodes at 3 .. KP + 2, zero children and prefetch rows past them
    // (the last internal node's children end at position 4 ((KP - 2) / 4) + 7; the sift-down guards
    // each 16-byte prefetch block separately, so the pitch stays minimal: c3 NCC keeps 2 CTAs / SM)
    a->hp = 4 * ((g.KP - 2) / 4) + 8;
    if (a->hp % 8 == 0) a->hp += 4;  // = 4 (mod 8): the lanes' 16-byte loads spread over the banks
  }
  // per warp: two staged offset groups (+ the heaps, or the output lists with WS = 1)
  a->scr = KR > 48 ? 64 * kFVY + rx * a->hp : ws == 2 ? 64 * kFVY : std::max(64 * kFVY, rx * (KR + 1));
  const size_t region = size_t(((g.z3 ? 2 : 1) * g.C * a->PL + 3) & ~3);  // (3D: + candidate planes; 16-B aligned)
  const size_t base = region + size_t(kFWarps) * ws * a->scr + (ws == 2 ? 2 * kFWarps * 32 : 0);
  // WS = 2: the per-row list areas reuse the staged region when it is large enough
  const size_t lists = size_t(kFWarps) * rx * (KR + 1);
  a->lofs = ws == 2 && lists > region ? int(base) : 0;
  return (base + (ws == 2 && lists > region ? lists : 0)) * 4;
}

// key bits of the window-relative index + 1 (values 1 .. Wn^2; 0 is the sentinel)
// key bits of the window-relative index + 1 (values 1 .. n slots; 0 is the sentinel)
int rel_bits_n(long long n) {
  int rb = 1;
  while ((1ll << rb) <= n) ++rb;
  return rb;
}
int boxf_rel_bits(int Wn) { return rel_bits_n((long long)Wn * Wn); }
// 3D search: (plane offset, window slot) = zwin Wn^2 slots
int boxf_rel_bits_g(const Geometry& g) { return rel_bits_n((long long)(g.z3 ? g.zwin : 1) * g.Wn * g.Wn); }

// register list length: the smallest instantiated size >= KP (an insertion costs 2 KR - 1 IMNMX)
int boxf_kr(const Geometry& g) {
  return g.KP <= 24 ? 24 : g.KP <= 32 ? 32 : g.KP <= 40 ? 40 : g.KP <= 48 ? 48 : g.KP <= 80 ? 80 : 0;
}

template <int S, int BK, int KR, bool NCC = false, typename TIN = float>
cudaError_t launch_boxf_t(const BoxfArgs& a, int F, size_t smem, cudaStream_t st, int ws = 1, bool z3 = false) {
  const int tiles_y = (a.iy_end - a.iy_begin + a.rows - 1) / a.rows;
  auto k = a.C == 1 ? bm_boxf_kernel<S, BK, kFVY, KR, true, NCC, TIN> : bm_boxf_kernel<S, BK, kFVY, KR, false, NCC, TIN>;
  if constexpr (KR <= 48 && !NCC) {
    if (ws == 2) k = a.C == 1 ? bm_boxf_kernel<S, BK, kFVY, KR, true, NCC, TIN, 2>
                              : bm_boxf_kernel<S, BK, kFVY, KR, false, NCC, TIN, 2>;
  }
  if constexpr (!NCC) {
    if (z3) k = a.C == 1 ? bm_boxf_kernel<S, BK, kFVY, KR, true, NCC, TIN, 1, true>
                         : bm_boxf_kernel<S, BK, kFVY, KR, false, NCC, TIN, 1, true>;
  }
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k<<<dim3(a.tiles_x * tiles_y, F), kFWarps * 32 * ws, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

bool boxf_supported(const Geometry& g) {
  // L2: float images (uint8 L2 has the dp4a box kernel); NCC: both dtypes, K + m <= 32
  if (g.metric == SC_METRIC_L2 && g.dtype != SC_DTYPE_F32) return false;
  // NCC: uint8 keeps the exact 128-bit re-rank of <= 32 kept keys; float input takes wider lists
  if (g.metric == SC_METRIC_NCC && g.KP > (g.dtype == SC_DTYPE_U8 ? 32 : 80)) return false;
  const bool shape = (g.s == 3 && g.b == 8) || (g.s == 1 && g.b == 7) || (g.s == 4 && g.b == 8) ||
                     (g.s == 2 && g.b == 8) || (g.s == 1 && g.b == 6);
  if (!shape) return false;
  const int kr = boxf_kr(g);
  if (kr == 0) return false;
  // keeps >= 20 distance bits in the 32-bit keys (>= 19 with the 3D search's plane offsets)
  if (boxf_rel_bits_g(g) > (g.z3 ? 13 : 12)) return false;
  if (g.z3 && (g.metric != SC_METRIC_L2 || kr > 48)) return false;  // 3D: L2 with register lists
  BoxfArgs a{};
  // up to the whole SM's shared memory (one channel with register lists normally fits two CTAs)
  return boxf_layout(g, kr, &a) <= 227 * 1024;
}

namespace {
// Tile height (reference rows per CTA): the grid is tiles_x x ceil(rows_in_band / R) CTAs per
// frame, each of which keeps one SM slot busy for a time ~ R rows; fewer rows than kFWarps pay off
// where the full-height grid leaves most of its last wave empty (c4: 384 CTAs at 1 CTA / SM =
// 2.6 waves -> R = 7: 444 CTAs = 3 full waves of 7/8 the work each). Cost model: waves x R.
int boxf_rows(long long tiles_x, long long band_rows, long long F, int per_sm) {
  static int n_sm = 0;
  if (n_sm == 0) {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
      n_sm = v;
    else
      n_sm = 148;
  }
  const long long slots = (long long)n_sm * per_sm;
  auto cost = [&](int r) {
    const long long units = tiles_x * ((band_rows + r - 1) / r) * F;
    return (double)((units + slots - 1) / slots) * r;
  };
  // SC_BM_BOXF_ROWS=r (1 .. kFWarps) forces the tile height (A/B timing, tests of short tiles)
  static const int forced = [] {
    const char* e = getenv("SC_BM_BOXF_ROWS");
    const int v = e ? atoi(e) : 0;
    return v >= 1 && v <= kFWarps ? v : 0;
  }();
  if (forced) return forced;
  // two CTAs per SM: a part-filled last wave is not idle time (its CTAs run alone on their SMs,
  // faster) -- the model does not hold there (m1, 2 CTAs / SM: R = 7 2.10 -> 2.30 ms)
  if (per_sm != 1) return kFWarps;
  int best = kFWarps;
  double best_c = cost(kFWarps);
  // one row fewer only, and only for a >= 8 % modelled gain: the model counts work, but an SM
  // with fewer active warps also issues less (measured: c4 R = 7 2.446 -> 2.398 ms for 12.5 %
  // modelled; m1 R = 5, 6 % modelled, 2.10 -> 2.29 ms)
  const double c = cost(kFWarps - 1);
  if (c < best_c * 0.92) best = kFWarps - 1;
  return best;
}

cudaError_t launch_boxf_kernel(const sc_bm_plan_s& p, const void* imgs, int F, int iy_begin, int iy_end,
                               int32_t* idx_out, void* dist_out, cudaStream_t st, int64_t* launches) {
  const Geometry& g = p.g;
  BoxfArgs a{};
  a.fix_count = p.ws.fix_count;
  a.fix_list = p.ws.fix_list;
  a.imgs = imgs;
  a.idx_out = idx_out;
  a.dist_out = static_cast<float*>(dist_out);
  a.H = g.H; a.W = g.W; a.C = g.C; a.Wn = g.Wn; a.K = g.K; a.KP = g.KP; a.lo = g.lo; a.hi = g.hi; a.nx = g.nx;
  a.iy_begin = iy_begin; a.iy_end = iy_end;
  const int ns = (g.b + g.s - 1) / g.s;
  a.tiles_x = (g.nx + (33 - ns) - 1) / (33 - ns);
  a.rb = boxf_rel_bits_g(g);
  a.z0 = int(p.batch_f0);
  a.sz = p.zstride;
  a.P = int(p.n_planes);
  a.zlo = p.zlo;
  a.zhi = p.zhi;
  a.zwin = g.zwin;
  const int kr = boxf_kr(g);  // the layout and the instantiation use the same list size
  const size_t smem = boxf_layout(g, kr, &a);
  if (launches) *launches += 1;
  const int ws = g.metric == SC_METRIC_NCC ? 1 : boxf_ws(g, kr);
  // CTAs per SM: 16-warp window-split CTAs (128 registers) take a whole SM; 8-warp CTAs two when
  // their shared memory fits twice
  const int per_sm = ws == 2 ? 1 : (2 * (smem + 1024) <= 228 * 1024 ? 2 : 1);
  a.rows = boxf_rows(a.tiles_x, iy_end - iy_begin, F, per_sm);
  if (g.metric == SC_METRIC_NCC) {  // uint8: K + m <= 32, exact re-rank; float: lists up to 80
#define SCBM_NCC_CASE(S_, B_)                                                                          \
  if (g.s == S_ && g.b == B_) {                                                                        \
    if (kr == 24)                                                                                      \
      return g.dtype == SC_DTYPE_U8 ? launch_boxf_t<S_, B_, 24, true, uint8_t>(a, F, smem, st)         \
                                    : launch_boxf_t<S_, B_, 24, true, float>(a, F, smem, st);          \
    if (kr == 32)                                                                                      \
      return g.dtype == SC_DTYPE_U8 ? launch_boxf_t<S_, B_, 32, true, uint8_t>(a, F, smem, st)         \
                                    : launch_boxf_t<S_, B_, 32, true, float>(a, F, smem, st);          \
    if (kr == 40) return launch_boxf_t<S_, B_, 40, true, float>(a, F, smem, st);                       \
    if (kr == 48) return launch_boxf_t<S_, B_, 48, true, float>(a, F, smem, st);                       \
    return launch_boxf_t<S_, B_, 80, true, float>(a, F, smem, st);                                     \
  }
    SCBM_NCC_CASE(3, 8)
    SCBM_NCC_CASE(1, 7)
    SCBM_NCC_CASE(4, 8)
    SCBM_NCC_CASE(2, 8)
    SCBM_NCC_CASE(1, 6)
#undef SCBM_NCC_CASE
    return cudaErrorInvalidValue;
  }
  const bool z3 = g.z3 != 0;
#define SCBM_BOXF_CASE(S_, B_)                                                    \
  if (g.s == S_ && g.b == B_) {                                                   \
    if (kr == 24) return launch_boxf_t<S_, B_, 24>(a, F, smem, st, ws, z3);       \
    if (kr == 32) return launch_boxf_t<S_, B_, 32>(a, F, smem, st, ws, z3);       \
    if (kr == 40) return launch_boxf_t<S_, B_, 40>(a, F, smem, st, ws, z3);       \
    if (kr == 48) return launch_boxf_t<S_, B_, 48>(a, F, smem, st, ws, z3);       \
    return launch_boxf_t<S_, B_, 80>(a, F, smem, st);                             \
  }
  SCBM_BOXF_CASE(3, 8)
  SCBM_BOXF_CASE(1, 7)
  SCBM_BOXF_CASE(4, 8)
  SCBM_BOXF_CASE(2, 8)
  SCBM_BOXF_CASE(1, 6)
#undef SCBM_BOXF_CASE
  return cudaErrorInvalidValue;
}
}  // namespace

cudaError_t launch_bm_boxf(const sc_bm_plan_s& p, const void* imgs, int F, int iy_begin, int iy_end,
                           int32_t* idx_out, void* dist_out, cudaStream_t st, int64_t* launches) {
  // matcher, then the exact fix-up of the references its quantised keys leave open
  cudaError_t e = cudaMemsetAsync(p.ws.fix_count, 0, sizeof(int), st);
  if (e == cudaSuccess) e = launch_boxf_kernel(p, imgs, F, iy_begin, iy_end, idx_out, dist_out, st, launches);
  if (e != cudaSuccess) return e;
  if (launches) *launches += 1;
  return launch_fixup(p, imgs, F, iy_begin, iy_end, idx_out, dist_out, st);
}

}  // namespace scbm
