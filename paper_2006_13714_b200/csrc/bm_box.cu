// bm_box.cu -- the box-sum Self-Convolution matcher (SC_KERNEL_BOX; uint8, patch b = 8,
// reference stride s = 4, one channel): steps a0, a2, a3, a4, a6 fused in one kernel.
//
// a2. For a fixed window offset delta = (dy, dx) the cross term of every reference (Eq. 5,
// PAPER.md:277-279; footnote 2) is an 8x8 box sum, over the reference's patch,
// of the product image P_delta(y, x) = x'(y, x) * x'(y + dy, x + dx): the image correlated
// with its own shifted copy. With s = 4 = b / 2 every 4x4 block of P_delta lies in 2 x 2
// references, so the kernel forms 4-row x 4-column block sums -- one dp4a per block row on
// packed centred int8 words (x' = x - 128, exact int32) -- and assembles each reference's
// cross term from its 2 x 2 blocks:
//   * horizontally, lane l holds the references of reference column ix0 + l; the right half
//     of its patch is the left half of lane l + 1's (shfl.down), so a lane only correlates
//     its own 4-column strip (lane 31 is a helper: it supplies column ix0 + 31's strip);
//   * vertically, a lane owns NY = 2 references (rows iy, iy + 1) that share their middle
//     4 patch rows: 12 dp4a rows per offset instead of 16.
// Per (reference, candidate) pair that is 6 dp4a instead of the 16 of a direct 8x8 dot product
// (8 with NY = 1). A lane slides over VY vertically adjacent offsets (dy0 .. dy0+VY-1, fixed dx),
// loading each candidate row once for all of them; candidate words come from four byte-shifted
// copies of the staged region, so any 4-byte run is one aligned shared-memory load.
//
// a1 in registers. The candidate norm h_X(.)h_X is the same kind of box sum of
// x'^2: a dp4a chain over the lane's candidate rows, P[t] = sum_{u<t} |row u|^2, gives each
// offset's strip norm as P[t+8] - P[t] (no norm map, no norm pass; exact int32).
// a3. d' = n_c - 2 C (Lemma 2; ||X_i||^2 is constant per reference and added
// back after selection) = E_l + E_{l+1} with E = strip norm - 2 strip cross term, so one shfl
// per pair. Window clipping: warp-uniform row masks and a per-lane column predicate.
// a4. Per-reference 32-bit register top-K (regtopk.cuh; Theorem 1's K largest b_i = K smallest
// d) fed by a per-lane threshold bitmask; references whose K-th key saturates
// go to the exact fix-up (fixup.cu). Offsets are visited centre-out (dy blocks, then dx), so
// thresholds tighten early. a6: rows of K (idx, dist) staged in shared memory and written
// coalesced (a warp's 31 references are contiguous in the output).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "ncc.cuh"
#include "regtopk.cuh"
#include "sc_internal.h"

namespace scbm {
namespace {

constexpr int kBoxWarps = 8;
constexpr int kBoxRefsX = 31;  // references per warp row (lane 31 is the helper strip)

struct BoxArgs {
  const uint8_t* imgs;  // [F][H][W]
  int32_t* idx_out;     // [F][band refs][K]
  int32_t* dist_out;
  int H, W, Wn, K, KP, lo, hi, nx, iy_begin, iy_end, tiles_x;
  int RH, WP, PL;  // staged region rows, words per region row, words per byte-shifted copy
  int nblk;        // dy blocks of VY offsets
  int scr;         // per-warp scratch words
  int T;           // temporal search radius (0: the reference's own frame only)
  int n_frames;    // frames reachable from imgs (temporal search: the whole batch)
  int frame0;      // batch index of the launch's first reference frame (temporal search)
  int idx_foff;    // temporal search: frame offset added to the batch-global idx (halo buffers)
  int rb;          // 32-bit keys: window-relative index bits
  uint32_t dsat;   // 32-bit keys: distance saturation value
  int* fix_count;
  int* fix_list;
  int packed;      // packed tables (sc_bm_set_packed): idx_out receives the row keys themselves
};

__device__ __forceinline__ int centre_out(int k) { return (k & 1) ? ((k + 1) >> 1) : -(k >> 1); }

#ifndef SCBM_BOX_SHFL_OUT
#define SCBM_BOX_SHFL_OUT 0  // 1: write the output rows through shuffles (no staging scratch)
#endif
#ifndef SCBM_BOX_JOINT_ROUNDS
#define SCBM_BOX_JOINT_ROUNDS 1  // both references of a lane inserted in the same survivor rounds
#endif
#ifndef SCBM_BOX_SENT
#define SCBM_BOX_SENT 1  // joint survivor rounds pick from a sentinel bit (bit 0 -> a scratch row whose
                         // slack yields a saturated no-op key): no clamp, no per-lane no-op select
                         // (90 instead of 96 instructions per round; c5 8.73 -> 8.65 ms)
#endif
#ifndef SCBM_BOX_SORTFILL
#define SCBM_BOX_SORTFILL 1  // the first flush with survivors builds the (empty) lists by a bitonic sort
                             // (c5 8.64 -> 8.45 ms: the first flush was 14 % of all survivor rounds)
#endif
#ifndef SCBM_BOX_MINB
#define SCBM_BOX_MINB 2  // CTAs per SM the register allocation targets (tuning builds override)
#endif

// WPC: the staged row pitch in words when known at compile time (0 = runtime a.WP); a constant
// pitch turns the candidate-row loads into [register + immediate] LDS (no per-load address math)
// dp4a on the staged words: signed int8 (centred, L2) or unsigned uint8 (raw, NCC)
template <bool U>
__device__ __forceinline__ int dp4(uint32_t x, uint32_t y, int acc) {
  if constexpr (U) return int(__dp4a(x, y, uint32_t(acc)));
  else return __dp4a(int(x), int(y), acc);
}

// NCC (SC_METRIC_NCC, Eq. 4): the same block sums on RAW bytes (unsigned dp4a, exact); a lane
// forms C = U_l + U_{l+1} and n_c = D_l + D_{l+1} (two shuffles), filters on the float score
// sqrt(n_r) - C / sqrt(n_c) >= 0 with quantised 32-bit keys (rel + 1, 0 sentinels), keeps K + m
// and re-ranks them exactly (ncc.cuh) from the staged bytes.
// WNC: the window side when known at compile time (0 = runtime): the window geometry, key widths
// and loop bounds then become immediates (no per-round constant reloads in the survivor loop)
// TEMP (3D / temporal search): the candidates of a reference in frame f are
// the window positions of frames f-T .. f+T of the batch (PAPER.md:661/697's video setting); the
// region is restaged per frame (time offsets visited centre-out: 0, +1, -1, ...), the keys'
// window-relative index becomes (tau + T) Wn^2 + slot, and idx is the batch-global
// frame * H * W + cy * W + cx.
template <int NY, int VY, int KR, int WPC = 0, bool NCC = false, int WNC = 0, bool TEMP = false>
__global__ void __launch_bounds__(kBoxWarps * 32, NY == 1 ? 3 : SCBM_BOX_MINB) bm_box_kernel(BoxArgs a) {
  const int WP = WPC > 0 ? WPC : a.WP;
  constexpr int kRB = WNC > 0 ? (WNC * WNC <= 2 ? 2 : 32 - __builtin_clz(unsigned(WNC * WNC - 1))) : 0;
  const int Wn = WNC > 0 ? WNC : a.Wn;
  const int lo = WNC > 0 ? -(WNC / 2) : a.lo, hi = WNC > 0 ? WNC - 1 - WNC / 2 : a.hi;
  const int nblk = WNC > 0 ? (WNC + VY - 1) / VY : a.nblk;
  const int rbits = WNC > 0 ? (kRB < 2 ? 2 : kRB) : a.rb;
  const uint32_t dsat = WNC > 0 ? uint32_t((uint64_t(1) << (32 - (kRB < 2 ? 2 : kRB))) - 1) : a.dsat;
  extern __shared__ __align__(16) uint32_t sm[];
  constexpr int NR = 4 * NY + 4;   // patch rows of the lane's NY references
  constexpr int NT = NR + VY - 1;  // candidate rows per (dy block, dx)
  const int f = blockIdx.y;
  const int ty = blockIdx.x / a.tiles_x, tx = blockIdx.x - ty * a.tiles_x;
  const int iy_first = a.iy_begin + ty * (kBoxWarps * NY);
  const int ix_first = tx * kBoxRefsX;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Ybase = iy_first * 4 + lo, Xbase = ix_first * 4 + lo;

  // ---- a0: four byte-shifted copies of the centred region. Copy k, row r, word w holds
  // region bytes [4w+k, 4w+k+3] as int8 x' = x ^ 0x80 = x - 128 (0 outside the image).
  const int fref = TEMP ? a.frame0 + f : f;  // frame of the references (index into imgs)
  auto stage = [&](int frame) {
  const uint8_t* img = a.imgs + size_t(frame) * a.H * a.W;
  for (int e = threadIdx.x; e < a.PL; e += blockDim.x) {
    const int r = e / WP, w = e - r * WP;
    const int y = Ybase + r, x = Xbase + 4 * w;
    uint32_t u0 = 0u, u1 = 0u;
    if (y >= 0 && y < a.H) {
      const uint8_t* row = img + size_t(y) * a.W;
      if (x >= 0 && x + 8 <= a.W && (reinterpret_cast<uintptr_t>(row + x) & 3) == 0) {
        u0 = __ldg(reinterpret_cast<const uint32_t*>(row + x)) ^ (NCC ? 0u : 0x80808080u);
        u1 = __ldg(reinterpret_cast<const uint32_t*>(row + x + 4)) ^ (NCC ? 0u : 0x80808080u);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int xx = x + j;
          const uint32_t v = (xx >= 0 && xx < a.W) ? uint32_t(row[xx] ^ (NCC ? 0u : 0x80u)) : 0u;
          if (j < 4) u0 |= v << (8 * j);
          else u1 |= v << (8 * (j - 4));
        }
      }
    }
    sm[e] = u0;
    sm[a.PL + e] = __funnelshift_r(u0, u1, 8);
    sm[2 * a.PL + e] = __funnelshift_r(u0, u1, 16);
    sm[3 * a.PL + e] = __funnelshift_r(u0, u1, 24);
  }
  };
  stage(fref);
  __syncthreads();

  const int iy0 = iy_first + warp * NY;
  const bool wact = iy0 < a.iy_end;  // warp-uniform (temporal: every warp joins the restaging)
  if (!TEMP && !wact) return;
  const int ix = ix_first + lane;
  const bool lane_ok = lane < kBoxRefsX && ix < a.nx;
  const int rx = ix * 4;
  const int rr0 = (iy0 - iy_first) * 4 - lo;  // region row of image row 4 * iy0

  // the lane's 4-column strip of its references' patch rows (reference side, aligned)
  uint32_t R[NR];
  {
    const int off = -lo;
    const uint32_t* src = sm + (off & 3) * a.PL + rr0 * WP + lane + (off >> 2);
#pragma unroll
    for (int r = 0; r < NR; ++r) R[r] = src[r * WP];
  }
  bool ref_ok[NY];
  int32_t nr[NY];  // ||X_i||^2 of the centred reference (left strip + lane l+1's right strip)
  int thr[NY];     // largest d' = d - ||X_i||^2 that may still enter the reference's top-K
  float thrf[NY];  // NCC: largest filter score that may still enter the top-(K+m)
  float nrs[NY];   // NCC: sqrt(n_r)
  float gsq[NY];   // NCC: the filter's bound on C^2 / n_c (0: keep everything)
  RegTopK32<KR> rt[NY];
  const Key32 key32{rbits, dsat};
#pragma unroll
  for (int q = 0; q < NY; ++q) {
    int n = 0;
#pragma unroll
    for (int r = 0; r < 8; ++r) n = dp4<NCC>(R[4 * q + r], R[4 * q + r], n);
    nr[q] = n + __shfl_down_sync(0xffffffffu, n, 1);
    ref_ok[q] = lane_ok && iy0 + q < a.iy_end;
    rt[q].init();
    thr[q] = int(dsat) - nr[q];
    thrf[q] = __int_as_float(0x7f800000);
    nrs[q] = sqrtf(float(nr[q]));
    gsq[q] = 0.f;
    if constexpr (NCC) {  // 0 sentinels: the (K+m)-th key sits in r[KR-1]
#pragma unroll
      for (int k = 0; k < KR; ++k) rt[q].r[k] = k < KR - a.KP ? 0u : 0xffffffffu;
    }
  }
  uint32_t* scratch = sm + 4 * a.PL + warp * a.scr;
  constexpr bool kSent = SCBM_BOX_SENT && SCBM_BOX_JOINT_ROUNDS && !NCC && NY == 2;
  constexpr int kQS = 64 * VY + (kSent ? 32 : 0);  // scratch words per reference row (kSent: + the sentinel row)
  if constexpr (kSent) {  // slack 2^31: dthr - slack wraps past dsat -> a saturated key (never kept over a real one)
    scratch[lane] = 0x80000000u;
    scratch[kQS + lane] = 0x80000000u;
  }

  bool fresh = true;  // SORTFILL: no survivor inserted yet (warp-uniform)
  const int b0 = (0 - lo) / VY;  // dy block holding dy = 0
  const int span = max(-lo, hi);
  const int nt = TEMP ? 2 * a.T + 1 : 1;
  for (int kt = 0; kt < nt; ++kt) {  // time offsets, centre-out (TEMP only; else one pass)
  const int tau = centre_out(kt);
  if (TEMP) {
    if (fref + tau < 0 || fref + tau >= a.n_frames) continue;  // CTA-uniform
    if (kt > 0) {
      __syncthreads();  // every warp is done with the previous frame's region
      stage(fref + tau);
      __syncthreads();
    }
    if (!wact) continue;
  }
  const int relt = TEMP ? (tau + a.T) * Wn * Wn : 0;  // window-relative index offset of this frame
  // two phases over the dy blocks: the near offsets (dx pairs j < kNearPairs: |dx| <= 5) of every
  // block first, then the rest -- the thresholds tighten sooner than with each block's whole dx
  // range in turn (a c5 simulation: 5 % fewer survivor rounds)
#ifndef SCBM_NEAR_PAIRS
#define SCBM_NEAR_PAIRS 5
#endif
  constexpr int kNearPairs = SCBM_NEAR_PAIRS;
  for (int ph = 0; ph < 2; ++ph) {
  const int j_begin = ph == 0 ? 0 : kNearPairs, j_end = ph == 0 ? min(kNearPairs, span + 1) : span + 1;
  for (int kb = 0; kb < 2 * nblk; ++kb) {
    const int bb = b0 + centre_out(kb);
    if (bb < 0 || bb >= nblk) continue;
    const int dy0 = lo + bb * VY;
    // offsets dy0 + i inside the window (dy <= hi) whose candidate row lies in [0, H-b]
    unsigned rows[NY];
    bool any_row = false;
#pragma unroll
    for (int q = 0; q < NY; ++q) {
      const int cy0 = 4 * (iy0 + q) + dy0;  // candidate row of offset i = 0
      const int ilo = max(0, -cy0), ihi = min(min(VY - 1, hi - dy0), a.H - 8 - cy0);
      rows[q] = ihi >= ilo ? (((2u << ihi) - 1u) & ~((1u << ilo) - 1u)) : 0u;
      any_row |= rows[q] != 0u;
    }
    if (!any_row) continue;  // warp-uniform
    const uint32_t* cbase = sm + (rr0 + dy0) * WP + lane;
    // a4 survivors of two consecutive offset groups are inserted together (fewer, fuller rounds:
    // a round lasts as long as the busiest lane); the bits of group h sit at h*VY .. h*VY+VY-1
    // and its distances in scratch rows q*2VY + h*VY + i
    unsigned pend[NY];
#pragma unroll
    for (int q = 0; q < NY; ++q) pend[q] = 0u;
    int rel0p = 0;
    unsigned rmask[NY];  // window rows of this dy block x reference validity
#pragma unroll
    for (int q = 0; q < NY; ++q) rmask[q] = ref_ok[q] ? rows[q] : 0u;
    auto flush = [&](int rel0c) {
#if SCBM_BOX_JOINT_ROUNDS
      if constexpr (!NCC && NY == 2) {
        // both references of a lane in the same rounds: one survivor of each per round (two insertion
        // networks), so a round lasts as long as the busiest lane's busier list instead of the
        // busiest lane of each list in turn (a c5 simulation: ~10 % less round work)
        if constexpr (kSent) {
          // survivor bits shifted up by one; bit 0 (always set) selects the sentinel row 0
          unsigned b0 = (pend[0] << 1) | 1u, b1 = (pend[1] << 1) | 1u;
          if (__any_sync(0xffffffffu, (b0 | b1) > 1u)) {
            const uint32_t s0 = uint32_t(__cvta_generic_to_shared(scratch + lane));
            const uint32_t s1 = s0 + 4u * uint32_t(kQS);
            const int relA = rel0p - Wn, relB = rel0c - VY * Wn - Wn;
            const uint32_t dthr0 = uint32_t(thr[0] + nr[0]), dthr1 = uint32_t(thr[1] + nr[1]);
            if (SCBM_BOX_SORTFILL && fresh) {
              // the lists are still empty: build them from the staged keys with a bitonic sort of
              // the first KR keys (absent ones = ~0) and insert the rest (c5: a 16-key network +
              // 6 insertions per list instead of 22 survivor rounds)
              const int relB0 = rel0c - VY * Wn;
              auto fill = [&](RegTopK32<KR>& L, unsigned pb, uint32_t sb, uint32_t dthr) {
                auto key_at = [&](int i) -> uint32_t {
                  uint32_t d;
                  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(d) : "r"(sb + 128u * uint32_t(i + 1)));
                  const uint32_t k = (min(dthr - d, dsat) << rbits) | uint32_t((i < VY ? rel0p : relB0) + i * Wn);
                  return ((pb >> i) & 1u) ? k : 0xffffffffu;
                };
#pragma unroll
                for (int i = 0; i < KR; ++i) L.r[i] = i < 2 * VY ? key_at(i) : 0xffffffffu;
#pragma unroll
                for (int k = 2; k <= KR; k <<= 1)
#pragma unroll
                  for (int jj = k >> 1; jj > 0; jj >>= 1)
#pragma unroll
                    for (int i = 0; i < KR; ++i) {
                      const int l = i ^ jj;
                      if (l > i) {
                        const uint32_t lo_ = min(L.r[i], L.r[l]), hi_ = max(L.r[i], L.r[l]);
                        const bool asc = (i & k) == 0;
                        L.r[i] = asc ? lo_ : hi_;
                        L.r[l] = asc ? hi_ : lo_;
                      }
                    }
#pragma unroll
                for (int i = KR; i < 2 * VY; ++i) L.insert(key_at(i));
              };
              fill(rt[0], pend[0], s0, dthr0);
              fill(rt[1], pend[1], s1, dthr1);
              fresh = false;
              b0 = b1 = 1u;  // (every survivor is in)
            }
            while (__any_sync(0xffffffffu, (b0 | b1) > 1u)) {
              uint32_t p0, p1, d0, d1;
              asm("bfind.u32 %0, %1;" : "=r"(p0) : "r"(b0));
              asm("bfind.u32 %0, %1;" : "=r"(p1) : "r"(b1));
              asm volatile("ld.shared.u32 %0, [%1];" : "=r"(d0) : "r"(s0 + 128u * p0));
              asm volatile("ld.shared.u32 %0, [%1];" : "=r"(d1) : "r"(s1 + 128u * p1));
              const int rel0 = (int(p0) <= VY ? relA : relB) + int(p0) * Wn;
              const int rel1 = (int(p1) <= VY ? relA : relB) + int(p1) * Wn;
              const uint32_t k0 = (min(dthr0 - d0, dsat) << rbits) | uint32_t(rel0);
              const uint32_t k1 = (min(dthr1 - d1, dsat) << rbits) | uint32_t(rel1);
              b0 &= ~(1u << p0) | 1u;
              b1 &= ~(1u << p1) | 1u;
              rt[0].insert(k0);
              rt[1].insert(k1);
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) thr[q] = key32.thr(a.K == KR ? rt[q].r[KR - 1] : rt[q].at(a.K - 1)) - nr[q];
            __syncwarp();
          }
          pend[0] = pend[1] = 0u;
          return;
        }
        unsigned b0 = pend[0], b1 = pend[1];
        if (__any_sync(0xffffffffu, (b0 | b1) != 0u)) {
          const uint32_t s0 = uint32_t(__cvta_generic_to_shared(scratch + lane));
          const uint32_t s1 = s0 + 4u * uint32_t(64 * VY);
          const int relB = rel0c - VY * Wn;
          const uint32_t dthr0 = uint32_t(thr[0] + nr[0]), dthr1 = uint32_t(thr[1] + nr[1]);
          while (__any_sync(0xffffffffu, (b0 | b1) != 0u)) {
            uint32_t p0, p1, d0, d1;
            asm("bfind.u32 %0, %1;" : "=r"(p0) : "r"(b0));
            asm("bfind.u32 %0, %1;" : "=r"(p1) : "r"(b1));
            const int i0 = int(min(p0, uint32_t(2 * VY - 1))), i1 = int(min(p1, uint32_t(2 * VY - 1)));
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(d0) : "r"(s0 + 128u * uint32_t(i0)));
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(d1) : "r"(s1 + 128u * uint32_t(i1)));
            const int rel0 = (i0 < VY ? rel0p : relB) + i0 * Wn, rel1 = (i1 < VY ? rel0p : relB) + i1 * Wn;
            const uint32_t k0 = ((min(dthr0 - d0, dsat) << rbits) | uint32_t(rel0)) | (b0 ? 0u : 0xffffffffu);
            const uint32_t k1 = ((min(dthr1 - d1, dsat) << rbits) | uint32_t(rel1)) | (b1 ? 0u : 0xffffffffu);
            b0 &= ~(1u << i0);
            b1 &= ~(1u << i1);
            rt[0].insert(k0);
            rt[1].insert(k1);
          }
#pragma unroll
          for (int q = 0; q < 2; ++q) thr[q] = key32.thr(a.K == KR ? rt[q].r[KR - 1] : rt[q].at(a.K - 1)) - nr[q];
          __syncwarp();
        }
        pend[0] = pend[1] = 0u;
        return;
      }
#endif
#pragma unroll
      for (int q = 0; q < NY; ++q) {
        unsigned bits = pend[q];
        if (__any_sync(0xffffffffu, bits != 0u)) {
          const uint32_t* sc = scratch + q * (64 * VY) + lane;
          const int relB = rel0c - VY * Wn;
          const uint32_t sc_s = uint32_t(__cvta_generic_to_shared(sc));
          const uint32_t dthr = uint32_t(thr[q] + nr[q]);  // L2: d = dthr - staged slack
          while (__any_sync(0xffffffffu, bits != 0u)) {
            // any survivor (insertion order is irrelevant): the highest set bit (bfind; ~0 if none,
            // clamped to a valid scratch row so the unconditional load of every lane stays in bounds);
            // lanes without a survivor insert the no-op key ~0 (branch-free round)
            uint32_t pos, d;
            asm("bfind.u32 %0, %1;" : "=r"(pos) : "r"(bits));
            const int i = int(min(pos, uint32_t(NCC ? VY - 1 : 2 * VY - 1)));
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(d) : "r"(sc_s + 128u * uint32_t(i)));
            if constexpr (NCC) {  // staged C and n_c -> filter score sqrt(n_r) - C / sqrt(n_c) (float bits)
              uint32_t nw;
              asm volatile("ld.shared.u32 %0, [%1];" : "=r"(nw) : "r"(sc_s + 128u * uint32_t(i + VY)));
              const float sc = nrs[q] - (nw > 0u ? float(d) * rsqrtf(float(nw)) : 0.f);
              d = __float_as_uint(fmaxf(sc, 0.f));
            }
            const int rel = (i < VY ? rel0p : relB) + i * Wn;
            const uint32_t none = bits ? 0u : 0xffffffffu;
            uint32_t key;
            if constexpr (NCC)  // float bits of the score, quantised; rel + 1 (0 = sentinel)
              key = (((d >> (rbits - 1)) << rbits) | uint32_t(rel + 1)) | none;
            else
              key = ((min(dthr - d, dsat) << rbits) | uint32_t(rel)) | none;
            bits &= ~(1u << i);
            rt[q].insert(key);
          }
          if constexpr (NCC) {
            const uint32_t kth = rt[q].r[KR - 1];
            if (kth != 0xffffffffu) {  // largest score of the (K+m)-th key's quantum + margin
              const float smax = __uint_as_float(((kth >> rbits) << (rbits - 1)) | ((1u << (rbits - 1)) - 1u));
              thrf[q] = fmaf(smax, 1.0f + 1e-5f, 1e-30f);
              const float g = nrs[q] - thrf[q];  // keep iff C / sqrt(n_c) >= g, i.e. C^2 >= g^2 n_c (C >= 0)
              gsq[q] = g > 0.f ? g * g * (1.0f - 1e-6f) : 0.f;
            }
          } else {
            thr[q] = key32.thr(a.K == KR ? rt[q].r[KR - 1] : rt[q].at(a.K - 1)) - nr[q];
          }
          __syncwarp();
        }
        pend[q] = 0u;
      }
    };
    // one offset group (fixed dx, offsets dy0 .. dy0+VY-1) into staging half H (compile time)
    auto group = [&](int dx, auto hc) -> int {
      constexpr int H = decltype(hc)::value;
      (void)H;  // (NCC stages one group per flush)
      const int off = dx - lo;
      const uint32_t* col = cbase + (off & 3) * a.PL + (off >> 2);
      uint32_t Cw[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t) Cw[t] = col[t * WP];
      // a1 in registers: P[t] = sum_{u < t} |candidate strip row u|^2 (a dp4a prefix chain),
      // so the strip norm of offset i of reference q is P[4q+i+8] - P[4q+i]
      int P[NT + 1];
      P[0] = 0;
#pragma unroll
      for (int t = 0; t < NT; ++t) P[t + 1] = dp4<NCC>(Cw[t], Cw[t], P[t]);
      // a2: block sums -> left-strip cross terms U[q][i] of reference q at offset (dy0 + i, dx)
      int U[NY][VY];
#pragma unroll
      for (int i = 0; i < VY; ++i) {
        if constexpr (NY == 1) {
          int acc = 0;
#pragma unroll
          for (int r = 0; r < 8; ++r) acc = dp4<NCC>(R[r], Cw[r + i], acc);
          U[0][i] = acc;
        } else {
          int m = 0;  // middle rows 4..7, shared by both references
#pragma unroll
          for (int r = 4; r < 8; ++r) m = dp4<NCC>(R[r], Cw[r + i], m);
          int t0 = m, t1 = m;
#pragma unroll
          for (int r = 0; r < 4; ++r) t0 = dp4<NCC>(R[r], Cw[r + i], t0);
#pragma unroll
          for (int r = 8; r < 12; ++r) t1 = dp4<NCC>(R[r], Cw[r + i], t1);
          U[0][i] = t0;
          U[1][i] = t1;
        }
      }
      const bool colok = unsigned(rx + dx) <= unsigned(a.W - 8);  // candidate column in [0, W-b]
      // strip norms of the 4(NY-1) + VY distinct candidate rows: D[j] = P[j + 8] - P[j]
      int D[4 * (NY - 1) + VY];
#pragma unroll
      for (int j = 0; j < 4 * (NY - 1) + VY; ++j) D[j] = P[j + 8] - P[j];
#pragma unroll
      for (int q = 0; q < NY; ++q) {
        // a3: d' = n_c - 2 C = E_l + E_{l+1}, E = strip norm - 2 * strip cross term
        // slack t = thr - d' (>= 0: the candidate may enter the top-K); fail bits = sign bits
        [[maybe_unused]] int t[VY];
        unsigned fails = 0u;
        if constexpr (NCC) {
          // raw bytes: 0 <= C, n_c < 2^22, so both convert to fp32 exactly and
          // the filter sqrt(n_r) - C / sqrt(n_c) <= thrf needs no square root: C^2 - gsq n_c >= 0
          // (gsq carries a 1e-6 relative margin, so rounding never drops a candidate). C and n_c
          // are staged for the flush, which scores the survivors.
          uint32_t* sc = scratch + q * (64 * VY) + lane;
#pragma unroll
          for (int i = VY - 1; i >= 0; --i) {
            const int cc = U[q][i] + __shfl_down_sync(0xffffffffu, U[q][i], 1);      // C
            const int nn = D[4 * q + i] + __shfl_down_sync(0xffffffffu, D[4 * q + i], 1);  // n_c
            const float fc = __int2float_rn(cc), fn = __int2float_rn(nn);  // exact: < 2^24 (one I2FP each)
            sc[32 * i] = uint32_t(cc);
            sc[32 * (i + VY)] = uint32_t(nn);
            fails = __funnelshift_l(__float_as_uint(fmaf(-gsq[q], fn, fc * fc)), fails, 1);
          }
        } else {
#pragma unroll
          for (int i = VY - 1; i >= 0; --i) {
            const int e = D[4 * q + i] - 2 * U[q][i];
            t[i] = thr[q] - e - __shfl_down_sync(0xffffffffu, e, 1);
            fails = __funnelshift_l(uint32_t(t[i]), fails, 1);  // (fails << 1) | sign(t): one SHF
          }
        }
        const unsigned bits = ~fails & (colok ? rmask[q] : 0u);
        if constexpr (NCC) {
          pend[q] |= bits;
        } else if (__any_sync(0xffffffffu, bits != 0u)) {
          uint32_t* sc = scratch + q * kQS + (kSent ? 32 : 0) + H * (32 * VY) + lane;
          // the slack t is staged; the flush recovers d = d' + ||X_i||^2 = (thr + n_r) - t (exact,
          // thr does not change between the two staged groups of a flush)
#pragma unroll
          for (int i = 0; i < VY; ++i) sc[32 * i] = uint32_t(t[i]);
          pend[q] |= bits << (H * VY);
        }
      }
      return relt + (dy0 - lo) * Wn + off;  // window-relative index of offset (dy0, dx)
    };
    // dx centre-out (0, 1, -1, 2, -2, ...), consecutive pairs (-j, j+1) staged in the two halves
    // and flushed together; a lone group (window edge) flushes alone. NCC: one group per flush
    // (the scratch holds its C and n_c).
    if constexpr (NCC) {
      for (int kx = 2 * j_begin; kx < 2 * j_end && kx <= 2 * span; ++kx) {
        const int dx = centre_out(kx);
        if (dx < lo || dx > hi) continue;
        rel0p = group(dx, std::integral_constant<int, 0>{});
        flush(0);
      }
    } else {
      for (int j = j_begin; j < j_end; ++j) {
        const bool va = -j >= lo, vb = j + 1 <= hi;
        if (!va && !vb) continue;  // warp-uniform
        rel0p = group(va ? -j : j + 1, std::integral_constant<int, 0>{});
        flush(va && vb ? group(j + 1, std::integral_constant<int, 1>{}) : 0);
      }
    }
  }
  }  // phases
  }  // time offsets

  const size_t band_refs = size_t(a.iy_end - a.iy_begin) * a.nx;
  const int nref = min(kBoxRefsX, a.nx - ix_first);
  if constexpr (NCC) {
    // ---- a5 + a6 (NCC): per reference, the kept K + m candidates re-scored EXACTLY from the staged
    // raw bytes (C, n_c, n_r by unsigned dp4a), one warp bitonic sort (ncc.cuh), K (idx, -NCC)
    const uint32_t relmask = (1u << rbits) - 1u;
    const int roff = -lo;
#pragma unroll
    for (int q = 0; q < NY; ++q) {
      const int iy = iy0 + q;
      if (iy >= a.iy_end) break;  // warp-uniform
      const size_t row0 = size_t(f) * band_refs + size_t(iy - a.iy_begin) * a.nx + ix_first;
      __syncwarp();
      if (lane_ok) {
#pragma unroll
        for (int k = 0; k < KR; ++k) scratch[lane * (KR + 1) + k] = rt[q].r[k];
      }
      __syncwarp();
      const int ry = 4 * iy;
      const uint32_t* refbase = sm + (roff & 3) * a.PL + (rr0 + 4 * q) * WP + (roff >> 2);
      const int kskip = KR - a.KP;  // leading 0 sentinels: lane k takes the k-th kept key
      for (int j = 0; j < nref; ++j) {
        const uint32_t kk = lane < a.KP ? scratch[j * (KR + 1) + kskip + lane] : 0xffffffffu;
        const bool have = kk != 0u && kk != 0xffffffffu;
        const int rel = have ? int(kk & relmask) - 1 : 0;
        const int dyy = rel / Wn, dxx = rel - dyy * Wn;
        const int cy = ry + dyy + lo, cx = (ix_first + j) * 4 + dxx + lo;
        const int ccol = cx - Xbase;  // region byte column of the candidate (>= 0)
        const uint32_t* cbase2 = sm + (ccol & 3) * a.PL + (cy - Ybase) * WP + (ccol >> 2);
        int ci = 0, nci = 0;
        const int nri = __shfl_sync(0xffffffffu, nr[q], j);  // ||X_i||^2 (raw bytes), lane j's reference
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            const uint32_t rv = refbase[r * WP + j + w];
            const uint32_t cv = have ? cbase2[r * WP + w] : 0u;
            ci = dp4<true>(rv, cv, ci);
            nci = dp4<true>(cv, cv, nci);
          }
        NccItem it;
        it.idx = have ? cy * a.W + cx : -1;
        const bool zero = nri == 0 || nci == 0;
        it.c = zero ? 0 : ci;
        it.n = zero ? 1 : nci;
        it.f = (zero || !have) ? 0.0 : double(ci) / sqrt(double(nri) * double(nci));
        // the kept keys were quantised (2^-(rbits-1)... relative): when the worst kept key's quantum
        // could still hold a score as good as the exact K-th one, a dropped candidate might belong
        // to the top-K -> exact re-rank over the whole window (fixup.cu)
        const uint32_t klast = __shfl_sync(0xffffffffu, kk, a.KP - 1);
        it = warp_repair_ncc<true>(it, lane);  // kept keys arrive in (quantised score, idx) order
        const double fK = __shfl_sync(0xffffffffu, it.f, a.K - 1);
        if (lane == 0 && klast != 0u && klast != 0xffffffffu && nri > 0) {
          const float smin = __uint_as_float((klast >> rbits) << (rbits - 1));  // quantum minimum
          const double nrd = sqrt(double(nri)), scK = nrd * (1.0 - fK);         // exact K-th score
          if (double(smin) <= scK * (1.0 + 1e-5) + 1e-6 * nrd) {
            const int pos = atomicAdd(a.fix_count, 1);
            a.fix_list[pos] = int(row0 + j);
          }
        }
        if (lane < a.K) {
          a.idx_out[(row0 + j) * a.K + lane] = it.idx;
          reinterpret_cast<float*>(a.dist_out)[(row0 + j) * a.K + lane] =
              it.idx < 0 ? __int_as_float(0x7f800000) : float(-it.f);
        }
      }
    }
    return;
  } else {
  // ---- a6: exact references -> staged rows of K keys -> coalesced (idx, dist) stores;
  // references whose K-th key is saturated or unfilled -> the fix-up list
#pragma unroll
  for (int q = 0; q < NY; ++q) {
    const int iy = iy0 + q;
    if (iy >= a.iy_end) break;  // warp-uniform
    const size_t row0 = size_t(f) * band_refs + size_t(iy - a.iy_begin) * a.nx + ix_first;
    const bool exact = key32.exact(rt[q].at(a.K - 1));
    if (ref_ok[q] && !exact) {
      const int pos = atomicAdd(a.fix_count, 1);
      a.fix_list[pos] = int(row0 + lane);
    }
    const int ry = 4 * iy;
#if SCBM_BOX_SHFL_OUT
    // transpose through shuffles: output element e = j K + k is lane j's k-th key
    for (int e0 = 0; e0 < nref * a.K; e0 += 32) {
      const int e = e0 + lane;
      const int j = min(e / a.K, 31), k = e - (e / a.K) * a.K;
      uint32_t kk = 0u;
#pragma unroll
      for (int kq = 0; kq < KR; ++kq) {
        const uint32_t v = __shfl_sync(0xffffffffu, rt[q].r[kq], j);
        if (kq == k) kk = v;
      }
      if (e < nref * a.K && !TEMP && a.packed) {
        reinterpret_cast<uint32_t*>(a.idx_out)[row0 * a.K + e] = kk;
      } else if (e < nref * a.K) {
        int rel = key32.rel(kk);
        const int tsl = TEMP ? rel / (Wn * Wn) : 0;  // frame slot tau + T
        rel -= tsl * Wn * Wn;
        const int dyy = rel / Wn, dxx = rel - dyy * Wn;
        a.idx_out[row0 * a.K + e] = (TEMP ? (fref + tsl - a.T + a.idx_foff) * a.H * a.W : 0) +
                                    (ry + dyy + lo) * a.W + (ix_first + j) * 4 + dxx + lo;
        a.dist_out[row0 * a.K + e] = key32.dist(kk);
      }
    }
#else
    __syncwarp();
    if (lane_ok) {
#pragma unroll
      for (int k = 0; k < KR; ++k)
        if (k < a.K) scratch[lane * (KR + 1) + k] = rt[q].r[k];
    }
    __syncwarp();
    auto emit = [&](int e, int j, int k) {
      const uint32_t kk = scratch[j * (KR + 1) + k];
      if (!TEMP && a.packed) {  // the key is the packed word (rows that do not fit: the fix-up's)
        reinterpret_cast<uint32_t*>(a.idx_out)[row0 * a.K + e] = kk;
        return;
      }
      int rel = key32.rel(kk);
      const int tsl = TEMP ? rel / (Wn * Wn) : 0;  // frame slot tau + T
      rel -= tsl * Wn * Wn;
      const int dyy = rel / Wn, dxx = rel - dyy * Wn;
      a.idx_out[row0 * a.K + e] = (TEMP ? (fref + tsl - a.T + a.idx_foff) * a.H * a.W : 0) +
                                  (ry + dyy + lo) * a.W + (ix_first + j) * 4 + dxx + lo;
      a.dist_out[row0 * a.K + e] = key32.dist(kk);
    };
    if (a.K == KR) {  // the list length is K (c5): element -> (reference, rank) by a constant divisor
      for (int e = lane; e < nref * KR; e += 32) emit(e, e / KR, e % KR);
    } else {
      for (int e = lane; e < nref * a.K; e += 32) {
        const int j = e / a.K;
        emit(e, j, e - j * a.K);
      }
    }
    __syncwarp();
#endif
  }
  }  // !NCC
}

int box_vy(const Geometry& g) { return g.Wn % 11 == 0 ? 11 : g.Wn % 7 == 0 ? 7 : g.Wn <= 8 ? 8 : 11; }

size_t box_layout(const Geometry& g, int NY, int VY, int KR, BoxArgs* a) {
  a->nblk = (g.Wn + VY - 1) / VY;
  a->RH = 4 * kBoxWarps * NY + a->nblk * VY + 3;  // deepest candidate row read + 1
  a->WP = 32 + (g.Wn - 1) / 4;                    // lane 31's last candidate word + 1
  a->PL = a->RH * a->WP;
  a->scr = std::max(64 * VY * NY + (SCBM_BOX_SENT ? 32 * NY : 0), SCBM_BOX_SHFL_OUT ? 0 : kBoxRefsX * (KR + 1));
  return size_t(4 * a->PL + kBoxWarps * a->scr) * 4;
}

template <int NY, int VY, int KR, int WPC = 0, bool NCC = false, int WNC = 0, bool TEMP = false>
cudaError_t launch_box_t(const BoxArgs& a, int F, size_t smem, cudaStream_t st) {
  const int tiles_y = (a.iy_end - a.iy_begin + kBoxWarps * NY - 1) / (kBoxWarps * NY);
  auto k = bm_box_kernel<NY, VY, KR, WPC, NCC, WNC, TEMP>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k<<<dim3(a.tiles_x * tiles_y, F), kBoxWarps * 32, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

int box_key_bits(const Geometry& g) { return std::max(2, key32_rel_bits(g.Wn)); }

// temporal search: the window-relative index spans (2T+1) Wn^2 slots
int box_key_bits_t(const Geometry& g, int T) {
  int rb = 2;
  while ((1 << rb) < (2 * T + 1) * g.Wn * g.Wn) ++rb;
  return rb;
}

bool box_temporal_supported(const Geometry& g, int T) {
  return T == 0 || (g.metric == SC_METRIC_L2 && box_supported(g) && box_key_bits_t(g, T) <= 12);
}

bool box_supported(const Geometry& g) {
  if (g.dtype != SC_DTYPE_U8 || g.b != 8 || g.s != 4 || g.C != 1 || g.K > 32) return false;
  if (key32_rel_bits(g.Wn) > 11) return false;  // keeps >= 21 distance bits in the 32-bit keys
  if (g.metric == SC_METRIC_NCC && (g.KP > 32 || (1 << key32_rel_bits(g.Wn)) <= g.Wn * g.Wn))
    return false;  // NCC: K + m <= 32 register keys, rel + 1 must fit
  BoxArgs a{};
  return box_layout(g, 2, box_vy(g), 32, &a) <= 227 * 1024;
}

cudaError_t launch_bm_box(const sc_bm_plan_s& p, const void* imgs, int F, int iy_begin, int iy_end,
                          int32_t* idx_out, void* dist_out, cudaStream_t st, int64_t* launches) {
  const Geometry& g = p.g;
  BoxArgs a{};
  a.imgs = static_cast<const uint8_t*>(imgs);
  a.idx_out = idx_out;
  a.dist_out = static_cast<int32_t*>(dist_out);
  a.H = g.H; a.W = g.W; a.Wn = g.Wn; a.K = g.K; a.KP = g.KP; a.lo = g.lo; a.hi = g.hi; a.nx = g.nx;
  a.iy_begin = iy_begin; a.iy_end = iy_end;
  a.tiles_x = (g.nx + kBoxRefsX - 1) / kBoxRefsX;
  a.rb = box_key_bits(g);
  a.dsat = uint32_t((uint64_t(1) << (32 - a.rb)) - 1);
  a.fix_count = p.ws.fix_count;
  a.fix_list = p.ws.fix_list;
  const int vy = box_vy(g), kr = g.KP <= 16 ? 16 : 32;
  const size_t smem = box_layout(g, 2, vy, kr, &a);
  if (p.T > 0) {  // temporal search (L2): batch-wide frame access, wider keys, runtime geometry
    a.imgs = static_cast<const uint8_t*>(p.batch_base);
    a.T = p.T;
    a.frame0 = int(p.batch_f0);
    a.n_frames = int(p.batch_n);
    a.idx_foff = int(p.idx_frame_off);
    a.rb = box_key_bits_t(g, p.T);
    a.dsat = uint32_t((uint64_t(1) << (32 - a.rb)) - 1);
    cudaError_t e = cudaMemsetAsync(p.ws.fix_count, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
    if (kr == 16 && vy == 11) e = launch_box_t<2, 11, 16, 0, false, 0, true>(a, F, smem, st);
    else if (kr == 16 && vy == 7) e = launch_box_t<2, 7, 16, 0, false, 0, true>(a, F, smem, st);
    else if (kr == 16) e = launch_box_t<2, 8, 16, 0, false, 0, true>(a, F, smem, st);
    else if (vy == 11) e = launch_box_t<2, 11, 32, 0, false, 0, true>(a, F, smem, st);
    else if (vy == 7) e = launch_box_t<2, 7, 32, 0, false, 0, true>(a, F, smem, st);
    else e = launch_box_t<2, 8, 32, 0, false, 0, true>(a, F, smem, st);
    if (launches) *launches += 2;
    if (e != cudaSuccess) return e;
    return launch_fixup(p, imgs, F, iy_begin, iy_end, idx_out, dist_out, st);
  }
  if (g.metric == SC_METRIC_NCC) {  // K + m <= 32; references the key quantisation leaves open -> fix-up
    cudaError_t e = cudaMemsetAsync(p.ws.fix_count, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
    if (g.Wn == 33 && g.KP <= 18) e = launch_box_t<2, 11, 18, 40, true, 33>(a, F, box_layout(g, 2, vy, 18, &a), st);
    else if (g.Wn == 33 && g.KP <= 20) e = launch_box_t<2, 11, 20, 40, true, 33>(a, F, box_layout(g, 2, vy, 20, &a), st);
    else if (g.Wn == 33 && g.KP <= 24) e = launch_box_t<2, 11, 24, 40, true, 33>(a, F, box_layout(g, 2, vy, 24, &a), st);
    else if (vy == 11 && a.WP == 40 && g.KP <= 24) e = launch_box_t<2, 11, 24, 40, true>(a, F, box_layout(g, 2, vy, 24, &a), st);
    else {  // 32-key lists: the layout (per-warp scratch for the KR + 1 pitch) must match KR
      const size_t smem32 = box_layout(g, 2, vy, 32, &a);
      if (vy == 11 && a.WP == 40) e = launch_box_t<2, 11, 32, 40, true>(a, F, smem32, st);
      else if (vy == 11) e = launch_box_t<2, 11, 32, 0, true>(a, F, smem32, st);
      else if (vy == 7) e = launch_box_t<2, 7, 32, 0, true>(a, F, smem32, st);
      else e = launch_box_t<2, 8, 32, 0, true>(a, F, smem32, st);
    }
    if (launches) *launches += 2;
    if (e != cudaSuccess) return e;
    return launch_fixup(p, imgs, F, iy_begin, iy_end, idx_out, dist_out, st);
  }
  a.packed = p.packed_cap > 0 ? 1 : 0;  // (T = 0, L2: the packed run checks)
  cudaError_t e = cudaMemsetAsync(p.ws.fix_count, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  if (kr == 16 && g.Wn == 33) e = launch_box_t<2, 11, 16, 40, false, 33>(a, F, smem, st);  // c5: all constant
  else if (kr == 16 && vy == 11 && a.WP == 40) e = launch_box_t<2, 11, 16, 40>(a, F, smem, st);  // Wn 29..33
  else if (kr == 16 && vy == 11) e = launch_box_t<2, 11, 16>(a, F, smem, st);
  else if (kr == 16 && vy == 7) e = launch_box_t<2, 7, 16>(a, F, smem, st);
  else if (kr == 16) e = launch_box_t<2, 8, 16>(a, F, smem, st);
  else if (vy == 11) e = launch_box_t<2, 11, 32>(a, F, smem, st);
  else if (vy == 7) e = launch_box_t<2, 7, 32>(a, F, smem, st);
  else e = launch_box_t<2, 8, 32>(a, F, smem, st);
  if (launches) *launches += 2;
  if (e != cudaSuccess) return e;
  return launch_fixup(p, imgs, F, iy_begin, iy_end, idx_out, dist_out, st);
}

}  // namespace scbm
