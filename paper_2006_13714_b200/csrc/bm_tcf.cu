// bm_tcf.cu -- the tensor-core float matcher (SC_KERNEL_TC_F32): f32 images, one channel, patch
// side b <= 8, any reference stride: steps a0, a2-a6 fused in one kernel, a1 from the norm map.
//
// a2 (the Self-Convolution cross term, Eq. 5) runs on the 5th-generation tensor
// cores as a 3xTF32 GEMM  D[ref][cand] = sum_k A[ref][k] B[cand][k]  with fp32 accumulation in TMEM:
// every operand is split x = hi + lo (hi = x with the 13 low mantissa bits cleared, exactly
// representable in tf32; lo = x - hi, exact in fp32) and D = A_hi B_hi + A_hi B_lo + A_lo B_hi, which
// keeps the products to ~2^-21 relative (fp32-class; bf16x3 would not meet the 1e-5 rule).
//   * A (M = 128 references of an 8 x 16 reference block; TMEM lane quadrant q = a 4 x 8 sub-block)
//     lives in TMEM, written once per CTA by tcgen05.st (lane m = reference m): the centred patch
//     x' = x - 0.5 as K = 8 b tf32 values, k = 8 u + v (patch row u, column v; v >= b is zero),
//     hi at columns [0, 8b), lo at [8b, 16b) -- so a CTA needs no shared memory for A and two CTAs
//     (8 epilogue warps) share an SM.
//   * B (N = 64 candidates: a 4-row x 16-column block of candidate top-left positions) is K-major
//     straight out of a "shift-expanded" tile E[y][jg][kc][j][t] = x'(cy0 + y, cx0 + 8 jg + j + 4 kc + t):
//     an 8-candidate group (8 consecutive columns jg of candidate row i) x 16 B of K (4 shifts v)
//     is one canonical core matrix, the K-group of patch row u of candidate row i is tile row i + u,
//     so ONE descriptor per patch row (start + 512 u, LBO = 128, SBO = 256) addresses the whole block --
//     no im2col; the tile is 4 + b - 1 rows x 512 B per copy (hi, lo). (MN-major B, which would need
//     no shifted copies along K, does not work for kind::tf32: tools/tf32_layout_test.cu; A from
//     TMEM: tools/tf32_tmem_a_test.cu.)
//   * per candidate tile, 3 b MMAs (tcgen05.mma.cta_group::1.kind::tf32 [d], [a_tmem], b_desc, K = 8)
//     into one of two 128 x 64 fp32 TMEM accumulators (double-buffered: the MMAs of tile t+1 overlap
//     the epilogue of tile t), issued by one thread, committed to mbarriers; three producer warps
//     stage the E tiles of a 2-slot ring from the CTA's staged image region.
// Epilogue (4 warps per CTA, one per TMEM lane quadrant; lane = reference, its list stays in
// registers or in its shared-memory heap for the whole kernel): tcgen05.ld 32 columns (two candidate rows),
// d' = n_c - 2 C (Lemma 2; n_c from the fp64-SAT norm map), slack = thr - d',
// sign bits packed into a fail mask (one SHF per pair), the window mask, and the u8 box kernel's
// branch-free survivor rounds into the reference's top-(K+m) of 32-bit keys (a4, Theorem 1,
// PAPER.md:322-330). Tiles are visited by distance to the block (thresholds tighten early); a warp
// skips tiles / candidate rows outside its quadrant's window union. a5 + a6 as in the float box
// kernel: the kept keys re-scored by direct differences, sorted, written; references whose kept
// keys cannot decide the K-th go to the exact fix-up (fixup.cu).
#include <algorithm>
#include <cstdio>

#include "regtopk.cuh"
#include "sc_internal.h"
#include "sm100.cuh"
#include "topk.cuh"

namespace scbm {
namespace {

constexpr int kTfEpi = 4;                       // epilogue warps = TMEM lane quadrants
constexpr int kTfWarps = 8;                     // 4 epilogue + the MMA / producer warp + 3 joining a5 only
constexpr int kTfThreads = kTfWarps * 32;
constexpr int kRBY = 8, kRBX = 16;  // reference block (M = 128)
constexpr int kTR = 4, kTC = 16;    // candidate tile (N = 64)
constexpr int kES = 2;              // E ring slots
#ifndef SCBM_TCF_STAGERS
#define SCBM_TCF_STAGERS 4  // warps staging the E tiles (warp kTfEpi issues the MMAs; the others idle until
                            // a5). c3: 3.33 ms with 4, 3.35 with 1
#endif
constexpr int kStg = SCBM_TCF_STAGERS;
// TMEM (256 columns per CTA, two CTAs per SM): A_hi at [0, 8b), A_lo at [8b, 16b) (the reference
// patches, written once by tcgen05.st), the two N = 64 accumulators at [128, 192) and [192, 256)
constexpr uint32_t kTmemD = 128;
constexpr int kScrPitch = 36;       // epilogue scratch words per lane (32 staged + pad; 16-B rows)
constexpr float kTcfErr = 2e-5f;    // bound on the 3xTF32 identity's error, relative to n_r + d
constexpr int kBinBase = (127 - 6) << 4;  // BOUND histogram: bin 0 = float bits >> 19 of 2^-6
#ifndef SCBM_TCF_PROF
#define SCBM_TCF_PROF 0  // timing experiments only: per-warp cycle counters printed by a few CTAs
#endif
#ifndef SCBM_TCF_SIFT
#define SCBM_TCF_SIFT 4  // 1: branch-free fixed-depth sift-downs, root in a register, next survivor prefetched;
                         // 2: + the grandchildren loaded one level ahead (one 16-byte load per level);
                         // 3: + the great-grandchildren two levels ahead (two 16-byte loads per level);
                         // 4: a 4-ary heap (three levels for K + m <= 85; the children of the four
                         //    children loaded one level ahead): c3 3.33 -> 3.13 ms against 2
#endif
#ifndef SCBM_TCF_FILLUP
#define SCBM_TCF_FILLUP 0  // 1: 4-ary heap, while not full, keys are appended and sifted up (a divergent loop:
                           // measured 3.25 ms on c3 against 3.13 with fixed-depth sift-downs only; off)
#endif
#ifndef SCBM_TCF_A5ILP
#define SCBM_TCF_A5ILP 1  // a5: a lane's 4 kept keys re-scored in one interleaved loop
#endif
#ifndef SCBM_TCF_BOUND
#define SCBM_TCF_BOUND 0  // 1: heap lists (K + m > 48) get a first sweep over the tiles that bounds the
                          // (K+m)-th distance (measured on c3: 42 % fewer insertions, 23 % fewer survivor
                          // rounds, but the extra sweep costs more than they save: 4.12 vs 3.33 ms; off)
#endif
#ifndef SCBM_TCF_SKIP
#define SCBM_TCF_SKIP 0  // timing experiments only: 1 no survivor rounds, 2 no epilogue math, 4 no a5
#endif

struct TcfArgs {
  const float* imgs;   // [F][H][W]
  const float* norm;   // norm map interior of frame 0 (centred, fp32), pitch Mx, frame stride nfs
  int32_t* idx_out;    // [F][band refs][K]
  float* dist_out;
  float* dense;        // debug: every window distance [refs][Wn^2] (nullptr: block matching)
  int H, W, s, Wn, K, KP, lo, hi, nx, iy_begin, iy_end, tiles_x;
  int Mx;
  long long nfs;
  int rb;              // window-relative index bits of the 32-bit keys (rel + 1, 0 = sentinel)
  int RH, RWp;         // staged region rows / row pitch (floats)
  uint32_t off_raw, off_A, off_E, off_heap, off_scr, off_order, off_nc;
  int hp;              // heap pitch (words per reference)
  int scr;             // epilogue scratch words per warp
  int* fix_count;
  int* fix_list;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t tf32_hi(float x) { return __float_as_uint(x) & 0xffffe000u; }

template <int BK, int KR, bool DENSE>
__global__ void __launch_bounds__(kTfThreads, 2) bm_tcf_kernel(TcfArgs a) {
  constexpr bool HEAP = KR > 48;
  constexpr int kSiftLevels = KR >= 128 ? 7 : KR >= 64 ? 6 : 5;  // sift-down levels below the root: floor(log2(KP))
  constexpr int kSift4 = KR > 85 ? 4 : 3;  // SIFT 4 (4-ary heap): levels below the root
  constexpr int kHB = SCBM_TCF_SIFT == 4 ? 3 : 1;  // heap position of the root
  constexpr int ER = kTR + BK - 1;                  // E tile rows
  constexpr uint32_t kEBytes = uint32_t(ER) * 512;  // one copy (hi or lo) of an E tile
  constexpr uint32_t kIdesc = sm100::idesc_tf32(128, kTR * kTC, /*a_mn=*/false, /*b_mn=*/false);
  constexpr uint32_t kKA = 8 * BK;                  // A columns per copy (hi, lo) in TMEM
  // BOUND: the tiles are swept twice. Sweep 1 only counts, per reference, the minimum distance of
  // every 2 x 16 group of window candidates in a histogram of 1/16-octave bins over [2^-6, 2^10)
  // (u8 counters in the reference's heap row); the upper edge of the bin where the count reaches
  // K + m bounds the (K+m)-th smallest distance from above (K + m group minima are distinct
  // candidates below it), so sweep 2 starts with that threshold instead of +inf and the heap sees
  // far fewer insertions (c3: ~350 -> ~150 per reference). The MMAs of sweep 2 recompute the same
  // values (deterministic), so the bound holds for the distances sweep 2 filters.
  constexpr bool BOUND = HEAP && !DENSE && SCBM_TCF_BOUND;
  constexpr int NSW = BOUND ? 2 : 1;  // sweeps over the tiles
  extern __shared__ __align__(1024) uint8_t smem[];
  const int f = blockIdx.y;
  const int by = blockIdx.x / a.tiles_x, bx = blockIdx.x - by * a.tiles_x;
  const int iy_first = a.iy_begin + by * kRBY;
  const int iy_last = min(a.iy_end, iy_first + kRBY) - 1;
  const int ix_first = bx * kRBX;
  const int ix_last = min(a.nx, ix_first + kRBX) - 1;
  const int s = a.s, H = a.H, W = a.W;
  const int cyA = max(0, iy_first * s + a.lo), cyB = min(H - BK, iy_last * s + a.hi);
  // (tile columns start at a multiple of 4: the norm-map loads are 16-byte vectors)
  const int cxA = max(0, ix_first * s + a.lo) & ~3, cxB = min(W - BK, ix_last * s + a.hi);
  const int NTI = (cyB - cyA) / kTR + 1;  // candidate tile rows / columns of the block's window union
  const int NTC = (cxB - cxA) / kTC + 1;
  const int ntiles = NTI * NTC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_full = sbase, bar_empty = sbase + 16, bar_ee = sbase + 56;
  const uint32_t tmem_slot = sbase + 80, bar_nc = sbase + 96;  // bar_nc[2]: the tile's candidate norms staged
  float* raw = reinterpret_cast<float*>(smem + a.off_raw);
  const uint32_t sE = sbase + a.off_E;

  if (warp == kTfWarps - 1) {
    sm100::tmem_alloc(tmem_slot, 256);
    sm100::tmem_relinquish();
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(bar_full + 8 * i, 1);
      sm100::mbar_init(bar_empty + 8 * i, kTfEpi);
    }
    for (int i = 0; i < kES; ++i) {
      sm100::mbar_init(bar_ee + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) sm100::mbar_init(bar_nc + 8 * i, 32);
    sm100::fence_barrier_init();
  }

  // ---- the block's image region as stored (0 outside the image): the A / E staging centres it
  // (a0: x' = x - 0.5), the a5 re-score reads the raw values
  const float* img = a.imgs + size_t(f) * H * W;
  const int RH = NTI * kTR + BK - 1, RW = NTC * kTC + 7;
  for (int e = threadIdx.x; e < RH * RW; e += kTfThreads) {
    const int r = e / RW, c = e - r * RW;
    const int y = cyA + r, x = cxA + c;
    raw[r * a.RWp + c] = (y < H && x < W) ? __ldg(img + size_t(y) * W + x) : 0.5f;
  }
  __syncthreads();
  // tile order: by L1 gap to the reference block's rectangle (every reference meets its own
  // neighbourhood first), ties by index
  int16_t* order = reinterpret_cast<int16_t*>(smem + a.off_order);
  {
    const int ry0 = iy_first * s, ry1 = iy_last * s, rx0 = ix_first * s, rx1 = ix_last * s;
    auto dist_of = [&](int t) {
      const int tr = t / NTC, tc = t - (t / NTC) * NTC;
      const int y0 = cyA + kTR * tr, y1 = y0 + kTR - 1, x0 = cxA + kTC * tc, x1 = x0 + kTC - 1;
      return max(0, max(ry0 - y1, y0 - ry1)) + max(0, max(rx0 - x1, x0 - rx1));
    };
    for (int t = threadIdx.x; t < ntiles; t += kTfThreads) {
      const int dt = dist_of(t);
      int rank = 0;
      for (int u = 0; u < ntiles; ++u) {
        const int du = dist_of(u);
        rank += (du < dt || (du == dt && u < t)) ? 1 : 0;
      }
      order[rank] = int16_t(t);
    }
  }
  sm100::fence_proxy_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + 80);
  // A into TMEM (epilogue warp q writes lanes 32q..32q+31 = its references): row m holds the centred
  // patch of reference m = 32 q + l -> (iy_first + 4 (q >> 1) + l / 8, ix_first + 8 (q & 1) + l % 8)
  // as K = 8 b tf32 values k = 8 u + v (v >= b: 0), hi at columns [0, 8b), lo at [8b, 16b)
  if (warp < kTfEpi) {
    const int iy = iy_first + 4 * (warp >> 1) + (lane >> 3), ix = ix_first + 8 * (warp & 1) + (lane & 7);
    const bool ok = iy <= iy_last && ix <= ix_last;
    const uint32_t ta = tmem + (uint32_t(32 * warp) << 16);
#pragma unroll 1
    for (int u = 0; u < BK; ++u) {
      uint32_t h[8], o[8];
      const float* src = raw + (iy * s - cyA + u) * a.RWp + (ix * s - cxA);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const float x = (ok && v < BK) ? src[v] - 0.5f : 0.f;
        h[v] = tf32_hi(x);
        o[v] = __float_as_uint(x - __uint_as_float(h[v]));
      }
      sm100::tmem_st8(ta + 8u * u, h);
      sm100::tmem_st8(ta + kKA + 8u * u, o);
    }
    sm100::tmem_wait_st();
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();

  if (warp >= kTfEpi && warp < kTfEpi + kStg) {
    // ---------------- MMA issuer (one elected thread of warp kTfEpi) + tile producers (kStg warps):
    // the producers stage the E tile of t + 1 (hi and lo, E[y][jg][kc][j][t] = x'(cy0 + y, cx0 + 8 jg
    // + j + 4 kc + t)) while the tensor core runs tile t (each warp a share of the tile's entries, then
    // a named barrier among them); warp kTfEpi also stages the tile's 4 x 16 candidate norms (a1, from
    // the L2-resident norm map, loaded one tile ahead) into ring slot t & 1 (bar_nc) once the epilogue
    // has freed that accumulator, and its lane 0 issues the MMAs.
    const bool issuer = warp == kTfEpi;
    const int sw = warp - kTfEpi;  // producer index
    float* ncring = reinterpret_cast<float*>(smem + a.off_nc);  // [2][4][16]
    const float* nsrc = a.norm + size_t(f) * a.nfs;
    const int rr = lane >> 2, cq = lane & 3;
    auto load_norms = [&](int t) -> float4 {
      const int ot = order[t];
      const int tr = ot / NTC, tc = ot - tr * NTC;
      if (rr >= kTR) return make_float4(0.f, 0.f, 0.f, 0.f);
      const int cy = min(cyA + kTR * tr + rr, H - BK);
      return __ldg(reinterpret_cast<const float4*>(nsrc + size_t(cy) * a.Mx + cxA + kTC * tc) + cq);
    };
    auto stage = [&](int t) {
      const int ot = order[t % ntiles];
      const int sl_ = t % kES;
      const int tr = ot / NTC, tc = ot - tr * NTC;
      const float* src0 = raw + (kTR * tr) * a.RWp + kTC * tc;
      uint8_t* eh = smem + a.off_E + size_t(sl_) * 2 * kEBytes;
      for (int e = sw * 32 + lane; e < ER * 32; e += kStg * 32) {
        const int y = e >> 5, jg = (e >> 4) & 1, kc = (e >> 3) & 1, j = e & 7;
        const float* sp = src0 + y * a.RWp + 8 * jg + j + 4 * kc;
        uint32_t h[4], o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float x = sp[q] - 0.5f;
          h[q] = tf32_hi(x);
          o[q] = __float_as_uint(x - __uint_as_float(h[q]));
        }
        *reinterpret_cast<uint4*>(eh + e * 16) = make_uint4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<uint4*>(eh + kEBytes + e * 16) = make_uint4(o[0], o[1], o[2], o[3]);
      }
      sm100::fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
      if constexpr (kStg > 1) asm volatile("bar.sync 1, %0;" ::"n"(kStg * 32) : "memory");
      else __syncwarp();
    };
    float4 nv_next = issuer ? load_norms(0) : make_float4(0.f, 0.f, 0.f, 0.f);
    stage(0);
    for (int t = 0; t < NSW * ntiles; ++t) {
      const int sl = t % kES, buf = t & 1;
      if (issuer) {
        const float4 nv = nv_next;
        if (t + 1 < NSW * ntiles) nv_next = load_norms((t + 1) % ntiles);
        if (t >= 2) sm100::mbar_wait_sleep(bar_empty + 8 * buf, uint32_t(((t >> 1) - 1) & 1), 16);
        if (rr < kTR) reinterpret_cast<float4*>(ncring + (buf * kTR + rr) * kTC)[cq] = nv;
        sm100::mbar_arrive(bar_nc + 8 * buf);
        if (lane == 0) {
          sm100::tc_fence_after();
          const uint32_t eh = sE + uint32_t(sl) * 2 * kEBytes, el = eh + kEBytes;
#pragma unroll 1
          for (int u = 0; u < BK; ++u) {
            const uint64_t bh = sm100::smem_desc(eh + 512u * u, 128u, 256u);
            const uint64_t bl = sm100::smem_desc(el + 512u * u, 128u, 256u);
            const uint32_t d = tmem + kTmemD + uint32_t(kTR * kTC) * buf;
            sm100::mma_tf32_ta(d, tmem + 8u * u, bh, kIdesc, u > 0);        // A_hi B_hi
            sm100::mma_tf32_ta(d, tmem + 8u * u, bl, kIdesc, 1);            // A_hi B_lo
            sm100::mma_tf32_ta(d, tmem + kKA + 8u * u, bh, kIdesc, 1);      // A_lo B_hi
          }
          sm100::mma_commit(bar_full + 8 * buf);
          sm100::mma_commit(bar_ee + 8 * sl);
        }
        __syncwarp();
      }
      if (t + 1 < NSW * ntiles) {  // the next tile's slot is free once the MMAs of tile t - 1 are done
        if (t + 1 >= kES) sm100::mbar_wait_sleep(bar_ee + 8 * ((t + 1) % kES), uint32_t((((t + 1) / kES) - 1) & 1), 16);
        stage(t + 1);
      }
    }
  } else if (warp < kTfEpi) {
    // ---------------- epilogue: warp q = TMEM lanes 32q..32q+31 = references of a 4 x 8 sub-block
    const int q = warp;
    const int wiy0 = iy_first + 4 * (q >> 1), wix0 = ix_first + 8 * (q & 1);
    const int iy = wiy0 + (lane >> 3), ix = wix0 + (lane & 7);
    const bool valid = iy <= iy_last && ix <= ix_last;
    const bool wvalid = wiy0 <= iy_last && wix0 <= ix_last;
    const int wiy1 = min(iy_last, wiy0 + 3), wix1 = min(ix_last, wix0 + 7);
    const int wy_lo = wiy0 * s + a.lo, wy_hi = wiy1 * s + a.hi;  // the quadrant's window union
    const int wx_lo = wix0 * s + a.lo, wx_hi = wix1 * s + a.hi;
    const int ry = iy * s, rx = ix * s;
    const float nr = valid ? __ldg(a.norm + size_t(f) * a.nfs + size_t(ry) * a.Mx + rx) : 0.f;  // ||X_i||^2 (centred)
    const int rb = a.rb;
    const size_t band_refs = size_t(a.iy_end - a.iy_begin) * a.nx;
    const size_t ref_band = size_t(iy - a.iy_begin) * a.nx + ix;
    uint32_t* scratch = reinterpret_cast<uint32_t*>(smem + a.off_scr) + warp * a.scr;
    RegTopK32<HEAP ? 1 : KR> rt;
    if constexpr (!HEAP) {
#pragma unroll
      for (int k = 0; k < KR; ++k) rt.r[k] = k < KR - a.KP ? 0u : 0xffffffffu;
    }
    uint32_t* heap = reinterpret_cast<uint32_t*>(smem + a.off_heap) + (warp * 32 + lane) * a.hp;
    auto heap_init = [&]() {
      if constexpr (SCBM_TCF_SIFT == 4) {  // nodes at positions 3 .. KP + 2, zeros to the end of the row
        for (int k = kHB; k < kHB + a.KP; ++k) heap[k] = 0xffffffffu;
        for (int k = kHB + a.KP; k < a.hp; ++k) heap[k] = 0u;
      } else {
        for (int k = 1; k <= a.KP; ++k) heap[k] = 0xffffffffu;
        for (int k = a.KP + 1; k <= a.KP + 7; ++k) heap[k] = 0u;  // padding children: never the larger one
      }
    };
    uint8_t* const hist = reinterpret_cast<uint8_t*>(heap);  // BOUND sweep 1: 256 u8 bins (heap row)
    if constexpr (BOUND) {
      for (int k = 0; k < 64; ++k) heap[k] = 0u;
    } else if constexpr (HEAP) {
      heap_init();
    }
    uint32_t root_r = 0xffffffffu;  // heap[1] (SCBM_TCF_SIFT)
    constexpr bool kFillUp = SCBM_TCF_FILLUP && SCBM_TCF_SIFT == 4;
    int hcnt = kFillUp ? 0 : 1 << 30;  // FILLUP: keys in the heap while it fills
    (void)root_r;
    if constexpr (DENSE) {
      if (valid)
        for (int k = 0; k < a.Wn * a.Wn; ++k) a.dense[ref_band * a.Wn * a.Wn + k] = -1.f;
    }
    float thr = __int_as_float(0x7f800000);  // largest d' that may still enter the top-KP
    const uint32_t tq = tmem + (uint32_t(32 * q) << 16);
    const uint32_t sc_s = smem_u32(scratch + lane * kScrPitch);

#if SCBM_TCF_PROF
    long long p_wait = 0, p_round = 0, p_dense = 0, n_rounds = 0, n_ins = 0;
    const long long p_t0 = clock64();
#endif
    for (int t = 0; t < NSW * ntiles; ++t) {
      const int buf = t & 1;
      const bool sweep1 = BOUND && t < ntiles;
      if (BOUND && t == ntiles) {
        // end of sweep 1: the first bin where the cumulative count of group minima reaches K + m
        int cum = 0, bsel = 256;
        for (int w = 0; w < 64; ++w) {
          const uint32_t v = heap[w];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            cum += int((v >> (8 * k)) & 0xffu);
            if (bsel == 256 && cum >= a.KP) bsel = 4 * w + k;
          }
        }
        __syncwarp();
        heap_init();
        if constexpr (kFillUp) hcnt = 0;
        if (bsel < 255) {  // (bin 255 also holds everything >= 2^10: no bound)
          const float edge = __uint_as_float(uint32_t(bsel + kBinBase + 1) << 19);  // the bin's upper edge
          thr = fmaf(edge, 1.0f + 1e-6f, -nr) + 1e-30f;  // (d' = d - ||X_i||^2; rounding margin)
        }
      }
#if SCBM_TCF_PROF
      const long long pw0 = clock64();
#endif
      sm100::mbar_wait(bar_full + 8 * buf, uint32_t((t >> 1) & 1));
      sm100::mbar_wait(bar_nc + 8 * buf, uint32_t((t >> 1) & 1));
      sm100::tc_fence_after();
#if SCBM_TCF_PROF
      p_wait += clock64() - pw0;
#endif
      const float4* ncr = reinterpret_cast<const float4*>(smem + a.off_nc) + buf * kTR * 4;
      const int ot = order[t % ntiles];
      const int tr = ot / NTC, tc = ot - tr * NTC;
      const int cy0 = cyA + kTR * tr, cx0 = cxA + kTC * tc;
      const bool xrel = wvalid && cx0 <= wx_hi && cx0 + kTC - 1 >= wx_lo && !(SCBM_TCF_SKIP & 2);
      if (xrel) {
        // this lane's window columns inside the tile (a 16-bit mask), the same for every row
        const int jlo = max(0, max(0, rx + a.lo) - cx0), jhi = min(15, min(W - BK, rx + a.hi) - cx0);
        const uint32_t cols = (valid && jhi >= jlo) ? (((2u << jhi) - 1u) & ~((1u << jlo) - 1u)) : 0u;
#pragma unroll 1
        for (int i2 = 0; i2 < kTR; i2 += 2) {
          const int cyp = cy0 + i2;
          const bool r0 = cyp >= wy_lo && cyp <= wy_hi && cyp <= cyB;
          const bool r1 = cyp + 1 >= wy_lo && cyp + 1 <= wy_hi && cyp + 1 <= cyB;
          if (!r0 && !r1) continue;  // warp-uniform
          uint32_t cv[32];
          sm100::tmem_ld32(tq + kTmemD + uint32_t(kTR * kTC) * buf + 16u * i2, cv);
          // candidate norms of the two rows (staged by the MMA warp; rows past the map are masked below)
          float4 nq[8];
#pragma unroll
          for (int v = 0; v < 8; ++v) nq[v] = ncr[i2 * 4 + v];
          sm100::tmem_wait_ld();
          const uint32_t m0 = (r0 && cyp - ry >= a.lo && cyp - ry <= a.hi) ? cols : 0u;
          const uint32_t m1 = (r1 && cyp + 1 - ry >= a.lo && cyp + 1 - ry <= a.hi) ? cols : 0u;
          const uint32_t wmask = m0 | (m1 << 16);
          float dp[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float4 n4 = nq[j >> 2];
            const float nc = (j & 3) == 0 ? n4.x : (j & 3) == 1 ? n4.y : (j & 3) == 2 ? n4.z : n4.w;
            dp[j] = fmaf(-2.f, __uint_as_float(cv[j]), nc);  // d' = n_c - 2 C
          }
          if constexpr (DENSE) {
            const int rel0 = (cyp - ry - a.lo) * a.Wn + (cx0 - rx - a.lo);
            float* drow = a.dense + ref_band * a.Wn * a.Wn;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if ((wmask >> j) & 1u) drow[rel0 + (j >> 4) * a.Wn + (j & 15)] = dp[j] + nr;
            continue;
          }
          if (sweep1) {  // the group's minimum distance -> its histogram bin
            float mn = __int_as_float(0x7f800000);
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if ((wmask >> j) & 1u) mn = fminf(mn, dp[j]);
            if (wmask != 0u) {
              const uint32_t bits = __float_as_uint(fmaxf(mn + nr, 0.f));
              const int bin = min(255, max(0, int(bits >> 19) - kBinBase));
              hist[bin] = uint8_t(min(255, int(hist[bin]) + 1));
            }
            continue;
          }
          uint32_t fails = 0u;
#pragma unroll
          for (int j = 31; j >= 0; --j) fails = __funnelshift_l(__float_as_uint(thr - dp[j]), fails, 1);
          uint32_t bits = ~fails & wmask;
          if (SCBM_TCF_SKIP & 1) bits = 0u;
          if (!__any_sync(0xffffffffu, bits != 0u)) continue;
          // stage the distances d = d' + ||X_i||^2 (>= 0) of the two rows, then insert one survivor per
          // lane per round (branch-free; lanes without one insert the no-op key ~0)
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 o = make_float4(fmaxf(dp[j] + nr, 0.f), fmaxf(dp[j + 1] + nr, 0.f),
                                         fmaxf(dp[j + 2] + nr, 0.f), fmaxf(dp[j + 3] + nr, 0.f));
            *reinterpret_cast<float4*>(scratch + lane * kScrPitch + j) = o;
          }
          __syncwarp();
          const int rel1b = (cyp - ry - a.lo) * a.Wn + (cx0 - rx - a.lo) + 1;
#if SCBM_TCF_PROF
          const long long pr0 = clock64();
          n_ins += __popc(bits);
#endif
#if SCBM_TCF_SIFT
          // one survivor per lane per round, the next one's distance loaded while this one sinks;
          // the heap root lives in a register (root_r) and the sift-down runs a fixed number of
          // levels with predicated loads / stores (no divergent early exit)
          int i = 31 - __clz(bits | 1u);
          uint32_t d;
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(d) : "r"(sc_s + 4u * uint32_t(i)));
          while (__any_sync(0xffffffffu, bits != 0u)) {
#if SCBM_TCF_PROF
            ++n_rounds;
#endif
            const int ic = i;
            const uint32_t qd = d >> (rb - 1);
            const int rel1 = rel1b + (ic >> 4) * a.Wn + (ic & 15);
            const uint32_t key = bits ? (qd << rb) | uint32_t(rel1) : 0xffffffffu;
            bits &= ~(1u << ic);
            i = 31 - __clz(bits | 1u);
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(d) : "r"(sc_s + 4u * uint32_t(i)));
            if constexpr (HEAP) {
              if (kFillUp && key < root_r && hcnt < a.KP) {
                // the heap is not full yet: the key goes to the next free node and sifts UP (a few
                // steps on average) instead of replacing the (+inf) root and sinking through every
                // level; the root register becomes the real maximum once the KP-th key is in
                int n = hcnt++;
                while (n > 0) {
                  const int p = (n - 1) >> 2;
                  const uint32_t pv = heap[3 + p];
                  if (pv >= key) break;
                  heap[3 + n] = pv;
                  n = p;
                }
                heap[3 + n] = key;
                if (hcnt == a.KP) root_r = heap[3];
              } else if (key < root_r) {  // replace the root, sift down (children of h: 2h, 2h+1)
                int h = 1;
                bool alive = true;
                uint32_t nroot = key;
#if SCBM_TCF_SIFT == 3
                // children of h in vv, grandchildren (4h .. 4h+3) in gq, great-grandchildren (8h .. 8h+7) in
                // g0, g1: a level's loads are consumed two levels later (heap rows 16-byte aligned, nodes
                // KP+1 .. KP+7 are 0: never the larger child)
                uint2 vv = *reinterpret_cast<const uint2*>(heap + 2);
                uint4 gq = *reinterpret_cast<const uint4*>(heap + 4);
                uint4 g0 = *reinterpret_cast<const uint4*>(heap + 8);
                uint4 g1 = *reinterpret_cast<const uint4*>(heap + 12);
#pragma unroll
                for (int lvl = 0; lvl < kSiftLevels; ++lvl) {
                  const int c = 2 * h;
                  const bool right = vv.y > vv.x;
                  const int cb = right ? c + 1 : c;
                  const uint32_t big = max(vv.x, vv.y);
                  const bool mv = alive && big > key;
                  const uint2 nv = right ? make_uint2(gq.z, gq.w) : make_uint2(gq.x, gq.y);
                  const uint4 nq = right ? g1 : g0;
                  if (lvl + 2 < kSiftLevels) {
                    g0 = g1 = make_uint4(0u, 0u, 0u, 0u);
                    if (mv && 8 * cb <= a.KP) {
                      g0 = *reinterpret_cast<const uint4*>(heap + 8 * cb);
                      g1 = *reinterpret_cast<const uint4*>(heap + 8 * cb + 4);
                    }
                  }
                  if (mv) heap[h] = big;
                  if (lvl == 0) nroot = mv ? big : key;
                  h = mv ? cb : h;
                  alive = mv && 2 * cb <= a.KP;
                  vv = nv;
                  gq = nq;
                }
#elif SCBM_TCF_SIFT == 4
                // 4-ary max-heap: node n at position n + 3, so the children of n (4n+1 .. 4n+4) sit at
                // positions 4n+4 .. 4n+7 -- one aligned 16-byte load; the children of the four children
                // (positions 16n+8 .. 16n+23) are loaded one level ahead. Three levels below the root
                // hold K + m <= 85 keys (binary: six). Positions past the last node are 0.
                int n = 0;
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
                    // (one guard for the four blocks: the row pitch is chosen so that a block group past the
                    // row holds no node -- see tcf_layout -- and such groups read as zeros)
                    if (mv && 16 * cb + 24 <= a.hp) {
                      g0 = *reinterpret_cast<const uint4*>(heap + 16 * cb + 8);
                      g1 = *reinterpret_cast<const uint4*>(heap + 16 * cb + 12);
                      g2 = *reinterpret_cast<const uint4*>(heap + 16 * cb + 16);
                      g3 = *reinterpret_cast<const uint4*>(heap + 16 * cb + 20);
                    }
                  }
                  if (mv) heap[3 + n] = big;
                  if (lvl == 0) nroot = mv ? big : key;
                  n = mv ? cb : n;
                  alive = mv && 4 * cb + 1 < a.KP;
                  vv = nv;
                }
                h = 3 + n;
#elif SCBM_TCF_SIFT == 2
                // children of h in vv, grandchildren (nodes 4h .. 4h+3) in gq: the next level's load is
                // issued before this level's comparison resolves (heap rows are 16-byte aligned, nodes
                // KP+1 .. KP+3 are 0: never the larger child)
                uint2 vv = *reinterpret_cast<const uint2*>(heap + 2);
                uint4 gq = *reinterpret_cast<const uint4*>(heap + 4);
#pragma unroll
                for (int lvl = 0; lvl < kSiftLevels; ++lvl) {
                  const int c = 2 * h;
                  const bool right = vv.y > vv.x;
                  const int cb = right ? c + 1 : c;
                  const uint32_t big = max(vv.x, vv.y);
                  const bool mv = alive && big > key;
                  const uint2 nv = right ? make_uint2(gq.z, gq.w) : make_uint2(gq.x, gq.y);
                  if (lvl + 1 < kSiftLevels) {
                    gq = make_uint4(0u, 0u, 0u, 0u);
                    if (mv && 4 * cb <= a.KP) gq = *reinterpret_cast<const uint4*>(heap + 4 * cb);
                  }
                  if (mv) heap[h] = big;
                  if (lvl == 0) nroot = mv ? big : key;
                  h = mv ? cb : h;
                  alive = mv && 2 * cb <= a.KP;
                  vv = nv;
                }
#else
#pragma unroll
                for (int lvl = 0; lvl < kSiftLevels; ++lvl) {
                  const int c = 2 * h;
                  uint2 vv = make_uint2(0u, 0u);
                  if (alive && c <= a.KP) vv = *reinterpret_cast<const uint2*>(heap + c);
                  const int cb = vv.y > vv.x ? c + 1 : c;
                  const uint32_t big = max(vv.x, vv.y);
                  const bool mv = big > key;  // (0 for a finished sift or past the last level)
                  if (mv) heap[h] = big;
                  if (lvl == 0) nroot = mv ? big : key;
                  h = mv ? cb : h;
                  alive = mv;
                }
#endif
                heap[h] = key;
                root_r = nroot;
              }
            } else {
              rt.insert(key);
            }
          }
#else
          while (__any_sync(0xffffffffu, bits != 0u)) {
#if SCBM_TCF_PROF
            ++n_rounds;
#endif
            const int i = 31 - __clz(bits | 1u);
            uint32_t d;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(d) : "r"(sc_s + 4u * uint32_t(i)));
            const uint32_t qd = d >> (rb - 1);
            const int rel1 = rel1b + (i >> 4) * a.Wn + (i & 15);
            const uint32_t key = bits ? (qd << rb) | uint32_t(rel1) : 0xffffffffu;
            bits &= ~(1u << i);
            if constexpr (HEAP) {
              if (key < heap[1]) {  // replace the root, sift down (children of h: 2h, 2h+1)
                int h = 1;
                for (int c = 2; c <= a.KP; c = 2 * h) {
                  const uint2 vv = *reinterpret_cast<const uint2*>(heap + c);
                  const int cb = vv.y > vv.x ? c + 1 : c;
                  const uint32_t big = max(vv.x, vv.y);
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
#endif
#if SCBM_TCF_PROF
          p_round += clock64() - pr0;
#endif
          const uint32_t kth = HEAP ? (SCBM_TCF_SIFT ? root_r : heap[1]) : rt.r[KR - 1];
          if (kth != 0xffffffffu) {
            // largest distance whose key can still tie the KP-th key, plus a rounding margin
            const float dmax = __uint_as_float(((kth >> rb) << (rb - 1)) | ((1u << (rb - 1)) - 1u));
            thr = fmaf(dmax, 1.0f + 1e-6f, -nr) + 1e-30f;
          }
          __syncwarp();
        }
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(bar_empty + 8 * buf);
    }

#if SCBM_TCF_PROF
    {
      const long long tot = clock64() - p_t0;
      long long ins = n_ins;
      for (int o = 16; o; o >>= 1) ins += __shfl_xor_sync(0xffffffffu, ins, o);
      if (lane == 0 && (blockIdx.x == 0 || blockIdx.x == 700 || blockIdx.x == 1500) && blockIdx.y == 0)
        printf("tcfprof cta %d warp %d tiles %d loop %lld wait %lld rounds_cyc %lld rounds %lld ins %lld\n",
               blockIdx.x, warp, ntiles, tot, p_wait, p_round, n_rounds, ins);
    }
#endif
    if constexpr (!DENSE) {  // hand the reference norms and register lists to the a5 stage
      float* nrs = reinterpret_cast<float*>(smem + a.off_E);
      uint32_t* lists = reinterpret_cast<uint32_t*>(smem + a.off_E) + 128;
      nrs[32 * warp + lane] = nr;
      if constexpr (!HEAP) {
#pragma unroll
        for (int k = 0; k < KR; ++k) lists[(32 * warp + lane) * (KR + 1) + k] = rt.r[k];
      }
    }
  }

#if SCBM_TCF_PROF
  long long pa0 = 0;
#endif
  if constexpr (!DENSE) {
    // ---- a5 + a6, all warps: per reference (one warp each), the KP kept keys re-scored by direct
    // differences from the staged region (the input values as stored), sorted by (distance, idx),
    // K written; references whose kept keys cannot decide the K-th go to the exact fix-up.
    __syncthreads();  // every tile's MMAs and epilogue are done: the E ring holds the handed-over lists
#if SCBM_TCF_PROF
    pa0 = clock64();
#endif
    const float* nrs = reinterpret_cast<const float*>(smem + a.off_E);
    const uint32_t* lists = reinterpret_cast<const uint32_t*>(smem + a.off_E) + 128;
    const uint32_t* heaps = reinterpret_cast<const uint32_t*>(smem + a.off_heap);
    const int rb = a.rb;
    const size_t band_refs = size_t(a.iy_end - a.iy_begin) * a.nx;
    constexpr int NJ = (KR + 31) / 32;
    for (int m = warp; m < ((SCBM_TCF_SKIP & 4) ? 0 : 128); m += kTfWarps) {
      const int q = m >> 5, l = m & 31;
      const int iyj = iy_first + 4 * (q >> 1) + (l >> 3), ixj = ix_first + 8 * (q & 1) + (l & 7);
      if (iyj > iy_last || ixj > ix_last) continue;  // warp-uniform
      const int ryj = iyj * s, rxj = ixj * s;
      const size_t row = size_t(f) * band_refs + size_t(iyj - a.iy_begin) * a.nx + ixj;
      const float* pr = raw + (ryj - cyA) * a.RWp + (rxj - cxA);
      // the kept keys re-scored exactly; 128-key sets (K + m > 64) sorted once, 4 per lane
      // (element e = 4 lane + i), smaller ones through the warp lists
      auto rescore = [&](uint32_t kk) -> uint64_t {
        if (kk == 0u || kk == 0xffffffffu) return kKeyInf;
        const int rel = int(kk & ((1u << rb) - 1u)) - 1;
        const int dyy = rel / a.Wn, dxx = rel - dyy * a.Wn;
        const int cy = ryj + dyy + a.lo, cx = rxj + dxx + a.lo;
        const float* pc = raw + (cy - cyA) * a.RWp + (cx - cxA);
        float d = 0.f;
#pragma unroll
        for (int r = 0; r < BK; ++r)
#pragma unroll
          for (int c = 0; c < BK; ++c) {
            const float df = pr[r * a.RWp + c] - pc[r * a.RWp + c];
            d = fmaf(df, df, d);
          }
        return (uint64_t(__float_as_uint(d)) << 32) | uint32_t(cy * W + cx);
      };
      auto kept = [&](int k) -> uint32_t {
        if constexpr (HEAP) return k < a.KP ? heaps[m * a.hp + kHB + k] : 0xffffffffu;
        else return k < KR ? lists[m * (KR + 1) + k] : 0xffffffffu;
      };
      uint64_t kv;  // the K-th exact key (broadcast)
      if constexpr (NJ >= 3) {
        uint64_t v[4];
#if SCBM_TCF_A5ILP
        {  // the lane's 4 kept keys re-scored together (each reference value loaded once, 4 chains)
          const float* pc[4];
          bool ok[4];
          int cidx[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint32_t kk = kept(4 * lane + i);
            ok[i] = kk != 0u && kk != 0xffffffffu;
            const int rel = ok[i] ? int(kk & ((1u << rb) - 1u)) - 1 : 0;
            const int dyy = rel / a.Wn, dxx = rel - dyy * a.Wn;
            const int cy = ryj + dyy + a.lo, cx = rxj + dxx + a.lo;
            cidx[i] = cy * W + cx;
            pc[i] = ok[i] ? raw + (cy - cyA) * a.RWp + (cx - cxA) : pr;
          }
          float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int r = 0; r < BK; ++r)
#pragma unroll
            for (int c = 0; c < BK; ++c) {
              const float rv = pr[r * a.RWp + c];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float df = rv - pc[i][r * a.RWp + c];
                d[i] = fmaf(df, df, d[i]);
              }
            }
#pragma unroll
          for (int i = 0; i < 4; ++i)
            v[i] = ok[i] ? (uint64_t(__float_as_uint(d[i])) << 32) | uint32_t(cidx[i]) : kKeyInf;
        }
#else
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = rescore(kept(4 * lane + i));
#endif
        warp_sort128(v, lane);
        uint64_t kq = v[0];
#pragma unroll
        for (int i = 1; i < 4; ++i)
          if (i == (a.K - 1) % 4) kq = v[i];
        kv = __shfl_sync(0xffffffffu, kq, (a.K - 1) / 4);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int k = 4 * lane + i;
          if (k < a.K) {
            const bool none = v[i] == kKeyInf;
            a.idx_out[row * a.K + k] = none ? -1 : int32_t(uint32_t(v[i]));
            a.dist_out[row * a.K + k] = none ? __int_as_float(0x7f800000) : __uint_as_float(uint32_t(v[i] >> 32));
          }
        }
      } else {
        WarpTopK<NJ> top;
        top.init();
#pragma unroll
        for (int sl = 0; sl < NJ; ++sl) top.merge(rescore(kept(sl * 32 + lane)), lane);
        kv = kKeyInf;
#pragma unroll
        for (int sl = 0; sl < NJ; ++sl)
          if (sl == (a.K - 1) / 32) kv = top.v[sl];
        kv = __shfl_sync(0xffffffffu, kv, (a.K - 1) % 32);
#pragma unroll
        for (int sl = 0; sl < NJ; ++sl) {
          const int k = sl * 32 + lane;
          if (k < a.K) {
            const uint64_t key = top.v[sl];
            const bool none = key == kKeyInf;
            a.idx_out[row * a.K + k] = none ? -1 : int32_t(uint32_t(key));
            a.dist_out[row * a.K + k] = none ? __int_as_float(0x7f800000) : __uint_as_float(uint32_t(key >> 32));
          }
        }
      }
      {  // worst kept key vs the exact K-th distance: the filter's error could hide a candidate
        const float nrj = nrs[m];
        const uint32_t klast = HEAP ? heaps[m * a.hp + kHB] : lists[m * (KR + 1) + KR - 1];  // heap root / last
        if (lane == 0 && klast != 0u && klast != 0xffffffffu && kv != kKeyInf) {
          const float dK = __uint_as_float(uint32_t(kv >> 32));
          const float smin = __uint_as_float((klast >> rb) << (rb - 1));
          if (smin <= fmaf(dK, 1.0f + 1e-5f, kTcfErr * (nrj + dK))) {
            const int pos = atomicAdd(a.fix_count, 1);
            a.fix_list[pos] = int(row);
          }
        }
      }
    }
  }
#if SCBM_TCF_PROF
  if constexpr (!DENSE) {
    if (lane == 0 && (blockIdx.x == 0 || blockIdx.x == 700 || blockIdx.x == 1500) && blockIdx.y == 0)
      printf("tcfprof cta %d warp %d a5 %lld\n", blockIdx.x, warp, clock64() - pa0);
  }
#endif
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == kTfWarps - 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem, 256);
  }
}

struct TcfLayout {
  int RHmax, RWp, NTImax, NTCmax, hp, scr;
  uint32_t off_order, off_raw, off_A, off_E, off_heap, off_scr, off_nc, bytes;
};

int tcf_kr(const Geometry& g) {
  return g.KP <= 24 ? 24 : g.KP <= 32 ? 32 : g.KP <= 40 ? 40 : g.KP <= 48 ? 48 : g.KP <= 80 ? 80 : 0;
}

int tcf_rel_bits(int Wn) {  // bits of rel + 1 (values 1 .. Wn^2; 0 = sentinel)
  int rb = 1;
  while ((1 << rb) <= Wn * Wn) ++rb;
  return rb;
}

TcfLayout tcf_layout(const Geometry& g) {
  TcfLayout L{};
  const int kr = tcf_kr(g);
  L.NTImax = ((kRBY - 1) * g.s + g.Wn - 1) / kTR + 1;
  L.NTCmax = ((kRBX - 1) * g.s + g.Wn - 1 + 3) / kTC + 1;  // + the alignment of cxA
  L.RHmax = L.NTImax * kTR + g.b - 1;
  L.RWp = L.NTCmax * kTC + 7 + 1;
  // heap pitch: nodes 1 .. KP + 7 (seven 0 padding nodes), a multiple of 4 words: 16-byte aligned rows
  // (the sift-down's grandchild / great-grandchild loads)
  // (4-ary: the last internal node's children end at position 4 ((KP - 2) / 4) + 7)
  // (4-ary: the last internal node's children end at position 4 ((KP - 2) / 4) + 7, and every
  // 64-byte prefetch group 16 c + 8 .. 16 c + 23 that starts at or before the last node (position
  // KP + 2) must lie inside the row, so the sift-down's single guard never skips a node: c3 3.13 ms,
  // against 3.27 with four per-block guards and the minimum pitch)
  L.hp = SCBM_TCF_SIFT == 4 ? std::max(4 * ((g.KP - 2) / 4) + 8, 16 * ((g.KP - 6) / 16) + 24)
                            : (g.KP + (SCBM_TCF_SIFT >= 3 ? 8 : 4) + 3) & ~3;
  if (kr > 48 && SCBM_TCF_BOUND && L.hp < 64) L.hp = 64;  // (the bound sweep's 256 u8 bins share the row)
  if (L.hp % 8 == 0) L.hp += 4;  // = 4 (mod 8): the 32 lanes' 16-byte loads spread over all banks
  L.scr = std::max(32 * kScrPitch, kr > 48 ? 0 : 32 * (kr + 1));
  uint32_t off = 128;  // barriers + TMEM slot
  L.off_order = off;
  off += uint32_t(L.NTImax * L.NTCmax) * 2;
  off = (off + 15) & ~15u;
  L.off_raw = off;
  off += uint32_t(L.RHmax * L.RWp) * 4;
  off = (off + 1023) & ~1023u;
  L.off_A = off;  // (A lives in TMEM)
  L.off_E = off;  // the E ring; after the last tile the a5 stage's norms + register lists
  // (the heaps stay in their own area: only the reference norms are handed over)
  off += std::max(uint32_t(kES) * 2u * uint32_t(kTR + g.b - 1) * 512u,
                  uint32_t(128 + (kr > 48 ? 0 : 128 * (kr + 1))) * 4u);
  L.off_nc = off;  // candidate-norm ring [2][8][16]
  off += 2u * kTR * kTC * 4u;
  L.off_heap = off;
  if (kr > 48) off += 128u * uint32_t(L.hp) * 4u;
  L.off_scr = off;
  off += uint32_t(kTfEpi * L.scr) * 4u;
  L.bytes = off;
  return L;
}

template <int BK, int KR, bool DENSE>
cudaError_t launch_tcf_t(const TcfArgs& a, int F, size_t smem, cudaStream_t st) {
  const int tiles_y = (a.iy_end - a.iy_begin + kRBY - 1) / kRBY;
  auto k = bm_tcf_kernel<BK, KR, DENSE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k<<<dim3(a.tiles_x * tiles_y, F), kTfThreads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

bool tcf_supported(const Geometry& g) {
  if (g.dtype != SC_DTYPE_F32 || g.metric != SC_METRIC_L2 || g.C != 1) return false;
  if (g.b < 1 || g.b > 8 || tcf_kr(g) == 0) return false;
  if (tcf_rel_bits(g.Wn) > 12) return false;  // keeps >= 20 distance bits in the 32-bit keys
  if (g.W - g.b + 1 < 16 && g.W < 24) return false;  // (tiles read 16 norm columns; tiny widths use others)
  // two CTAs per SM (4 + 4 epilogue warps) up to 113 KB; larger layouts run one CTA per SM
  return tcf_layout(g).bytes <= 227 * 1024;
}

bool tcf_preferred(const Geometry& g) {
  return tcf_supported(g) && g.s == 1 && !g.z3 && tcf_layout(g).bytes <= 113 * 1024;
}

cudaError_t launch_bm_tcf(const sc_bm_plan_s& p, const void* imgs, int F, int iy_begin, int iy_end,
                          int32_t* idx_out, void* dist_out, void* dense, cudaStream_t st, int64_t* launches) {
  const Geometry& g = p.g;
  const TcfLayout L = tcf_layout(g);
  TcfArgs a{};
  a.imgs = static_cast<const float*>(imgs);
  a.norm = static_cast<const float*>(p.ws.norm);
  a.idx_out = idx_out;
  a.dist_out = static_cast<float*>(dist_out);
  a.dense = static_cast<float*>(dense);
  a.H = g.H; a.W = g.W; a.s = g.s; a.Wn = g.Wn; a.K = g.K; a.KP = g.KP; a.lo = g.lo; a.hi = g.hi; a.nx = g.nx;
  a.iy_begin = iy_begin; a.iy_end = iy_end;
  a.tiles_x = (g.nx + kRBX - 1) / kRBX;
  a.Mx = g.Mxp;
  a.nfs = g.NFS;
  a.rb = tcf_rel_bits(g.Wn);
  a.RH = L.RHmax; a.RWp = L.RWp;
  a.off_raw = L.off_raw; a.off_A = L.off_A; a.off_E = L.off_E; a.off_heap = L.off_heap; a.off_scr = L.off_scr;
  a.off_order = L.off_order;
  a.off_nc = L.off_nc;
  a.hp = L.hp;
  a.scr = L.scr;
  a.fix_count = p.ws.fix_count;
  a.fix_list = p.ws.fix_list;
  const int kr = tcf_kr(g);
  cudaError_t e = cudaSuccess;
  if (!dense) e = cudaMemsetAsync(p.ws.fix_count, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  if (launches) *launches += 1;
#define SCBM_TCF_B(B_)                                                                 \
  if (g.b == B_) {                                                                     \
    if (dense) return launch_tcf_t<B_, 24, true>(a, F, L.bytes, st);                   \
    if (kr == 24) e = launch_tcf_t<B_, 24, false>(a, F, L.bytes, st);                  \
    else if (kr == 32) e = launch_tcf_t<B_, 32, false>(a, F, L.bytes, st);             \
    else if (kr == 40) e = launch_tcf_t<B_, 40, false>(a, F, L.bytes, st);             \
    else if (kr == 48) e = launch_tcf_t<B_, 48, false>(a, F, L.bytes, st);             \
    else e = launch_tcf_t<B_, 80, false>(a, F, L.bytes, st);                           \
  }
  SCBM_TCF_B(8)
  else SCBM_TCF_B(7)
  else SCBM_TCF_B(6)
  else SCBM_TCF_B(5)
  else SCBM_TCF_B(4)
  else SCBM_TCF_B(3)
  else SCBM_TCF_B(2)
  else SCBM_TCF_B(1)
#undef SCBM_TCF_B
  if (e != cudaSuccess) return e;
  if (launches) *launches += 1;
  return launch_fixup(p, imgs, F, iy_begin, iy_end, idx_out, dist_out, st);
}

}  // namespace scbm
