// bm_tc.cu -- the tensor-core matcher (SC_KERNEL_TC_I8): uint8 images, b = 8, C = 1.
//
// a2 (the Self-Convolution cross term, Eq. 5) runs on the 5th-generation
// tensor cores as an int8 GEMM  D[ref][cand] = sum_k A[ref][k] * B[cand][k]  (k = 8*l + m over
// the 8x8 patch, centred x' = x - 128 as signed int8, exact int32 accumulation in TMEM):
//
//   * A (M = 128 references of an 8 x 16 reference block) is K-major in shared memory: one
//     64-byte centred patch per reference in canonical 8-row x 16-byte core matrices.
//   * B (N = 128 candidates: an 8-row x 16-column block of candidate top-left positions) is
//     MN-major straight out of a "shift-expanded" copy of the image region E[y][c][m][t] =
//     x'(y, X0 + 16c + t + m): K-group l of candidate row i is image row y0 + i + l, so ONE
//     descriptor (LBO = SBO = row pitch) addresses the whole 8 x 16 candidate block -- no
//     im2col materialisation, 8 bytes of E per image byte.
//   * each tile is two tcgen05.mma.cta_group::1.kind::i8 (K = 32 each) into a 128 x 128 int32
//     TMEM accumulator, double-buffered (256 TMEM columns) so the MMA of tile t+1 overlaps the
//     epilogue of tile t; one elected thread of the MMA warp issues them and commits to an
//     mbarrier.
//
// Epilogue (4 warps, TMEM lane quarter q = references 32q..32q+31 = a 4 x 8 sub-block):
// tcgen05.ld 16 columns (one candidate row of the tile), d' = n_c - 2C (Lemma 2),
// one compare per pair against the reference's heap root into a bitmask; rows where some lane
// passed go through the window check and the survivor queue / per-reference heaps of refq.cuh
// (a4). Tiles outside a warp's window union are skipped. a6 as in bm_lanes.cu (exact int32).
#include <cstdio>
#include <cstdlib>

#include "refq.cuh"
#include "regtopk.cuh"
#include "sc_internal.h"
#include "sm100.cuh"
#include "topk.cuh"

namespace scbm {
namespace {

constexpr int kEpiWarps = 8;
constexpr int kThreads = (kEpiWarps + 1) * 32;
constexpr int kRBY = 8, kRBX = 16;   // reference block (M = 128)
constexpr int kTR = 8, kTC = 16;     // candidate tile: 8 rows x 16 columns (N = 128)
constexpr uint32_t kIdesc = sm100::idesc_i8(128, 128, /*a_mn=*/false, /*b_mn=*/true);

struct TcArgs {
  const uint8_t* imgs;
  const int32_t* norm;
  int32_t* idx_out;
  int32_t* dist_out;
  int H, W, s, Wn, K, KP, lo, hi, nx, My, Mx, iy_begin, iy_end, tiles_x;
  int NCmax, NTImax;
  long long nfs;  // norm-map frame stride
  uint32_t off_A, off_E, off_N, off_heap, off_q;  // shared byte offsets
  int heap_pitch;
  int rb;          // 32-bit keys: window-relative index bits
  uint32_t dsat;   // 32-bit keys: distance saturation value
  int* fix_count;  // exact fix-up list (fixup.cu)
  int* fix_list;
  int dbg;  // SCBM_TC_DEBUG: bit0 skip epilogue work, bit1 skip MMA (timing experiments only)
};

__device__ unsigned long long g_tc_stats[8];  // debug counters (SCBM_TC_DEBUG & 4)
__device__ unsigned long long g_tc_clk[8];    // debug cycle accumulators (SCBM_TC_DEBUG & 8)
#define TCLK(i, t0) do { if (a.dbg & 8) { const long long _t = clock64(); if (lane == 0) atomicAdd(&g_tc_clk[i], (unsigned long long)(_t - (t0))); (t0) = _t; } } while (0)


__global__ void __launch_bounds__(kThreads, 2) bm_tc_i8_kernel(TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  long long t0 = clock64();
  const int f = blockIdx.y;
  const int by = blockIdx.x / a.tiles_x, bx = blockIdx.x - by * a.tiles_x;
  const int iy_first = a.iy_begin + by * kRBY;
  const int iy_last = min(a.iy_end, iy_first + kRBY) - 1;
  const int ix_first = bx * kRBX;
  const int ix_last = min(a.nx, ix_first + kRBX) - 1;
  const int s = a.s, H = a.H, W = a.W, b = 8;
  const int cyA = max(0, iy_first * s + a.lo), cyB = min(H - b, iy_last * s + a.hi);
  const int cxA = max(0, ix_first * s + a.lo), cxB = min(W - b, ix_last * s + a.hi);
  const int X0 = cxA & ~15;
  const int NC = (cxB - X0) / kTC + 1;           // candidate column chunks
  const int NTI = (cyB - cyA) / kTR + 1;         // candidate row blocks
  const int RH = NTI * kTR + 7;                  // image rows of E
  const uint32_t RP = uint32_t(NC) * 128u;       // E row pitch (bytes)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const uint32_t sbase = smem_addr(smem);
  const uint32_t bar_full = sbase, bar_empty = sbase + 16;  // 2 + 2 mbarriers
  const uint32_t tmem_slot = sbase + 32;
  const uint32_t bar_nc = sbase + 40;  // 2 mbarriers: norm values of the tile staged (count 32)
  const uint32_t sA = sbase + a.off_A, sE = sbase + a.off_E;
  uint64_t* heaps = reinterpret_cast<uint64_t*>(smem + a.off_heap);

  if (warp == kEpiWarps) {
    sm100::tmem_alloc(tmem_slot, 256);
    sm100::tmem_relinquish();
  }
  if (threadIdx.x == 0) {
    sm100::mbar_init(bar_full, 1);
    sm100::mbar_init(bar_full + 8, 1);
    sm100::mbar_init(bar_empty, kEpiWarps);
    sm100::mbar_init(bar_empty + 8, kEpiWarps);
    sm100::mbar_init(bar_nc, 32);
    sm100::mbar_init(bar_nc + 8, 32);
    sm100::fence_barrier_init();
  }

  // ---- a0 staging: A (reference patches), E (shift-expanded image), norm tile, heaps
  const uint8_t* img = a.imgs + size_t(f) * H * W;
  for (int e = threadIdx.x; e < 128 * 4; e += kThreads) {
    const int m = e >> 2, kc = e & 3;
    const int w = m >> 5, L = m & 31;
    const int iy = iy_first + 4 * (w >> 1) + (L >> 3), ix = ix_first + 8 * (w & 1) + (L & 7);
    uint32_t v[4] = {0, 0, 0, 0};
    if (iy <= iy_last && ix <= ix_last) {
      const uint8_t* p = img + size_t(iy * s + 2 * kc) * W + ix * s;
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          uint32_t wd = 0;
#pragma unroll
          for (int e2 = 0; e2 < 4; ++e2) wd |= uint32_t(p[h * W + 4 * q + e2]) << (8 * e2);
          v[2 * h + q] = wd ^ 0x80808080u;
        }
    }
    uint4* dst = reinterpret_cast<uint4*>(smem + a.off_A + (m >> 3) * 512 + kc * 128 + (m & 7) * 16);
    *dst = make_uint4(v[0], v[1], v[2], v[3]);
  }
  for (int e = threadIdx.x; e < RH * NC; e += kThreads) {
    const int yr = e / NC, c = e - yr * NC;
    const int y = cyA + yr;
    uint32_t w[8];
    const int x0 = X0 + 16 * c;
    const uint8_t* rowp = img + size_t(y) * W + x0;
    if (y < H && x0 + 32 <= W && (reinterpret_cast<uintptr_t>(rowp) & 15) == 0) {
      const uint4* src = reinterpret_cast<const uint4*>(rowp);
      const uint4 q0 = src[0], q1 = src[1];
      w[0] = q0.x; w[1] = q0.y; w[2] = q0.z; w[3] = q0.w; w[4] = q1.x; w[5] = q1.y; w[6] = q1.z; w[7] = q1.w;
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] ^= 0x80808080u;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint32_t wd = 0;
#pragma unroll
        for (int e2 = 0; e2 < 4; ++e2) {
          const int x = x0 + 4 * i + e2;
          const uint32_t v = (y < H && x < W) ? uint32_t(img[size_t(y) * W + x] ^ 0x80u) : 0u;
          wd |= v << (8 * e2);
        }
        w[i] = wd;
      }
    }
    uint8_t* row = smem + a.off_E + size_t(yr) * RP + c * 128;
#pragma unroll
    for (int mm = 0; mm < 8; ++mm) {
      const int q = mm >> 2, sh = 8 * (mm & 3);
      uint4 o;
      o.x = __funnelshift_r(w[q + 0], w[q + 1], sh);
      o.y = __funnelshift_r(w[q + 1], w[q + 2], sh);
      o.z = __funnelshift_r(w[q + 2], w[q + 3], sh);
      o.w = __funnelshift_r(w[q + 3], w[q + 4], sh);
      *reinterpret_cast<uint4*>(row + mm * 16) = o;
    }
  }
  const int32_t* nsrc = a.norm + size_t(f) * a.nfs;  // a.Mx = norm-map row pitch

  for (int e = threadIdx.x; e < 2 * 128; e += kThreads)  // published thresholds: +inf until set
    reinterpret_cast<uint64_t*>(smem + a.off_q)[e] = kKeyInf;
  // Tile order: by L1 gap to the rectangle of the block's own reference positions, so every
  // reference meets its spatial neighbourhood (including itself) first and its top-K threshold
  // tightens early (fewer survivors); ties by index.
  int16_t* order = reinterpret_cast<int16_t*>(smem + 64);
  {
    const int ry0 = iy_first * s, ry1 = iy_last * s, rx0 = ix_first * s, rx1 = ix_last * s;
    auto dist_of = [&](int t) {
      const int tr = t / NC, tc = t - (t / NC) * NC;
      const int y0 = cyA + kTR * tr, y1 = y0 + kTR - 1, x0 = X0 + kTC * tc, x1 = x0 + kTC - 1;
      const int gy = max(0, max(ry0 - y1, y0 - ry1)), gx = max(0, max(rx0 - x1, x0 - rx1));
      return gy + gx;
    };
    const int nt = NTI * NC;
    for (int t = threadIdx.x; t < nt; t += kThreads) {
      const int dt = dist_of(t);
      int rank = 0;
      for (int u = 0; u < nt; ++u) {
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
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + 32);
  const int ntiles = NTI * NC;
  const int lane_ = threadIdx.x & 31;
  { const int lane = lane_; TCLK(0, t0); }

  if (warp == kEpiWarps) {
    // ---------------- MMA issuer (one elected thread) + norm producer (all 32 lanes):
    // before tile t's MMA the warp stages the tile's 8 x 16 candidate norms into ring slot t & 1
    // (16-byte loads from the L2-resident norm map) and arrives on bar_nc[slot].
    int32_t* ncring = reinterpret_cast<int32_t*>(smem + a.off_N);  // [2][8][16]
    for (int t = 0; t < ntiles; ++t) {
      const int ot = order[t];
      const int tr = ot / NC, tc = ot - tr * NC;
      const int buf = t & 1;
      if (t >= 2) sm100::mbar_wait(bar_empty + 8 * buf, uint32_t(((t >> 1) - 1) & 1));
      {
        const int rr = lane >> 2, cq = lane & 3;
        const int cy = min(cyA + kTR * tr + rr, H - b);
        const int4 v = __ldg(reinterpret_cast<const int4*>(nsrc + size_t(cy) * a.Mx + X0 + kTC * tc) + cq);
        reinterpret_cast<int4*>(ncring + (buf * kTR + rr) * kTC)[cq] = v;
        sm100::mbar_arrive(bar_nc + 8 * buf);
      }
      if (lane == 0) {
        TCLK(5, t0);
        sm100::tc_fence_after();
        if (a.dbg & 2) {
          sm100::mbar_arrive(bar_full + 8 * buf);
        } else {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const uint64_t ad = sm100::smem_desc(sA + 256u * j, 128u, 512u);
            const uint64_t bd =
                sm100::smem_desc(sE + uint32_t(kTR * tr + 4 * j) * RP + uint32_t(tc) * 128u, RP, RP);
            sm100::mma_i8(tmem + 128u * buf, ad, bd, kIdesc, j);
          }
          sm100::mma_commit(bar_full + 8 * buf);
        }
      }
      __syncwarp();
    }
    __syncwarp();
  } else {
    // ---------------- epilogue warps: e = warp; lane quarter q = e % 4 (TMEM lanes 32q..32q+31
    // = references 32q..32q+31, a 4 x 8 sub-block); half hh = e / 4 takes tile rows 4hh..4hh+3.
    // Each lane keeps the best 16 keys of ITS reference over ITS half in registers (branch-free
    // insertion network, no memory latency, no divergence). The filter threshold is
    // min(own 16th, partner's published 16th): each list holds KP keys of the reference, so the
    // KP-th best of their union is <= either (a valid upper bound).
    const int q = warp & 3, hh = warp >> 2;
    const int wy = q >> 1, wx = q & 1;
    const int iy = iy_first + 4 * wy + (lane >> 3), ix = ix_first + 8 * wx + (lane & 7);
    const bool valid = iy <= iy_last && ix <= ix_last;
    const int ry = iy * s, rx = ix * s;
    const int wiy0 = iy_first + 4 * wy, wiy1 = min(iy_last, wiy0 + 3);
    const int wix0 = ix_first + 8 * wx, wix1 = min(ix_last, wix0 + 7);
    const bool wvalid = wiy0 <= iy_last && wix0 <= ix_last;
    const int wy_lo = wiy0 * s + a.lo, wy_hi = wiy1 * s + a.hi;  // candidate rows of this warp
    const int wx_lo = wix0 * s + a.lo, wx_hi = wix1 * s + a.hi;
    const int ref_local = q * 32 + lane;
    uint32_t* pub = reinterpret_cast<uint32_t*>(smem + a.off_q);  // [2][128] published K-th keys
    RegTopK32<16> rt;
    rt.init();
    const Key32 key32{a.rb, a.dsat};
    const int kp1 = a.KP - 1;
    const int32_t nr = valid ? __ldg(nsrc + size_t(ry) * a.Mx + rx) : 0;  // ||X_i||^2 (centred)
    uint32_t other = 0xffffffffu;
    int32_t thr = 0x7fffffff;  // d' threshold (d' = d - ||X_i||^2)
    const uint32_t tq = tmem + (uint32_t(32 * q) << 16);
    uint32_t* scratch = reinterpret_cast<uint32_t*>(smem + a.off_q + kEpiWarps * 64 * 12) + warp * 32 * 16;

    for (int t = 0; t < ntiles; ++t) {
      const int ot = order[t];
      const int tr = ot / NC, tc = ot - tr * NC;
      const int buf = t & 1;
      TCLK(2, t0);
      sm100::mbar_wait(bar_full + 8 * buf, uint32_t((t >> 1) & 1));
      sm100::mbar_wait(bar_nc + 8 * buf, uint32_t((t >> 1) & 1));
      sm100::tc_fence_after();
      TCLK(1, t0);
      const int cx0 = X0 + kTC * tc;
      const int4* ncr = reinterpret_cast<const int4*>(smem + a.off_N) + buf * kTR * 4;
      const bool xrel = !(a.dbg & 1) && wvalid && cx0 <= wx_hi && cx0 + kTC - 1 >= wx_lo;
      if (xrel) {
        // exchange thresholds with the partner half once per tile (stale reads are conservative)
        const uint32_t mine = rt.at(kp1);
        pub[hh * 128 + ref_local] = mine;
        other = pub[(1 - hh) * 128 + ref_local];
        thr = key32.thr(min(mine, other)) - nr;
#pragma unroll 1
        for (int i2 = 4 * hh; i2 < 4 * hh + 4; i2 += 2) {
          const int cyp = cyA + kTR * tr + i2;
          const bool r0 = !(cyp < wy_lo || cyp > wy_hi || cyp > cyB);
          const bool r1 = !(cyp + 1 < wy_lo || cyp + 1 > wy_hi || cyp + 1 > cyB);
          if (!r0 && !r1) continue;  // warp-uniform
          uint32_t c2[32];
          sm100::tmem_ld32(tq + 128u * buf + 16u * i2, c2);
          int4 nq[8];
#pragma unroll
          for (int v = 0; v < 8; ++v) nq[v] = ncr[i2 * 4 + v];
          sm100::tmem_wait_ld();
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (!(h ? r1 : r0)) continue;
            const int cy = cyp + h;
            if ((a.dbg & 4) && lane == 0) atomicAdd(&g_tc_stats[0], 1ull);
            int dp[16];
            unsigned bits = 0;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const int4 x = nq[4 * h + v];
              dp[4 * v + 0] = x.x - 2 * int(c2[16 * h + 4 * v + 0]);
              dp[4 * v + 1] = x.y - 2 * int(c2[16 * h + 4 * v + 1]);
              dp[4 * v + 2] = x.z - 2 * int(c2[16 * h + 4 * v + 2]);
              dp[4 * v + 3] = x.w - 2 * int(c2[16 * h + 4 * v + 3]);
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) bits |= (dp[j] <= thr ? 1u : 0u) << j;
            // window of this lane's reference (rows and columns)
            const bool yok = valid && cy - ry >= a.lo && cy - ry <= a.hi;
            const int jlo = max(0, rx + a.lo - cx0), jhi = min(15, min(rx + a.hi, W - b) - cx0);
            const unsigned cols = (yok && jhi >= jlo) ? (((2u << jhi) - 1u) & ~((1u << jlo) - 1u)) : 0u;
            bits &= cols;
            if (a.dbg & 4) {
              const int tot = __reduce_add_sync(0xffffffffu, __popc(bits));
              if (lane == 0) { atomicAdd(&g_tc_stats[1], tot ? 1ull : 0ull); atomicAdd(&g_tc_stats[2], (unsigned long long)tot); }
            }
            TCLK(2, t0);
            if (__any_sync(0xffffffffu, bits != 0)) {
              // slow path: stage the 16 distances, then insert one survivor per lane per round
              // into the 32-bit register list
              uint32_t* sc = scratch + lane;
#pragma unroll
              for (int j = 0; j < 16; ++j) sc[32 * j] = uint32_t(dp[j] + nr);
              const int rel0 = (cy - ry - a.lo) * a.Wn + (cx0 - rx - a.lo);
              while (__any_sync(0xffffffffu, bits != 0)) {
                const int j = bits ? __ffs(bits) - 1 : 0;
                const uint32_t x = bits ? key32.make(int(sc[32 * j]), rel0 + j) : 0xffffffffu;
                bits &= bits - 1;
                rt.insert(x);
              }
              thr = key32.thr(min(rt.at(kp1), other)) - nr;
              __syncwarp();
              TCLK(3, t0);
            }
          }
        }
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(bar_empty + 8 * buf);
    }
    TCLK(2, t0);
    // merge the partner half's list into half 0's, then output (or flag for the exact fix-up)
    uint32_t* lists = reinterpret_cast<uint32_t*>(heaps);  // [128][17] half-1 lists
    if (hh == 1) {
#pragma unroll
      for (int i = 0; i < 16; ++i) lists[ref_local * 17 + i] = rt.r[i];
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32));
    if (hh == 0) {
      for (int i = 0; i < 16; ++i) rt.insert(lists[ref_local * 17 + i]);
      if (valid) {
        const size_t band_refs = size_t(a.iy_end - a.iy_begin) * a.nx;
        const size_t ref_band = size_t(iy - a.iy_begin) * a.nx + ix;
        if (!key32.exact(rt.at(kp1))) {
          const int pos = atomicAdd(a.fix_count, 1);
          a.fix_list[pos] = int(size_t(f) * band_refs + ref_band);
        } else {
          const size_t o = (size_t(f) * band_refs + ref_band) * a.K;
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            if (k < a.K) {
              const uint32_t kk = rt.r[k];
              const int rel = key32.rel(kk);
              const int dyy = rel / a.Wn, dxx = rel - dyy * a.Wn;
              a.idx_out[o + k] = (ry + dyy + a.lo) * W + rx + dxx + a.lo;
              a.dist_out[o + k] = key32.dist(kk);
            }
          }
        }
      }
    }
  }
  { const int lane = lane_; if (warp < kEpiWarps) TCLK(4, t0); }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == kEpiWarps) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem, 256);
  }
}

struct TcLayout {
  int NCmax, NTImax, heap_pitch;
  uint32_t off_A, off_E, off_N, off_heap, off_q, bytes;
};

TcLayout tc_layout(const Geometry& g) {
  TcLayout L{};
  const int span_x = (kRBX - 1) * g.s + g.Wn;  // candidate columns of a full block
  const int span_y = (kRBY - 1) * g.s + g.Wn;
  L.NCmax = (span_x + 15) / kTC + 1;
  L.NTImax = (span_y + kTR - 1) / kTR;
  L.heap_pitch = 17;  // 16 register-list keys per reference, odd pitch
  uint32_t off = 1024;  // barriers + TMEM slot
  L.off_A = off;
  off += 128 * 64;
  L.off_E = off;
  off += uint32_t(L.NTImax * kTR + 7) * L.NCmax * 128;
  L.off_N = off;  // 2-slot ring of the current tiles' candidate norms [2][8][16] int32
  off += 2 * kTR * kTC * 4;
  L.off_heap = off;
  off += uint32_t(128 * L.heap_pitch) * 4;  // half-1 32-bit lists for the final merge
  off = (off + 15) & ~15u;
  L.off_q = off;
  off += kEpiWarps * 64 * (8 + 4);
  off += kEpiWarps * 32 * 16 * 4;  // per-warp slow-path scratch (16 ordered distances per lane)
  L.bytes = off;
  return L;
}

}  // namespace

bool tc_supported(const Geometry& g) {
  if (g.dtype != SC_DTYPE_U8 || g.b != 8 || g.C != 1 || g.KP > 16 || g.Wn > 45) return false;
  return tc_layout(g).bytes <= 227 * 1024;
}

cudaError_t launch_bm_tc(const sc_bm_plan_s& p, const void* imgs, int F, int iy_begin, int iy_end,
                         int32_t* idx_out, void* dist_out, cudaStream_t st, int64_t* launches) {
  const Geometry& g = p.g;
  const TcLayout L = tc_layout(g);
  TcArgs a{};
  a.imgs = static_cast<const uint8_t*>(imgs);
  a.norm = static_cast<const int32_t*>(p.ws.norm);
  a.idx_out = idx_out;
  a.dist_out = static_cast<int32_t*>(dist_out);
  a.H = g.H; a.W = g.W; a.s = g.s; a.Wn = g.Wn; a.K = g.K; a.KP = g.KP;
  a.lo = g.lo; a.hi = g.hi; a.nx = g.nx; a.My = g.My; a.Mx = g.Mxp;  // Mx = norm-map row pitch
  a.nfs = g.NFS;
  a.iy_begin = iy_begin; a.iy_end = iy_end;
  a.tiles_x = (g.nx + kRBX - 1) / kRBX;
  a.NCmax = L.NCmax; a.NTImax = L.NTImax;
  a.off_A = L.off_A; a.off_E = L.off_E; a.off_N = L.off_N; a.off_heap = L.off_heap; a.off_q = L.off_q;
  a.heap_pitch = L.heap_pitch;
  a.rb = key32_rel_bits(g.Wn);
  a.dsat = uint32_t((uint64_t(1) << (32 - a.rb)) - 1);
  a.fix_count = p.ws.fix_count;
  a.fix_list = p.ws.fix_list;
  {
    const char* e = getenv("SCBM_TC_DEBUG");
    a.dbg = e ? atoi(e) : 0;
  }
  const int tiles_y = (iy_end - iy_begin + kRBY - 1) / kRBY;
  cudaFuncSetAttribute(bm_tc_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.bytes));
  cudaError_t e0 = cudaMemsetAsync(a.fix_count, 0, sizeof(int), st);
  if (e0 != cudaSuccess) return e0;
  bm_tc_i8_kernel<<<dim3(a.tiles_x * tiles_y, F), kThreads, L.bytes, st>>>(a);
  if (a.dbg & 12) {
    unsigned long long h[8];
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(h, g_tc_stats, sizeof(h));
    unsigned long long c[8];
    cudaMemcpyFromSymbol(c, g_tc_clk, sizeof(c));
    fprintf(stderr, "tc clk (warp-cycles): staging %llu wait_full %llu fast %llu slow %llu tail %llu mma_wait_empty %llu\n",
            c[0], c[1], c[2], c[3], c[4], c[5]);
    fprintf(stderr, "tc stats: rows %llu rows_with_surv %llu survivors %llu warmup_survivors %llu\n", h[0], h[1],
            h[2], h[3]);
  }
  if (launches) *launches += 2;
  cudaError_t e1 = cudaGetLastError();
  if (e1 != cudaSuccess) return e1;
  return launch_fixup(p, imgs, F, iy_begin, iy_end, idx_out, dist_out, st);
}

}  // namespace scbm
