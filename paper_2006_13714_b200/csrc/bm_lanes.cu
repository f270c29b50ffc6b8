// bm_lanes.cu -- the CUDA-core matcher with LANES = REFERENCES (default SIMT kernel).
//
// Steps a0, a2, a3, a4 (+ a5 for f32), a6 fused (see bm_simt.cu for the step definitions;
// this kernel differs in how work maps to lanes):
//
//   * a warp owns 32 consecutive references of one reference-grid row; all 32 lanes visit the
//     same window offset (dy, dx) at the same time, so no lane idles on window remainders
//     (only references clipped at the image border mask offsets);
//   * each lane keeps its own reference patch in registers and slides over VY vertically
//     adjacent candidates (dy0..dy0+VY-1, dx), reusing every loaded image row for up to VY
//     patch rows (u8: dp4a on packed int8 from four byte-shifted copies; f32: FMA);
//   * offsets are visited centre-out (dy blocks and dx ordered by distance from 0), so good
//     matches arrive early and the top-K threshold tightens fast (fewer survivors);
//   * survivors go through the per-warp queue of refq.cuh into per-reference shared lists.
//
// Arithmetic is identical to bm_simt.cu: u8 exact int32, f32 fp32 FMA + fp32 re-score.
#include "sc_internal.h"
#include "refq.cuh"
#include "regtopk.cuh"
#include "topk.cuh"

namespace scbm {
namespace {

struct LanesArgs {
  const void* imgs;   // [F][C][H][W]
  const void* norm;   // [F][My][Mx]
  int32_t* idx_out;   // [F][band refs][K]
  void* dist_out;
  void* dense;        // debug [refs][Wn*Wn] or nullptr
  int H, W, C, b, s, Wn, K, KP, lo, hi, nx, My, Mx;
  long long nfs;      // norm-map frame stride
  int iy_begin, iy_end;
  int NWY, tiles_x;   // warps (reference rows) per CTA; CTAs across x (32 refs each)
  int RWp, RHp;       // image region pitch (elements) and padded height
  int WP, PL;         // u8: words per copy row, words per copy plane
  int NP, NPs, NQ, NHp;  // norm tile: phase planes (x mod NP, NP = 1 << NPs), words per plane row, height
  int PADT;           // zero rows above both tiles
  int img_words, norm_words, list_pitch;
  int rb;             // R32 path: window-relative index bits of the 32-bit keys
  uint32_t dsat;      // R32 path: distance saturation value
  int* fix_count;     // R32 path: references needing the exact fix-up (count + list)
  int* fix_list;
};

template <typename In> struct LPath;

template <> struct LPath<float> {
  using T = float;
  template <int BK> struct Ref { float r[BK][BK]; };
  template <int BK>
  __device__ static void load_ref(Ref<BK>& R, const uint32_t* tile, const LanesArgs& a, int c, int y, int x) {
    const float* t = reinterpret_cast<const float*>(tile) + size_t(c) * a.RHp * a.RWp + y * a.RWp + x;
#pragma unroll
    for (int l = 0; l < BK; ++l)
#pragma unroll
      for (int m = 0; m < BK; ++m) R.r[l][m] = (l < a.b && m < a.b) ? t[l * a.RWp + m] : 0.f;
  }
  template <int BK, int VY>
  __device__ static void cross(float (&acc)[VY], const Ref<BK>& R, const uint32_t* tile, const LanesArgs& a,
                               int c, int y0, int x0) {
    const float* col = reinterpret_cast<const float*>(tile) + size_t(c) * a.RHp * a.RWp + y0 * a.RWp + x0;
#pragma unroll
    for (int t = 0; t < BK + VY - 1; ++t) {
      float xr[BK];
#pragma unroll
      for (int m = 0; m < BK; ++m) xr[m] = col[t * a.RWp + m];
#pragma unroll
      for (int i = 0; i < VY; ++i) {
        const int l = t - i;
        if (l >= 0 && l < BK) {
#pragma unroll
          for (int m = 0; m < BK; ++m) acc[i] = fmaf(R.r[l][m], xr[m], acc[i]);
        }
      }
    }
  }
  __device__ static uint32_t ord(float v) { return ord_f32(v); }
};

template <> struct LPath<uint8_t> {
  using T = int32_t;
  template <int BK> struct Ref { uint32_t r[BK][BK / 4]; };
  // One packed copy of the centred bytes (word w of a row = bytes 4w..4w+3); any 4-byte run
  // starting at byte x is funnelshift(word[x>>2], word[(x>>2)+1], 8*(x&3)).
  template <int BK>
  __device__ static void load_ref(Ref<BK>& R, const uint32_t* tile, const LanesArgs& a, int c, int y, int x) {
    const uint32_t* t = tile + size_t(c) * a.PL + y * a.WP + (x >> 2);
    const int sh = 8 * (x & 3);
#pragma unroll
    for (int l = 0; l < BK; ++l)
#pragma unroll
      for (int q = 0; q < BK / 4; ++q) {
        uint32_t w = l < a.b ? __funnelshift_r(t[l * a.WP + q], t[l * a.WP + q + 1], sh) : 0u;
        const int nb = a.b - 4 * q;
        if (nb < 4) w = nb <= 0 ? 0u : (w & ((1u << (8 * nb)) - 1u));
        R.r[l][q] = w;
      }
  }
  template <int BK, int VY>
  __device__ static void cross(int32_t (&acc)[VY], const Ref<BK>& R, const uint32_t* tile, const LanesArgs& a,
                               int c, int y0, int x0) {
    const uint32_t* col = tile + size_t(c) * a.PL + y0 * a.WP + (x0 >> 2);
    const int sh = 8 * (x0 & 3);
#pragma unroll
    for (int t = 0; t < BK + VY - 1; ++t) {
      uint32_t w[BK / 4 + 1], xw[BK / 4];
#pragma unroll
      for (int q = 0; q <= BK / 4; ++q) w[q] = col[t * a.WP + q];
#pragma unroll
      for (int q = 0; q < BK / 4; ++q) xw[q] = __funnelshift_r(w[q], w[q + 1], sh);
#pragma unroll
      for (int i = 0; i < VY; ++i) {
        const int l = t - i;
        if (l >= 0 && l < BK) {
#pragma unroll
          for (int q = 0; q < BK / 4; ++q) acc[i] = __dp4a(int(R.r[l][q]), int(xw[q]), acc[i]);
        }
      }
    }
  }
  __device__ static uint32_t ord(int32_t v) { return ord_i32(v); }
};

// Offset k of a centre-out enumeration of [lo, hi]: 0, 1, -1, 2, -2, ... (skips outside values).
__device__ __forceinline__ int centre_out(int k) { return (k & 1) ? ((k + 1) >> 1) : -(k >> 1); }

// KR == 0: shared heaps + survivor queue (refq.cuh); KR in {16, 32}: per-lane 32-bit register
// top-KR (regtopk.cuh, u8 only) with the exact fix-up for saturated / short references.
template <typename In, int BK, int VY, bool ONE_CH, int KR>
__global__ void __launch_bounds__(256, KR > 0 ? 3 : 1) bm_lanes_kernel(LanesArgs a) {
  using P = LPath<In>;
  using T = typename P::T;
  extern __shared__ __align__(16) uint32_t smem_u32[];
  const int f = blockIdx.y;
  const int ty = blockIdx.x / a.tiles_x, tx = blockIdx.x - ty * a.tiles_x;
  const int iy_first = a.iy_begin + ty * a.NWY;
  const int iy_last = min(a.iy_end, iy_first + a.NWY) - 1;
  const int ix_first = tx * 32;
  const int ix_last = min(a.nx, ix_first + 32) - 1;
  const int s = a.s, b = a.b;
  const int Y0 = max(0, iy_first * s + a.lo), Y1 = min(a.H - 1, iy_last * s + a.hi + b - 1);
  const int X0 = max(0, ix_first * s + a.lo), X1 = min(a.W - 1, ix_last * s + a.hi + b - 1);
  const int RH = Y1 - Y0 + 1, RW = X1 - X0 + 1;
  const int NY1 = min(a.H - b, iy_last * s + a.hi), NX1 = min(a.W - b, ix_last * s + a.hi);
  const int NH = NY1 - Y0 + 1, NW = NX1 - X0 + 1;

  uint32_t* tile = smem_u32;
  T* ntile = reinterpret_cast<T*>(smem_u32 + a.img_words);
  uint64_t* lists = reinterpret_cast<uint64_t*>(smem_u32 + a.img_words + a.norm_words);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  uint64_t* qkeys = lists + size_t(nwarps) * 32 * a.list_pitch;
  int32_t* qrefs = reinterpret_cast<int32_t*>(qkeys + nwarps * 64);

  // ---- a0: stage the centred image region and the norm tile
  const size_t plane_px = size_t(a.H) * a.W;
  const int PADT = a.PADT;  // zero rows above the region (blocks may start above the image)
  if constexpr (sizeof(In) == 1) {
    // packed centred bytes, 4 words (16 B) per thread-iteration: one 16-byte global load when the
    // row segment is 16-byte aligned and in range (c5: X0 = 128 tx - 16), else byte loads
    const uint8_t* img = static_cast<const uint8_t*>(a.imgs) + size_t(f) * a.C * plane_px;
    const int WQ = (a.WP + 3) >> 2;  // 16-byte groups per row
    const int total = a.C * a.RHp * WQ;
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      const int c = e / (a.RHp * WQ), r = e - c * (a.RHp * WQ);
      const int y2 = r / WQ, g4 = r - y2 * WQ;
      const int yy = y2 - PADT;
      uint32_t wv[4] = {0u, 0u, 0u, 0u};
      if (yy >= 0 && yy < RH) {
        const uint8_t* row = img + size_t(c) * plane_px + size_t(Y0 + yy) * a.W + X0;
        const int xb = 16 * g4;
        if (xb + 16 <= RW && (reinterpret_cast<uintptr_t>(row + xb) & 15) == 0) {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(row + xb));
          wv[0] = v.x ^ 0x80808080u; wv[1] = v.y ^ 0x80808080u; wv[2] = v.z ^ 0x80808080u; wv[3] = v.w ^ 0x80808080u;
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int e2 = 0; e2 < 4; ++e2) {
              const int xx = xb + 4 * q + e2;
              wv[q] |= (xx < RW ? uint32_t(row[xx] ^ 0x80u) : 0u) << (8 * e2);
            }
        }
      }
      uint32_t* dst = tile + size_t(c) * a.PL + y2 * a.WP + 4 * g4;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (4 * g4 + q < a.WP) dst[q] = wv[q];
    }
  } else {
    const float* img = static_cast<const float*>(a.imgs) + size_t(f) * a.C * plane_px;
    float* ft = reinterpret_cast<float*>(tile);
    for (int c = 0; c < a.C; ++c) {
      const float* src = img + size_t(c) * plane_px;
      float* dst = ft + size_t(c) * a.RHp * a.RWp;
      for (int y2 = warp; y2 < a.RHp; y2 += nwarps) {
        const int yy = y2 - PADT;
        for (int xx = lane; xx < a.RWp; xx += 32)
          dst[y2 * a.RWp + xx] =
              (yy >= 0 && yy < RH && xx < RW) ? src[size_t(Y0 + yy) * a.W + X0 + xx] - 0.5f : 0.f;
      }
    }
  }
  const T* nsrc_g = static_cast<const T*>(a.norm) + size_t(f) * a.nfs;  // a.Mx = norm-map row pitch
  if (KR == 0) {
    // norm tile in NP phase planes: element (y, x) at plane x % NP, word x / NP
    const T* nsrc = nsrc_g;
    const int per_plane = a.NHp * a.NQ;
    for (int e = threadIdx.x; e < a.NP * per_plane; e += blockDim.x) {
      const int ph = e / per_plane, r = e - ph * per_plane;
      const int y2 = r / a.NQ, q = r - y2 * a.NQ;
      const int yy = y2 - PADT;
      const int xx = (q << a.NPs) + ph;
      ntile[e] = (yy >= 0 && yy < NH && xx < NW) ? nsrc[size_t(Y0 + yy) * a.Mx + X0 + xx] : T(0);
    }
  }
  // lists: all +inf
  for (int e = threadIdx.x; e < nwarps * 32 * a.list_pitch; e += blockDim.x) lists[e] = kKeyInf;
  __syncthreads();

  const int iy = iy_first + warp;
  if (iy > iy_last) return;
  const int ix = ix_first + lane;
  const bool lane_ok = ix <= ix_last;
  const int ry = iy * s, rx = (lane_ok ? ix : ix_last) * s;
  const int cy0 = max(0, ry + a.lo), cy1 = min(a.H - b, ry + a.hi);  // warp-uniform
  const int cx0 = max(0, rx + a.lo), cx1 = min(a.W - b, rx + a.hi);  // per lane
  const int ref_local = warp * 32 + lane;
  RefHeaps hp{smem_addr(lists), a.list_pitch, a.KP, heap_depth(a.KP)};
  WarpQueue q{smem_addr(qkeys + warp * 64), smem_addr(qrefs + warp * 64)};
  const uint32_t myheap = hp.heap(ref_local);
  uint32_t thr = 0xffffffffu;  // hi32 of this reference's heap root (its current KP-th key)
  int qcnt = 0;
  const int ry_l = ry - Y0 + PADT, rx_l = rx - X0;  // tile coordinates (rows include PADT)
  const int nplane = a.NHp * a.NQ, npm = a.NP - 1;
  auto nidx = [&](int yl, int xl) { return (xl & npm) * nplane + yl * a.NQ + (xl >> a.NPs); };
  constexpr bool R32 = KR > 0;
  const T nr = R32 ? __ldg(nsrc_g + size_t(ry) * a.Mx + rx) : ntile[nidx(ry_l, rx_l)];
  RegTopK32<(KR > 0 ? KR : 1)> rt;
  const Key32 key32{a.rb, a.dsat};
  int thr_dp = 0;  // R32: largest d' that may still pass (d' = d - ||X_i||^2)
  if constexpr (R32) {
    rt.init();
    thr_dp = int(a.dsat) - int(nr);
  }
  uint32_t* r32scratch = reinterpret_cast<uint32_t*>(qkeys) + warp * 32 * 16;  // VY <= 16 values per lane

  typename P::template Ref<BK> R;
  if (ONE_CH) P::template load_ref<BK>(R, tile, a, 0, ry_l, rx_l);
  T* dense_row = nullptr;
  if (a.dense && lane_ok) {
    dense_row = static_cast<T*>(a.dense) + size_t((iy - a.iy_begin) * a.nx + ix) * a.Wn * a.Wn;
    for (int i = 0; i < a.Wn * a.Wn; ++i) dense_row[i] = T(-1);
  }

  const int nblk = (a.Wn + VY - 1) / VY;
  const int b0 = (0 - a.lo) / VY;  // block holding dy = 0
  const int span = max(-a.lo, a.hi);
  for (int kb = 0; kb < 2 * nblk; ++kb) {
    const int bb = b0 + centre_out(kb);
    if (bb < 0 || bb >= nblk) continue;
    const int dyb = a.lo + bb * VY;
    const int cyb = ry + dyb;
    if (cyb + VY - 1 < cy0 || cyb > cy1) continue;  // whole block clipped (warp-uniform)
    for (int kx = 0; kx <= 2 * span; ++kx) {
      const int dx = centre_out(kx);
      if (dx < a.lo || dx > a.hi) continue;
      const int cx = rx + dx;
      const bool xok = lane_ok && cx >= cx0 && cx <= cx1;
      if (!__any_sync(0xffffffffu, xok)) continue;
      const int cxl = min(max(cx, 0), a.W - b) - X0;  // clamp for safe addressing
      T acc[VY];
#pragma unroll
      for (int i = 0; i < VY; ++i) acc[i] = T(0);
      const int nch = ONE_CH ? 1 : a.C;
      for (int c = 0; c < nch; ++c) {
        if (!ONE_CH) P::template load_ref<BK>(R, tile, a, c, ry_l, rx_l);
        P::template cross<BK, VY>(acc, R, tile, a, c, cyb - Y0 + PADT, cxl);
      }
      const int ny_l = cyb - Y0 + PADT;  // tile row of candidate row 0 of this block
      if (a.dense) {
#pragma unroll
        for (int i = 0; i < VY; ++i) {
          const int cy = cyb + i;
          const T dp = ntile[nidx(ny_l + i, cxl)] - T(2) * acc[i];
          if (xok && cy >= cy0 && cy <= cy1) dense_row[(cy - ry - a.lo) * a.Wn + (cx - rx - a.lo)] = dp + nr;
        }
        continue;
      }
      // rows inside the (warp-uniform) vertical window, columns inside this lane's window
      const int i_lo = max(0, cy0 - cyb), i_hi = min(VY - 1, cy1 - cyb);
      const unsigned rows = (i_hi >= i_lo) ? (((2u << i_hi) - 1u) & ~((1u << i_lo) - 1u)) : 0u;
      if constexpr (R32) {
        // fast path: d' <= thr_dp into a bitmask; survivors inserted into the register list.
        // Candidate norms come straight from the L1/L2-resident norm map (no shared tile).
        const T* nbg = nsrc_g + size_t(min(max(cyb, 0), a.H - b)) * a.Mx + (cxl + X0);
        int dpv[VY];
        unsigned bits = 0;
#pragma unroll
        for (int i = 0; i < VY; ++i) {
          const int cyi = min(max(cyb + i, 0), a.H - b);
          dpv[i] = int(__ldg(nsrc_g + size_t(cyi) * a.Mx + (cxl + X0))) - 2 * int(acc[i]);
          bits |= (dpv[i] <= thr_dp ? 1u : 0u) << i;
        }
        bits &= xok ? rows : 0u;
        if (__any_sync(0xffffffffu, bits != 0)) {
          uint32_t* sc = r32scratch + lane;
#pragma unroll
          for (int i = 0; i < VY; ++i) sc[32 * i] = uint32_t(dpv[i] + int(nr));
          const int rel0 = (dyb - a.lo) * a.Wn + (dx - a.lo);
          while (__any_sync(0xffffffffu, bits != 0)) {
            const int i = bits ? __ffs(bits) - 1 : 0;
            const uint32_t x = bits ? key32.make(int(sc[32 * i]), rel0 + i * a.Wn) : 0xffffffffu;
            bits &= bits - 1;
            rt.insert(x);
          }
          thr_dp = key32.thr(rt.at(a.KP - 1)) - int(nr);
          __syncwarp();
        }
        continue;
      }
      const T* nb = ntile + nidx(ny_l, cxl);
      // fast path: one compare per candidate into a per-lane bitmask of passing rows
      uint32_t u[VY];
      unsigned bits = 0;
#pragma unroll
      for (int i = 0; i < VY; ++i) {
        u[i] = P::ord(nb[i * a.NQ] - T(2) * acc[i]);
        bits |= (u[i] <= thr ? 1u : 0u) << i;
      }
      bits &= xok ? rows : 0u;
      const unsigned any = __reduce_or_sync(0xffffffffu, bits);
      if (any) {
        bool refresh = false;
#pragma unroll
        for (int i = 0; i < VY; ++i) {
          if (!(any & (1u << i))) continue;  // warp-uniform
          const bool pb = (bits >> i) & 1u;
          const uint64_t key = (uint64_t(u[i]) << 32) | uint32_t((cyb + i) * a.W + cx);
          // warm-up: while its heap is not full (root = +inf) a lane pushes its own candidates
          // directly (all lanes in parallel, no queue); afterwards the warp queue.
          const bool fill = pb && thr == 0xffffffffu;
          if (fill) {
            heap_push_cold(myheap, a.KP, hp.depth, key);
            thr = hp.thr_hi(ref_local);
          }
          const bool pass = pb && !fill && u[i] <= thr;
          refresh |= queue_push(q, hp, qcnt, pass, key, ref_local, lane);
        }
        if (refresh) thr = hp.thr_hi(ref_local);
      }
    }
  }
  if constexpr (R32) {
    if (a.dense) return;
    // a6 from registers; references whose K-th key is saturated / unfilled go to the fix-up
    const size_t band_refs = size_t(a.iy_end - a.iy_begin) * a.nx;
    if (lane_ok) {
      const size_t ref_band = size_t(iy - a.iy_begin) * a.nx + ix;
      if (!key32.exact(rt.at(a.KP - 1))) {
        const int pos = atomicAdd(a.fix_count, 1);
        a.fix_list[pos] = int(size_t(f) * band_refs + ref_band);
      } else {
        const size_t o = (size_t(f) * band_refs + ref_band) * a.K;
        int32_t* dist = static_cast<int32_t*>(a.dist_out);
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          if (k < a.K) {
            const uint32_t kk = rt.r[k];
            const int rel = key32.rel(kk);
            const int dyy = rel / a.Wn, dxx = rel - dyy * a.Wn;
            a.idx_out[o + k] = (ry + dyy + a.lo) * a.W + rx + dxx + a.lo;
            dist[o + k] = key32.dist(kk);
          }
        }
      }
    }
    return;
  }
  if (a.dense) return;
  while (qcnt > 0) qcnt = queue_drain(q, hp, qcnt, lane);
  heap_sort(myheap, a.KP, hp.depth);  // each lane sorts its own reference's heap
  __syncwarp();

  // ---- a5/a6: outputs, one reference at a time across the warp (coalesced rows of K)
  const int n_ref_lanes = min(32, ix_last - ix_first + 1);
  const size_t band_refs = size_t(a.iy_end - a.iy_begin) * a.nx;
  if constexpr (sizeof(In) == 1) {
    int32_t* dist = static_cast<int32_t*>(a.dist_out);
    for (int r = 0; r < n_ref_lanes; ++r) {
      const T nr_r = __shfl_sync(0xffffffffu, nr, r);
      const uint64_t* L = lists + size_t(warp * 32 + r) * a.list_pitch;
      const size_t o = (size_t(f) * band_refs + size_t(iy - a.iy_begin) * a.nx + ix_first + r) * a.K;
      for (int k = lane; k < a.K; k += 32) {
        const uint64_t key = L[k];
        const bool none = key == kKeyInf;
        a.idx_out[o + k] = none ? -1 : int32_t(uint32_t(key));
        dist[o + k] = none ? 0x7fffffff : unord_i32(uint32_t(key >> 32)) + nr_r;
      }
    }
  } else {
    // a5: re-score the KP keys of each reference by direct differences, re-sort, keep K
    const float* img = static_cast<const float*>(a.imgs) + size_t(f) * a.C * plane_px;
    float* dist = static_cast<float*>(a.dist_out);
    for (int r = 0; r < n_ref_lanes; ++r) {
      const int rxr = (ix_first + r) * s;
      uint64_t* L = lists + size_t(warp * 32 + r) * a.list_pitch;
      const float nr_r = __shfl_sync(0xffffffffu, float(nr), r);
      const uint64_t kp_key = L[0];  // heap root: the KP-th identity key (kKeyInf: list not full)
      __syncwarp();
      for (int k = lane; k < a.KP; k += 32) {
        const uint64_t key = L[k];
        if (key == kKeyInf) continue;
        const uint32_t idx = uint32_t(key);
        const int cyk = int(idx) / a.W, cxk = int(idx) - cyk * a.W;
        float d = 0.f;
        for (int c = 0; c < a.C; ++c) {
          const float* pr = img + c * plane_px + size_t(ry) * a.W + rxr;
          const float* pc = img + c * plane_px + size_t(cyk) * a.W + cxk;
          for (int l = 0; l < b; ++l)
#pragma unroll 4
            for (int m = 0; m < b; ++m) {
              const float df = __ldg(pr + l * a.W + m) - __ldg(pc + l * a.W + m);
              d = fmaf(df, df, d);
            }
        }
        L[k] = (uint64_t(__float_as_uint(d)) << 32) | idx;
      }
      __syncwarp();
      // sort the KP re-scored keys: WarpTopK over ceil(KP/32) slots (one merge per slot)
      WarpTopK<5> t;
      t.init();
      for (int j = 0; j * 32 < a.KP; ++j) {
        const int k = j * 32 + lane;
        t.merge(k < a.KP ? L[k] : kKeyInf, lane);
      }
      const size_t o = (size_t(f) * band_refs + size_t(iy - a.iy_begin) * a.nx + ix_first + r) * a.K;
      {  // identity-rounding check (bm_simt.cu a5): a hidden top-K candidate -> exact fix-up
        uint64_t kk = kKeyInf;
#pragma unroll
        for (int j = 0; j < 5; ++j)
          if (j == (a.K - 1) / 32) kk = t.v[j];
        kk = __shfl_sync(0xffffffffu, kk, (a.K - 1) % 32);
        if (lane == 0 && kp_key != kKeyInf && kk != kKeyInf) {
          const float dK = __uint_as_float(uint32_t(kk >> 32));
          const float dKP = unord_f32(uint32_t(kp_key >> 32)) + nr_r;
          const float kappa = 2.f * float(b * b * a.C) * 5.96e-8f;
          if (dKP - kappa * (6.f * fmaxf(nr_r, 0.f) + 4.f * dK) <= dK * (1.f + 1e-5f)) {
            const int pos = atomicAdd(a.fix_count, 1);
            a.fix_list[pos] = int(o / a.K);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        const int k = j * 32 + lane;
        if (k < a.K) {
          const uint64_t key = t.v[j];
          const bool none = key == kKeyInf;
          a.idx_out[o + k] = none ? -1 : int32_t(uint32_t(key));
          dist[o + k] = none ? __int_as_float(0x7f800000) : __uint_as_float(uint32_t(key >> 32));
        }
      }
    }
  }
}

int bk_for(int b, bool u8) {
  if (u8) return b <= 4 ? 4 : b <= 8 ? 8 : 16;
  return b == 7 ? 7 : b <= 4 ? 4 : b <= 8 ? 8 : 16;
}

// VY: rows of candidates per lane step; configs pick a divisor of Wn where possible.
int vy_for(const Geometry& g) {
  const int bk = bk_for(g.b, g.dtype == SC_DTYPE_U8);
  if (bk == 16) return 4;
  if (bk == 8 && g.dtype == SC_DTYPE_U8) return g.Wn % 11 == 0 ? 11 : g.Wn % 7 == 0 ? 7 : 8;
  if (bk == 8 && g.dtype == SC_DTYPE_F32) return g.Wn % 13 == 0 ? 13 : (g.Wn + 1) % 7 == 0 ? 7 : 8;
  return 8;
}

}  // namespace
int lanes_r32_slots(const Geometry& g);
namespace {

// r32: the register top-K instantiation (no norm tile, no heaps); dense tables always use heaps' layout
size_t lanes_smem(const Geometry& g, int NWY, int VY, bool r32, LanesArgs* a) {
  const bool u8 = g.dtype == SC_DTYPE_U8;
  const int BK = bk_for(g.b, u8);
  const int pad = BK - g.b;
  a->PADT = VY - 1;
  a->RWp = 31 * g.s + g.Wn + g.b - 1 + pad;
  a->RHp = (NWY - 1) * g.s + g.Wn + g.b - 1 + pad + 2 * (VY - 1);
  if (u8) {
    a->WP = (a->RWp + 3) / 4 + 2;
    a->PL = a->RHp * a->WP;
    a->img_words = g.C * a->PL;
  } else {
    a->WP = a->PL = 0;
    a->img_words = g.C * a->RHp * a->RWp;
  }
  a->img_words = (a->img_words + 3) & ~3;
  a->NPs = (g.s % 8 == 0) ? 3 : (g.s % 4 == 0) ? 2 : (g.s % 2 == 0) ? 1 : 0;
  a->NP = 1 << a->NPs;
  const int NW = 31 * g.s + g.Wn;
  a->NQ = (NW + a->NP - 1) / a->NP + 1;
  a->NHp = (NWY - 1) * g.s + g.Wn + 2 * (VY - 1);
  a->norm_words = r32 ? 0 : ((a->NP * a->NHp * a->NQ + 3) & ~3);
  a->list_pitch = r32 ? 0 : (g.KP | 1);  // the register top-K path needs no heaps
  size_t bytes = size_t(a->img_words + a->norm_words) * 4;
  bytes += size_t(NWY) * 32 * a->list_pitch * 8;  // reference lists
  bytes += size_t(NWY) * 32 * 16 * 4;           // survivor queues (64 x 12 B) / R32 scratch (32 x 16 x 4 B)
  return bytes;
}

template <typename In, int BK, int VY, int KR>
cudaError_t launch_t(const LanesArgs& a, int F, size_t smem, cudaStream_t st) {
  const int tiles_y = (a.iy_end - a.iy_begin + a.NWY - 1) / a.NWY;
  dim3 grid(a.tiles_x * tiles_y, F);
  if (a.C == 1) {
    auto k = bm_lanes_kernel<In, BK, VY, true, KR>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    k<<<grid, 32 * a.NWY, smem, st>>>(a);
  } else {
    auto k = bm_lanes_kernel<In, BK, VY, false, KR>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    k<<<grid, 32 * a.NWY, smem, st>>>(a);
  }
  return cudaGetLastError();
}

template <typename In>
cudaError_t dispatch(const LanesArgs& a, int F, size_t smem, cudaStream_t st, int bk, int vy, int kr) {
  if constexpr (sizeof(In) == 1) {
    if (bk == 8 && kr == 16) {
      if (vy == 11) return launch_t<In, 8, 11, 16>(a, F, smem, st);
      if (vy == 7) return launch_t<In, 8, 7, 16>(a, F, smem, st);
      return launch_t<In, 8, 8, 16>(a, F, smem, st);
    }
    if (bk == 8 && kr == 32) {
      if (vy == 11) return launch_t<In, 8, 11, 32>(a, F, smem, st);
      return launch_t<In, 8, 8, 32>(a, F, smem, st);
    }
    if (bk == 8 && vy == 11) return launch_t<In, 8, 11, 0>(a, F, smem, st);
    if (bk == 8 && vy == 7) return launch_t<In, 8, 7, 0>(a, F, smem, st);
    if (bk == 8) return launch_t<In, 8, 8, 0>(a, F, smem, st);
    if (bk == 4) return launch_t<In, 4, 8, 0>(a, F, smem, st);
    return launch_t<In, 16, 4, 0>(a, F, smem, st);
  } else {
    if (bk == 8 && vy == 13) return launch_t<In, 8, 13, 0>(a, F, smem, st);
    if (bk == 8 && vy == 7) return launch_t<In, 8, 7, 0>(a, F, smem, st);
    if (bk == 8) return launch_t<In, 8, 8, 0>(a, F, smem, st);
    if (bk == 7) return launch_t<In, 7, 8, 0>(a, F, smem, st);
    if (bk == 4) return launch_t<In, 4, 8, 0>(a, F, smem, st);
    return launch_t<In, 16, 4, 0>(a, F, smem, st);
  }
}

}  // namespace

int lanes_warps_for(const Geometry& g, int sm_count, int n_images) {
  // 8 reference rows per CTA unless shared memory or the grid size says fewer
  for (int nwy : {8, 4, 2, 1}) {
    LanesArgs a{};
    const size_t sm = lanes_smem(g, nwy, vy_for(g), lanes_r32_slots(g) > 0, &a);
    const long long ctas = (long long)((g.ny + nwy - 1) / nwy) * ((g.nx + 31) / 32) * n_images;
    if (sm <= 110 * 1024 && ctas >= 4LL * sm_count) return nwy;
    if (nwy == 1) return 1;
  }
  return 1;
}

size_t lanes_smem_bytes(const Geometry& g, int nwy) {
  LanesArgs a{};
  return lanes_smem(g, nwy, vy_for(g), lanes_r32_slots(g) > 0, &a);
}

// Register 32-bit top-K eligibility (u8, exact patch side 8, K <= 32, Wn^2 <= 2^11 so that the
// distance field keeps >= 21 bits).
int lanes_r32_slots(const Geometry& g) {
  if (g.dtype != SC_DTYPE_U8 || g.b != 8 || g.KP > 32) return 0;
  if (key32_rel_bits(g.Wn) > 11) return 0;
  return g.KP <= 16 ? 16 : 32;
}

cudaError_t launch_bm_lanes(const sc_bm_plan_s& p, const void* imgs, int F, int iy_begin, int iy_end,
                            int32_t* idx_out, void* dist_out, void* dense, cudaStream_t st,
                            int64_t* launches) {
  const Geometry& g = p.g;
  LanesArgs a{};
  a.imgs = imgs;
  a.norm = p.ws.norm;
  a.idx_out = idx_out;
  a.dist_out = dist_out;
  a.dense = dense;
  a.H = g.H; a.W = g.W; a.C = g.C; a.b = g.b; a.s = g.s; a.Wn = g.Wn; a.K = g.K; a.KP = g.KP;
  a.lo = g.lo; a.hi = g.hi; a.nx = g.nx; a.My = g.My; a.Mx = g.Mxp;  // Mx = norm-map row pitch
  a.nfs = g.NFS;
  a.iy_begin = iy_begin; a.iy_end = iy_end;
  a.NWY = p.lanes_nwy;
  a.tiles_x = (g.nx + 31) / 32;
  const int vy = vy_for(g);
  const int kr = dense ? 0 : lanes_r32_slots(g);  // dense tables: the heap instantiation's layout
  const size_t smem = lanes_smem(g, a.NWY, vy, kr > 0, &a);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  a.rb = key32_rel_bits(g.Wn);
  a.dsat = (a.rb >= 32) ? 0u : uint32_t((uint64_t(1) << (32 - a.rb)) - 1);
  a.fix_count = p.ws.fix_count;
  a.fix_list = p.ws.fix_list;
  if (launches) *launches += 1;
  const int bk = bk_for(g.b, g.dtype == SC_DTYPE_U8);
  cudaError_t e;
  // fix-up: u8 register keys (saturation), float top-K (identity rounding, see bm_simt.cu a5)
  const bool fix = kr > 0 || (g.dtype == SC_DTYPE_F32 && dense == nullptr);
  if (fix) {
    e = cudaMemsetAsync(p.ws.fix_count, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
  }
  if (g.dtype == SC_DTYPE_U8) e = dispatch<uint8_t>(a, F, smem, st, bk, vy, kr);
  else e = dispatch<float>(a, F, smem, st, bk, vy, kr);
  if (e != cudaSuccess || !fix) return e;
  if (launches) *launches += 1;
  return launch_fixup(p, imgs, F, iy_begin, iy_end, idx_out, dist_out, st);
}

}  // namespace scbm
