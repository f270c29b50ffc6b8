// bm_simt.cu -- steps a0, a2, a3, a4 (+ a5 for f32), a6 fused in one CUDA-core kernel.
//
//   a0 staging   one CTA owns a TRY x TRX tile of references; it stages the image region
//                covering the union of their clipped windows plus the patch extent (the
//                "window halo"), centred, in shared memory, and the matching tile of the norm
//                map. u8: x' = x ^ 0x80 (= x - 128 as int8) stored as FOUR byte-shifted copies of
//                packed int8 words so any 4-byte run of a row is one aligned 32-bit load
//                (copies interleaved 8 banks apart: conflict-free across a warp); f32: x - 0.5.
//   a2 cross     C_i(j) = <X'_i, X'_j> (Self-Convolution, Eq. 5; channels
//                summed, Eq. 12): one warp per reference, the reference patch in registers;
//                each lane slides over VY vertically adjacent candidates of one column, so every
//                image row it loads feeds up to VY patch rows. u8 uses dp4a (4 int8 MACs per
//                instruction, exact int32); f32 uses fp32 FMA.
//   a3 assembly  d' = n_c - 2 C (Lemma 2, ||X_i||^2 deferred: constant per
//                reference; Theorem 1's b_i = -d'/2).
//   a4 top-K     32-bit threshold filter (ord(d') <= ord of the KP-th key: a superset, exact
//                ties resolved in the merge) + register-resident warp merges (topk.cuh).
//   a5 re-score  f32 only: the best KP = K+8 keys are re-scored by direct differences
//                sum (x_r - x_c)^2 in fp32 from the uncentred input and re-sorted.
//   a6 output    coalesced stores of K idx + K dist per reference; u8 dist = d' + n_r exact.
#include "nlm.cuh"
#include "sc_internal.h"
#include "topk.cuh"

namespace scbm {
namespace {

constexpr int kWarpKeys = 32 + 32 * 5;  // per-warp shared keys: survivor buffer + list

struct SimtArgs {
  const void* imgs;   // [F][C][H][W]
  const void* norm;   // [F][My][Mx] int32 / float (centred norm map)
  int32_t* idx_out;   // [F][band refs][K]
  void* dist_out;     // [F][band refs][K]
  void* dense;        // dense tables: [refs][Wn*Wn] (one image) or nullptr
  float nlm_inv_h2;   // > 0: normalise each dense row into NLM weights in the epilogue (nlm.cuh)
  float* avg_out;     // NL-means estimate [band refs][C][b][b] (AVG instantiation), 1 / h^2 in nlm_inv_h2
  int* fix_count;     // float L2: references whose identity rounding could hide a top-K candidate
  int* fix_list;      // (exact fix-up, fixup.cu); nullptr: no check
  int H, W, C, b, s, Wn, K, KP, lo, hi, nx, My, Mx;
  long long nfs;      // norm-map frame stride
  int iy_begin, iy_end;
  int TRY, TRX, tiles_x;
  int RWp, RHp;       // logical image-region pitch (elements) / padded height
  int WP, PL;         // u8: words per row of one shifted copy, words per copy plane
  int NWp, NHp;       // norm-tile pitch / padded height
  int img_words;      // shared words of the image tile
};

template <typename In> struct Path;

// -------- f32: fp32 FMA on centred floats
template <> struct Path<float> {
  using T = float;     // norm / accumulator type
  template <int BK> struct Ref { float r[BK][BK]; };
  template <int BK>
  __device__ static void load_ref(Ref<BK>& R, const uint32_t* tile, const SimtArgs& a, int c, int ry0, int rx0) {
    const float* t = reinterpret_cast<const float*>(tile) + size_t(c) * a.RHp * a.RWp + ry0 * a.RWp + rx0;
#pragma unroll
    for (int l = 0; l < BK; ++l)
#pragma unroll
      for (int m = 0; m < BK; ++m) R.r[l][m] = (l < a.b && m < a.b) ? t[l * a.RWp + m] : 0.f;
  }
  template <int BK, int VY>
  __device__ static void cross(float (&acc)[VY], const Ref<BK>& R, const uint32_t* tile, const SimtArgs& a,
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

// -------- u8: dp4a on packed centred int8 (x ^ 0x80), four byte-shifted copies
template <> struct Path<uint8_t> {
  using T = int32_t;
  template <int BK> struct Ref { uint32_t r[BK][BK / 4]; };
  __device__ static const uint32_t* plane(const uint32_t* tile, const SimtArgs& a, int c, int k) {
    return tile + size_t(c * 4 + k) * a.PL;
  }
  template <int BK>
  __device__ static void load_ref(Ref<BK>& R, const uint32_t* tile, const SimtArgs& a, int c, int ry0, int rx0) {
    const uint32_t* t = plane(tile, a, c, rx0 & 3) + ry0 * a.WP + (rx0 >> 2);
#pragma unroll
    for (int l = 0; l < BK; ++l)
#pragma unroll
      for (int q = 0; q < BK / 4; ++q) {
        uint32_t w = l < a.b ? t[l * a.WP + q] : 0u;
        const int nb = a.b - 4 * q;  // valid bytes in this word
        if (nb < 4) w = nb <= 0 ? 0u : (w & ((1u << (8 * nb)) - 1u));
        R.r[l][q] = w;
      }
  }
  template <int BK, int VY>
  __device__ static void cross(int32_t (&acc)[VY], const Ref<BK>& R, const uint32_t* tile, const SimtArgs& a,
                               int c, int y0, int x0) {
    const uint32_t* col = plane(tile, a, c, x0 & 3) + y0 * a.WP + (x0 >> 2);
#pragma unroll
    for (int t = 0; t < BK + VY - 1; ++t) {
      uint32_t xw[BK / 4];
#pragma unroll
      for (int q = 0; q < BK / 4; ++q) xw[q] = col[t * a.WP + q];
#pragma unroll
      for (int i = 0; i < VY; ++i) {
        const int l = t - i;
        if (l >= 0 && l < BK) {
#pragma unroll
          for (int q = 0; q < BK / 4; ++q)
            acc[i] = __dp4a(int(R.r[l][q]), int(xw[q]), acc[i]);
        }
      }
    }
  }
  __device__ static uint32_t ord(int32_t v) { return ord_i32(v); }
};

// AVG (NL-means, sc_bm_nlm_average): patch elements per lane, ceil(b^2 C / 32) rounded up to
// 2, 4 or 8 (b^2 C <= 256); 0 = block matching / dense tables
template <typename In, int BK, int VY, int NJ, bool ONE_CH, int AVG>
__device__ __forceinline__ void process_ref(const SimtArgs& a, int f, int ref_band, int iy, int ix,
                                            const uint32_t* __restrict__ tile,
                                            const typename Path<In>::T* __restrict__ ntile,
                                            uint64_t* __restrict__ buf, int Y0, int X0, int lane) {
  using P = Path<In>;
  using T = typename P::T;
  const int s = a.s, b = a.b;
  const int ry = iy * s, rx = ix * s;
  const int cy0 = max(0, ry + a.lo), cy1 = min(a.H - b, ry + a.hi);
  const int cx0 = max(0, rx + a.lo), cx1 = min(a.W - b, rx + a.hi);
  const int ncols = cx1 - cx0 + 1, nrows = cy1 - cy0 + 1;
  const int nby = (nrows + VY - 1) / VY;
  const int nitems = nby * ncols;
  const T nr = ntile[(ry - Y0) * a.NWp + (rx - X0)];

  uint64_t* lst = buf + 32;  // 32*NJ sorted keys (shared)
  for (int j = lane; j < 32 * NJ; j += 32) lst[j] = kKeyInf;
  __syncwarp();
  uint32_t thr = 0xffffffffu;  // ord(d') of the KP-th key (inclusive superset filter)
  int cnt = 0;

  typename P::template Ref<BK> R;
  if (ONE_CH) P::template load_ref<BK>(R, tile, a, 0, ry - Y0, rx - X0);

  T* dense_row = nullptr;
  if (a.dense) {
    dense_row = static_cast<T*>(a.dense) + size_t(ref_band) * a.Wn * a.Wn;
    for (int i = lane; i < a.Wn * a.Wn; i += 32) dense_row[i] = T(-1);
    __syncwarp();
  }
  // NL-means estimate (AVG, PAPER.md:252 after Eq. 2): X_i ~ sum_j s_i(j) X_j over the clipped
  // window, fused -- no weight table. Streaming softmax over the candidate blocks: running minimum
  // distance m (weights exp(-(d - m)/h^2) <= 1, rescaled when m drops), lane-partial Theta, and
  // the weighted sum of the raw candidate patches with lanes over the b^2 C patch elements.
  // The candidate pixels come from the CTA's staged (centred) tile; the centring constant is added
  // back after the normalisation (sum_j s_i(j) (x'_j + c) = sum_j s_i(j) x'_j + c).
  constexpr int EPL = AVG > 0 ? AVG : 1;
  float avg_acc[EPL];
  int avg_c[EPL], avg_l[EPL], avg_m[EPL];  // element -> (channel, row, column); channel -1: none
  float m_run = __int_as_float(0x7f800000), theta = 0.f;
  if constexpr (AVG > 0) {
    const int bb2 = b * b;
#pragma unroll
    for (int k = 0; k < EPL; ++k) {
      const int e = lane + 32 * k;
      const int c = e / bb2, l = (e - c * bb2) / b, m = e - c * bb2 - l * b;
      const bool in = e < bb2 * a.C;
      avg_c[k] = in ? c : 0;  // out-of-patch elements read a valid pixel and are never stored
      avg_l[k] = in ? l : 0;
      avg_m[k] = in ? m : 0;
      avg_acc[k] = 0.f;
    }
  }

  for (int base = 0; base < nitems; base += 32) {
    const int item = base + lane;
    const bool ivalid = item < nitems;
    const int it = ivalid ? item : nitems - 1;
    const int by = it / ncols;
    const int cy = cy0 + by * VY, cx = cx0 + (it - by * ncols);
    T acc[VY];
#pragma unroll
    for (int i = 0; i < VY; ++i) acc[i] = T(0);
    const int nch = ONE_CH ? 1 : a.C;
    for (int c = 0; c < nch; ++c) {
      if (!ONE_CH) P::template load_ref<BK>(R, tile, a, c, ry - Y0, rx - X0);
      P::template cross<BK, VY>(acc, R, tile, a, c, cy - Y0, cx - X0);
    }
    if constexpr (AVG > 0) {
      float dv[VY], wv[VY];
      float bmin = __int_as_float(0x7f800000);
#pragma unroll
      for (int i = 0; i < VY; ++i) {
        const int cyi = cy + i;
        const bool ok = ivalid && cyi <= cy1;
        const T nc = ntile[(cyi - Y0) * a.NWp + (cx - X0)];
        dv[i] = ok ? fmaxf(float(nc - T(2) * acc[i] + nr), 0.f) : __int_as_float(0x7f800000);
        bmin = fminf(bmin, dv[i]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) bmin = fminf(bmin, __shfl_xor_sync(0xffffffffu, bmin, o));
      if (bmin < m_run) {  // warp-uniform: rescale what was accumulated against the old minimum
        const float sc = expf(-(m_run - bmin) * a.nlm_inv_h2);
        theta *= sc;
#pragma unroll
        for (int k = 0; k < EPL; ++k) avg_acc[k] *= sc;
        m_run = bmin;
      }
      unsigned any = 0u;
#pragma unroll
      for (int i = 0; i < VY; ++i) {
        wv[i] = dv[i] < __int_as_float(0x7f800000) ? expf(-(dv[i] - m_run) * a.nlm_inv_h2) : 0.f;
        theta += wv[i];
        any |= (wv[i] > 0.f ? 1u : 0u) << i;
      }
      // every lane's candidates in turn: broadcast weights and position, lanes over patch elements
      // (zero weights of clipped rows multiply finite staged pixels: no branch, loads batched)
      for (unsigned lanes = __ballot_sync(0xffffffffu, any != 0u); lanes; lanes &= lanes - 1) {
        const int L = __ffs(lanes) - 1;
        const int yL = __shfl_sync(0xffffffffu, cy, L) - Y0, xL = __shfl_sync(0xffffffffu, cx, L) - X0;
        float wj[VY];
#pragma unroll
        for (int i = 0; i < VY; ++i) wj[i] = __shfl_sync(0xffffffffu, wv[i], L);
#pragma unroll
        for (int k = 0; k < EPL; ++k) {
          const int y = yL + avg_l[k], x = xL + avg_m[k];
          if constexpr (sizeof(In) == 1) {  // packed centred bytes: copy x & 3, byte 0 of word x >> 2
            const uint32_t* col = P::plane(tile, a, avg_c[k], x & 3) + y * a.WP + (x >> 2);
#pragma unroll
            for (int i = 0; i < VY; ++i)
              avg_acc[k] = fmaf(wj[i], float(int8_t(col[i * a.WP] & 0xffu)), avg_acc[k]);
          } else {
            const float* col = reinterpret_cast<const float*>(tile) + (size_t(avg_c[k]) * a.RHp + y) * a.RWp + x;
#pragma unroll
            for (int i = 0; i < VY; ++i) avg_acc[k] = fmaf(wj[i], col[i * a.RWp], avg_acc[k]);
          }
        }
      }
      continue;
    }
#pragma unroll
    for (int i = 0; i < VY; ++i) {
      const int cyi = cy + i;
      const bool ok = ivalid && cyi <= cy1;
      const T nc = ntile[(cyi - Y0) * a.NWp + (cx - X0)];
      const T dp = nc - T(2) * acc[i];
      if (a.dense) {
        if (ok) dense_row[(cyi - ry - a.lo) * a.Wn + (cx - rx - a.lo)] = dp + nr;
        continue;
      }
      const uint32_t u = P::ord(dp);
      const bool pass = ok && u <= thr;
      const unsigned msk = __ballot_sync(0xffffffffu, pass);
      if (msk) {
        const int n = __popc(msk);
        if (cnt + n > 32) {  // flush the buffer first
          thr = smem_list_merge<NJ>(lst, buf, cnt, a.KP, lane);
          cnt = 0;
        }
        if (pass) buf[cnt + __popc(msk & ((1u << lane) - 1u))] = (uint64_t(u) << 32) | uint32_t(cyi * a.W + cx);
        cnt += n;
        __syncwarp();
      }
    }
  }
  if constexpr (AVG > 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) theta += __shfl_xor_sync(0xffffffffu, theta, o);
    const float inv = 1.f / theta, centre = sizeof(In) == 1 ? 128.f : 0.5f;
    float* out = a.avg_out + size_t(ref_band) * a.C * b * b;
#pragma unroll
    for (int k = 0; k < EPL; ++k)
      if (lane + 32 * k < a.C * b * b) out[lane + 32 * k] = fmaf(avg_acc[k], inv, centre);
    return;
  }
  if (a.dense) {
    if (a.nlm_inv_h2 > 0.f) {  // fused NLM epilogue: the warp's own row, just written (L2-hot)
      __syncwarp();
      const NlmRowGeom gm{ry, rx, a.H - b, a.W - b, a.Wn, a.lo};
      nlm_normalize_row<T>(dense_row, gm, a.nlm_inv_h2, lane);
    }
    return;
  }
  if (cnt > 0) smem_list_merge<NJ>(lst, buf, cnt, a.KP, lane);

  const size_t out_base = (size_t(f) * ((a.iy_end - a.iy_begin) * a.nx) + ref_band) * a.K;
  if constexpr (sizeof(In) == 1) {
    int32_t* dist = static_cast<int32_t*>(a.dist_out);
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int k = lane + 32 * j;
      if (k < a.K) {
        const uint64_t key = lst[k];
        const bool none = key == kKeyInf;
        a.idx_out[out_base + k] = none ? -1 : int32_t(uint32_t(key));
        dist[out_base + k] = none ? 0x7fffffff : unord_i32(uint32_t(key >> 32)) + nr;
      }
    }
  } else {
    // a5: re-score the best KP keys by direct differences from the uncentred input.
    const float* img = static_cast<const float*>(a.imgs) + size_t(f) * a.C * a.H * a.W;
    const size_t pl = size_t(a.H) * a.W;
    const uint64_t kp_key = lst[a.KP - 1];  // the KP-th identity key (filter boundary)
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int k = lane + 32 * j;
      const uint64_t key = lst[k];
      if (k >= a.KP || key == kKeyInf) {
        lst[k] = kKeyInf;
        continue;
      }
      const uint32_t idx = uint32_t(key);
      const int cyk = int(idx) / a.W, cxk = int(idx) - cyk * a.W;
      float d = 0.f;
      for (int c = 0; c < a.C; ++c) {
        const float* pr = img + c * pl + size_t(ry) * a.W + rx;
        const float* pc = img + c * pl + size_t(cyk) * a.W + cxk;
        for (int l = 0; l < b; ++l)
#pragma unroll 4
          for (int m = 0; m < b; ++m) {
            const float df = __ldg(pr + l * a.W + m) - __ldg(pc + l * a.W + m);
            d = fmaf(df, df, d);
          }
      }
      lst[k] = (uint64_t(__float_as_uint(d)) << 32) | idx;  // d >= +0: bits are monotone
    }
    __syncwarp();
    smem_list_sort<NJ>(lst, lane);
    // A candidate the fp32 identity pushed beyond the KP-th key could still be a true top-K one
    // when the identity's rounding (relative to the norms, ~b^2 C ulps: it matters only for
    // near-degenerate data, e.g. b = 1 on smooth images) reaches the exact K-th distance: then
    // the reference goes to the exact fix-up (fixup.cu). Threat candidates have d <= d_K, so
    // n_c <= 2 n_r + 2 d_K and the identity's terms are <= 6 n_r + 4 d_K.
    if (lane == 0 && kp_key != kKeyInf && a.fix_count != nullptr) {
      const uint64_t kk = lst[a.K - 1];
      const float dK = __uint_as_float(uint32_t(kk >> 32));
      const float dKP = unord_f32(uint32_t(kp_key >> 32)) + nr;
      const float kappa = 2.f * float(b * b * a.C) * 5.96e-8f;
      if (kk != kKeyInf && dKP - kappa * (6.f * fmaxf(nr, 0.f) + 4.f * dK) <= dK * (1.f + 1e-5f)) {
        const int pos = atomicAdd(a.fix_count, 1);
        a.fix_list[pos] = int(size_t(f) * ((a.iy_end - a.iy_begin) * a.nx) + ref_band);
      }
    }
    float* dist = static_cast<float*>(a.dist_out);
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int k = lane + 32 * j;
      if (k < a.K) {
        const uint64_t key = lst[k];
        const bool none = key == kKeyInf;
        a.idx_out[out_base + k] = none ? -1 : int32_t(uint32_t(key));
        dist[out_base + k] = none ? __int_as_float(0x7f800000) : __uint_as_float(uint32_t(key >> 32));
      }
    }
  }
}

template <typename In, int BK, int VY, int NJ, bool ONE_CH, int AVG>
__global__ void __launch_bounds__(256) bm_simt_kernel(SimtArgs a) {
  using T = typename Path<In>::T;
  extern __shared__ __align__(16) uint32_t smem_u32[];
  const int f = blockIdx.y;
  const int ty = blockIdx.x / a.tiles_x, tx = blockIdx.x - ty * a.tiles_x;
  const int iy_first = a.iy_begin + ty * a.TRY;
  const int iy_last = min(a.iy_end, iy_first + a.TRY) - 1;
  const int ix_first = tx * a.TRX;
  const int ix_last = min(a.nx, ix_first + a.TRX) - 1;
  const int s = a.s, b = a.b;
  // image region: rows [Y0, Y1], cols [X0, X1]
  const int Y0 = max(0, iy_first * s + a.lo), Y1 = min(a.H - 1, iy_last * s + a.hi + b - 1);
  const int X0 = max(0, ix_first * s + a.lo), X1 = min(a.W - 1, ix_last * s + a.hi + b - 1);
  const int RH = Y1 - Y0 + 1, RW = X1 - X0 + 1;
  // candidate (norm) region: rows [Y0, NY1], cols [X0, NX1]
  const int NY1 = min(a.H - b, iy_last * s + a.hi), NX1 = min(a.W - b, ix_last * s + a.hi);
  const int NH = NY1 - Y0 + 1, NW = NX1 - X0 + 1;

  uint32_t* tile = smem_u32;
  T* ntile = reinterpret_cast<T*>(smem_u32 + a.img_words);
  uint64_t* bufs = reinterpret_cast<uint64_t*>(smem_u32 + a.img_words + ((a.NHp * a.NWp + 1) & ~1));

  const size_t plane_px = size_t(a.H) * a.W;
  if constexpr (sizeof(In) == 1) {
    const uint8_t* img = static_cast<const uint8_t*>(a.imgs) + size_t(f) * a.C * plane_px;
    const int total = a.C * 4 * a.PL;
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      const int pk = e / a.PL, r = e - pk * a.PL;
      const int c = pk >> 2, k = pk & 3;
      const int yy = r / a.WP, w = r - yy * a.WP;
      uint32_t word = 0;
      if (yy < RH) {
        const uint8_t* row = img + size_t(c) * plane_px + size_t(Y0 + yy) * a.W + X0;
#pragma unroll
        for (int e2 = 0; e2 < 4; ++e2) {
          const int xx = 4 * w + k + e2;
          const uint32_t v = xx < RW ? uint32_t(row[xx] ^ 0x80u) : 0u;
          word |= v << (8 * e2);
        }
      }
      tile[e] = word;
    }
  } else {
    const float* img = static_cast<const float*>(a.imgs) + size_t(f) * a.C * plane_px;
    float* ft = reinterpret_cast<float*>(tile);
    for (int c = 0; c < a.C; ++c) {
      const float* src = img + size_t(c) * plane_px;
      float* dst = ft + size_t(c) * a.RHp * a.RWp;
      for (int yy = threadIdx.x / 32; yy < a.RHp; yy += blockDim.x / 32)
        for (int xx = threadIdx.x & 31; xx < a.RWp; xx += 32)
          dst[yy * a.RWp + xx] = (yy < RH && xx < RW) ? src[size_t(Y0 + yy) * a.W + X0 + xx] - 0.5f : 0.f;
    }
  }
  const T* nsrc = static_cast<const T*>(a.norm) + size_t(f) * a.nfs;
  for (int yy = threadIdx.x / 32; yy < a.NHp; yy += blockDim.x / 32)
    for (int xx = threadIdx.x & 31; xx < a.NWp; xx += 32)
      ntile[yy * a.NWp + xx] = (yy < NH && xx < NW) ? nsrc[size_t(Y0 + yy) * a.Mx + X0 + xx] : T(0);
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  uint64_t* buf = bufs + warp * kWarpKeys;
  const int ty_n = iy_last - iy_first + 1, tx_n = ix_last - ix_first + 1;
  for (int r = warp; r < ty_n * tx_n; r += nwarps) {
    const int iy = iy_first + r / tx_n, ix = ix_first + r % tx_n;
    const int ref_band = (iy - a.iy_begin) * a.nx + ix;
    process_ref<In, BK, VY, NJ, ONE_CH, AVG>(a, f, ref_band, iy, ix, tile, ntile, buf, Y0, X0, lane);
  }
}

template <typename In, int BK, int VY, int NJ, int AVG = 0>
cudaError_t launch_t(const SimtArgs& a, int F, size_t smem, cudaStream_t st) {
  const int tiles_y = (a.iy_end - a.iy_begin + a.TRY - 1) / a.TRY;
  dim3 grid(a.tiles_x * tiles_y, F);
  if (a.C == 1) {
    auto k = bm_simt_kernel<In, BK, VY, NJ, true, AVG>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    k<<<grid, 256, smem, st>>>(a);
  } else {
    auto k = bm_simt_kernel<In, BK, VY, NJ, false, AVG>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    k<<<grid, 256, smem, st>>>(a);
  }
  return cudaGetLastError();
}

int nj_for(int KP) { return KP <= 32 ? 1 : KP <= 64 ? 2 : KP <= 96 ? 3 : 5; }

template <typename In, int BK, int VY, bool SPEC>
cudaError_t dispatch_nj(const SimtArgs& a, int F, size_t smem, cudaStream_t st) {
  if (a.avg_out) {  // NL-means: no lists; elements per lane for b^2 C <= 64 / 128 / 256
    const int n = a.b * a.b * a.C;
    if (n <= 64) return launch_t<In, BK, VY, 1, 2>(a, F, smem, st);
    if (n <= 128) return launch_t<In, BK, VY, 1, 4>(a, F, smem, st);
    return launch_t<In, BK, VY, 1, 8>(a, F, smem, st);
  }
  const int nj = nj_for(a.KP);
  if constexpr (SPEC) {
    if (nj == 1) return launch_t<In, BK, VY, 1>(a, F, smem, st);
    if (nj == 2) return launch_t<In, BK, VY, 2>(a, F, smem, st);
    if (nj == 3) return launch_t<In, BK, VY, 3>(a, F, smem, st);
  }
  return launch_t<In, BK, VY, 5>(a, F, smem, st);
}

// Compile-time patch extent: exact for the configs' sides, zero-padded generic otherwise.
int bk_for(int b, bool u8) {
  if (u8) return b <= 4 ? 4 : b <= 8 ? 8 : 16;
  return b == 7 ? 7 : b <= 4 ? 4 : b <= 8 ? 8 : 16;
}
int vy_for(int b) { return b <= 8 ? 8 : 4; }

template <typename In>
cudaError_t dispatch_b(const SimtArgs& a, int F, size_t smem, cudaStream_t st) {
  constexpr bool u8 = sizeof(In) == 1;
  const int bk = bk_for(a.b, u8);
  if (bk == 8 && a.b == 8) return dispatch_nj<In, 8, 8, true>(a, F, smem, st);
  if (bk == 8) return dispatch_nj<In, 8, 8, false>(a, F, smem, st);
  if constexpr (!u8) {
    if (bk == 7) return dispatch_nj<In, 7, 8, true>(a, F, smem, st);
  }
  if (bk == 4) return dispatch_nj<In, 4, 8, false>(a, F, smem, st);
  return dispatch_nj<In, 16, 4, false>(a, F, smem, st);
}

size_t smem_bytes(const Geometry& g, int TRY, int TRX, SimtArgs* a) {
  const bool u8 = g.dtype == SC_DTYPE_U8;
  const int BK = bk_for(g.b, u8), VY = vy_for(g.b);
  const int pad = BK - g.b;
  a->RWp = (TRX - 1) * g.s + g.Wn + g.b - 1 + pad;
  a->RHp = (TRY - 1) * g.s + g.Wn + g.b - 1 + pad + VY - 1;
  if (u8) {
    a->WP = (a->RWp + 3) / 4 + 1;
    int pl = a->RHp * a->WP;
    pl += ((8 - pl % 32) + 32) % 32;  // plane size == 8 (mod 32) words: copies 8 banks apart
    a->PL = pl;
    a->img_words = g.C * 4 * pl;
  } else {
    a->WP = a->PL = 0;
    a->img_words = g.C * a->RHp * a->RWp;
  }
  a->img_words = (a->img_words + 3) & ~3;
  a->NWp = (TRX - 1) * g.s + g.Wn;
  a->NHp = (TRY - 1) * g.s + g.Wn + VY - 1;
  size_t bytes = size_t(a->img_words) * 4 + size_t((a->NHp * a->NWp + 1) & ~1) * 4;
  bytes += size_t(8) * kWarpKeys * 8;  // 8 warps x (32 survivors + 32*NJ list)
  return bytes;
}

}  // namespace

TileCfg choose_simt_tile(const Geometry& g, int sm_count, int n_images) {
  TileCfg t{};
  t.warps = 8;
  t.VY = vy_for(g.b);
  int best_try = 1, best_trx = 1;
  // largest square-ish tile that fits ~100 KB and still gives >= 8 CTAs per SM
  const int cands[][2] = {{8, 8}, {4, 8}, {4, 4}, {2, 4}, {2, 2}, {1, 2}, {1, 1}};
  for (auto& c : cands) {
    SimtArgs a{};
    const size_t sm = smem_bytes(g, c[0], c[1], &a);
    const long long tiles = (long long)((g.ny + c[0] - 1) / c[0]) * ((g.nx + c[1] - 1) / c[1]) * n_images;
    best_try = c[0];
    best_trx = c[1];
    if (sm <= 100 * 1024 && tiles >= 8LL * sm_count) break;
  }
  t.TRY = best_try;
  t.TRX = best_trx;
  SimtArgs a{};
  t.smem = smem_bytes(g, t.TRY, t.TRX, &a);
  return t;
}

cudaError_t launch_bm_simt(const sc_bm_plan_s& p, const void* imgs, int F, int iy_begin, int iy_end,
                           int32_t* idx_out, void* dist_out, void* dense, cudaStream_t st,
                           int64_t* launches) {
  const Geometry& g = p.g;
  SimtArgs a{};
  a.imgs = imgs;
  a.norm = p.ws.norm;
  a.idx_out = idx_out;
  a.dist_out = dist_out;
  a.dense = dense;
  a.nlm_inv_h2 = (dense || p.nlm_avg_out) ? p.nlm_inv_h2 : 0.f;
  a.avg_out = static_cast<float*>(p.nlm_avg_out);
  a.H = g.H; a.W = g.W; a.C = g.C; a.b = g.b; a.s = g.s; a.Wn = g.Wn; a.K = g.K; a.KP = g.KP;
  a.lo = g.lo; a.hi = g.hi; a.nx = g.nx; a.My = g.My; a.Mx = g.Mxp;  // Mx = norm-map row pitch
  a.nfs = g.NFS;
  a.iy_begin = iy_begin; a.iy_end = iy_end;
  a.TRY = p.tile.TRY; a.TRX = p.tile.TRX;
  a.tiles_x = (g.nx + a.TRX - 1) / a.TRX;
  const size_t smem = smem_bytes(g, a.TRY, a.TRX, &a);
  if (launches) *launches += 1;
  if (g.dtype == SC_DTYPE_U8) return dispatch_b<uint8_t>(a, F, smem, st);
  const bool fix = dense == nullptr && a.avg_out == nullptr;  // float top-K: identity-rounding check
  if (fix) {
    a.fix_count = p.ws.fix_count;
    a.fix_list = p.ws.fix_list;
    cudaError_t e = cudaMemsetAsync(p.ws.fix_count, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = dispatch_b<float>(a, F, smem, st);
  if (e != cudaSuccess || !fix) return e;
  if (launches) *launches += 1;
  return launch_fixup(p, imgs, F, iy_begin, iy_end, idx_out, dist_out, st);
}

}  // namespace scbm
