// bm_simt.cu -- steps a0, a2, a3, a4 (+ a5 for f32) fused in one CUDA-core kernel.
//
//   a0 staging   one CTA owns a TRY x TRX tile of references; it stages the image region
//                covering the union of their clipped windows plus the patch extent
//                (the "window halo"), centred (u8: x-128, f32: x-0.5), and the matching
//                tile of the norm map, in shared memory.
//   a2 cross     C_i(j) = <X'_i, X'_j> (Self-Convolution, Eq. 5, channels
//                summed, Eq. 12): one warp per reference; the reference patch lives in
//                registers; each lane slides over VY vertically adjacent candidates of one
//                column, so every image row it loads feeds up to VY patch rows
//                (VY*b^2 FMAs per (b+VY-1)*b shared loads).
//   a3 assembly  d' = n_c - 2 C (Lemma 2, with ||X_i||^2 deferred: it is
//                constant per reference, so ranking by d' is ranking by d; Theorem 1's
//                b_i = -d'/2).
//   a4 top-K     threshold filter + warp bitonic merges on packed keys (topk.cuh).
//   a5 re-score  f32 only: the best K+8 keys are re-scored by direct differences
//                sum (x_r - x_c)^2 in fp32 from the uncentred input and re-sorted.
//   a6 output    coalesced stores of K idx + K dist per reference; u8 dist = d' + n_r exact.
//
// u8 arithmetic is exact int32 (|C'| <= 64*128^2 = 2^20 per channel); f32 is fp32 FMA.
#include "sc_internal.h"
#include "topk.cuh"

namespace scbm {
namespace {

template <typename In> struct Elem;
template <> struct Elem<uint8_t> {
  using T = int32_t;
  __device__ static T centre(uint8_t x) { return T(x) - 128; }
  __device__ static uint32_t ord(T v) { return ord_i32(v); }
};
template <> struct Elem<float> {
  using T = float;
  __device__ static T centre(float x) { return x - 0.5f; }
  __device__ static uint32_t ord(T v) { return ord_f32(v); }
};

struct SimtArgs {
  const void* imgs;   // [F][C][H][W]
  const void* norm;   // [F][My][Mx] int32 / float (centred norm map)
  int32_t* idx_out;   // [F][band refs][K]
  void* dist_out;     // [F][band refs][K]
  void* dense;        // debug: [refs][Wn*Wn] (one image) or nullptr
  int H, W, C, b, s, Wn, K, KP, MS, lo, hi, nx, My, Mx;
  int iy_begin, iy_end;
  int TRY, TRX, tiles_x;
  int RWp, RHp, NWp, NHp;  // shared tile pitches / padded heights
};

template <int n> struct Pow2 { static constexpr int v = n; };

// BK: compile-time patch extent; EXACT: b == BK (else the reference is zero-padded to BK).
template <typename In, int BK, int VY, bool ONE_CH>
__device__ __forceinline__ void process_ref(const SimtArgs& a, int f, int ref_band, int iy, int ix,
                                            const typename Elem<In>::T* __restrict__ tile,
                                            const typename Elem<In>::T* __restrict__ ntile,
                                            uint64_t* arr, int Y0, int X0, int lane) {
  using T = typename Elem<In>::T;
  const int s = a.s, b = a.b;
  const int ry = iy * s, rx = ix * s;
  const int cy0 = max(0, ry + a.lo), cy1 = min(a.H - b, ry + a.hi);
  const int cx0 = max(0, rx + a.lo), cx1 = min(a.W - b, rx + a.hi);
  const int ncols = cx1 - cx0 + 1, nrows = cy1 - cy0 + 1;
  const int nby = (nrows + VY - 1) / VY;
  const int nitems = nby * ncols;
  const int plane = a.RHp * a.RWp;
  const T nr = ntile[(ry - Y0) * a.NWp + (rx - X0)];

  for (int i = lane; i < a.MS; i += 32) arr[i] = kKeyInf;
  __syncwarp();
  uint64_t thr = kKeyInf;
  int cnt = 0;

  T refv[BK][BK];
  auto load_ref = [&](int c) {
    const T* rp = tile + c * plane + (ry - Y0) * a.RWp + (rx - X0);
#pragma unroll
    for (int l = 0; l < BK; ++l)
#pragma unroll
      for (int m = 0; m < BK; ++m) refv[l][m] = (l < b && m < b) ? rp[l * a.RWp + m] : T(0);
  };
  if (ONE_CH) load_ref(0);

  int32_t* dense_i = nullptr;
  T* dense_row = nullptr;
  if (a.dense) {
    const size_t ref_g = size_t(ref_band);
    dense_row = static_cast<T*>(a.dense) + ref_g * a.Wn * a.Wn;
    for (int i = lane; i < a.Wn * a.Wn; i += 32) dense_row[i] = T(-1);
    __syncwarp();
  }
  (void)dense_i;

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
      if (!ONE_CH) load_ref(c);
      const T* col = tile + c * plane + (cy - Y0) * a.RWp + (cx - X0);
#pragma unroll
      for (int t = 0; t < BK + VY - 1; ++t) {
        T xr[BK];
#pragma unroll
        for (int m = 0; m < BK; ++m) xr[m] = col[t * a.RWp + m];
#pragma unroll
        for (int i = 0; i < VY; ++i) {
          const int l = t - i;
          if (l >= 0 && l < BK) {
#pragma unroll
            for (int m = 0; m < BK; ++m) acc[i] += refv[l][m] * xr[m];
          }
        }
      }
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
      const uint64_t key = (uint64_t(Elem<In>::ord(dp)) << 32) | uint32_t(cyi * a.W + cx);
      const bool pass = ok && key < thr;
      const unsigned msk = __ballot_sync(0xffffffffu, pass);
      if (pass) arr[a.KP + cnt + __popc(msk & ((1u << lane) - 1u))] = key;
      cnt += __popc(msk);
      if (cnt >= 32) {
        __syncwarp();
        thr = warp_topk_merge(arr, a.KP, a.MS, lane);
        cnt = 0;
      }
    }
  }
  if (a.dense) return;
  __syncwarp();
  if (cnt > 0) warp_topk_merge(arr, a.KP, a.MS, lane);

  const size_t out_base = (size_t(f) * ((a.iy_end - a.iy_begin) * a.nx) + ref_band) * a.K;
  if constexpr (sizeof(In) == 1) {
    int32_t* dist = static_cast<int32_t*>(a.dist_out);
    for (int k = lane; k < a.K; k += 32) {
      const uint64_t key = arr[k];
      if (key == kKeyInf) {
        a.idx_out[out_base + k] = -1;
        dist[out_base + k] = 0x7fffffff;
      } else {
        a.idx_out[out_base + k] = int32_t(uint32_t(key));
        dist[out_base + k] = unord_i32(uint32_t(key >> 32)) + nr;
      }
    }
  } else {
    // a5: re-score the best KP keys by direct differences from the uncentred input.
    const float* img = static_cast<const float*>(a.imgs) + size_t(f) * a.C * a.H * a.W;
    const size_t pl = size_t(a.H) * a.W;
    for (int k = lane; k < a.KP; k += 32) {
      const uint64_t key = arr[k];
      if (key == kKeyInf) continue;
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
      arr[k] = (uint64_t(__float_as_uint(d)) << 32) | idx;  // d >= +0: bits are monotone
    }
    __syncwarp();
    int n2 = 32;
    while (n2 < a.KP) n2 <<= 1;
    for (int i = a.KP + lane; i < n2; i += 32) arr[i] = kKeyInf;
    __syncwarp();
    warp_bitonic_sort(arr, n2, lane);
    float* dist = static_cast<float*>(a.dist_out);
    for (int k = lane; k < a.K; k += 32) {
      const uint64_t key = arr[k];
      if (key == kKeyInf) {
        a.idx_out[out_base + k] = -1;
        dist[out_base + k] = __int_as_float(0x7f800000);
      } else {
        a.idx_out[out_base + k] = int32_t(uint32_t(key));
        dist[out_base + k] = __uint_as_float(uint32_t(key >> 32));
      }
    }
  }
  __syncwarp();
}

template <typename In, int BK, int VY, bool ONE_CH>
__global__ void __launch_bounds__(256) bm_simt_kernel(SimtArgs a) {
  using T = typename Elem<In>::T;
  extern __shared__ __align__(16) unsigned char smem[];
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

  T* tile = reinterpret_cast<T*>(smem);
  T* ntile = tile + size_t(a.C) * a.RHp * a.RWp;
  uint64_t* keys = reinterpret_cast<uint64_t*>(ntile + size_t(a.NHp) * a.NWp + 2);
  keys = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(keys) + 15) & ~uintptr_t(15));

  const In* img = static_cast<const In*>(a.imgs) + size_t(f) * a.C * a.H * a.W;
  for (int c = 0; c < a.C; ++c) {
    const In* src = img + size_t(c) * a.H * a.W;
    T* dst = tile + size_t(c) * a.RHp * a.RWp;
    for (int yy = threadIdx.x / 32; yy < a.RHp; yy += blockDim.x / 32)
      for (int xx = threadIdx.x & 31; xx < a.RWp; xx += 32)
        dst[yy * a.RWp + xx] =
            (yy < RH && xx < RW) ? Elem<In>::centre(src[size_t(Y0 + yy) * a.W + X0 + xx]) : T(0);
  }
  const T* nsrc = static_cast<const T*>(a.norm) + size_t(f) * a.My * a.Mx;
  for (int yy = threadIdx.x / 32; yy < a.NHp; yy += blockDim.x / 32)
    for (int xx = threadIdx.x & 31; xx < a.NWp; xx += 32)
      ntile[yy * a.NWp + xx] = (yy < NH && xx < NW) ? nsrc[size_t(Y0 + yy) * a.Mx + X0 + xx] : T(0);
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  uint64_t* arr = keys + warp * a.MS;
  const int ty_n = iy_last - iy_first + 1, tx_n = ix_last - ix_first + 1;
  for (int r = warp; r < ty_n * tx_n; r += nwarps) {
    const int iy = iy_first + r / tx_n, ix = ix_first + r % tx_n;
    const int ref_band = (iy - a.iy_begin) * a.nx + ix;
    process_ref<In, BK, VY, ONE_CH>(a, f, ref_band, iy, ix, tile, ntile, arr, Y0, X0, lane);
  }
}

template <typename In, int BK, int VY>
cudaError_t launch_t(const SimtArgs& a, int F, size_t smem, cudaStream_t st) {
  const int tiles_y = (a.iy_end - a.iy_begin + a.TRY - 1) / a.TRY;
  dim3 grid(a.tiles_x * tiles_y, F);
  if (a.C == 1) {
    auto k = bm_simt_kernel<In, BK, VY, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    k<<<grid, 256, smem, st>>>(a);
  } else {
    auto k = bm_simt_kernel<In, BK, VY, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    k<<<grid, 256, smem, st>>>(a);
  }
  return cudaGetLastError();
}

template <typename In>
cudaError_t dispatch_b(const SimtArgs& a, int F, size_t smem, cudaStream_t st, int VY) {
  // exact instantiations for the configs' patch sides, zero-padded generic ones otherwise
  if (a.b == 8) return launch_t<In, 8, 8>(a, F, smem, st);
  if (a.b == 7) return launch_t<In, 7, 8>(a, F, smem, st);
  if (a.b <= 4) return launch_t<In, 4, 8>(a, F, smem, st);
  if (a.b <= 8) return launch_t<In, 8, 8>(a, F, smem, st);
  return launch_t<In, 16, 4>(a, F, smem, st);
}

int bk_for(int b) { return b == 7 ? 7 : b <= 4 ? 4 : b <= 8 ? 8 : 16; }
int vy_for(int b) { return b <= 8 ? 8 : 4; }

size_t smem_bytes(const Geometry& g, int TRY, int TRX, int* RWp, int* RHp, int* NWp, int* NHp,
                  int* MS) {
  const int BK = bk_for(g.b), VY = vy_for(g.b);
  const int pad = BK - g.b;
  *RWp = (TRX - 1) * g.s + g.Wn + g.b - 1 + pad;
  *RHp = (TRY - 1) * g.s + g.Wn + g.b - 1 + pad + VY - 1;
  *NWp = (TRX - 1) * g.s + g.Wn;
  *NHp = (TRY - 1) * g.s + g.Wn + VY - 1;
  int ms = 64;
  while (ms < g.KP + 64) ms <<= 1;
  *MS = ms;
  size_t bytes = size_t(g.C) * (*RHp) * (*RWp) * 4 + size_t(*NHp) * (*NWp) * 4 + 8 + 16;
  bytes += size_t(8) * ms * 8;  // 8 warps
  return bytes;
}

}  // namespace

TileCfg choose_simt_tile(const Geometry& g, int sm_count, int n_images) {
  TileCfg t{};
  t.warps = 8;
  t.VY = vy_for(g.b);
  int best_try = 1, best_trx = 1;
  // largest square-ish tile that fits ~100 KB and still gives >= 4 waves of 2 CTAs/SM
  const int cands[][2] = {{8, 8}, {4, 8}, {4, 4}, {2, 4}, {2, 2}, {1, 2}, {1, 1}};
  for (auto& c : cands) {
    int a, bb, cc, d, ms;
    const size_t sm = smem_bytes(g, c[0], c[1], &a, &bb, &cc, &d, &ms);
    const long long tiles = (long long)((g.ny + c[0] - 1) / c[0]) * ((g.nx + c[1] - 1) / c[1]) * n_images;
    best_try = c[0];
    best_trx = c[1];
    if (sm <= 100 * 1024 && tiles >= 8LL * sm_count) break;
  }
  t.TRY = best_try;
  t.TRX = best_trx;
  int a, bb, cc, d, ms;
  t.smem = smem_bytes(g, t.TRY, t.TRX, &a, &bb, &cc, &d, &ms);
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
  a.H = g.H; a.W = g.W; a.C = g.C; a.b = g.b; a.s = g.s; a.Wn = g.Wn; a.K = g.K; a.KP = g.KP;
  a.lo = g.lo; a.hi = g.hi; a.nx = g.nx; a.My = g.My; a.Mx = g.Mx;
  a.iy_begin = iy_begin; a.iy_end = iy_end;
  a.TRY = p.tile.TRY; a.TRX = p.tile.TRX;
  a.tiles_x = (g.nx + a.TRX - 1) / a.TRX;
  const size_t smem = smem_bytes(g, a.TRY, a.TRX, &a.RWp, &a.RHp, &a.NWp, &a.NHp, &a.MS);
  if (launches) *launches += 1;
  if (g.dtype == SC_DTYPE_U8) return dispatch_b<uint8_t>(a, F, smem, st, p.tile.VY);
  return dispatch_b<float>(a, F, smem, st, p.tile.VY);
}

}  // namespace scbm
