// fixup.cu -- exact top-K for references flagged by the 32-bit register top-K paths.
//
// The fast paths keep 32-bit register keys. uint8 L2 (bm_box, bm_lanes, bm_tc): the distance
// field saturates at DSAT (regtopk.cuh), so a reference whose K-th key is saturated -- or still
// +inf because its window has fewer than K candidates -- is appended to a flag list. Quantised
// keys (NCC on both box kernels, float L2 on bm_boxf): a reference whose worst kept key's quantum
// could still hold a candidate as good as its exact K-th one is flagged. This kernel recomputes
// exactly those references from scratch over the whole window: L2 by direct differences (Eq. 3,
// PAPER.md:255-262; exact integers for uint8, fp32 for float) with 64-bit (distance, idx) keys
// and warp top-K merges (topk.cuh); NCC by exact re-ranking (ncc.cuh). It runs after every
// matching launch; with nothing flagged (the normal case) each warp reads the count and exits.
#include "sc_internal.h"
#include "ncc.cuh"
#include "topk.cuh"

namespace scbm {
namespace {

struct FixArgs {
  const void* imgs;  // uint8 or float [frames][C][H][W]
  const int* fix_count;
  const int* fix_list;
  int32_t* idx_out;
  void* dist_out;    // int32 (uint8 L2) or float (float L2, NCC: -NCC)
  int H, W, C, b, s, K, lo, hi, nx, iy_begin, iy_end;
  int T, n_frames, frame0;  // temporal search: frames fref-T..fref+T of the batch at imgs
  int ncc;                  // SC_METRIC_NCC: exact NCC re-rank (K <= 32), dist_out = -NCC (float)
  int idx_foff;             // temporal search: frame offset added to the batch-global idx
  // 3D search (sc_bm_plan3d): reference plane (frame0 + f) * sz of a P-plane volume at imgs,
  // candidates at plane offsets [zlo, zhi] (clipped to [0, P - C]), idx = (z H + y) W + x
  int z3, sz, P, zlo, zhi;
  // packed tables (uint8 L2, K <= 32; packed.cu): idx_out receives the row words
  // (dist << prb) | slot, rows that do not fit -> escape words + an overflow record in ptail
  int packed, Wn, prb;
  uint32_t pdsat;
  uint32_t* ptail;
  long long pk_f0;  // image index (in the run) of the chunk's first frame
  int nref_full;    // references per image
};

// NCC (Eq. 4): a reference whose kept top-(K+8) could have lost a top-K candidate to the 32-bit
// key quantisation (bm_box.cu / bm_boxf.cu a5) is re-ranked over its whole window: per candidate
// C, n_c, n_r (exact integers for uint8, fp64 for float), chunks of 32 ranked by warp_rank_ncc and
// merged into the running best 32 (float input: ordered by the reported float32 NCC, as in a5).
template <typename TIN>
__device__ void fixup_ncc_ref(const FixArgs& a, int code, int lane) {
  constexpr bool EXACT = sizeof(TIN) == 1;
  const int band_refs = (a.iy_end - a.iy_begin) * a.nx;
  const int f = code / band_refs, rb = code - f * band_refs;
  const int iy = a.iy_begin + rb / a.nx, ix = rb % a.nx;
  const int ry = iy * a.s, rx = ix * a.s;
  const int cy0 = max(0, ry + a.lo), cy1 = min(a.H - a.b, ry + a.hi);
  const int cx0 = max(0, rx + a.lo), cx1 = min(a.W - a.b, rx + a.hi);
  const int ncols = cx1 - cx0 + 1, nwin = (cy1 - cy0 + 1) * ncols;
  const size_t plane = size_t(a.H) * a.W;
  const TIN* img = static_cast<const TIN*>(a.imgs) + size_t(a.frame0 + f) * a.C * plane;
  if constexpr (!EXACT) {
    if (a.K > 32) {  // float input with K > 32 (wide lists): (float32 d_NCC, idx) 64-bit keys, K <= 128
      WarpTopK<4> top;
      top.init();
      for (int base = 0; base < nwin; base += 32) {
        const int k = base + lane;
        uint64_t key = kKeyInf;
        if (k < nwin) {
          const int cy = cy0 + k / ncols, cx = cx0 + k % ncols;
          double cd = 0.0, ncd = 0.0, nrd = 0.0;
          for (int c = 0; c < a.C; ++c)
            for (int l = 0; l < a.b; ++l) {
              const TIN* pr = img + c * plane + size_t(ry + l) * a.W + rx;
              const TIN* pc = img + c * plane + size_t(cy + l) * a.W + cx;
              for (int m = 0; m < a.b; ++m) {
                cd = fma(double(pr[m]), double(pc[m]), cd);
                ncd = fma(double(pc[m]), double(pc[m]), ncd);
                nrd = fma(double(pr[m]), double(pr[m]), nrd);
              }
            }
          const double den = sqrt(nrd * ncd);
          const float dn = -float(den > 0.0 ? cd / den : 0.0);
          key = (uint64_t(ord_f32(dn)) << 32) | uint32_t(cy * a.W + cx);
        }
        top.merge(key, lane);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = lane + 32 * j;
        if (k < a.K) {
          const uint64_t key = top.v[j];
          const bool none = key == kKeyInf;
          const size_t o = size_t(code) * a.K + k;
          a.idx_out[o] = none ? -1 : int32_t(uint32_t(key));
          static_cast<float*>(a.dist_out)[o] = none ? __int_as_float(0x7f800000) : unord_f32(uint32_t(key >> 32));
        }
      }
      return;
    }
  }
  NccItem best;
  best.c = 0; best.n = 1; best.f = 0.0; best.idx = -1;
  for (int base = 0; base < nwin; base += 32) {
    const int k = base + lane;
    NccItem it;
    it.c = 0; it.n = 1; it.f = 0.0; it.idx = -1;
    if (k < nwin) {
      const int cy = cy0 + k / ncols, cx = cx0 + k % ncols;
      int cc = 0, nc = 0, nr = 0;
      double cd = 0.0, ncd = 0.0, nrd = 0.0;
      for (int c = 0; c < a.C; ++c)
        for (int l = 0; l < a.b; ++l) {
          const TIN* pr = img + c * plane + size_t(ry + l) * a.W + rx;
          const TIN* pc = img + c * plane + size_t(cy + l) * a.W + cx;
          for (int m = 0; m < a.b; ++m) {
            if constexpr (EXACT) {
              cc += int(pr[m]) * int(pc[m]);
              nc += int(pc[m]) * int(pc[m]);
              nr += int(pr[m]) * int(pr[m]);
            } else {
              cd = fma(double(pr[m]), double(pc[m]), cd);
              ncd = fma(double(pc[m]), double(pc[m]), ncd);
              nrd = fma(double(pr[m]), double(pr[m]), nrd);
            }
          }
        }
      if constexpr (EXACT) {
        const bool zero = nr == 0 || nc == 0;
        it.c = zero ? 0 : cc;
        it.n = zero ? 1 : nc;
        it.f = zero ? 0.0 : double(cc) / sqrt(double(nr) * double(nc));
      } else {
        const double den = sqrt(nrd * ncd);
        it.f = double(float(den > 0.0 ? cd / den : 0.0));
      }
      it.idx = cy * a.W + cx;
    }
    it = warp_rank_ncc<EXACT>(it, lane);
    // the best 32 of (running list, chunk): both sorted, so pair lane l with the chunk's 31 - l
    NccItem r;
    r.c = __shfl_sync(0xffffffffu, it.c, 31 - lane);
    r.n = __shfl_sync(0xffffffffu, it.n, 31 - lane);
    r.f = __shfl_sync(0xffffffffu, it.f, 31 - lane);
    r.idx = __shfl_sync(0xffffffffu, it.idx, 31 - lane);
    if (ncc_better<EXACT>(r, best)) best = r;
    best = warp_rank_ncc<EXACT>(best, lane);
  }
  if (lane < a.K) {
    const size_t o = size_t(code) * a.K + lane;
    a.idx_out[o] = best.idx;
    static_cast<float*>(a.dist_out)[o] = best.idx < 0 ? __int_as_float(0x7f800000) : float(-best.f);
  }
}

template <typename TIN>
__global__ void __launch_bounds__(256) fixup_kernel(FixArgs a) {
  constexpr bool U8 = sizeof(TIN) == 1;
  const int count = *a.fix_count;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int band_refs = (a.iy_end - a.iy_begin) * a.nx;
  for (int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < count; e += nw) {
    const int code = a.fix_list[e];
    if (a.ncc) {
      fixup_ncc_ref<TIN>(a, code, lane);
      continue;
    }
    const int f = code / band_refs, rb = code - f * band_refs;
    const int iy = a.iy_begin + rb / a.nx, ix = rb % a.nx;
    const int ry = iy * a.s, rx = ix * a.s;
    const int cy0 = max(0, ry + a.lo), cy1 = min(a.H - a.b, ry + a.hi);
    const int cx0 = max(0, rx + a.lo), cx1 = min(a.W - a.b, rx + a.hi);
    const int ncols = cx1 - cx0 + 1, nwin = (cy1 - cy0 + 1) * ncols;
    const size_t plane = size_t(a.H) * a.W;
    const int fref = a.frame0 + f;  // the reference's frame (temporal: index into the batch)
    // candidate frames (planes with the 3D search) fa .. fb; zunit = planes per frame step
    const int zr = a.z3 ? fref * a.sz : fref;
    const int fa = a.z3 ? max(0, zr + a.zlo) : max(0, fref - a.T);
    const int fb = a.z3 ? min(a.P - a.C, zr + a.zhi) : min(a.n_frames - 1, fref + a.T);
    const int zunit = a.z3 ? 1 : a.C;
    const int ncand = nwin * (fb - fa + 1);
    const TIN* imgs = static_cast<const TIN*>(a.imgs);
    const TIN* rimg = imgs + size_t(zr) * zunit * plane;
    WarpTopK<4> top;  // K <= 128
    top.init();
    for (int base = 0; base < ncand; base += 32) {
      const int k = base + lane;
      uint64_t key = kKeyInf;
      if (k < ncand) {
        const int fr = fa + k / nwin, kw = k - (k / nwin) * nwin;
        const int cy = cy0 + kw / ncols, cx = cx0 + kw % ncols;
        const TIN* cimg = imgs + size_t(fr) * zunit * plane;
        int di = 0;      // uint8: exact integers
        float df = 0.f;  // float: direct differences in fp32 (as the a5 re-score)
        for (int c = 0; c < a.C; ++c)
          for (int l = 0; l < a.b; ++l) {
            const TIN* pr = rimg + c * plane + size_t(ry + l) * a.W + rx;
            const TIN* pc = cimg + c * plane + size_t(cy + l) * a.W + cx;
            for (int m = 0; m < a.b; ++m) {
              if constexpr (U8) {
                const int v = int(pr[m]) - int(pc[m]);
                di += v * v;
              } else {
                const float v = float(pr[m]) - float(pc[m]);
                df = fmaf(v, v, df);
              }
            }
          }
        // idx: frame-local without temporal search, batch-global with it
        const int idx = (a.z3 ? fr * int(plane) : a.T > 0 ? (fr + a.idx_foff) * int(plane) : 0) + cy * a.W + cx;
        const uint32_t dbits = U8 ? uint32_t(di) : __float_as_uint(df);  // d >= 0: monotone bits
        key = (uint64_t(dbits) << 32) | uint32_t(idx);
      }
      top.merge(key, lane);
    }
    const size_t o = size_t(code) * a.K;
    if (U8 && a.packed) {  // K <= 32: lane k holds rank k
      const uint64_t key = top.v[0];
      const bool none = key == kKeyInf;
      const uint32_t d = uint32_t(key >> 32), ci = uint32_t(key);
      uint32_t* pk = reinterpret_cast<uint32_t*>(a.idx_out);
      if (__all_sync(0xffffffffu, lane >= a.K || (!none && d < a.pdsat))) {
        if (lane < a.K) {
          const int cy = int(ci) / a.W, cx = int(ci) - (int(ci) / a.W) * a.W;
          pk[o + lane] = (d << a.prb) | uint32_t((cy - ry - a.lo) * a.Wn + (cx - rx - a.lo));
        }
      } else {  // escape row + its exact record
        if (lane < a.K) pk[o + lane] = 0xffffffffu;
        uint32_t pos = 0u;
        if (lane == 0) pos = atomicAdd(a.ptail, 1u);
        pos = __shfl_sync(0xffffffffu, pos, 0);
        if (pos < a.ptail[1]) {
          uint32_t* rec = a.ptail + 2 + size_t(pos) * (2 + 2 * a.K);
          const long long row = (a.pk_f0 + f) * a.nref_full + (long long)iy * a.nx + ix;
          if (lane == 0) {
            rec[0] = uint32_t(row);
            rec[1] = uint32_t(row >> 32);
          }
          if (lane < a.K) {
            rec[2 + lane] = none ? 0xffffffffu : ci;
            rec[2 + a.K + lane] = none ? 0x7fffffffu : d;
          }
        }
      }
      continue;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = lane + 32 * j;
      if (k < a.K) {
        const uint64_t key = top.v[j];
        const bool none = key == kKeyInf;
        a.idx_out[o + k] = none ? -1 : int32_t(uint32_t(key));
        if constexpr (U8)
          static_cast<int32_t*>(a.dist_out)[o + k] = none ? 0x7fffffff : int32_t(key >> 32);
        else
          static_cast<float*>(a.dist_out)[o + k] = none ? __int_as_float(0x7f800000) : __uint_as_float(uint32_t(key >> 32));
      }
    }
  }
}

}  // namespace

cudaError_t launch_fixup(const sc_bm_plan_s& p, const void* imgs, int F, int iy_begin, int iy_end,
                         int32_t* idx_out, void* dist_out, cudaStream_t st) {
  const Geometry& g = p.g;
  FixArgs a{};
  a.imgs = imgs;
  a.fix_count = p.ws.fix_count;
  a.fix_list = p.ws.fix_list;
  a.idx_out = idx_out;
  a.dist_out = dist_out;
  a.H = g.H; a.W = g.W; a.C = g.C; a.b = g.b; a.s = g.s; a.K = g.K; a.lo = g.lo; a.hi = g.hi;
  a.nx = g.nx; a.iy_begin = iy_begin; a.iy_end = iy_end;
  a.T = p.T;
  a.ncc = g.metric == SC_METRIC_NCC;
  a.z3 = g.z3;
  a.sz = p.zstride;
  a.P = int(p.n_planes);
  a.zlo = p.zlo;
  a.zhi = p.zhi;
  if (p.T > 0 || g.z3) {  // temporal / 3D search: the batch (volume) base and the chunk's first frame
    a.imgs = p.batch_base;
    a.frame0 = int(p.batch_f0);
    a.n_frames = int(p.batch_n);
    a.idx_foff = int(p.idx_frame_off);
  } else {
    a.frame0 = 0;
    a.n_frames = 1 << 30;
  }
  (void)F;
  if (p.packed_cap > 0 && g.dtype == SC_DTYPE_U8 && !a.ncc && p.T == 0 && !g.z3) {
    a.packed = 1;
    a.Wn = g.Wn;
    a.prb = packed_rel_bits(g);
    a.pdsat = uint32_t((uint64_t(1) << (32 - a.prb)) - 1);
    a.ptail = p.packed_tail;
    a.pk_f0 = p.packed_f0;
    a.nref_full = g.ny * g.nx;
  }
  if (g.dtype == SC_DTYPE_U8) fixup_kernel<uint8_t><<<p.sm_count * 2, 256, 0, st>>>(a);
  else fixup_kernel<float><<<p.sm_count * 2, 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace scbm
