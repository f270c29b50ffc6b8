// fixup.cu -- exact top-K for references flagged by the 32-bit register top-K paths.
//
// The u8 fast paths (bm_lanes.cu with KR > 0, bm_tc.cu) keep 32-bit keys whose distance field
// saturates at DSAT (regtopk.cuh). A reference whose K-th key is saturated -- or still +inf
// because its window has fewer than K candidates -- is appended to a flag list instead of
// being written. This kernel recomputes exactly those references from scratch: every window
// candidate's distance by direct differences (Eq. 3; exact integers),
// 64-bit (distance, idx) keys, warp top-K merges (topk.cuh). It runs after every matching
// launch; with nothing flagged (the normal case) each warp reads the count and exits.
#include "sc_internal.h"
#include "topk.cuh"

namespace scbm {
namespace {

struct FixArgs {
  const uint8_t* imgs;
  const int* fix_count;
  const int* fix_list;
  int32_t* idx_out;
  int32_t* dist_out;
  int H, W, C, b, s, K, lo, hi, nx, iy_begin, iy_end;
  int T, n_frames, frame0;  // temporal search: frames fref-T..fref+T of the batch at imgs
};

__global__ void __launch_bounds__(256) fixup_kernel(FixArgs a) {
  const int count = *a.fix_count;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int band_refs = (a.iy_end - a.iy_begin) * a.nx;
  for (int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < count; e += nw) {
    const int code = a.fix_list[e];
    const int f = code / band_refs, rb = code - f * band_refs;
    const int iy = a.iy_begin + rb / a.nx, ix = rb % a.nx;
    const int ry = iy * a.s, rx = ix * a.s;
    const int cy0 = max(0, ry + a.lo), cy1 = min(a.H - a.b, ry + a.hi);
    const int cx0 = max(0, rx + a.lo), cx1 = min(a.W - a.b, rx + a.hi);
    const int ncols = cx1 - cx0 + 1, nwin = (cy1 - cy0 + 1) * ncols;
    const size_t plane = size_t(a.H) * a.W;
    const int fref = a.frame0 + f;  // the reference's frame (temporal: index into the batch)
    const int fa = max(0, fref - a.T), fb = min(a.n_frames - 1, fref + a.T);
    const int ncand = nwin * (fb - fa + 1);
    const uint8_t* rimg = a.imgs + size_t(fref) * a.C * plane;
    WarpTopK<4> top;  // K <= 128
    top.init();
    for (int base = 0; base < ncand; base += 32) {
      const int k = base + lane;
      uint64_t key = kKeyInf;
      if (k < ncand) {
        const int fr = fa + k / nwin, kw = k - (k / nwin) * nwin;
        const int cy = cy0 + kw / ncols, cx = cx0 + kw % ncols;
        const uint8_t* cimg = a.imgs + size_t(fr) * a.C * plane;
        int d = 0;
        for (int c = 0; c < a.C; ++c)
          for (int l = 0; l < a.b; ++l) {
            const uint8_t* pr = rimg + c * plane + size_t(ry + l) * a.W + rx;
            const uint8_t* pc = cimg + c * plane + size_t(cy + l) * a.W + cx;
            for (int m = 0; m < a.b; ++m) {
              const int v = int(pr[m]) - int(pc[m]);
              d += v * v;
            }
          }
        // idx: frame-local without temporal search, batch-global with it
        const int idx = (a.T > 0 ? fr * int(plane) : 0) + cy * a.W + cx;
        key = (uint64_t(uint32_t(d)) << 32) | uint32_t(idx);
      }
      top.merge(key, lane);
    }
    const size_t o = size_t(code) * a.K;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = lane + 32 * j;
      if (k < a.K) {
        const uint64_t key = top.v[j];
        const bool none = key == kKeyInf;
        a.idx_out[o + k] = none ? -1 : int32_t(uint32_t(key));
        a.dist_out[o + k] = none ? 0x7fffffff : int32_t(key >> 32);
      }
    }
  }
}

}  // namespace

cudaError_t launch_fixup(const sc_bm_plan_s& p, const void* imgs, int F, int iy_begin, int iy_end,
                         int32_t* idx_out, void* dist_out, cudaStream_t st) {
  const Geometry& g = p.g;
  FixArgs a{};
  a.imgs = static_cast<const uint8_t*>(imgs);
  a.fix_count = p.ws.fix_count;
  a.fix_list = p.ws.fix_list;
  a.idx_out = idx_out;
  a.dist_out = static_cast<int32_t*>(dist_out);
  a.H = g.H; a.W = g.W; a.C = g.C; a.b = g.b; a.s = g.s; a.K = g.K; a.lo = g.lo; a.hi = g.hi;
  a.nx = g.nx; a.iy_begin = iy_begin; a.iy_end = iy_end;
  a.T = p.T;
  if (p.T > 0) {  // temporal search: the batch base and the chunk's first frame
    a.imgs = static_cast<const uint8_t*>(p.batch_base);
    a.frame0 = int(p.batch_f0);
    a.n_frames = int(p.batch_n);
  } else {
    a.frame0 = 0;
    a.n_frames = 1 << 30;
  }
  (void)F;
  fixup_kernel<<<p.sm_count * 2, 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace scbm
