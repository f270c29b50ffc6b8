// plan.cpp -- the C ABI of include/sc_bm.h: validation, geometry, workspace, chunked
// norm -> match scheduling on the caller's stream, and the pipelined host-buffer path.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <new>

#include "sc_internal.h"

using namespace scbm;

namespace {

// keys re-ranked beyond K (every kernel checks whether the margin could have
// hidden a top-K candidate and sends such references to the exact fix-up): 4 (measured on c2, c4,
// c5-NCC: no reference reaches the fix-up, the shorter lists save 3-5 %), 8 for large K (c3's
// K = 70: margin 4 sends near-tie references to the fix-up, which costs more than it saves)
constexpr int kRescoreMargin = 4;
constexpr int kRescoreMarginLargeK = 8;
// NCC: 2 for uint8 (the integer fix-up is cheap: c5 sends 489 of 8.2M references to it and
// still gains 4 %), 4 for float input (its fp64 fix-up costs more than the shorter list saves)
constexpr int kNccMarginU8 = 2;
constexpr int kNccMarginF32 = 4;

sc_status_t cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return SC_OK;
  if (e == cudaErrorMemoryAllocation) return SC_ERR_OUT_OF_MEMORY;
  return SC_ERR_CUDA;
}

size_t elem_size(int dtype) { return dtype == SC_DTYPE_U8 ? 1 : 4; }

// Clipped window extent along one axis for a reference at r (readings R1/R3).
int64_t span(int r, int lo, int hi, int maxpos) {
  const int a = std::max(0, r + lo), b = std::min(maxpos, r + hi);
  return b >= a ? int64_t(b - a + 1) : 0;
}

// u8 norms come from a direct box filter (no integral image workspace); f32 from an fp64 SAT.
size_t per_frame_ws(const Geometry& g, int nbands) {
  const size_t SP = size_t((g.W + 15) / 16 * 16);
  const size_t nmap = size_t(g.NFS) * 4;
  if (g.dtype == SC_DTYPE_U8) return nmap;
  return SP * g.H * 8 + SP * nbands * 8 + nmap;
}

sc_status_t check_device(const sc_bm_plan_s* p) {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) return SC_ERR_CUDA;
  return dev == p->device ? SC_OK : SC_ERR_WRONG_DEVICE;
}

void free_ws(sc_bm_plan_s* p) {
  if (p->ws.sat) cudaFree(p->ws.sat);
  if (p->ws.bandsum) cudaFree(p->ws.bandsum);
  if (p->ws.norm_base) cudaFree(p->ws.norm_base);
  if (p->ws.fix_count) cudaFree(p->ws.fix_count);
  if (p->ws.fix_list) cudaFree(p->ws.fix_list);
  p->ws = Workspace{};
}

void free_host(sc_bm_plan_s* p) {
  HostStaging& h = p->host;
  if (!h.ready) return;
  for (int i = 0; i < 2; ++i) {
    cudaFree(h.d_img[i]);
    cudaFree(h.d_idx[i]);
    cudaFree(h.d_dist[i]);
    cudaEventDestroy(h.ev_in[i]);
    cudaEventDestroy(h.ev_done[i]);
    cudaEventDestroy(h.ev_out[i]);
  }
  cudaStreamDestroy(h.copy_in);
  cudaStreamDestroy(h.copy_out);
  if (h.d_tail) cudaFree(h.d_tail);
  h = HostStaging{};
}

// Enqueue norm + match for images [0, n) of imgs, chunked so the norm workspace of a chunk
// stays resident in L2 while its matching kernel runs.
sc_status_t enqueue(sc_bm_plan_s* p, const void* imgs, int64_t n, int iy_begin, int iy_end,
                    int32_t* idx, void* dist, void* dense, cudaStream_t st, int64_t f_begin = 0,
                    int64_t f_end = -1) {
  // reference frames [f_begin, f_end) of the n-frame batch at imgs (outputs start at f_begin);
  // temporal search reads candidates from every frame of the batch
  if (f_end < 0) f_end = n;
  const Geometry& g = p->g;
  const size_t img_bytes = size_t(g.C) * g.H * g.W * elem_size(g.dtype);
  const size_t out_elems = size_t(iy_end - iy_begin) * g.nx * g.K;
  const bool avg = p->nlm_avg_out != nullptr;  // sc_bm_nlm_average: the one-warp-per-reference matcher
  const int chunk = ((p->kernel == SC_KERNEL_BOX || p->kernel == SC_KERNEL_BOXF) && dense == nullptr && !avg) ? p->FB : p->F;
  for (int64_t f0 = f_begin; f0 < f_end; f0 += chunk) {
    const int F = int(std::min<int64_t>(chunk, f_end - f0));
    // (3D search: every launch reads the whole volume; its chunk of reference planes starts at f0)
    const void* src = g.z3 ? imgs : static_cast<const char*>(imgs) + f0 * img_bytes;
    cudaEvent_t* ev = nullptr;
    Timing& tm = p->timing;
    if (tm.enabled && size_t(tm.n_used + 1) * 3 <= tm.ev.size()) {
      ev = &tm.ev[size_t(tm.n_used) * 3];
      ++tm.n_used;
      cudaEventRecord(ev[0], st);
    }
    // the box-sum matcher forms the norms in registers; every other matcher reads the norm map
    const bool box = (p->kernel == SC_KERNEL_BOX || p->kernel == SC_KERNEL_BOXF) && dense == nullptr && !avg;
    cudaError_t e = box ? cudaSuccess : launch_norm(*p, src, F, st, &p->launches);
    if (e != cudaSuccess) return cuda_status(e);
    if (ev) cudaEventRecord(ev[1], st);
    p->batch_base = imgs;  // temporal search reads the neighbouring frames of the whole batch
    p->batch_f0 = f0;
    p->batch_n = n;
    p->packed_f0 = p->packed_base + (f0 - f_begin);  // packed tables: overflow records' row numbers
    int32_t* io = idx ? idx + (f0 - f_begin) * out_elems : nullptr;
    void* dd = dist ? static_cast<char*>(dist) + (f0 - f_begin) * out_elems * 4 : nullptr;
    if (avg)
      e = launch_bm_simt(*p, src, F, iy_begin, iy_end, io, dd, nullptr, st, &p->launches);
    else if (p->kernel == SC_KERNEL_TC_I8 && dense == nullptr)
      e = launch_bm_tc(*p, src, F, iy_begin, iy_end, io, dd, st, &p->launches);
    else if (p->kernel == SC_KERNEL_TC_F32 && !(dense != nullptr && p->nlm_inv_h2 > 0.f))
      e = launch_bm_tcf(*p, src, F, iy_begin, iy_end, io, dd, dense, st, &p->launches);
    else if (p->kernel == SC_KERNEL_BOX && dense == nullptr)
      e = launch_bm_box(*p, src, F, iy_begin, iy_end, io, dd, st, &p->launches);
    else if (p->kernel == SC_KERNEL_BOXF && dense == nullptr)
      e = launch_bm_boxf(*p, src, F, iy_begin, iy_end, io, dd, st, &p->launches);
    else if (p->kernel == SC_KERNEL_SIMT_WARP ||
             (dense != nullptr && (p->kernel == SC_KERNEL_BOX || p->kernel == SC_KERNEL_BOXF ||
                                   p->kernel == SC_KERNEL_TC_F32)))
      // dense tables (NLM weights, debug): one warp per reference, lanes along its window row, so
      // the [refs][Wn^2] rows are written contiguously
      e = launch_bm_simt(*p, src, F, iy_begin, iy_end, io, dd, dense, st, &p->launches);
    else
      e = launch_bm_lanes(*p, src, F, iy_begin, iy_end, io, dd, dense, st, &p->launches);
    if (e != cudaSuccess) return cuda_status(e);
    if (ev) cudaEventRecord(ev[2], st);
  }
  return SC_OK;
}

// packed tables: the plan can pack now (matcher, temporal radius) -- checked at every packed run
bool packed_ok(const sc_bm_plan_s* p) { return p->kernel == SC_KERNEL_BOX && p->T == 0; }

}  // namespace

extern "C" {

const char* sc_status_string(sc_status_t s) {
  switch (s) {
    case SC_OK: return "SC_OK";
    case SC_ERR_INVALID_ARGUMENT: return "SC_ERR_INVALID_ARGUMENT";
    case SC_ERR_UNSUPPORTED: return "SC_ERR_UNSUPPORTED";
    case SC_ERR_OUT_OF_MEMORY: return "SC_ERR_OUT_OF_MEMORY";
    case SC_ERR_CUDA: return "SC_ERR_CUDA";
    case SC_ERR_WRONG_DEVICE: return "SC_ERR_WRONG_DEVICE";
    case SC_ERR_OVERFLOW: return "SC_ERR_OVERFLOW";
  }
  return "SC_ERR_UNKNOWN";
}

sc_status_t sc_bm_plan(int H, int W, int C, int b, int stride, int window, int K, sc_dtype_t dtype,
                       sc_bm_plan_t* plan_out) {
  return sc_bm_plan_ex(H, W, C, b, stride, window, K, dtype, SC_METRIC_L2, plan_out);
}

sc_status_t sc_bm_plan_ex(int H, int W, int C, int b, int stride, int window, int K, sc_dtype_t dtype,
                          sc_metric_t metric, sc_bm_plan_t* plan_out) {
  if (!plan_out) return SC_ERR_INVALID_ARGUMENT;
  *plan_out = nullptr;
  if (b < 1 || b > 16 || C < 1 || C > 8 || stride < 1 || window < 1 || window > 255 || K < 1 ||
      K > 128 || H < b || W < b || int64_t(H) * W >= (int64_t(1) << 31) ||
      (dtype != SC_DTYPE_U8 && dtype != SC_DTYPE_F32) || (metric != SC_METRIC_L2 && metric != SC_METRIC_NCC))
    return SC_ERR_INVALID_ARGUMENT;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return SC_ERR_CUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return SC_ERR_CUDA;
  if (prop.major < 10) return SC_ERR_UNSUPPORTED;  // built for sm_100a only

  sc_bm_plan_s* p = new (std::nothrow) sc_bm_plan_s();
  if (!p) return SC_ERR_OUT_OF_MEMORY;
  p->device = dev;
  p->sm_count = prop.multiProcessorCount;
  Geometry& g = p->g;
  g.H = H; g.W = W; g.C = C; g.b = b; g.s = stride; g.Wn = window; g.K = K;
  g.dtype = dtype;
  g.ny = (H - b) / stride + 1;
  g.nx = (W - b) / stride + 1;
  g.lo = -(window / 2);
  g.hi = window - 1 - window / 2;
  g.My = H - b + 1;
  g.Mx = W - b + 1;
  // norm-map border: wide enough for every out-of-image candidate the box-sum matcher touches
  // (window offsets + its 8-row / 16-row register blocks), a multiple of 4 so rows stay 16-B aligned
  g.NPAD = (std::max(-g.lo, g.hi) + 24 + 3) & ~3;
  g.Mxp = (g.Mx + 2 * g.NPAD + 3) & ~3;
  g.NFS = (long long)(g.My + 2 * g.NPAD) * g.Mxp;
  g.metric = metric;
  g.KP = metric == SC_METRIC_NCC ? K + (dtype == SC_DTYPE_U8 ? kNccMarginU8 : kNccMarginF32)
         : dtype == SC_DTYPE_F32 ? K + (K > 48 ? kRescoreMarginLargeK : kRescoreMargin) : K;
  if (metric == SC_METRIC_NCC && !boxf_supported(g) && !box_supported(g)) {  // NCC: box kernels only
    delete p;
    return SC_ERR_UNSUPPORTED;
  }

  // candidate counts (separable: clipped rows x clipped cols)
  int64_t sy = 0, sx = 0, ymin = INT64_MAX, ymax = 0, xmin = INT64_MAX, xmax = 0;
  for (int iy = 0; iy < g.ny; ++iy) {
    const int64_t v = span(iy * stride, g.lo, g.hi, H - b);
    sy += v; ymin = std::min(ymin, v); ymax = std::max(ymax, v);
  }
  for (int ix = 0; ix < g.nx; ++ix) {
    const int64_t v = span(ix * stride, g.lo, g.hi, W - b);
    sx += v; xmin = std::min(xmin, v); xmax = std::max(xmax, v);
  }
  p->total_cand = sy * sx;
  p->min_cand = ymin * xmin;
  p->max_cand = ymax * xmax;

  p->nbands = (H + kSatBand - 1) / kSatBand;
  // frames per chunk: keep one chunk's workspace (u8: norm map; f32: SAT + norm map) L2-resident
  // between the norm kernels and the matcher (126 MB L2)
  const size_t pf = per_frame_ws(g, p->nbands);
  const size_t budget = (dtype == SC_DTYPE_U8 ? 80u : 48u) << 20;
  p->F = int(std::max<size_t>(1, std::min<size_t>(64, budget / std::max<size_t>(pf, 1))));
  p->tile = choose_simt_tile(g, p->sm_count, p->F);
  p->lanes_nwy = lanes_warps_for(g, p->sm_count, p->F);
  // Default matcher: lanes = references where its 32-reference-wide CTA keeps >= 4 warps per
  // CTA in shared memory (u8 frames such as c5); the one-warp-per-reference kernel otherwise
  // (f32 / multi-channel / large K / narrow images, where it measured faster: DESIGN.md s7).
  const bool lanes_ok = dtype == SC_DTYPE_U8 && g.nx >= 64 && p->lanes_nwy >= 4 &&
                        lanes_smem_bytes(g, p->lanes_nwy) <= 227 * 1024;
  p->kernel = lanes_ok ? SC_KERNEL_SIMT : SC_KERNEL_SIMT_WARP;
  // u8, b = 8, s = 4 (config c5): the box-sum matcher (7 dp4a per pair instead of 16 + norm pass).
  // Its CTA covers 16 x 31 references; on small images (c1: 15 x 15 references = 1 CTA) the
  // one-warp-per-reference kernel spreads the work over more SMs and measured faster.
  const int64_t box_ctas = int64_t((g.ny + 15) / 16) * ((g.nx + 30) / 31);
  if (box_supported(g) && box_ctas >= 16) p->kernel = SC_KERNEL_BOX;
  // f32, one channel, (s, b) in {(3,8), (1,7), (4,8), (2,8)}, K + 8 <= 80 (c2, c3): the float
  // box-sum matcher
  if (boxf_supported(g)) p->kernel = SC_KERNEL_BOXF;
  // f32, one channel, stride 1 (c3): the 3xTF32 tensor-core matcher, where its layout leaves two
  // CTAs per SM -- stride-1 strips cost the float box kernel a 4-shuffle tree per pair (c3: 4.60 vs
  // 5.02 ms); with larger strides the box kernel's shared strips win (c2)
  if (metric == SC_METRIC_L2 && tcf_preferred(g)) p->kernel = SC_KERNEL_TC_F32;
  if (metric == SC_METRIC_NCC)  // uint8 stride 4: the dp4a box kernel; else the float one
    p->kernel = (box_supported(g) && (box_ctas >= 16 || !boxf_supported(g))) ? SC_KERNEL_BOX : SC_KERNEL_BOXF;

  const size_t SP = size_t((W + 15) / 16 * 16);
  cudaError_t e = cudaSuccess;
  if (dtype == SC_DTYPE_F32) {
    e = cudaMalloc(&p->ws.sat, SP * H * 8 * p->F);
    if (e == cudaSuccess) e = cudaMalloc(&p->ws.bandsum, SP * p->nbands * 8 * p->F);
  }
  const size_t nbytes = (size_t(g.NFS) * p->F + 64) * 4;
  if (e == cudaSuccess) e = cudaMalloc(&p->ws.norm_base, nbytes);
  // border value 0x7f7f7f7f (u8: 2.14e9, far above any threshold; f32: 3.4e38); the interior is
  // rewritten by every run
  if (e == cudaSuccess) e = cudaMemset(p->ws.norm_base, 0x7f, nbytes);
  if (e == cudaSuccess)
    p->ws.norm = static_cast<char*>(p->ws.norm_base) + (size_t(g.NPAD) * g.Mxp + g.NPAD) * 4;
  if (e == cudaSuccess) e = cudaMalloc(&p->ws.fix_count, sizeof(int));
  // box matchers: up to 64 frames per launch, the fix-up list capped at 16 M entries
  p->FB = int(std::max<int64_t>(1, std::min<int64_t>(64, (int64_t(16) << 20) / (int64_t(g.ny) * g.nx))));
  if (e == cudaSuccess)
    e = cudaMalloc(&p->ws.fix_list, size_t(g.ny) * g.nx * sizeof(int) * std::max(p->F, p->FB));
  if (e == cudaSuccess) e = cudaMemset(p->ws.fix_count, 0, sizeof(int));
  if (e != cudaSuccess) {
    free_ws(p);
    delete p;
    cudaGetLastError();
    return cuda_status(e);
  }
  p->ws.bytes = per_frame_ws(g, p->nbands) * p->F;
  *plan_out = p;
  return SC_OK;
}

sc_status_t sc_bm_run_rows(sc_bm_plan_t p, const void* imgs, int64_t n_images, int32_t iy_begin,
                           int32_t iy_end, int32_t* idx_out, void* dist_out, sc_stream_t stream) {
  if (!p || !imgs || !idx_out || n_images < 0) return SC_ERR_INVALID_ARGUMENT;
  // packed tables: idx_out is the packed buffer, dist_out NULL, whole images only
  if ((p->packed_cap > 0) != (dist_out == nullptr)) return SC_ERR_INVALID_ARGUMENT;
  if (p->packed_cap > 0 && !(packed_ok(p) && iy_begin == 0 && iy_end == p->g.ny)) return SC_ERR_UNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(imgs) & 15) != 0) return SC_ERR_INVALID_ARGUMENT;
  if (iy_begin < 0 || iy_end > p->g.ny || iy_end < iy_begin) return SC_ERR_INVALID_ARGUMENT;
  if (p->g.z3) return SC_ERR_UNSUPPORTED;  // a 3D plan runs volumes (sc_bm_run3d)
  // temporal search reports batch-global idx = frame * H * W + pixel, which must stay int32
  if (p->T > 0 && n_images * int64_t(p->g.H) * p->g.W > (int64_t(1) << 31)) return SC_ERR_INVALID_ARGUMENT;
  sc_status_t s = check_device(p);
  if (s != SC_OK) return s;
  if (p->packed_cap > 0) {  // the overflow area follows the rows: header first
    p->packed_tail = reinterpret_cast<uint32_t*>(idx_out) + size_t(n_images) * p->g.ny * p->g.nx * p->g.K;
    p->packed_base = 0;
    cudaError_t e = launch_packed_init(p->packed_tail, p->packed_cap, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_status(e);
    ++p->launches;
  }
  if (n_images == 0 || iy_end == iy_begin) return SC_OK;
  return enqueue(p, imgs, n_images, iy_begin, iy_end, idx_out, dist_out, nullptr,
                 reinterpret_cast<cudaStream_t>(stream));
}

sc_status_t sc_bm_run_temporal(sc_bm_plan_t p, const void* imgs, int64_t n_images, int64_t f_begin,
                               int64_t f_end, int64_t frame_offset, int32_t* idx_out, void* dist_out,
                               sc_stream_t stream) {
  if (p && p->g.z3) return SC_ERR_UNSUPPORTED;  // a 3D plan runs volumes (sc_bm_run3d)
  if (!p || !imgs || !idx_out || !dist_out || n_images < 0) return SC_ERR_INVALID_ARGUMENT;
  if (p->packed_cap > 0) return SC_ERR_UNSUPPORTED;  // (batch-global idx: plain tables only)
  if ((reinterpret_cast<uintptr_t>(imgs) & 15) != 0) return SC_ERR_INVALID_ARGUMENT;
  if (f_begin < 0 || f_end > n_images || f_end < f_begin) return SC_ERR_INVALID_ARGUMENT;
  if (p->T == 0) return SC_ERR_UNSUPPORTED;  // sc_bm_run_batch on imgs + f_begin frames does it
  if (frame_offset < 0 || (frame_offset + n_images) * int64_t(p->g.H) * p->g.W > (int64_t(1) << 31))
    return SC_ERR_INVALID_ARGUMENT;  // the offset batch-global idx must stay int32
  sc_status_t s = check_device(p);
  if (s != SC_OK) return s;
  if (f_end == f_begin) return SC_OK;
  p->idx_frame_off = frame_offset;
  s = enqueue(p, imgs, n_images, 0, p->g.ny, idx_out, dist_out, nullptr, reinterpret_cast<cudaStream_t>(stream),
              f_begin, f_end);
  p->idx_frame_off = 0;
  return s;
}

sc_status_t sc_bm_plan3d(int H, int W, int d, int b, int stride, int window, int z_stride, int z_window, int K,
                         sc_dtype_t dtype, sc_bm_plan_t* plan_out) {
  if (!plan_out) return SC_ERR_INVALID_ARGUMENT;
  *plan_out = nullptr;
  if (z_stride < 1 || z_window < 1 || z_window > 64) return SC_ERR_INVALID_ARGUMENT;
  if (dtype != SC_DTYPE_F32) return SC_ERR_UNSUPPORTED;  // (uint8 video: sc_bm_set_temporal)
  sc_bm_plan_t p = nullptr;
  sc_status_t st = sc_bm_plan_ex(H, W, d, b, stride, window, K, dtype, SC_METRIC_L2, &p);
  if (st != SC_OK) return st;
  p->g.z3 = 1;
  p->g.zwin = z_window;
  p->zstride = z_stride;
  p->zlo = -(z_window / 2);
  p->zhi = z_window - 1 - z_window / 2;
  if (!boxf_supported(p->g)) {
    sc_bm_destroy(p);
    return SC_ERR_UNSUPPORTED;
  }
  p->kernel = SC_KERNEL_BOXF;
  *plan_out = p;
  return SC_OK;
}

sc_status_t sc_bm_run3d(sc_bm_plan_t p, const void* vol, int64_t n_planes, int32_t* idx_out, void* dist_out,
                        sc_stream_t stream) {
  if (!p || !vol || !idx_out || !dist_out) return SC_ERR_INVALID_ARGUMENT;
  if (!p->g.z3) return SC_ERR_UNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(vol) & 15) != 0) return SC_ERR_INVALID_ARGUMENT;
  if (n_planes < p->g.C || n_planes * int64_t(p->g.H) * p->g.W > (int64_t(1) << 31)) return SC_ERR_INVALID_ARGUMENT;
  sc_status_t s = check_device(p);
  if (s != SC_OK) return s;
  const int64_t nz = (n_planes - p->g.C) / p->zstride + 1;
  p->n_planes = n_planes;
  return enqueue(p, vol, nz, 0, p->g.ny, idx_out, dist_out, nullptr, reinterpret_cast<cudaStream_t>(stream));
}

sc_status_t sc_bm_run_batch(sc_bm_plan_t p, const void* imgs, int64_t n_images, int32_t* idx_out,
                            void* dist_out, sc_stream_t stream) {
  if (!p) return SC_ERR_INVALID_ARGUMENT;
  return sc_bm_run_rows(p, imgs, n_images, 0, p->g.ny, idx_out, dist_out, stream);
}

sc_status_t sc_bm_run(sc_bm_plan_t p, const void* img, int32_t* idx_out, void* dist_out,
                      sc_stream_t stream) {
  return sc_bm_run_batch(p, img, 1, idx_out, dist_out, stream);
}

sc_status_t sc_bm_run_dense_debug(sc_bm_plan_t p, const void* img, void* dist_all, sc_stream_t stream) {
  if (p && p->g.z3) return SC_ERR_UNSUPPORTED;  // a 3D plan runs volumes (sc_bm_run3d)
  if (!p || !img || !dist_all) return SC_ERR_INVALID_ARGUMENT;
  if (p->g.metric != SC_METRIC_L2) return SC_ERR_UNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(img) & 15) != 0) return SC_ERR_INVALID_ARGUMENT;
  sc_status_t s = check_device(p);
  if (s != SC_OK) return s;
  return enqueue(p, img, 1, 0, p->g.ny, nullptr, nullptr, dist_all,
                 reinterpret_cast<cudaStream_t>(stream));
}

sc_status_t sc_bm_debug_fix_count(sc_bm_plan_t p, int32_t* count_out) {
  if (!p || !count_out) return SC_ERR_INVALID_ARGUMENT;
  sc_status_t s = check_device(p);
  if (s != SC_OK) return s;
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(count_out, p->ws.fix_count, sizeof(int32_t), cudaMemcpyDeviceToHost);
  return cuda_status(e);
}

sc_status_t sc_bm_nlm_weights(sc_bm_plan_t p, const void* img, float h, float* weights_out, sc_stream_t stream) {
  if (p && p->g.z3) return SC_ERR_UNSUPPORTED;  // a 3D plan runs volumes (sc_bm_run3d)
  if (!p || !img || !weights_out || !(h > 0.f) || !std::isfinite(h)) return SC_ERR_INVALID_ARGUMENT;
  if (p->g.metric != SC_METRIC_L2) return SC_ERR_UNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(img) & 15) != 0 || (reinterpret_cast<uintptr_t>(weights_out) & 3) != 0)
    return SC_ERR_INVALID_ARGUMENT;
  sc_status_t s = check_device(p);
  if (s != SC_OK) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // the window distances of every reference (Self-Convolution identity), written into the output;
  // the one-warp-per-reference dense matcher normalises its own row in its epilogue (nlm.cuh),
  // the lanes matcher (an explicit SC_KERNEL_SIMT choice) is followed by nlm_normalize
  const bool fused = p->kernel == SC_KERNEL_SIMT_WARP || p->kernel == SC_KERNEL_BOX || p->kernel == SC_KERNEL_BOXF ||
                     p->kernel == SC_KERNEL_TC_F32;
  p->nlm_inv_h2 = fused ? 1.f / (h * h) : 0.f;
  s = enqueue(p, img, 1, 0, p->g.ny, nullptr, nullptr, weights_out, st);
  p->nlm_inv_h2 = 0.f;
  if (s != SC_OK || fused) return s;
  return cuda_status(launch_nlm_normalize(*p, weights_out, h, st, &p->launches));
}

sc_status_t sc_bm_nlm_average(sc_bm_plan_t p, const void* img, float h, float* out, sc_stream_t stream) {
  if (p && p->g.z3) return SC_ERR_UNSUPPORTED;  // a 3D plan runs volumes (sc_bm_run3d)
  if (!p || !img || !out || !(h > 0.f) || !std::isfinite(h)) return SC_ERR_INVALID_ARGUMENT;
  if (p->g.metric != SC_METRIC_L2 || p->g.b * p->g.b * p->g.C > 256) return SC_ERR_UNSUPPORTED;
  if ((reinterpret_cast<uintptr_t>(img) & 15) != 0 || (reinterpret_cast<uintptr_t>(out) & 3) != 0)
    return SC_ERR_INVALID_ARGUMENT;
  sc_status_t s = check_device(p);
  if (s != SC_OK) return s;
  // window distances from the Self-Convolution identity, weights and the weighted patch sum fused
  // in the one-warp-per-reference matcher's epilogue (bm_simt.cu, AVG): no weight table
  p->nlm_inv_h2 = 1.f / (h * h);
  p->nlm_avg_out = out;
  s = enqueue(p, img, 1, 0, p->g.ny, nullptr, nullptr, nullptr, reinterpret_cast<cudaStream_t>(stream));
  p->nlm_avg_out = nullptr;
  p->nlm_inv_h2 = 0.f;
  return s;
}

sc_status_t sc_bm_norm_map(sc_bm_plan_t p, const void* img, void* norm_out, sc_stream_t stream) {
  if (p && p->g.z3) return SC_ERR_UNSUPPORTED;  // a 3D plan runs volumes (sc_bm_run3d)
  if (!p || !img || !norm_out) return SC_ERR_INVALID_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(img) & 15) != 0) return SC_ERR_INVALID_ARGUMENT;
  sc_status_t s = check_device(p);
  if (s != SC_OK) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = launch_norm(*p, img, 1, st, &p->launches);
  if (e != cudaSuccess) return cuda_status(e);
  e = cudaMemcpy2DAsync(norm_out, size_t(p->g.Mx) * 4, p->ws.norm, size_t(p->g.Mxp) * 4, size_t(p->g.Mx) * 4,
                        p->g.My, cudaMemcpyDeviceToDevice, st);
  return cuda_status(e);
}

sc_status_t sc_bm_run_host(sc_bm_plan_t p, const void* h_imgs, int64_t n_images, int32_t* h_idx,
                           void* h_dist, sc_stream_t stream) {
  if (p && p->g.z3) return SC_ERR_UNSUPPORTED;  // a 3D plan runs volumes (sc_bm_run3d)
  if (!p || !h_imgs || !h_idx || n_images < 0) return SC_ERR_INVALID_ARGUMENT;
  if ((p->packed_cap > 0) != (h_dist == nullptr)) return SC_ERR_INVALID_ARGUMENT;  // packed: h_idx only
  if (p->T > 0) return SC_ERR_UNSUPPORTED;  // chunked staging has no neighbouring frames
  if (p->packed_cap > 0 && !packed_ok(p)) return SC_ERR_UNSUPPORTED;
  sc_status_t s = check_device(p);
  if (s != SC_OK) return s;
  if (n_images == 0) return SC_OK;
  const Geometry& g = p->g;
  HostStaging& h = p->host;
  const size_t img_bytes = size_t(g.C) * g.H * g.W * elem_size(g.dtype);
  const size_t out_elems = size_t(g.ny) * g.nx * g.K;
  cudaError_t e = cudaSuccess;
  if (!h.ready) {
    // frames per pipeline stage: small enough that filling (first H2D + match) and draining (last
    // D2H) the pipeline stay short against the PCIe-bound copies (~24 MB of results per stage:
    // one c5 frame; 48 and 100 MB measured 1-3 % slower),
    // at most the plan's workspace chunk
    const size_t out_frame = out_elems * 8;
#ifndef SCBM_HOST_STAGE_MB
#define SCBM_HOST_STAGE_MB 24
#endif
    h.F = int(std::max<size_t>(1, std::min<size_t>(size_t(p->F), (size_t(SCBM_HOST_STAGE_MB) << 20) / std::max<size_t>(out_frame, 1))));
    // packed tables (box matcher only): stages of several frames -- one frame's box launch (c5: 270
    // CTAs, one partial wave) would take longer than its 8 MB copy
#ifndef SCBM_HOST_STAGE_MB_PACKED
#define SCBM_HOST_STAGE_MB_PACKED 40
#endif
    h.Fp = int(std::max<size_t>(1, std::min<size_t>(size_t(p->FB), (size_t(SCBM_HOST_STAGE_MB_PACKED) << 20) / std::max<size_t>(out_elems * 4, 1))));
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
      e = cudaMalloc(&h.d_img[i], img_bytes * std::max(h.F, h.Fp));
      if (e == cudaSuccess) e = cudaMalloc(&h.d_idx[i], out_elems * 4 * std::max(h.F, h.Fp));
      if (e == cudaSuccess) e = cudaMalloc(&h.d_dist[i], out_elems * 4 * h.F);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h.ev_in[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h.ev_done[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h.ev_out[i], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h.copy_in, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h.copy_out, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      h.ready = true;
      free_host(p);
      cudaGetLastError();
      return cuda_status(e);
    }
    h.ready = true;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool packed = p->packed_cap > 0;
  const size_t rec_words = size_t(packed_record_words(g));
  if (packed) {  // the run's overflow area lives on the device until the end of the run
    if (h.tail_cap != p->packed_cap) {
      if (h.d_tail) cudaFree(h.d_tail);
      h.d_tail = nullptr;
      h.tail_cap = -1;
      e = cudaMalloc(&h.d_tail, (2 + size_t(p->packed_cap) * rec_words) * 4);
      if (e != cudaSuccess) {
        h.d_tail = nullptr;
        cudaGetLastError();
        return cuda_status(e);
      }
      h.tail_cap = p->packed_cap;
    }
    p->packed_tail = h.d_tail;
    e = launch_packed_init(h.d_tail, p->packed_cap, st);
    if (e != cudaSuccess) return cuda_status(e);
    ++p->launches;
  }
  // double-buffered pipeline: H2D(chunk k+1) || match(chunk k) || D2H(chunk k-1)
  int64_t k = 0;
  const int FS = packed ? h.Fp : h.F;
  for (int64_t f0 = 0; f0 < n_images; f0 += FS, ++k) {
    const int slot = int(k & 1);
    const int F = int(std::min<int64_t>(FS, n_images - f0));
    if (k >= 2) cudaStreamWaitEvent(h.copy_in, h.ev_out[slot], 0);  // slot's D2H finished
    e = cudaMemcpyAsync(h.d_img[slot], static_cast<const char*>(h_imgs) + f0 * img_bytes,
                        img_bytes * F, cudaMemcpyHostToDevice, h.copy_in);
    if (e != cudaSuccess) return cuda_status(e);
    cudaEventRecord(h.ev_in[slot], h.copy_in);
    cudaStreamWaitEvent(st, h.ev_in[slot], 0);
    // one-frame stages with a large table (c3: 143 MB) are split into reference-row bands so the
    // D2H of band b overlaps the matching of band b+1
    const size_t row_elems = size_t(g.nx) * g.K;
    const size_t stage_bytes = size_t(48) << 20;
    const int nb = F == 1 ? int(std::max<size_t>(1, std::min<size_t>(size_t(g.ny), (out_elems * 8 + stage_bytes - 1) / stage_bytes))) : 1;
    for (int bi = 0; bi < nb; ++bi) {
      const int y0 = int(int64_t(g.ny) * bi / nb), y1 = int(int64_t(g.ny) * (bi + 1) / nb);
      const size_t off = size_t(y0) * row_elems, cnt = (nb == 1 ? out_elems * F : size_t(y1 - y0) * row_elems);
      p->packed_base = f0;
      s = enqueue(p, h.d_img[slot], F, nb == 1 ? 0 : y0, nb == 1 ? g.ny : y1, h.d_idx[slot] + off,
                  packed ? nullptr : static_cast<char*>(h.d_dist[slot]) + off * 4, nullptr, st);
      p->packed_base = 0;
      if (s != SC_OK) return s;
      cudaEventRecord(h.ev_done[slot], st);
      cudaStreamWaitEvent(h.copy_out, h.ev_done[slot], 0);
      e = cudaMemcpyAsync(h_idx + f0 * out_elems + off, h.d_idx[slot] + off, cnt * 4, cudaMemcpyDeviceToHost,
                          h.copy_out);
      if (e == cudaSuccess && !packed)
        e = cudaMemcpyAsync(static_cast<char*>(h_dist) + (f0 * out_elems + off) * 4,
                            static_cast<char*>(h.d_dist[slot]) + off * 4, cnt * 4, cudaMemcpyDeviceToHost, h.copy_out);
      if (e != cudaSuccess) return cuda_status(e);
    }
    cudaEventRecord(h.ev_out[slot], h.copy_out);
  }
  e = cudaStreamSynchronize(h.copy_out);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess && packed) {  // the overflow area after the host rows: header, then the records
    uint32_t* htail = reinterpret_cast<uint32_t*>(h_idx) + size_t(n_images) * out_elems;
    e = cudaMemcpy(htail, h.d_tail, 8, cudaMemcpyDeviceToHost);
    const size_t nrec = e == cudaSuccess ? std::min<size_t>(htail[0], size_t(p->packed_cap)) : 0;
    if (e == cudaSuccess && nrec > 0)
      e = cudaMemcpy(htail + 2, h.d_tail + 2, nrec * rec_words * 4, cudaMemcpyDeviceToHost);
  }
  return cuda_status(e);
}

sc_status_t sc_bm_group(sc_bm_plan_t p, const void* imgs, int64_t n_images, const int32_t* idx,
                        void* groups_out, sc_stream_t stream) {
  if (p && p->g.z3) return SC_ERR_UNSUPPORTED;  // a 3D plan runs volumes (sc_bm_run3d)
  if (!p || !imgs || !idx || !groups_out || n_images < 0) return SC_ERR_INVALID_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(imgs) & 15) != 0 || (reinterpret_cast<uintptr_t>(groups_out) & 15) != 0 ||
      (reinterpret_cast<uintptr_t>(idx) & 3) != 0)
    return SC_ERR_INVALID_ARGUMENT;
  sc_status_t s = check_device(p);
  if (s != SC_OK) return s;
  if (n_images == 0) return SC_OK;
  return cuda_status(launch_group(*p, imgs, n_images, idx, groups_out, reinterpret_cast<cudaStream_t>(stream),
                                  &p->launches));
}

sc_status_t sc_bm_plan_info(sc_bm_plan_t p, sc_bm_info_t* info) {
  if (!p || !info) return SC_ERR_INVALID_ARGUMENT;
  std::memset(info, 0, sizeof(*info));
  info->n_ref_y = p->g.ny;
  info->n_ref_x = p->g.nx;
  info->n_refs = int64_t(p->g.ny) * p->g.nx;
  info->min_candidates = p->min_cand;
  info->max_candidates = p->max_cand;
  info->total_candidates = p->total_cand;
  info->workspace_bytes = int64_t(p->ws.bytes);
  info->frames_per_chunk = (p->kernel == SC_KERNEL_BOX || p->kernel == SC_KERNEL_BOXF) ? p->FB : p->F;
  info->launches = p->launches;
  info->kernel = p->kernel;
  info->device = p->device;
  return SC_OK;
}

sc_status_t sc_bm_set_packed(sc_bm_plan_t p, int64_t cap_rows) {
  if (!p || cap_rows < 0 || cap_rows > (int64_t(1) << 30)) return SC_ERR_INVALID_ARGUMENT;
  const Geometry& g = p->g;
  if (cap_rows > 0 && (g.dtype != SC_DTYPE_U8 || g.metric != SC_METRIC_L2 || g.z3 || !box_supported(g)))
    return SC_ERR_UNSUPPORTED;
  p->packed_cap = cap_rows;
  return SC_OK;
}

sc_status_t sc_bm_packed_words(sc_bm_plan_t p, int64_t n_images, int64_t* words_out, int32_t* rel_bits_out) {
  if (!p || n_images < 0 || !words_out) return SC_ERR_INVALID_ARGUMENT;
  if (p->packed_cap <= 0) return SC_ERR_UNSUPPORTED;
  const Geometry& g = p->g;
  *words_out = n_images * g.ny * g.nx * g.K + 2 + p->packed_cap * packed_record_words(g);
  if (rel_bits_out) *rel_bits_out = packed_rel_bits(g);
  return SC_OK;
}

sc_status_t sc_bm_unpack(sc_bm_plan_t p, const uint32_t* packed, int64_t n_images, int32_t* idx_out,
                         int32_t* dist_out, sc_stream_t stream) {
  if (!p || !packed || !idx_out || !dist_out || n_images < 0) return SC_ERR_INVALID_ARGUMENT;
  if (p->packed_cap <= 0) return SC_ERR_UNSUPPORTED;
  sc_status_t s = check_device(p);
  if (s != SC_OK) return s;
  const Geometry& g = p->g;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint32_t hdr[2] = {0u, 0u};
  cudaError_t e = cudaMemcpyAsync(hdr, packed + size_t(n_images) * g.ny * g.nx * g.K, 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_status(e);
  if (hdr[0] > hdr[1]) return SC_ERR_OVERFLOW;  // escape rows whose records were lost
  e = launch_unpack(*p, packed, n_images, int64_t(hdr[0]), idx_out, dist_out, st);
  p->launches += hdr[0] > 0 ? 2 : 1;
  return cuda_status(e);
}

sc_status_t sc_bm_unpack_host(int H, int W, int b, int stride, int window, int K, const uint32_t* packed,
                              int64_t n_images, int32_t* idx_out, int32_t* dist_out) {
  if (!packed || !idx_out || !dist_out || n_images < 0) return SC_ERR_INVALID_ARGUMENT;
  if (H < b || W < b || b < 1 || stride < 1 || window < 1 || window > 255 || K < 1 || K > 128)
    return SC_ERR_INVALID_ARGUMENT;
  const int64_t ny = (H - b) / stride + 1, nx = (W - b) / stride + 1, nref = ny * nx;
  const int lo = -(window / 2), hi = window - 1 - window / 2;
  int rb = 0;
  while ((int64_t(1) << rb) < int64_t(window) * window) ++rb;
  if (rb < 2) rb = 2;
  const uint32_t mask = (1u << rb) - 1u;
  const int64_t rows = n_images * nref;
  for (int64_t r = 0; r < rows; ++r) {
    const int64_t j = r % nref;
    const int64_t ry = (j / nx) * stride, rx = (j % nx) * stride;
    for (int k = 0; k < K; ++k) {
      const uint32_t w = packed[r * K + k];
      int32_t idx = -1, dist = 0x7fffffff;
      if (w != 0xffffffffu) {
        const int slot = int(w & mask);
        if (slot >= window * window) return SC_ERR_INVALID_ARGUMENT;
        const int dy = slot / window + lo, dx = slot % window + lo;
        if (dy > hi || ry + dy < 0 || ry + dy > H - b || rx + dx < 0 || rx + dx > W - b) return SC_ERR_INVALID_ARGUMENT;
        idx = int32_t((ry + dy) * W + rx + dx);
        dist = int32_t(w >> rb);
      }
      idx_out[r * K + k] = idx;
      dist_out[r * K + k] = dist;
    }
  }
  const uint32_t* tail = packed + rows * K;
  if (tail[0] > tail[1]) return SC_ERR_OVERFLOW;
  for (uint32_t i = 0; i < tail[0]; ++i) {
    const uint32_t* rec = tail + 2 + size_t(i) * (2 + 2 * size_t(K));
    const int64_t row = int64_t(rec[0]) | (int64_t(rec[1]) << 32);
    if (row < 0 || row >= rows) return SC_ERR_INVALID_ARGUMENT;
    for (int k = 0; k < K; ++k) {
      idx_out[row * K + k] = int32_t(rec[2 + k]);
      dist_out[row * K + k] = int32_t(rec[2 + K + k]);
    }
  }
  return SC_OK;
}

sc_status_t sc_bm_set_temporal(sc_bm_plan_t p, int32_t T) {
  if (!p || T < 0) return SC_ERR_INVALID_ARGUMENT;
  if (p->g.z3) return SC_ERR_UNSUPPORTED;
  if (T > 0 && !box_temporal_supported(p->g, T)) return SC_ERR_UNSUPPORTED;
  if (T > 0 && p->T == 0) p->kernel_before_T = p->kernel;
  if (T == 0 && p->T > 0 && p->kernel_before_T >= 0) {  // back to the matcher the plan had
    p->kernel = p->kernel_before_T;
    p->kernel_before_T = -1;
  }
  p->T = T;
  if (T > 0) p->kernel = SC_KERNEL_BOX;  // the only matcher with a temporal window
  return SC_OK;
}

sc_status_t sc_bm_set_kernel(sc_bm_plan_t p, int32_t kernel) {
  if (!p) return SC_ERR_INVALID_ARGUMENT;
  if (p->T > 0 && kernel != SC_KERNEL_BOX) return SC_ERR_UNSUPPORTED;
  if (p->g.z3 && kernel != SC_KERNEL_BOXF) return SC_ERR_UNSUPPORTED;
  if (p->g.metric == SC_METRIC_NCC && kernel != SC_KERNEL_BOXF && kernel != SC_KERNEL_BOX) return SC_ERR_UNSUPPORTED;
  if (kernel == SC_KERNEL_SIMT && lanes_smem_bytes(p->g, p->lanes_nwy) > 227 * 1024) return SC_ERR_UNSUPPORTED;
  if (kernel == SC_KERNEL_TC_I8 && !tc_supported(p->g)) return SC_ERR_UNSUPPORTED;
  if (kernel == SC_KERNEL_BOX && !box_supported(p->g)) return SC_ERR_UNSUPPORTED;
  if (kernel == SC_KERNEL_BOXF && !boxf_supported(p->g)) return SC_ERR_UNSUPPORTED;
  if (kernel == SC_KERNEL_TC_F32 && !tcf_supported(p->g)) return SC_ERR_UNSUPPORTED;
  if (kernel != SC_KERNEL_SIMT && kernel != SC_KERNEL_SIMT_WARP && kernel != SC_KERNEL_TC_I8 &&
      kernel != SC_KERNEL_BOX && kernel != SC_KERNEL_BOXF && kernel != SC_KERNEL_TC_F32)
    return SC_ERR_UNSUPPORTED;
  p->kernel = kernel;
  return SC_OK;
}

sc_status_t sc_bm_set_timing(sc_bm_plan_t p, int32_t enable) {
  if (!p) return SC_ERR_INVALID_ARGUMENT;
  Timing& tm = p->timing;
  if (enable && tm.ev.empty()) {
    tm.ev.resize(3 * 8192);
    for (auto& e : tm.ev)
      if (cudaEventCreate(&e) != cudaSuccess) return SC_ERR_CUDA;
  }
  tm.enabled = enable != 0;
  tm.n_used = 0;
  return SC_OK;
}

sc_status_t sc_bm_get_timing(sc_bm_plan_t p, sc_bm_timing_t* out) {
  if (!p || !out) return SC_ERR_INVALID_ARGUMENT;
  std::memset(out, 0, sizeof(*out));
  Timing& tm = p->timing;
  for (int i = 0; i < tm.n_used; ++i) {
    cudaEvent_t* ev = &tm.ev[size_t(i) * 3];
    if (cudaEventSynchronize(ev[2]) != cudaSuccess) return SC_ERR_CUDA;
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    out->norm_ms += a;
    out->match_ms += b;
  }
  out->norm_chunks = tm.n_used;
  out->match_launches = tm.n_used;
  tm.n_used = 0;
  return SC_OK;
}

sc_status_t sc_bm_destroy(sc_bm_plan_t p) {
  if (!p) return SC_OK;
  for (auto& e : p->timing.ev) cudaEventDestroy(e);
  free_host(p);
  free_ws(p);
  delete p;
  return SC_OK;
}

}  // extern "C"
