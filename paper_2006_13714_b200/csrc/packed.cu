// packed.cu -- packed tables (sc_bm_set_packed): a lossless one-word-per-result
// encoding of the uint8 L2 output (Eq. 3) for the device->host copy and the
// multi-GPU gather, which the plain int32 (idx, dist) pair makes twice as large.
//
// Row word w = (dist << rb) | slot, slot = (cy - ry - lo) * Wn + (cx - rx - lo): exactly the box
// matcher's 32-bit register key (regtopk.cuh) for a row whose K-th key is unsaturated, so the
// matcher writes its keys as they are; the fix-up kernel (fixup.cu) encodes the rows it recomputes
// and sends rows that do not fit (a distance >= 2^(32-rb) - 1, or fewer than K candidates) to the
// overflow records after the rows (escape words 0xFFFFFFFF in the row). This file holds the
// overflow-area header and the device decode: idx = (ry + dy + lo) W + rx + dx + lo with
// (dy, dx) = (slot / Wn, slot % Wn), dist = w >> rb; then the records are patched in.
#include "sc_internal.h"

namespace scbm {
namespace {

__global__ void packed_init_kernel(uint32_t* tail, uint32_t cap) {
  tail[0] = 0u;  // escape rows written
  tail[1] = cap;
}

struct UnpackArgs {
  const uint32_t* pk;
  int32_t* idx;
  int32_t* dist;
  int per_img;  // n_refs * K words per image
  int K, nx, s, W, Wn, lo, rb;
};

// grid (x: words of an image, y: images); HBM-bound (4 B read, 8 B written per result)
__global__ void __launch_bounds__(256) unpack_kernel(UnpackArgs a) {
  const size_t base = size_t(blockIdx.y) * a.per_img;
  const uint32_t mask = (1u << a.rb) - 1u;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < a.per_img; e += gridDim.x * blockDim.x) {
    const uint32_t w = a.pk[base + e];
    const int r = e / a.K;
    const int iy = r / a.nx, ix = r - iy * a.nx;
    int32_t idx = -1, dist = 0x7fffffff;  // escape: patched from the overflow records
    if (w != 0xffffffffu) {
      const int slot = int(w & mask);
      const int dy = slot / a.Wn, dx = slot - dy * a.Wn;
      idx = (iy * a.s + dy + a.lo) * a.W + ix * a.s + dx + a.lo;
      dist = int32_t(w >> a.rb);
    }
    a.idx[base + e] = idx;
    a.dist[base + e] = dist;
  }
}

// one warp per overflow record: row (low, high), K idx, K dist
__global__ void __launch_bounds__(256) patch_kernel(const uint32_t* tail, int64_t n_records, int K, int32_t* idx,
                                                    int32_t* dist) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < n_records; r += nw) {
    const uint32_t* rec = tail + 2 + r * (2 + 2 * int64_t(K));
    const int64_t row = int64_t(rec[0]) | (int64_t(rec[1]) << 32);
    for (int k = lane; k < K; k += 32) {
      idx[row * K + k] = int32_t(rec[2 + k]);
      dist[row * K + k] = int32_t(rec[2 + K + k]);
    }
  }
}

}  // namespace

int packed_rel_bits(const Geometry& g) {
  int rb = 0;
  while ((1ll << rb) < (long long)g.Wn * g.Wn) ++rb;
  return rb < 2 ? 2 : rb;
}

int64_t packed_record_words(const Geometry& g) { return 2 + 2 * int64_t(g.K); }

cudaError_t launch_packed_init(uint32_t* tail, int64_t cap, cudaStream_t st) {
  packed_init_kernel<<<1, 1, 0, st>>>(tail, uint32_t(cap));
  return cudaGetLastError();
}

cudaError_t launch_unpack(const sc_bm_plan_s& p, const uint32_t* packed, int64_t n_images, int64_t n_records,
                          int32_t* idx_out, int32_t* dist_out, cudaStream_t st) {
  const Geometry& g = p.g;
  UnpackArgs a{};
  a.pk = packed;
  a.idx = idx_out;
  a.dist = dist_out;
  a.per_img = g.ny * g.nx * g.K;
  a.K = g.K; a.nx = g.nx; a.s = g.s; a.W = g.W; a.Wn = g.Wn; a.lo = g.lo;
  a.rb = packed_rel_bits(g);
  for (int64_t i0 = 0; i0 < n_images; i0 += 65535) {  // grid.y limit
    const int ni = int(n_images - i0 < 65535 ? n_images - i0 : 65535);
    UnpackArgs b = a;
    b.pk = a.pk + size_t(i0) * a.per_img;
    b.idx = a.idx + size_t(i0) * a.per_img;
    b.dist = a.dist + size_t(i0) * a.per_img;
    const int gx = (a.per_img + 255) / 256 < 4 * p.sm_count ? (a.per_img + 255) / 256 : 4 * p.sm_count;
    unpack_kernel<<<dim3(gx > 0 ? gx : 1, ni), 256, 0, st>>>(b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (n_records > 0) {
    const uint32_t* tail = packed + size_t(n_images) * a.per_img;
    const int64_t blocks = (n_records * 32 + 255) / 256;
    patch_kernel<<<int(blocks < 8 * p.sm_count ? blocks : 8 * p.sm_count), 256, 0, st>>>(tail, n_records, g.K,
                                                                                          idx_out, dist_out);
    return cudaGetLastError();
  }
  return cudaSuccess;
}

}  // namespace scbm
