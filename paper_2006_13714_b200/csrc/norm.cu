// norm.cu -- step a1: h_X (.) h_X (used by Lemma 2) for every
// candidate position, via an integral image (summed-area table) of the squared centred image.
//
//   v(y,x)  = sum_c x'_c(y,x)^2          x' = x - 128 (u8) or x - 0.5 (f32)
//   S       = inclusive 2D prefix sum of v        (stored as buf[y][x] = S(y+1, x+1))
//   n(y,x)  = S(y+b,x+b) - S(y,x+b) - S(y+b,x) + S(y,x)   for y <= H-b, x <= W-b
//
// u8 : uint32 wrap-around arithmetic. Every box sum is < 2^32 (<= 8*16*16*128^2 < 2^25), so
//      the 4-corner combination modulo 2^32 equals the exact value even though S itself
//      wraps.
// f32: fp64 SAT (an fp32 SAT loses 1e-3 relative distance accuracy at full size).
//
// u8 frames use ONE kernel instead (norm_direct_u8): the same box sums formed directly by a
// separable box filter (vertical b-sums, then horizontal b-sums) of x'^2 staged in shared
// memory -- exact int32, bit-identical to the integral-image values, and 1 pass over the
// image instead of 4 passes over a 4-byte/pixel SAT (c5: 2.05 -> ~0.15 ms per 64 frames).
//
// The map is written into the interior of a padded buffer (NPAD rows / columns of a huge
// value on every side, set once at plan creation) so that the box-sum matcher can read
// norms of out-of-image candidates without clamping: they never pass a threshold.
//
// f32 kernels (per chunk of F frames, all coalesced):
//   sat_rows     one warp per image row; 16-byte vector loads, register prefix per lane,
//                warp shuffle scan across lanes, vector stores.
//   sat_bands    column totals of 32-row bands (thread per column).
//   sat_cols     carry-in from earlier bands + in-place inclusive column scan of one band.
//   norm_box     the 4-corner box sums.
#include "sc_internal.h"

namespace scbm {
namespace {

template <typename In> struct NormTraits;
template <> struct NormTraits<uint8_t> {
  using Acc = uint32_t;
  using Out = int32_t;
  static constexpr int kVec = 16;  // pixels per 16-byte vector
  __device__ static Acc sq(uint8_t x) {
    int v = int(x) - 128;
    return Acc(v * v);
  }
};
template <> struct NormTraits<float> {
  using Acc = double;
  using Out = float;
  static constexpr int kVec = 4;
  __device__ static Acc sq(float x) {
    double v = double(x - 0.5f);  // the same fp32 centring as the cross-term path
    return v * v;
  }
};

// One warp per row: buf[y][x] = sum_{x' <= x} v(y, x').
template <typename In>
__global__ void __launch_bounds__(128) sat_rows(const In* __restrict__ imgs, int C, int H, int W,
                                                int SP, typename NormTraits<In>::Acc* __restrict__ buf) {
  using T = NormTraits<In>;
  using Acc = typename T::Acc;
  constexpr int V = T::kVec;
  const int lane = threadIdx.x & 31;
  const int y = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int f = blockIdx.y;
  if (y >= H) return;
  const size_t plane = size_t(H) * W;
  const In* img = imgs + size_t(f) * C * plane + size_t(y) * W;
  Acc* out = buf + (size_t(f) * H + y) * SP;
  const bool vec_ok = (W % V == 0) && ((reinterpret_cast<uintptr_t>(imgs) & 15) == 0);
  Acc carry = 0;
  for (int x0 = 0; x0 < W; x0 += 32 * V) {
    const int x = x0 + lane * V;
    Acc v[V];
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = 0;
    if (x < W) {
      for (int c = 0; c < C; ++c) {
        const In* row = img + size_t(c) * plane;
        if (vec_ok) {
          uint4 q = *reinterpret_cast<const uint4*>(row + x);
          const In* e = reinterpret_cast<const In*>(&q);
#pragma unroll
          for (int i = 0; i < V; ++i) v[i] += T::sq(e[i]);
        } else {
#pragma unroll
          for (int i = 0; i < V; ++i)
            if (x + i < W) v[i] += T::sq(row[x + i]);
        }
      }
    }
#pragma unroll
    for (int i = 1; i < V; ++i) v[i] += v[i - 1];
    Acc tot = v[V - 1], inc = tot;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      Acc t = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += t;
    }
    const Acc base = carry + inc - tot;
    carry += __shfl_sync(0xffffffffu, inc, 31);
    if (x < W) {
      if (x + V <= SP) {
#pragma unroll
        for (int i = 0; i < V; ++i) out[x + i] = base + v[i];  // contiguous; compiler vectorises
      }
    }
  }
}

// Column totals of band k: tot[f][k][x] = sum_{y in band k} buf[y][x].
template <typename Acc>
__global__ void sat_bands(const Acc* __restrict__ buf, int H, int W, int SP, int nb,
                          Acc* __restrict__ tot) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y, f = blockIdx.z;
  if (x >= W) return;
  const int y0 = k * kSatBand, y1 = min(H, y0 + kSatBand);
  const Acc* p = buf + size_t(f) * H * SP + x;
  Acc s = 0;
#pragma unroll 8
  for (int y = y0; y < y1; ++y) s += p[size_t(y) * SP];
  tot[(size_t(f) * nb + k) * SP + x] = s;
}

// In-place inclusive column scan of band k with the carry of bands < k.
template <typename Acc>
__global__ void sat_cols(Acc* __restrict__ buf, int H, int W, int SP, int nb,
                         const Acc* __restrict__ tot) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y, f = blockIdx.z;
  if (x >= W) return;
  Acc s = 0;
  for (int kk = 0; kk < k; ++kk) s += tot[(size_t(f) * nb + kk) * SP + x];
  const int y0 = k * kSatBand, y1 = min(H, y0 + kSatBand);
  Acc* p = buf + size_t(f) * H * SP + x;
  for (int y = y0; y < y1; ++y) {
    s += p[size_t(y) * SP];
    p[size_t(y) * SP] = s;
  }
}

template <typename Acc>
__device__ __forceinline__ Acc sat_at(const Acc* __restrict__ buf, int SP, int y, int x) {
  return (y == 0 || x == 0) ? Acc(0) : buf[size_t(y - 1) * SP + (x - 1)];
}

template <typename In>
__global__ void norm_box(const typename NormTraits<In>::Acc* __restrict__ buf, int H, int W, int SP,
                         int b, int Mxp, long long nfs, typename NormTraits<In>::Out* __restrict__ norm) {
  using Acc = typename NormTraits<In>::Acc;
  using Out = typename NormTraits<In>::Out;
  const int My = H - b + 1, Mx = W - b + 1;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  const int f = blockIdx.z;
  if (x >= Mx || y >= My) return;
  const Acc* S = buf + size_t(f) * H * SP;
  Acc v = sat_at(S, SP, y + b, x + b) - sat_at(S, SP, y, x + b) - sat_at(S, SP, y + b, x) +
          sat_at(S, SP, y, x);
  norm[size_t(f) * nfs + size_t(y) * Mxp + x] = Out(v);
}

// u8: direct separable box sums of x'^2 (exact int32; identical to the integral-image values).
// One CTA per 32-row x 128-column output tile: the squared centred tile (+ b-1 halo) summed
// over channels goes to shared memory, then vertical b-sums, then horizontal b-sums.
constexpr int kNdRows = 32, kNdCols = 128;
__global__ void __launch_bounds__(256) norm_direct_u8(const uint8_t* __restrict__ imgs, int C, int H, int W,
                                                      int b, int Mxp, long long nfs, int32_t* __restrict__ norm) {
  __shared__ int sq[kNdRows + 15][kNdCols + 16];
  __shared__ int vs[kNdRows][kNdCols + 16];
  const int My = H - b + 1, Mx = W - b + 1;
  const int y0 = blockIdx.y * kNdRows, x0 = blockIdx.x * kNdCols, f = blockIdx.z;
  const int rows = min(kNdRows, My - y0) + b - 1, cols = min(kNdCols, Mx - x0) + b - 1;
  const size_t plane = size_t(H) * W;
  const uint8_t* img = imgs + size_t(f) * C * plane;
  for (int e = threadIdx.x; e < rows * cols; e += blockDim.x) {
    const int r = e / cols, c = e - r * cols;
    int v = 0;
    for (int ch = 0; ch < C; ++ch) {
      const int t = int(img[ch * plane + size_t(y0 + r) * W + x0 + c]) - 128;
      v += t * t;
    }
    sq[r][c] = v;
  }
  __syncthreads();
  const int orows = rows - b + 1;
  for (int e = threadIdx.x; e < orows * cols; e += blockDim.x) {
    const int r = e / cols, c = e - r * cols;
    int v = 0;
    for (int l = 0; l < b; ++l) v += sq[r + l][c];
    vs[r][c] = v;
  }
  __syncthreads();
  const int ocols = cols - b + 1;
  for (int e = threadIdx.x; e < orows * ocols; e += blockDim.x) {
    const int r = e / ocols, c = e - r * ocols;
    int v = 0;
    for (int m = 0; m < b; ++m) v += vs[r][c + m];
    norm[size_t(f) * nfs + size_t(y0 + r) * Mxp + x0 + c] = v;
  }
}

template <typename In>
cudaError_t launch_norm_t(const sc_bm_plan_s& p, const In* imgs, int F, cudaStream_t st,
                          int64_t* launches) {
  using Acc = typename NormTraits<In>::Acc;
  using Out = typename NormTraits<In>::Out;
  const Geometry& g = p.g;
  if constexpr (sizeof(In) == 1) {
    norm_direct_u8<<<dim3((g.Mx + kNdCols - 1) / kNdCols, (g.My + kNdRows - 1) / kNdRows, F), 256, 0, st>>>(
        imgs, g.C, g.H, g.W, g.b, g.Mxp, g.NFS, static_cast<int32_t*>(p.ws.norm));
    if (launches) *launches += 1;
    return cudaGetLastError();
  }
  const int SP = (g.W + 15) / 16 * 16;
  Acc* buf = static_cast<Acc*>(p.ws.sat);
  Acc* tot = static_cast<Acc*>(p.ws.bandsum);
  sat_rows<In><<<dim3((g.H + 3) / 4, F), 128, 0, st>>>(imgs, g.C, g.H, g.W, SP, buf);
  const int nb = p.nbands;
  dim3 cg((g.W + 127) / 128, nb, F);
  sat_bands<Acc><<<cg, 128, 0, st>>>(buf, g.H, g.W, SP, nb, tot);
  sat_cols<Acc><<<cg, 128, 0, st>>>(buf, g.H, g.W, SP, nb, tot);
  norm_box<In><<<dim3((g.Mx + 127) / 128, g.My, F), 128, 0, st>>>(buf, g.H, g.W, SP, g.b, g.Mxp, g.NFS,
                                                                  static_cast<Out*>(p.ws.norm));
  if (launches) *launches += 4;
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_norm(const sc_bm_plan_s& p, const void* imgs, int F, cudaStream_t st,
                        int64_t* launches) {
  if (p.g.dtype == SC_DTYPE_U8)
    return launch_norm_t<uint8_t>(p, static_cast<const uint8_t*>(imgs), F, st, launches);
  return launch_norm_t<float>(p, static_cast<const float*>(imgs), F, st, launches);
}

}  // namespace scbm
