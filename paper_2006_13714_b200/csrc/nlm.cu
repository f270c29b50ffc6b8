// nlm.cu -- NLM weights (the "next" row SURVEY.md 8f rank 3): Eq. 2
//     s_i(j) = exp(-||X_j - X_i||_F^2 / h^2) / Theta_i,   Theta_i = sum_j exp(-||X_j - X_i||^2 / h^2)
// over the reference's clipped search window (footnote 2), computed the paper's
// way (Proposition 1): the window distances come from the Self-Convolution
// identity (the matcher's dense mode writes n_c + n_r - 2 C_i for every window slot, Lemma 2), and
// this kernel turns each reference's row into normalised weights in place.
//
// Stabilisation: the row minimum d_min is subtracted before the exponential -- exp(-(d - d_min)/h^2)
// has the same ratio (numerator and Theta share the factor exp(d_min / h^2)) and cannot underflow
// to 0/0. One warp per reference row, coalesced, in place (int32 u8 distances / float distances ->
// float weights of the same size).
#include <math.h>

#include <algorithm>

#include "nlm.cuh"
#include "sc_internal.h"

namespace scbm {
namespace {

template <typename T>
__global__ void __launch_bounds__(256) nlm_normalize(void* rows, long long n_refs, int nx, int s, int cy_max,
                                                     int cx_max, int Wn, int lo, float inv_h2) {
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long r = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n_refs; r += nw) {
    const NlmRowGeom gm{int(r / nx) * s, int(r % nx) * s, cy_max, cx_max, Wn, lo};
    nlm_normalize_row<T>(static_cast<T*>(rows) + r * Wn * Wn, gm, inv_h2, lane);
  }
}

}  // namespace

cudaError_t launch_nlm_normalize(const sc_bm_plan_s& p, void* rows, float h, cudaStream_t st, int64_t* launches) {
  const Geometry& g = p.g;
  const long long n_refs = (long long)g.ny * g.nx;
  const int slots = g.Wn * g.Wn;
  const float inv_h2 = 1.f / (h * h);
  const long long blocks = std::min<long long>((n_refs + 7) / 8, (long long)p.sm_count * 16);
  if (launches) *launches += 1;
  const int lo = -(g.Wn / 2);
  (void)slots;
  if (g.dtype == SC_DTYPE_U8)
    nlm_normalize<int32_t><<<unsigned(blocks), 256, 0, st>>>(rows, n_refs, g.nx, g.s, g.H - g.b, g.W - g.b, g.Wn, lo,
                                                             inv_h2);
  else
    nlm_normalize<float><<<unsigned(blocks), 256, 0, st>>>(rows, n_refs, g.nx, g.s, g.H - g.b, g.W - g.b, g.Wn, lo,
                                                           inv_h2);
  return cudaGetLastError();
}

}  // namespace scbm
