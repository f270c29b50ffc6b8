// sc_internal.h -- plan struct and kernel launchers shared by plan.cpp and the .cu files.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/sc_bm.h"

namespace scbm {

struct Geometry {
  int H, W, C, b, s, Wn, K;
  int dtype;          // SC_DTYPE_*
  int ny, nx;         // reference grid
  int lo, hi;         // window offsets
  int My, Mx;         // valid candidate positions (H-b+1, W-b+1)
  int Mxp;            // norm-map row pitch (Mx + 2*NPAD rounded up to 4 ints: 16-byte aligned rows)
  int NPAD;           // norm-map border (rows and columns) on every side, filled with a huge value
  long long NFS;      // norm-map frame stride in elements ((My + 2*NPAD) * Mxp)
  int KP;             // keys kept per ref before output (K, or K+rescore margin for f32 / NCC)
  int metric;         // SC_METRIC_L2 (Eq. 3) or SC_METRIC_NCC (Eq. 4)
  int z3 = 0;         // 3D search over volume planes (sc_bm_plan3d): C = the patch depth d
  int zwin = 1;       // 3D: plane offsets per reference (the window depth c)
};

// Workspace for one chunk of frames.
struct Workspace {
  void* sat = nullptr;      // [F][H+1][W+1] uint32 (u8) or double (f32)
  void* bandsum = nullptr;  // [F][nbands][W+1] column band totals
  void* norm_base = nullptr;  // allocation of the padded norm map [F][My+2*NPAD][Mxp]
  void* norm = nullptr;     // interior of frame 0: element (f, y, x) at norm[f*NFS + y*Mxp + x]
  int* fix_count = nullptr; // exact fix-up: number of flagged references of the current chunk
  int* fix_list = nullptr;  // [F * n_refs] flagged (frame * band_refs + band ref) indices
  size_t bytes = 0;
};

struct HostStaging {
  bool ready = false;
  int F = 0;                 // frames per chunk
  int Fp = 0;                // frames per chunk with packed tables (half the bytes per frame)
  void* d_img[2] = {nullptr, nullptr};
  int32_t* d_idx[2] = {nullptr, nullptr};
  void* d_dist[2] = {nullptr, nullptr};
  cudaStream_t copy_in = nullptr, copy_out = nullptr;
  cudaEvent_t ev_in[2], ev_done[2], ev_out[2];
  uint32_t* d_tail = nullptr;  // packed tables: the run's overflow area (header + records)
  int64_t tail_cap = -1;       // cap_rows d_tail was allocated for
};

struct Timing {
  bool enabled = false;
  int n_used = 0;                  // event triples used since the last read
  std::vector<cudaEvent_t> ev;     // 3 events per chunk: before norm, between, after match
};

struct TileCfg {
  int TRY, TRX;  // reference tile (ref-grid units) per CTA
  int VY;        // vertical candidates per lane
  int warps;     // warps per CTA
  size_t smem;   // dynamic shared memory bytes
};

}  // namespace scbm

struct sc_bm_plan_s {
  scbm::Geometry g;
  int device = 0;
  int sm_count = 148;
  int kernel = SC_KERNEL_SIMT;
  int F = 1;  // frames per chunk (norm-map matchers: the chunk's norm workspace stays in L2)
  int FB = 64;  // frames per launch of the box-sum matchers (no workspace: one big grid, one tail)
  int nbands = 1;
  scbm::Workspace ws;
  scbm::TileCfg tile;
  int lanes_nwy = 4;  // reference rows (warps) per CTA of the lanes = references kernel
  scbm::HostStaging host;
  scbm::Timing timing;
  int64_t launches = 0;
  int T = 0;                          // temporal search radius (sc_bm_set_temporal)
  int kernel_before_T = -1;           // the matcher T > 0 replaced (restored by T = 0)
  float nlm_inv_h2 = 0.f;             // > 0 while sc_bm_nlm_weights / sc_bm_nlm_average run
  void* nlm_avg_out = nullptr;        // set while sc_bm_nlm_average runs (float [refs][C][b][b])
  const void* batch_base = nullptr;   // temporal search: the run's whole batch ...
  int64_t batch_f0 = 0, batch_n = 0;  // ... the current chunk's first frame and the batch size
  int64_t idx_frame_off = 0;          // sc_bm_run_temporal: frame offset of the batch-global idx
  int64_t min_cand = 0, max_cand = 0, total_cand = 0;
  int zstride = 1, zlo = 0, zhi = 0;  // 3D search: reference plane stride, plane offsets [zlo, zhi]
  int64_t n_planes = 0;               // 3D search: planes of the volume of the current sc_bm_run3d
  int64_t packed_cap = 0;             // sc_bm_set_packed: overflow rows (0: plain tables)
  uint32_t* packed_tail = nullptr;    // packed run: its overflow area (header word 0 = count)
  int64_t packed_f0 = 0;              // packed run: image index of the current chunk in the run
  int64_t packed_base = 0;            // packed run: image index (in the run) of the enqueued batch
};

namespace scbm {

constexpr int kSatBand = 32;  // rows per column-scan band

// norm.cu: integral image of x'^2 and the 4-corner norm map for F frames.
cudaError_t launch_norm(const sc_bm_plan_s& p, const void* imgs, int F, cudaStream_t st,
                        int64_t* launches);

// bm_simt.cu: fused cross term + distance assembly + top-K (+ f32 re-score) for F frames.
// dense != nullptr selects the debug mode that writes every window distance instead.
cudaError_t launch_bm_simt(const sc_bm_plan_s& p, const void* imgs, int F, int iy_begin,
                           int iy_end, int32_t* idx_out, void* dist_out, void* dense,
                           cudaStream_t st, int64_t* launches);
TileCfg choose_simt_tile(const Geometry& g, int sm_count, int n_images);

// bm_lanes.cu: the lanes = references matcher (SC_KERNEL_SIMT).
cudaError_t launch_bm_lanes(const sc_bm_plan_s& p, const void* imgs, int F, int iy_begin,
                            int iy_end, int32_t* idx_out, void* dist_out, void* dense,
                            cudaStream_t st, int64_t* launches);
int lanes_warps_for(const Geometry& g, int sm_count, int n_images);
int lanes_r32_slots(const Geometry& g);

// fixup.cu: exact top-K (64-bit keys, direct differences) for references flagged by the
// 32-bit register top-K paths (saturated distance field or fewer than K candidates).
cudaError_t launch_fixup(const sc_bm_plan_s& p, const void* imgs, int F, int iy_begin, int iy_end,
                         int32_t* idx_out, void* dist_out, cudaStream_t st);

// bm_tc.cu: the tcgen05 kind::i8 matcher (SC_KERNEL_TC_I8; u8, b = 8, C = 1).
bool tc_supported(const Geometry& g);
cudaError_t launch_bm_tc(const sc_bm_plan_s& p, const void* imgs, int F, int iy_begin, int iy_end,
                         int32_t* idx_out, void* dist_out, cudaStream_t st, int64_t* launches);
size_t lanes_smem_bytes(const Geometry& g, int nwy);

// bm_tcf.cu: the tensor-core float matcher (SC_KERNEL_TC_F32; f32, C = 1, b <= 8, 3xTF32 on tcgen05).
// dense != nullptr: the debug mode writing every window distance [refs][Wn^2] (-1 in clipped slots).
bool tcf_supported(const Geometry& g);
bool tcf_preferred(const Geometry& g);  // the default matcher where it measured faster (stride 1)
cudaError_t launch_bm_tcf(const sc_bm_plan_s& p, const void* imgs, int F, int iy_begin, int iy_end,
                          int32_t* idx_out, void* dist_out, void* dense, cudaStream_t st, int64_t* launches);

// bm_box.cu: the box-sum matcher (SC_KERNEL_BOX; u8, b = 8, s = 4, C = 1, K <= 32).
bool box_supported(const Geometry& g);
bool box_temporal_supported(const Geometry& g, int T);
cudaError_t launch_bm_box(const sc_bm_plan_s& p, const void* imgs, int F, int iy_begin, int iy_end,
                          int32_t* idx_out, void* dist_out, cudaStream_t st, int64_t* launches);

// packed.cu: packed tables (sc_bm_set_packed): overflow-area header, device decode.
// Row words w = (dist << rb) | slot; escape rows (0xFFFFFFFF) come from the overflow records.
int packed_rel_bits(const Geometry& g);
int64_t packed_record_words(const Geometry& g);
cudaError_t launch_packed_init(uint32_t* tail, int64_t cap, cudaStream_t st);
cudaError_t launch_unpack(const sc_bm_plan_s& p, const uint32_t* packed, int64_t n_images, int64_t n_records,
                          int32_t* idx_out, int32_t* dist_out, cudaStream_t st);

// nlm.cu: NLM weights (Eq. 2 / Prop. 1) from a dense window-distance table, normalised in place.
cudaError_t launch_nlm_normalize(const sc_bm_plan_s& p, void* rows, float h, cudaStream_t st, int64_t* launches);

// group.cu: patch grouping Y_i from a run's idx table.
cudaError_t launch_group(const sc_bm_plan_s& p, const void* imgs, int64_t n_images, const int32_t* idx,
                         void* out, cudaStream_t st, int64_t* launches);

// bm_boxf.cu: the float box-sum matcher (SC_KERNEL_BOXF; f32, C = 1, (s, b) in a small set).
bool boxf_supported(const Geometry& g);
cudaError_t launch_bm_boxf(const sc_bm_plan_s& p, const void* imgs, int F, int iy_begin, int iy_end,
                           int32_t* idx_out, void* dist_out, cudaStream_t st, int64_t* launches);

}  // namespace scbm
