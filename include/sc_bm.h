/*
 * sc_bm.h -- C ABI of the B200-native Self-Convolution block-matching library (libscbm.so).
 *
 * The operation (arXiv 2006.13714):
 *   For every reference patch X_i on a stride grid, find the K candidate patches X_j of
 *   its search window with the smallest squared Euclidean distance
 *       d_E(X_j, X_i) = ||X_j - X_i||_F^2                         (Eq. 3)
 *   restricted to the window Omega_i (footnote 2), channels summed jointly
 *   (Eq. 12's S(.)). The library evaluates it the paper's way:
 *       d_E = h_X(j)^2 + ||X_i||^2 - 2 C_i(j)                     (Lemma 2)
 *   with the norms h_X (.) h_X from an integral image of the squared image
 *   and the cross term C_i the image self-convolved with X_i (Eq. 5);
 *   selection keeps the K largest values of b_i = C_i - 1/2 h_X (.) h_X, i.e. the K
 *   smallest d_E (Theorem 1, proof PAPER.md:487-502).
 *
 * Geometry:
 *   reference grid  ry = 0, s, 2s, ... <= H-b;  rx = 0, s, ... <= W-b;  n_ref_y * n_ref_x refs,
 *                   reference j = iy * n_ref_x + ix (raster), images outermost.
 *   window          candidate top-left (cy, cx) with cy - ry, cx - rx in [lo, hi],
 *                   lo = -floor(Wn/2), hi = Wn - 1 - floor(Wn/2), clipped to [0,H-b] x [0,W-b];
 *                   every position (candidate stride 1).
 *   index           idx = cy * W + cx (pixel raster of the top-left corner, per image).
 *   order           each row of K results is sorted ascending by (distance, idx).
 *   short windows   if a window has fewer than K candidates the tail is idx = -1 and
 *                   dist = INT32_MAX (u8) or +inf (f32).
 *
 * Layouts (all row-major, contiguous):
 *   img      [n_images][C][H][W]  uint8 (SC_DTYPE_U8) or float (SC_DTYPE_F32), planar channels.
 *   idx_out  [n_images][n_refs][K] int32.
 *   dist_out [n_images][n_refs][K] int32 (u8: exact integer distances) or float (f32).
 *
 * Ownership and threading:
 *   The plan owns its device workspace, allocated by sc_bm_plan on the current CUDA device
 *   and freed by sc_bm_destroy. The caller owns img / idx_out / dist_out (device memory
 *   unless stated otherwise) and the stream. The device-pointer run calls never allocate,
 *   never synchronise and are CUDA-graph capturable. Runs sharing one plan must be ordered
 *   on one stream (the workspace is shared); distinct plans are independent.
 *
 * Errors:
 *   Argument validation is synchronous and returns a status. Kernel launch failures return
 *   SC_ERR_CUDA; asynchronous device faults surface at the caller's next synchronisation.
 *   The library never prints and never exits. There is no CPU fallback: without a usable
 *   sm_100 device sc_bm_plan returns SC_ERR_CUDA / SC_ERR_UNSUPPORTED.
 *
 * Numerics:
 *   u8  : values are shifted by -128 (d is a difference, Eq. 3, so it is unchanged); the
 *         integral image is uint32 (wrap-around, box sums exact), the cross term int32; all
 *         distances are exact integers -- bit-identical to the definition.
 *   f32 : values are centred by -0.5; the integral image is fp64; the cross term fp32; the
 *         top-(K+m) survivors (m = 4, or 8 for K > 48) are re-scored by direct differences in
 *         fp32 and re-sorted; references where the margin could hide a top-K candidate are
 *         recomputed exactly over their whole window.
 *         Distances are within relative 1e-5 of the exact value (BASELINE.json north_star).
 */
#ifndef SC_BM_H
#define SC_BM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SC_BM_ABI_VERSION 1

typedef struct CUstream_st* sc_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum { SC_DTYPE_U8 = 0, SC_DTYPE_F32 = 1 } sc_dtype_t;

/* Similarity metric: SC_METRIC_L2 = squared Euclidean distance (Eq. 3, the default);
 * SC_METRIC_NCC = normalised cross-correlation (Eq. 4, Lemma 1) on
 * the raw values: the K LARGEST NCC = C_i(j) / (||X_i|| ||X_j||) per window, NCC := 0 when a
 * norm is 0; dist_out holds d_NCC = -NCC as float32 for both dtypes; uint8 orderings are exact. */
typedef enum { SC_METRIC_L2 = 0, SC_METRIC_NCC = 1 } sc_metric_t;

typedef enum {
    SC_OK = 0,
    SC_ERR_INVALID_ARGUMENT = 1, /* null pointer, misaligned pointer, parameter out of range */
    SC_ERR_UNSUPPORTED = 2,      /* valid request this build cannot serve (e.g. no sm_100 device) */
    SC_ERR_OUT_OF_MEMORY = 3,    /* workspace allocation failed */
    SC_ERR_CUDA = 4,             /* CUDA runtime / launch error */
    SC_ERR_WRONG_DEVICE = 5,     /* current device differs from the plan's device */
    SC_ERR_OVERFLOW = 6          /* packed tables: more escape rows than the overflow area holds */
} sc_status_t;

typedef struct sc_bm_plan_s* sc_bm_plan_t;

typedef struct {
    int64_t n_ref_y, n_ref_x, n_refs;   /* reference grid per image */
    int64_t min_candidates;             /* smallest clipped window (candidates of one ref) */
    int64_t max_candidates;             /* largest clipped window */
    int64_t total_candidates;           /* sum over the refs of one image: the pair count */
    int64_t workspace_bytes;            /* device workspace owned by the plan */
    int64_t frames_per_chunk;           /* images processed per norm->match chunk */
    int64_t launches;                   /* kernels launched by this plan so far (counter) */
    int32_t kernel;                     /* SC_KERNEL_* selected for the cross-term/top-K step */
    int32_t device;                     /* CUDA device ordinal the plan is bound to */
} sc_bm_info_t;

#define SC_KERNEL_SIMT 0       /* CUDA-core matcher, lanes = references */
#define SC_KERNEL_TC_I8 1      /* tcgen05 kind::i8 cross term (TMEM) + fused top-K (u8 only) */
#define SC_KERNEL_SIMT_WARP 2  /* CUDA-core matcher, one warp per reference (lanes = candidates) */
#define SC_KERNEL_BOX 3        /* box-sum matcher: 4x4 block sums of the shifted product image
                                  (u8, b = 8, stride 4, C = 1, K <= 32; default where supported) */
#define SC_KERNEL_TC_F32 5     /* tcgen05 3xTF32 cross term (TMEM) + fused top-K (f32, C = 1, b <= 8) */
#define SC_KERNEL_BOXF 4       /* float box-sum matcher (f32, any C, (stride, b) in {(3,8), (1,7), (1,6),
                                  (4,8), (2,8)}, K + m <= 80; default where supported) */

/*
 * Create a plan. H, W: image size (H, W >= b, H*W < 2^31); C: channels (1..8); b: patch
 * side (1..16); stride: reference stride (>= 1); window: Wn (1..255); K: matches (1..128);
 * dtype: SC_DTYPE_U8 or SC_DTYPE_F32. *plan_out receives the handle (NULL on failure).
 */
sc_status_t sc_bm_plan(int H, int W, int C, int b, int stride, int window, int K,
                       sc_dtype_t dtype, sc_bm_plan_t* plan_out);

/* Same with an explicit metric. SC_METRIC_NCC (Eq. 4) runs on the box-sum
 * kernels: uint8 with stride 4, b = 8, one channel on the dp4a kernel; otherwise the float kernel,
 * which needs (stride, b) in {(3,8), (1,7), (4,8), (2,8)}, any channel count; K <= 30 for uint8
 * (exact 128-bit ordering of the kept keys), K <= 76 for float (else SC_ERR_UNSUPPORTED). */
sc_status_t sc_bm_plan_ex(int H, int W, int C, int b, int stride, int window, int K,
                          sc_dtype_t dtype, sc_metric_t metric, sc_bm_plan_t* plan_out);

/*
 * Block matching of one image (Eq. 3, over the window of footnote 2,
 * PAPER.md:280; evaluated through Lemma 2, and Theorem 1):
 * img [C][H][W] -> idx_out / dist_out [n_refs][K]. Device pointers; img 16-B aligned, outputs
 * 4-B aligned. SC_ERR_INVALID_ARGUMENT for a null / misaligned pointer, SC_ERR_WRONG_DEVICE off
 * the plan's device, SC_ERR_CUDA when the launch fails. Asynchronous on `stream`.
 */
sc_status_t sc_bm_run(sc_bm_plan_t plan, const void* img, int32_t* idx_out, void* dist_out,
                      sc_stream_t stream);

/*
 * Block matching (Eq. 3; footnote 2) of n_images independent
 * images [n][C][H][W] -> [n][n_refs][K] (the video batch of config c5; the paper's video
 * setting). Device pointers, errors as sc_bm_run. With sc_bm_set_temporal(T > 0)
 * idx is batch-global, so n_images * H * W must stay <= 2^31 (SC_ERR_INVALID_ARGUMENT).
 */
sc_status_t sc_bm_run_batch(sc_bm_plan_t plan, const void* imgs, int64_t n_images,
                            int32_t* idx_out, void* dist_out, sc_stream_t stream);

/*
 * Row band of Eq. 3: the multi-GPU partitioner's spatial split (DESIGN.md
 * "Multi-GPU"; every reference is independent given its window, footnote 2): only the
 * references of reference-grid rows [iy_begin, iy_end) of each image; idx_out / dist_out
 * are [n_images][(iy_end - iy_begin) * n_ref_x][K]. The full image is read (replicated).
 */
sc_status_t sc_bm_run_rows(sc_bm_plan_t plan, const void* imgs, int64_t n_images,
                           int32_t iy_begin, int32_t iy_end, int32_t* idx_out, void* dist_out,
                           sc_stream_t stream);

/*
 * Same as sc_bm_run_batch but imgs / idx_out / dist_out are HOST pointers (pinned memory
 * gives full overlap; pageable memory works but serialises the copies). The library
 * pipelines host->device copies, matching and device->host copies over frame chunks on
 * the given stream plus plan-owned streams, and returns when the results are in host
 * memory. The first call allocates the plan's staging buffers (a documented exception
 * to "run never allocates").
 */
sc_status_t sc_bm_run_host(sc_bm_plan_t plan, const void* h_imgs, int64_t n_images,
                           int32_t* h_idx_out, void* h_dist_out, sc_stream_t stream);

/*
 * Patch grouping (the step after block matching): Y_i = [y_{S_i(1)}, ..., y_{S_i(K)}]
 * (footnote PAPER.md:548). For every reference i of the n_images images and
 * each of its K matches (idx: the idx_out of a run on the same images, [n][n_refs][K] int32),
 * copy the matched b x b x C patch of imgs into
 *     groups_out [n_images][n_refs][K][C][b][b]   (input dtype, uncentred; column k of Y_i is
 *                                                 the channel-major vectorisation of patch k)
 * idx = -1 (fewer than K candidates) gives a zero column. Device pointers: imgs and groups_out
 * 16-byte aligned, idx 4-byte aligned; idx entries must be valid indices from a run of this plan
 * (not checked on the device). Asynchronous on `stream`, never allocates.
 */
sc_status_t sc_bm_group(sc_bm_plan_t plan, const void* imgs, int64_t n_images, const int32_t* idx,
                        void* groups_out, sc_stream_t stream);

/*
 * NLM weights (Eq. 2, via Proposition 1) of ONE image:
 *     weights_out[i][(dy-lo)*Wn + (dx-lo)] = exp(-||X_j - X_i||_F^2 / h^2) / Theta_i
 * over reference i's clipped window (0 in clipped slots; every row sums to 1), float32
 * [n_refs][Wn*Wn], device pointers (img 16-byte, weights_out 4-byte aligned), h > 0 the NLM
 * bandwidth (the paper's b in Eq. 2). The window distances come from the Self-Convolution
 * identity (Lemma 2), written into weights_out and normalised in place. L2 plans only.
 */
sc_status_t sc_bm_nlm_weights(sc_bm_plan_t plan, const void* img, float h, float* weights_out,
                              sc_stream_t stream);

/*
 * NL-means estimate of every reference patch (after Eq. 2): the weighted average
 *     X_hat_i = sum_j s_i(j) X_j,   s_i(j) = exp(-||X_j - X_i||_F^2 / h^2) / Theta_i,
 * j over the reference's clipped window (footnote 2), the distances from the
 * Self-Convolution identity (Proposition 1), X_j the raw input patches.
 * One image img [C][H][W] (device, 16-byte aligned) -> out [n_refs][C][b][b] float32 (device,
 * 4-byte aligned), reference raster order. The weights are never materialised (streaming
 * softmax in the matcher's epilogue). SC_ERR_UNSUPPORTED for the NCC metric or b*b*C > 256.
 * Asynchronous on `stream`, never allocates.
 */
sc_status_t sc_bm_nlm_average(sc_bm_plan_t plan, const void* img, float h, float* out,
                              sc_stream_t stream);

/*
 * 3D / temporal search (the video setting of PAPER.md:661, 697): with T > 0, the candidates of a
 * reference in image f of a sc_bm_run_batch / sc_bm_run_rows call are the window positions of
 * images f-T .. f+T of that call (clipped to the batch), and idx_out holds the BATCH-GLOBAL
 * index frame * H * W + cy * W + cx (ties by it: earlier frames first). uint8, b = 8, stride 4,
 * one channel, L2 metric, (2T+1) Wn^2 <= 4096 (else SC_ERR_UNSUPPORTED); T = 0 (default)
 * restores per-image search and the matcher the plan used before T > 0 forced the box kernel.
 * sc_bm_run_host is unsupported with T > 0.
 */
sc_status_t sc_bm_set_temporal(sc_bm_plan_t plan, int32_t T);

/*
 * Temporal search over part of a batch (a frame shard plus its halo): references from frames
 * [f_begin, f_end) of the n_images-frame batch imgs [n_images][C][H][W]; the candidates of a
 * reference in frame f are the clipped window positions of frames max(0, f-T) .. min(n_images-1,
 * f+T) of that batch (T from sc_bm_set_temporal, > 0, else SC_ERR_UNSUPPORTED). idx_out /
 * dist_out hold f_end - f_begin frames ([f][n_refs][K], as sc_bm_run_batch); idx is
 * (frame + frame_offset) * H * W + cy * W + cx, so a rank whose buffer starts at global frame
 * frame_offset (its halo) reports global indices. frame_offset >= 0 and the largest idx must fit
 * int32 (SC_ERR_INVALID_ARGUMENT otherwise). Device pointers, asynchronous on `stream`.
 */
sc_status_t sc_bm_run_temporal(sc_bm_plan_t plan, const void* imgs, int64_t n_images, int64_t f_begin,
                               int64_t f_end, int64_t frame_offset, int32_t* idx_out, void* dist_out,
                               sc_stream_t stream);

/*
 * 3D search (3D Self-Convolution "searching across channels" with patches of d < p
 * channels; the video setting, 6 x 6 x 1 patches in a 30 x 30 x c window, c = 9
 * frames). A volume vol [n_planes][H][W] (float, device, 16-B aligned) -- the channels of one
 * multi-channel image or the frames of a video -- is matched in 3D: a patch is d consecutive planes
 * x b x b; references start at planes 0, z_stride, 2 z_stride, ... <= n_planes - d (n_zref of them)
 * and on the usual spatial grid; the candidates of a reference at plane z are the patches starting
 * at planes z + dz, dz in [-floor(z_window/2), z_window - 1 - floor(z_window/2)] (clipped to
 * [0, n_planes - d]), at every clipped window position; the distance sums the d planes
 * (oracle.bm3d). Outputs [n_zref][n_refs][K] (idx int32, dist float), idx = (z_c H + cy) W + cx
 * (the volume raster of the candidate's first voxel), rows sorted by (dist, idx).
 * sc_bm_plan3d: float only (uint8 video search: sc_bm_set_temporal), z_window <= 64, the float
 * box-sum kernel's shapes ((stride, b) in {(3,8), (1,7), (4,8), (2,8), (1,6)}), K + 4 <= 48,
 * z_window Wn^2 < 2^13 (else SC_ERR_UNSUPPORTED). A 3D plan refuses every other run call.
 * sc_bm_run3d: n_planes >= d and n_planes H W <= 2^31 (SC_ERR_INVALID_ARGUMENT otherwise);
 * asynchronous on `stream`, never allocates.
 */
sc_status_t sc_bm_plan3d(int H, int W, int d, int b, int stride, int window, int z_stride, int z_window, int K,
                         sc_dtype_t dtype, sc_bm_plan_t* plan_out);
sc_status_t sc_bm_run3d(sc_bm_plan_t plan, const void* vol, int64_t n_planes, int32_t* idx_out, void* dist_out,
                        sc_stream_t stream);

/*
 * Packed tables (halve the device->host copy and the gather of the results; a
 * LOSSLESS re-encoding of the Eq. 3 output, not a different result).
 * sc_bm_set_packed(plan, cap_rows > 0) switches a uint8 L2 plan with one channel on the box-sum
 * matcher (SC_KERNEL_BOX; b = 8, stride 4) to writing every (idx, dist) result as ONE uint32 word
 *     w = (dist << rb) | slot,   slot = (cy - ry - lo) * Wn + (cx - rx - lo)   (the window slot),
 * rb = ceil(log2(Wn^2)) (>= 2, from sc_bm_packed_words), for every row whose K distances are all
 * < 2^(32 - rb) - 1 (the matcher's own 32-bit keys: the words ARE its register keys). A row that
 * does not fit (a distance >= 2^(32-rb) - 1, or fewer than K candidates) is written as K escape
 * words 0xFFFFFFFF and its exact row goes to the overflow area after the rows. Buffer layout
 * (uint32 words; sc_bm_packed_words(plan, n_images) gives the total):
 *     [0, R)          R = n_images * n_refs * K row words, rows in the order of idx_out,
 *     R + 0           escape rows written by the run (may exceed cap_rows: the excess is lost),
 *     R + 1           cap_rows,
 *     R + 2 + r (2 + 2K)   record r < min(count, cap_rows): the row number (n_refs * image +
 *                     reference; low, high 32 bits), its K idx, its K dist (as sc_bm_run_batch).
 * In packed mode sc_bm_run / sc_bm_run_batch / sc_bm_run_host take the packed buffer as
 * idx_out (device / host) and dist_out = NULL (else SC_ERR_INVALID_ARGUMENT); sc_bm_run_rows
 * over a partial band, sc_bm_run_temporal, T > 0 and any other matcher return SC_ERR_UNSUPPORTED.
 * cap_rows = 0 restores the plain tables. SC_ERR_UNSUPPORTED for a plan that cannot pack.
 * Records are in no particular order (device atomics); decoded tables are identical to the plain
 * run's. run_host allocates its overflow staging on the first packed call.
 */
sc_status_t sc_bm_set_packed(sc_bm_plan_t plan, int64_t cap_rows);
/* Words of a packed buffer for n_images images and the slot bits rb (host pointers). */
sc_status_t sc_bm_packed_words(sc_bm_plan_t plan, int64_t n_images, int64_t* words_out, int32_t* rel_bits_out);
/*
 * Decode a packed buffer of n_images images (device pointers) into idx_out / dist_out
 * [n_images][n_refs][K] int32 (the plain tables, bit-identical). Reads the overflow count first
 * (synchronises `stream`): SC_ERR_OVERFLOW when escape rows were lost (re-run unpacked or with a
 * larger cap_rows); then two kernels, asynchronous on `stream`.
 */
sc_status_t sc_bm_unpack(sc_bm_plan_t plan, const uint32_t* packed, int64_t n_images, int32_t* idx_out,
                         int32_t* dist_out, sc_stream_t stream);
/*
 * The same decode on the host (plain C++; no device, no plan: the geometry is passed): for a
 * packed buffer of n_images images of H x W with patch b, stride, window Wn, K results per row.
 * SC_ERR_INVALID_ARGUMENT for a bad geometry or a slot outside the window, SC_ERR_OVERFLOW when
 * escape rows were lost.
 */
sc_status_t sc_bm_unpack_host(int H, int W, int b, int stride, int window, int K, const uint32_t* packed,
                              int64_t n_images, int32_t* idx_out, int32_t* dist_out);

/* Plan geometry and bookkeeping. */
sc_status_t sc_bm_plan_info(sc_bm_plan_t plan, sc_bm_info_t* info);

/* Force a kernel (SC_KERNEL_*) for the cross-term/top-K step; for tests and benchmarks. */
sc_status_t sc_bm_set_kernel(sc_bm_plan_t plan, int32_t kernel);

/*
 * Per-kernel device timing (bench.py's roofline): when enabled, every chunk enqueued by a
 * run call records CUDA events on the run stream around its norm kernels and around its
 * matching kernel. sc_bm_get_timing waits for the recorded events, returns the summed
 * durations (milliseconds) and launch counts since the last call, and resets them.
 * Enabling pre-creates the event pool (allocation); it is off by default.
 */
typedef struct {
    double norm_ms, match_ms;     /* summed device time of the norm kernels / matching kernel */
    int64_t norm_chunks, match_launches;
} sc_bm_timing_t;
sc_status_t sc_bm_set_timing(sc_bm_plan_t plan, int32_t enable);
sc_status_t sc_bm_get_timing(sc_bm_plan_t plan, sc_bm_timing_t* out);

/* Free the plan and its workspace (NULL is a no-op). */
sc_status_t sc_bm_destroy(sc_bm_plan_t plan);

/* Static string for a status code. */
const char* sc_status_string(sc_status_t s);

/*
 * Test export of step a1: the norm map h_X (.) h_X of the CENTRED image
 * (u8: x - 128; f32: x - 0.5), channels summed, built from the integral image:
 * norm_out [(H-b+1)][(W-b+1)] int32 (u8) or float (f32). One image, device pointers.
 */
sc_status_t sc_bm_norm_map(sc_bm_plan_t plan, const void* img, void* norm_out, sc_stream_t stream);

/*
 * Test export of steps a2+a3 (Eq. 5 + Lemma 2) without selection: every window distance
 * dist_all [n_refs][Wn*Wn] (slot (dy-lo)*Wn + (dx-lo)), int32 (u8) or float (f32), -1 in
 * clipped slots. Computed by the same cross-term code as the matching kernel. One image.
 */
sc_status_t sc_bm_run_dense_debug(sc_bm_plan_t plan, const void* img, void* dist_all,
                                  sc_stream_t stream);

/*
 * Test export: the number of references the LAST matching launch of the plan (its last frame
 * chunk) sent to the exact fix-up kernel (u8 L2: saturated or unfilled 32-bit keys; NCC: key
 * quantisation that could hide a top-K candidate). Synchronises the device; host pointer.
 */
sc_status_t sc_bm_debug_fix_count(sc_bm_plan_t plan, int32_t* count_out);

#ifdef __cplusplus
}
#endif

#endif /* SC_BM_H */
