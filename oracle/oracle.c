/*
 * oracle.c -- plain, slow, obviously-correct CPU block matching (TEST INFRASTRUCTURE ONLY).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library. The product path (paper_2006_13714_b200/) never does,
 * and this file shares no code, header, table or helper with it.
 *
 * What it computes is the plain definition the paper proves Self-Convolution reaches
 * exactly (Theorem 1, proof PAPER.md:468-521; Lemma 2):
 *
 *   Euclidean block matching, Eq. 3:
 *       S_i = argmin_{|S| <= K} sum_{j in S} ||X_j - X_i||_F^2
 *   restricted to the search window Omega_i (footnote 2), with the
 *   multi-channel distance summed over channels (Eq. 12's S(.)).
 *
 * Readings of the paper:
 *   R1 window = Wn x Wn candidate top-left offsets dy,dx in [lo, hi],
 *      lo = -floor(Wn/2), hi = Wn-1-floor(Wn/2), centred on the reference's top-left;
 *   R3 window clipped to valid positions [0,H-b] x [0,W-b];
 *   R5 reference grid {0, s, 2s, ...} <= H-b (and W-b), raster order, images outermost;
 *   R6 every candidate position (candidate stride 1);
 *   R7 ties broken by (distance, idx) lexicographic, idx = cy*W + cx (pixel raster);
 *   R8 K smallest distances (= K largest values of b_i);
 *   R9 fewer than K candidates: idx = -1, dist = INT32_MAX (u8) / +inf (float).
 *
 * Arithmetic: distances by DIRECT differences (not the identity), int64 for uint8
 * input, double for float/double input. A full sort of every window candidate per
 * reference (qsort), first K kept. OpenMP over references only; the result does not
 * depend on the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define SCO_U8 0
#define SCO_F32 1
#define SCO_F64 2

typedef struct {
    double d;
    int64_t di; /* exact integer distance for u8 */
    int32_t idx;
} sco_key;

static double px(const void* img, int dtype, size_t off) {
    if (dtype == SCO_U8) return (double)((const uint8_t*)img)[off];
    if (dtype == SCO_F32) return (double)((const float*)img)[off];
    return ((const double*)img)[off];
}

static int cmp_key_int(const void* a, const void* b) {
    const sco_key* x = (const sco_key*)a;
    const sco_key* y = (const sco_key*)b;
    if (x->di != y->di) return x->di < y->di ? -1 : 1;
    return (x->idx > y->idx) - (x->idx < y->idx);
}

static int cmp_key_dbl(const void* a, const void* b) {
    const sco_key* x = (const sco_key*)a;
    const sco_key* y = (const sco_key*)b;
    if (x->d != y->d) return x->d < y->d ? -1 : 1;
    return (x->idx > y->idx) - (x->idx < y->idx);
}

/* Reference grid size along one axis (R5). */
static int grid_n(int extent, int b, int s) { return (extent - b) / s + 1; }

/* ||X_c - X_r||_F^2 by direct differences, summed over channels (Eq. 3 + Eq. 12). */
static void patch_dist(const void* img, int dtype, int C, int H, int W, int b,
                       int ry, int rx, int cy, int cx, int64_t* di, double* d) {
    if (dtype == SCO_U8) {
        const uint8_t* p = (const uint8_t*)img;
        int64_t acc = 0;
        for (int c = 0; c < C; ++c)
            for (int l = 0; l < b; ++l)
                for (int m = 0; m < b; ++m) {
                    size_t base = (size_t)c * H * W;
                    int64_t v = (int64_t)p[base + (size_t)(ry + l) * W + rx + m] -
                                (int64_t)p[base + (size_t)(cy + l) * W + cx + m];
                    acc += v * v;
                }
        *di = acc;
        *d = (double)acc;
    } else {
        double acc = 0.0;
        for (int c = 0; c < C; ++c)
            for (int l = 0; l < b; ++l)
                for (int m = 0; m < b; ++m) {
                    size_t base = (size_t)c * H * W;
                    double v = px(img, dtype, base + (size_t)(ry + l) * W + rx + m) -
                               px(img, dtype, base + (size_t)(cy + l) * W + cx + m);
                    acc += v * v;
                }
        *di = 0;
        *d = acc;
    }
}

/*
 * Brute-force BM for images [img_begin, img_end) and reference-grid rows [iy_begin, iy_end)
 * of each image. Outputs are [n_img][n_rows * n_ref_x][K] in reference raster order:
 * idx_out int32; dist_out int32 (u8 input) or double (float input).
 * Returns 0 on success, -1 on bad arguments.
 */
int sco_bm_rows(const void* imgs, int dtype, int C, int H, int W, int b, int s, int Wn, int K,
                int img_begin, int img_end, int iy_begin, int iy_end,
                int32_t* idx_out, void* dist_out, int nthreads) {
    if (!imgs || !idx_out || !dist_out || b < 1 || s < 1 || Wn < 1 || K < 1 || C < 1 ||
        H < b || W < b || img_end < img_begin)
        return -1;
    const int ny = grid_n(H, b, s), nx = grid_n(W, b, s);
    if (iy_begin < 0 || iy_end > ny || iy_end < iy_begin) return -1;
    const int lo = -(Wn / 2), hi = Wn - 1 - Wn / 2;
    const int rows = iy_end - iy_begin;
    const long long refs_per_img = (long long)rows * nx;
    const long long total = refs_per_img * (img_end - img_begin);
    const size_t img_elems = (size_t)C * H * W;
    const size_t esz = dtype == SCO_U8 ? 1 : dtype == SCO_F32 ? 4 : 8;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif

#pragma omp parallel
    {
        sco_key* keys = (sco_key*)malloc(sizeof(sco_key) * (size_t)Wn * (size_t)Wn);
#pragma omp for schedule(dynamic, 16)
        for (long long t = 0; t < total; ++t) {
            const int n = img_begin + (int)(t / refs_per_img);
            const long long j = t % refs_per_img;
            const int iy = iy_begin + (int)(j / nx), ix = (int)(j % nx);
            const int ry = iy * s, rx = ix * s;
            const void* img = (const char*)imgs + (size_t)n * img_elems * esz;
            /* R1 + R3: clipped window of candidate top-left positions. */
            const int cy0 = ry + lo < 0 ? 0 : ry + lo;
            const int cy1 = ry + hi > H - b ? H - b : ry + hi;
            const int cx0 = rx + lo < 0 ? 0 : rx + lo;
            const int cx1 = rx + hi > W - b ? W - b : rx + hi;
            int cnt = 0;
            for (int cy = cy0; cy <= cy1; ++cy)
                for (int cx = cx0; cx <= cx1; ++cx) {
                    patch_dist(img, dtype, C, H, W, b, ry, rx, cy, cx, &keys[cnt].di, &keys[cnt].d);
                    keys[cnt].idx = cy * W + cx;
                    ++cnt;
                }
            qsort(keys, (size_t)cnt, sizeof(sco_key), dtype == SCO_U8 ? cmp_key_int : cmp_key_dbl);
            const long long o = t * K;
            for (int k = 0; k < K; ++k) {
                if (k < cnt) {
                    idx_out[o + k] = keys[k].idx;
                    if (dtype == SCO_U8) ((int32_t*)dist_out)[o + k] = (int32_t)keys[k].di;
                    else ((double*)dist_out)[o + k] = keys[k].d;
                } else {
                    idx_out[o + k] = -1;
                    if (dtype == SCO_U8) ((int32_t*)dist_out)[o + k] = INT32_MAX;
                    else ((double*)dist_out)[o + k] = INFINITY;
                }
            }
        }
        free(keys);
    }
    return 0;
}

/* All references of all n_img images. */
int sco_bm(const void* imgs, int dtype, int n_img, int C, int H, int W, int b, int s, int Wn,
           int K, int32_t* idx_out, void* dist_out, int nthreads) {
    if (H < b || s < 1) return -1;
    return sco_bm_rows(imgs, dtype, C, H, W, b, s, Wn, K, 0, n_img, 0, grid_n(H, b, s),
                       idx_out, dist_out, nthreads);
}

/*
 * Every window distance (debug / cross-term check): dist_all[n_refs][Wn*Wn], slot
 * (dy-lo)*Wn + (dx-lo); clipped slots hold -1. One image.
 */
int sco_bm_dense(const void* img, int dtype, int C, int H, int W, int b, int s, int Wn,
                 double* dist_all, int nthreads) {
    if (!img || !dist_all || b < 1 || s < 1 || Wn < 1 || H < b || W < b) return -1;
    const int ny = grid_n(H, b, s), nx = grid_n(W, b, s);
    const int lo = -(Wn / 2);
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel for schedule(dynamic, 16)
    for (long long t = 0; t < (long long)ny * nx; ++t) {
        const int ry = (int)(t / nx) * s, rx = (int)(t % nx) * s;
        for (int a = 0; a < Wn; ++a)
            for (int c = 0; c < Wn; ++c) {
                const int cy = ry + lo + a, cx = rx + lo + c;
                double* out = &dist_all[t * Wn * Wn + (long long)a * Wn + c];
                if (cy < 0 || cx < 0 || cy > H - b || cx > W - b) {
                    *out = -1.0;
                    continue;
                }
                int64_t di;
                patch_dist(img, dtype, C, H, W, b, ry, rx, cy, cx, &di, out);
            }
    }
    return 0;
}

/*
 * h_X (.) h_X: ||X_j||_F^2 for every valid position j (used in Lemma 2),
 * summed over channels; by direct summation. out[(H-b+1)*(W-b+1)] (double).
 */
int sco_norm_map(const void* img, int dtype, int C, int H, int W, int b, double* out) {
    if (!img || !out || b < 1 || H < b || W < b) return -1;
    const int My = H - b + 1, Mx = W - b + 1;
    for (int y = 0; y < My; ++y)
        for (int x = 0; x < Mx; ++x) {
            double acc = 0.0;
            for (int c = 0; c < C; ++c)
                for (int l = 0; l < b; ++l)
                    for (int m = 0; m < b; ++m) {
                        double v = px(img, dtype, (size_t)c * H * W + (size_t)(y + l) * W + x + m);
                        acc += v * v;
                    }
            out[(size_t)y * Mx + x] = acc;
        }
    return 0;
}

/*
 * Self-Convolution, Eq. 5 summed over channels (Eq. 12):
 *   C_i(q, r) = sum_{c,l,m} X_i(l, m) X(q + l, r + m)   (0-based)
 * for the reference patch at (ry, rx), over the whole image: out[(H-b+1)*(W-b+1)].
 */
int sco_selfconv(const void* img, int dtype, int C, int H, int W, int b, int ry, int rx,
                 double* out) {
    if (!img || !out || b < 1 || H < b || W < b || ry < 0 || rx < 0 || ry > H - b || rx > W - b)
        return -1;
    const int My = H - b + 1, Mx = W - b + 1;
    for (int q = 0; q < My; ++q)
        for (int r = 0; r < Mx; ++r) {
            double acc = 0.0;
            for (int c = 0; c < C; ++c)
                for (int l = 0; l < b; ++l)
                    for (int m = 0; m < b; ++m) {
                        size_t base = (size_t)c * H * W;
                        acc += px(img, dtype, base + (size_t)(ry + l) * W + rx + m) *
                               px(img, dtype, base + (size_t)(q + l) * W + r + m);
                    }
            out[(size_t)q * Mx + r] = acc;
        }
    return 0;
}

/*
 * Direct distances for an explicit list of (reference, candidate) pairs of one image:
 * out[k] = ||X_{(cy,cx)} - X_{(ry,rx)}||_F^2 by direct differences (Eq. 3), channels summed.
 * Used to check sampled GPU outputs one by one at full size.
 */
int sco_pair_dist(const void* img, int dtype, int C, int H, int W, int b, long long n,
                  const int32_t* ry, const int32_t* rx, const int32_t* cy, const int32_t* cx,
                  double* out) {
    if (!img || !out || b < 1 || H < b || W < b) return -1;
    for (long long k = 0; k < n; ++k) {
        if (ry[k] < 0 || rx[k] < 0 || cy[k] < 0 || cx[k] < 0 || ry[k] > H - b || cy[k] > H - b ||
            rx[k] > W - b || cx[k] > W - b)
            return -1;
        int64_t di;
        patch_dist(img, dtype, C, H, W, b, ry[k], rx[k], cy[k], cx[k], &di, &out[k]);
    }
    return 0;
}

/*
 * -NCC of explicit (reference, candidate) pairs (Eq. 4, on the raw values,
 * channels summed; NCC := 0 when a norm is 0, R15), double -- the same arithmetic as
 * sco_ncc_rows' reported value, for full-size checks of sampled or selected pairs.
 */
int sco_pair_ncc(const void* img, int dtype, int C, int H, int W, int b, long long n,
                 const int32_t* ry, const int32_t* rx, const int32_t* cy, const int32_t* cx,
                 double* out) {
    if (!img || !out || b < 1 || H < b || W < b) return -1;
    for (long long k = 0; k < n; ++k) {
        if (ry[k] < 0 || rx[k] < 0 || cy[k] < 0 || cx[k] < 0 || ry[k] > H - b || cy[k] > H - b ||
            rx[k] > W - b || cx[k] > W - b)
            return -1;
        double nr = 0.0, nc = 0.0, cc = 0.0;
        for (int c = 0; c < C; ++c)
            for (int l = 0; l < b; ++l)
                for (int m = 0; m < b; ++m) {
                    const size_t base = (size_t)c * H * W;
                    const double vr = px(img, dtype, base + (size_t)(ry[k] + l) * W + rx[k] + m);
                    const double vc = px(img, dtype, base + (size_t)(cy[k] + l) * W + cx[k] + m);
                    cc += vr * vc;
                    nr += vr * vr;
                    nc += vc * vc;
                }
        const double den = sqrt(nr * nc);
        out[k] = den > 0.0 ? -(cc / den) : 0.0;
    }
    return 0;
}

/*
 * NCC block matching (the "next" row): Eq. 4,
 *   S_i = argmin_{|S| <= K} sum_{j in S} d_NCC(X_j, X_i),
 *   d_NCC(X_j, X_i) = - vec(X_j)^T vec(X_i) / (||X_j||_F ||X_i||_F)
 * on the RAW (uncentred, "non-negative natural image") values, channels summed jointly, over
 * the same clipped window, i.e. the K LARGEST normalised cross-correlations. Readings
 * (R14-R16): NCC := 0 when ||X_j|| ||X_i|| = 0; ties by (d_NCC, idx).
 * Ordering is EXACT for uint8 input: NCC_a > NCC_b is decided on integers, comparing
 * C_a |C_a| n_b with C_b |C_b| n_a in 128-bit arithmetic (n = squared norms); double for
 * float input. dist_out = d_NCC = -NCC (double), idx -1 / +inf for missing candidates.
 */
typedef struct {
    int64_t c, n;  /* exact cross term / candidate squared norm (u8) */
    double f;      /* NCC (float input, and the reported value) */
    int32_t idx;
} sco_nkey;

static int cmp_ncc_int(const void* a, const void* b) {
    const sco_nkey* x = (const sco_nkey*)a;
    const sco_nkey* y = (const sco_nkey*)b;
    /* larger NCC first: sign(c) c^2 / n, cross-multiplied (n > 0 here: zero norms map to c=0, n=1) */
    const __int128 lx = (__int128)(x->c < 0 ? -x->c : x->c) * x->c * y->n;
    const __int128 ly = (__int128)(y->c < 0 ? -y->c : y->c) * y->c * x->n;
    if (lx != ly) return lx > ly ? -1 : 1;
    return (x->idx > y->idx) - (x->idx < y->idx);
}

static int cmp_ncc_dbl(const void* a, const void* b) {
    const sco_nkey* x = (const sco_nkey*)a;
    const sco_nkey* y = (const sco_nkey*)b;
    if (x->f != y->f) return x->f > y->f ? -1 : 1;
    return (x->idx > y->idx) - (x->idx < y->idx);
}

int sco_ncc_rows(const void* imgs, int dtype, int C, int H, int W, int b, int s, int Wn, int K,
                 int img_begin, int img_end, int iy_begin, int iy_end,
                 int32_t* idx_out, double* dist_out, int nthreads) {
    if (!imgs || !idx_out || !dist_out || b < 1 || s < 1 || Wn < 1 || K < 1 || C < 1 ||
        H < b || W < b || img_end < img_begin)
        return -1;
    const int ny = grid_n(H, b, s), nx = grid_n(W, b, s);
    if (iy_begin < 0 || iy_end > ny || iy_end < iy_begin) return -1;
    const int lo = -(Wn / 2), hi = Wn - 1 - Wn / 2;
    const long long refs_per_img = (long long)(iy_end - iy_begin) * nx;
    const long long total = refs_per_img * (img_end - img_begin);
    const size_t img_elems = (size_t)C * H * W;
    const size_t esz = dtype == SCO_U8 ? 1 : dtype == SCO_F32 ? 4 : 8;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel
    {
        sco_nkey* keys = (sco_nkey*)malloc(sizeof(sco_nkey) * (size_t)Wn * (size_t)Wn);
#pragma omp for schedule(dynamic, 16)
        for (long long t = 0; t < total; ++t) {
            const int n = img_begin + (int)(t / refs_per_img);
            const long long j = t % refs_per_img;
            const int ry = (iy_begin + (int)(j / nx)) * s, rx = (int)(j % nx) * s;
            const void* img = (const char*)imgs + (size_t)n * img_elems * esz;
            const int cy0 = ry + lo < 0 ? 0 : ry + lo, cy1 = ry + hi > H - b ? H - b : ry + hi;
            const int cx0 = rx + lo < 0 ? 0 : rx + lo, cx1 = rx + hi > W - b ? W - b : rx + hi;
            /* reference squared norm */
            int64_t nri = 0;
            double nrd = 0.0;
            for (int c = 0; c < C; ++c)
                for (int l = 0; l < b; ++l)
                    for (int m = 0; m < b; ++m) {
                        const double v = px(img, dtype, (size_t)c * H * W + (size_t)(ry + l) * W + rx + m);
                        nrd += v * v;
                        nri += (int64_t)v * (int64_t)v;
                    }
            int cnt = 0;
            for (int cy = cy0; cy <= cy1; ++cy)
                for (int cx = cx0; cx <= cx1; ++cx) {
                    int64_t ci = 0, nci = 0;
                    double cd = 0.0, ncd = 0.0;
                    for (int c = 0; c < C; ++c)
                        for (int l = 0; l < b; ++l)
                            for (int m = 0; m < b; ++m) {
                                const size_t base = (size_t)c * H * W;
                                const double vr = px(img, dtype, base + (size_t)(ry + l) * W + rx + m);
                                const double vc = px(img, dtype, base + (size_t)(cy + l) * W + cx + m);
                                cd += vr * vc;
                                ncd += vc * vc;
                                if (dtype == SCO_U8) {
                                    ci += (int64_t)vr * (int64_t)vc;
                                    nci += (int64_t)vc * (int64_t)vc;
                                }
                            }
                    sco_nkey* k = &keys[cnt++];
                    k->idx = cy * W + cx;
                    const double den = sqrt(nrd * ncd);
                    k->f = den > 0.0 ? cd / den : 0.0;
                    if (nri == 0 || nci == 0) {  /* NCC := 0 */
                        k->c = 0;
                        k->n = 1;
                    } else {
                        k->c = ci;
                        k->n = nci;
                    }
                }
            qsort(keys, (size_t)cnt, sizeof(sco_nkey), dtype == SCO_U8 ? cmp_ncc_int : cmp_ncc_dbl);
            const long long o = t * K;
            for (int k = 0; k < K; ++k) {
                idx_out[o + k] = k < cnt ? keys[k].idx : -1;
                dist_out[o + k] = k < cnt ? -keys[k].f : INFINITY;
            }
        }
        free(keys);
    }
    return 0;
}

/*
 * 3D / temporal block matching (the video setting of PAPER.md:661, 697):
 * Eq. 3 with the candidate set of a reference in frame f = the clipped window positions of
 * frames f-T .. f+T of the batch (clipped to [0, n_img)), idx = frame * H * W + cy * W + cx
 * (batch-global), ties by (d, idx). uint8 / float as sco_bm_rows; all references of all frames.
 */
int sco_bm_temporal(const void* imgs, int dtype, int n_img, int C, int H, int W, int b, int s, int Wn,
                    int K, int T, int32_t* idx_out, void* dist_out, int nthreads) {
    if (!imgs || !idx_out || !dist_out || b < 1 || s < 1 || Wn < 1 || K < 1 || C < 1 || H < b ||
        W < b || n_img < 1 || T < 0)
        return -1;
    const int ny = grid_n(H, b, s), nx = grid_n(W, b, s);
    const int lo = -(Wn / 2), hi = Wn - 1 - Wn / 2;
    const long long refs_per_img = (long long)ny * nx, total = refs_per_img * n_img;
    const size_t img_elems = (size_t)C * H * W;
    const size_t esz = dtype == SCO_U8 ? 1 : dtype == SCO_F32 ? 4 : 8;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel
    {
        sco_key* keys = (sco_key*)malloc(sizeof(sco_key) * (size_t)Wn * (size_t)Wn * (size_t)(2 * T + 1));
#pragma omp for schedule(dynamic, 16)
        for (long long t = 0; t < total; ++t) {
            const int f = (int)(t / refs_per_img);
            const long long j = t % refs_per_img;
            const int ry = (int)(j / nx) * s, rx = (int)(j % nx) * s;
            const int cy0 = ry + lo < 0 ? 0 : ry + lo, cy1 = ry + hi > H - b ? H - b : ry + hi;
            const int cx0 = rx + lo < 0 ? 0 : rx + lo, cx1 = rx + hi > W - b ? W - b : rx + hi;
            const char* rimg = (const char*)imgs + (size_t)f * img_elems * esz;
            int cnt = 0;
            for (int fr = f - T; fr <= f + T; ++fr) {
                if (fr < 0 || fr >= n_img) continue;
                const char* cimg = (const char*)imgs + (size_t)fr * img_elems * esz;
                for (int cy = cy0; cy <= cy1; ++cy)
                    for (int cx = cx0; cx <= cx1; ++cx) {
                        /* direct differences between frame f's reference and frame fr's candidate */
                        int64_t acc = 0;
                        double accd = 0.0;
                        for (int c = 0; c < C; ++c)
                            for (int l = 0; l < b; ++l)
                                for (int m = 0; m < b; ++m) {
                                    const size_t base = (size_t)c * H * W;
                                    const double vr = px(rimg, dtype, base + (size_t)(ry + l) * W + rx + m);
                                    const double vc = px(cimg, dtype, base + (size_t)(cy + l) * W + cx + m);
                                    accd += (vr - vc) * (vr - vc);
                                    if (dtype == SCO_U8) acc += (int64_t)(vr - vc) * (int64_t)(vr - vc);
                                }
                        keys[cnt].di = acc;
                        keys[cnt].d = accd;
                        keys[cnt].idx = (int32_t)((long long)fr * H * W + (long long)cy * W + cx);
                        ++cnt;
                    }
            }
            qsort(keys, (size_t)cnt, sizeof(sco_key), dtype == SCO_U8 ? cmp_key_int : cmp_key_dbl);
            const long long o = t * K;
            for (int k = 0; k < K; ++k) {
                idx_out[o + k] = k < cnt ? keys[k].idx : -1;
                if (dtype == SCO_U8) ((int32_t*)dist_out)[o + k] = k < cnt ? (int32_t)keys[k].di : INT32_MAX;
                else ((double*)dist_out)[o + k] = k < cnt ? keys[k].d : INFINITY;
            }
        }
        free(keys);
    }
    return 0;
}

/*
 * NLM weights, Eq. 2 restricted to the search window (footnote 2,
 * PAPER.md:280; the SAME clipped window as BM):
 *   s_i(j) = exp(-||X_j - X_i||_F^2 / h^2) / Theta_i,  Theta_i = sum_j exp(-||X_j - X_i||^2 / h^2)
 * with direct-difference distances (double). out[n_refs][Wn*Wn], slot (dy-lo)*Wn + (dx-lo), 0 in
 * clipped slots. The common factor exp(d_min / h^2) is taken out of numerator and Theta_i
 * (s_i(j) = exp(-(d_j - d_min)/h^2) / sum_k exp(-(d_k - d_min)/h^2): the same ratio) so that
 * large d / h^2 cannot underflow to 0/0. One image.
 */
int sco_nlm_weights(const void* img, int dtype, int C, int H, int W, int b, int s, int Wn, double h,
                    double* out, int nthreads) {
    if (!img || !out || b < 1 || s < 1 || Wn < 1 || H < b || W < b || !(h > 0.0)) return -1;
    const int ny = grid_n(H, b, s), nx = grid_n(W, b, s);
    const int lo = -(Wn / 2);
    const int nslot = Wn * Wn;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel for schedule(dynamic, 16)
    for (long long t = 0; t < (long long)ny * nx; ++t) {
        const int ry = (int)(t / nx) * s, rx = (int)(t % nx) * s;
        double* row = &out[t * nslot];
        double dmin = INFINITY;
        for (int a = 0; a < Wn; ++a)
            for (int c = 0; c < Wn; ++c) {
                const int cy = ry + lo + a, cx = rx + lo + c;
                double* o = &row[a * Wn + c];
                if (cy < 0 || cx < 0 || cy > H - b || cx > W - b) {
                    *o = -1.0;
                    continue;
                }
                int64_t di;
                patch_dist(img, dtype, C, H, W, b, ry, rx, cy, cx, &di, o);
                if (*o < dmin) dmin = *o;
            }
        double theta = 0.0;
        for (int k = 0; k < nslot; ++k) {
            row[k] = row[k] < 0.0 ? 0.0 : exp(-(row[k] - dmin) / (h * h));
            theta += row[k];
        }
        for (int k = 0; k < nslot; ++k) row[k] /= theta;
    }
    return 0;
}

int sco_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/*
 * 3D block matching (the "next" row SURVEY.md 8f rank 4): the paper's 3D Self-Convolution
 * (patches Y_i of sqrt(n) x sqrt(n) x d with d < p, searched "across channels" by a
 * 3D FFT instead of the channel sum S(.)) and its video setting (SALT: 6 x 6 x 1 patches in a
 * 30 x 30 x c window, c = 9 frames). A volume V[P][H][W] of planes (the channels of
 * one image, or the frames of a video); a patch is d consecutive planes x b x b; references start at
 * planes z in {0, sz, 2 sz, ...} <= P - d and on the usual spatial grid; the candidates of a
 * reference at plane z are the patches starting at planes z + dz, dz in [lo_z, hi_z]
 * (lo_z = -floor(c/2), hi_z = c - 1 - floor(c/2), reading R4 for even c), clipped to [0, P - d],
 * and at the clipped spatial window positions (footnote 2);
 *     d(r, c) = sum_{t < d} sum_{l, m} (V[z_r + t][ry + l][rx + m] - V[z_c + t][cy + l][cx + m])^2
 * by direct differences (int64 for uint8, double otherwise), idx = (z_c H + cy) W + cx (the volume
 * raster of the candidate's first voxel), ties by (d, idx), output [n_zref][n_refs][K] with
 * n_zref = floor((P - d) / sz) + 1. d = P, c = 1 is multi-channel 2D BM; d = 1, c = 2T + 1,
 * sz = 1 is the temporal search of sco_bm_temporal.
 */
int sco_bm3d(const void* vol, int dtype, int P, int H, int W, int d, int b, int s, int sz, int Wn, int c,
             int K, int32_t* idx_out, void* dist_out, int nthreads) {
    if (!vol || !idx_out || !dist_out || P < 1 || d < 1 || d > P || b < 1 || s < 1 || sz < 1 || Wn < 1 ||
        c < 1 || K < 1 || H < b || W < b)
        return -1;
    const int ny = grid_n(H, b, s), nx = grid_n(W, b, s), nz = (P - d) / sz + 1;
    const int lo = -(Wn / 2), hi = Wn - 1 - Wn / 2, loz = -(c / 2), hiz = c - 1 - c / 2;
    const long long refs2d = (long long)ny * nx, total = refs2d * nz;
    const size_t plane = (size_t)H * W;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel
    {
        sco_key* keys = (sco_key*)malloc(sizeof(sco_key) * (size_t)Wn * (size_t)Wn * (size_t)c);
#pragma omp for schedule(dynamic, 16)
        for (long long t = 0; t < total; ++t) {
            const int zr = (int)(t / refs2d) * sz;
            const long long j = t % refs2d;
            const int ry = (int)(j / nx) * s, rx = (int)(j % nx) * s;
            const int cy0 = ry + lo < 0 ? 0 : ry + lo, cy1 = ry + hi > H - b ? H - b : ry + hi;
            const int cx0 = rx + lo < 0 ? 0 : rx + lo, cx1 = rx + hi > W - b ? W - b : rx + hi;
            int cnt = 0;
            for (int zc = zr + loz; zc <= zr + hiz; ++zc) {
                if (zc < 0 || zc > P - d) continue;
                for (int cy = cy0; cy <= cy1; ++cy)
                    for (int cx = cx0; cx <= cx1; ++cx) {
                        int64_t acc = 0;
                        double accd = 0.0;
                        for (int q = 0; q < d; ++q)
                            for (int l = 0; l < b; ++l)
                                for (int m = 0; m < b; ++m) {
                                    const double vr = px(vol, dtype, (size_t)(zr + q) * plane + (size_t)(ry + l) * W + rx + m);
                                    const double vc = px(vol, dtype, (size_t)(zc + q) * plane + (size_t)(cy + l) * W + cx + m);
                                    accd += (vr - vc) * (vr - vc);
                                    if (dtype == SCO_U8) acc += (int64_t)(vr - vc) * (int64_t)(vr - vc);
                                }
                        keys[cnt].di = acc;
                        keys[cnt].d = accd;
                        keys[cnt].idx = (int32_t)(((long long)zc * H + cy) * W + cx);
                        ++cnt;
                    }
            }
            qsort(keys, (size_t)cnt, sizeof(sco_key), dtype == SCO_U8 ? cmp_key_int : cmp_key_dbl);
            const long long o = t * K;
            for (int k = 0; k < K; ++k) {
                idx_out[o + k] = k < cnt ? keys[k].idx : -1;
                if (dtype == SCO_U8) ((int32_t*)dist_out)[o + k] = k < cnt ? (int32_t)keys[k].di : INT32_MAX;
                else ((double*)dist_out)[o + k] = k < cnt ? keys[k].d : INFINITY;
            }
        }
        free(keys);
    }
    return 0;
}

/* Direct distances of explicit 3D pairs (d-plane patches starting at planes zr / zc of a P-plane
 * volume), double -- the definition of sco_bm3d for full-size parity checks of selected pairs. */
int sco_pair_dist3d(const void* vol, int dtype, int P, int H, int W, int d, int b, long long n,
                    const int32_t* zr, const int32_t* ry, const int32_t* rx, const int32_t* zc,
                    const int32_t* cy, const int32_t* cx, double* out) {
    if (!vol || !out || d < 1 || d > P || b < 1 || H < b || W < b) return -1;
    const size_t plane = (size_t)H * W;
    for (long long k = 0; k < n; ++k) {
        if (zr[k] < 0 || zc[k] < 0 || zr[k] > P - d || zc[k] > P - d || ry[k] < 0 || rx[k] < 0 || cy[k] < 0 ||
            cx[k] < 0 || ry[k] > H - b || cy[k] > H - b || rx[k] > W - b || cx[k] > W - b)
            return -1;
        double acc = 0.0;
        for (int q = 0; q < d; ++q)
            for (int l = 0; l < b; ++l)
                for (int m = 0; m < b; ++m) {
                    const double vr = px(vol, dtype, (size_t)(zr[k] + q) * plane + (size_t)(ry[k] + l) * W + rx[k] + m);
                    const double vc = px(vol, dtype, (size_t)(zc[k] + q) * plane + (size_t)(cy[k] + l) * W + cx[k] + m);
                    acc += (vr - vc) * (vr - vc);
                }
        out[k] = acc;
    }
    return 0;
}
