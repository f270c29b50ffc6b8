"""CPU oracle for Self-Convolution block matching -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package. The product path
(``paper_2006_13714_b200``) never imports it and shares no code with it.

``oracle.c`` is the plain brute-force definition (Eq. 3, restricted
to the window of footnote 2, channels summed as in Eq. 12,
PAPER.md:540-547); see its header for the readings it follows. Pins:
tests/test_oracle.py (hand-worked fixture, closed forms, invariants, exhaustive
8x8 vs an independent numpy brute force, torch conv2d special case).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

U8, F32, F64 = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc -O2 -fopenmp, no intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=c11",
                               _SRC, "-o", _LIB, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        vp, i32p, dp = ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_double)
        ci = ctypes.c_int
        L.sco_bm_rows.argtypes = [vp, ci, ci, ci, ci, ci, ci, ci, ci, ci, ci, ci, ci, i32p, vp, ci]
        L.sco_bm.argtypes = [vp, ci, ci, ci, ci, ci, ci, ci, ci, ci, i32p, vp, ci]
        L.sco_bm_dense.argtypes = [vp, ci, ci, ci, ci, ci, ci, ci, dp, ci]
        L.sco_norm_map.argtypes = [vp, ci, ci, ci, ci, ci, dp]
        L.sco_selfconv.argtypes = [vp, ci, ci, ci, ci, ci, ci, ci, dp]
        L.sco_pair_dist.argtypes = [vp, ci, ci, ci, ci, ci, ctypes.c_longlong, i32p, i32p, i32p, i32p, dp]
        L.sco_pair_ncc.argtypes = [vp, ci, ci, ci, ci, ci, ctypes.c_longlong, i32p, i32p, i32p, i32p, dp]
        L.sco_bm3d.argtypes = [vp, ci, ci, ci, ci, ci, ci, ci, ci, ci, ci, ci, i32p, vp, ci]
        L.sco_pair_dist3d.argtypes = [vp, ci, ci, ci, ci, ci, ci, ctypes.c_longlong] + [i32p] * 6 + [dp]
        L.sco_num_threads.restype = ci
        L.sco_ncc_rows.argtypes = [vp, ci, ci, ci, ci, ci, ci, ci, ci, ci, ci, ci, ci, i32p, dp, ci]
        L.sco_bm_temporal.argtypes = [vp, ci, ci, ci, ci, ci, ci, ci, ci, ci, ci, i32p, vp, ci]
        L.sco_nlm_weights.argtypes = [vp, ci, ci, ci, ci, ci, ci, ci, ctypes.c_double, dp, ci]
        _lib = L
    return _lib


def _dtype_code(a: np.ndarray) -> int:
    if a.dtype == np.uint8:
        return U8
    if a.dtype == np.float32:
        return F32
    if a.dtype == np.float64:
        return F64
    raise TypeError(f"oracle: unsupported dtype {a.dtype}")


def grid(H: int, W: int, b: int, s: int):
    return (H - b) // s + 1, (W - b) // s + 1


def bm(img: np.ndarray, b: int, s: int, Wn: int, K: int, *, images=None, rows=None,
       nthreads: int = 0):
    """Brute-force BM. img: [N, C, H, W] (or [C,H,W] / [H,W]) uint8/float32/float64.

    Returns (idx int32 [n, refs, K], dist int32 (uint8 input) or float64 [n, refs, K]).
    ``images=(i0, i1)`` and ``rows=(iy0, iy1)`` restrict to a subset (reference-grid rows).
    """
    a = np.ascontiguousarray(img)
    if a.ndim == 2:
        a = a[None, None]
    elif a.ndim == 3:
        a = a[None]
    N, C, H, W = a.shape
    ny, nx = grid(H, W, b, s)
    i0, i1 = images if images is not None else (0, N)
    r0, r1 = rows if rows is not None else (0, ny)
    n = i1 - i0
    refs = (r1 - r0) * nx
    idx = np.empty((n, refs, K), dtype=np.int32)
    code = _dtype_code(a)
    dist = np.empty((n, refs, K), dtype=np.int32 if code == U8 else np.float64)
    rc = lib().sco_bm_rows(a.ctypes.data, code, C, H, W, b, s, Wn, K, i0, i1, r0, r1,
                           idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                           dist.ctypes.data, nthreads)
    if rc != 0:
        raise ValueError("oracle.bm: invalid arguments")
    return idx, dist


def ncc(img: np.ndarray, b: int, s: int, Wn: int, K: int, *, images=None, rows=None,
        nthreads: int = 0):
    """NCC block matching (Eq. 4): the K largest normalised cross-correlations
    of raw values per reference window. Returns (idx int32, dist float64 = d_NCC = -NCC)
    [n, refs, K]; exact integer ordering for uint8 input (see oracle.c sco_ncc_rows)."""
    a = np.ascontiguousarray(img)
    if a.ndim == 2:
        a = a[None, None]
    elif a.ndim == 3:
        a = a[None]
    N, C, H, W = a.shape
    ny, nx = grid(H, W, b, s)
    i0, i1 = images if images is not None else (0, N)
    r0, r1 = rows if rows is not None else (0, ny)
    n, refs = i1 - i0, (r1 - r0) * nx
    idx = np.empty((n, refs, K), dtype=np.int32)
    dist = np.empty((n, refs, K), dtype=np.float64)
    rc = lib().sco_ncc_rows(a.ctypes.data, _dtype_code(a), C, H, W, b, s, Wn, K, i0, i1, r0, r1,
                            idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                            dist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), nthreads)
    if rc != 0:
        raise ValueError("oracle.ncc: invalid arguments")
    return idx, dist


def bm_temporal(img: np.ndarray, b: int, s: int, Wn: int, K: int, T: int, nthreads: int = 0):
    """Temporal BM over a batch [N, C, H, W]: candidates in frames f-T..f+T; idx batch-global
    (frame * H * W + cy * W + cx). Returns (idx int32, dist int32 | float64) [N, refs, K]."""
    a = np.ascontiguousarray(img)
    N, C, H, W = a.shape
    ny, nx = grid(H, W, b, s)
    idx = np.empty((N, ny * nx, K), dtype=np.int32)
    code = _dtype_code(a)
    dist = np.empty((N, ny * nx, K), dtype=np.int32 if code == U8 else np.float64)
    rc = lib().sco_bm_temporal(a.ctypes.data, code, N, C, H, W, b, s, Wn, K, T,
                               idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), dist.ctypes.data, nthreads)
    if rc != 0:
        raise ValueError("oracle.bm_temporal: invalid arguments")
    return idx, dist


def bm3d(vol: np.ndarray, d: int, b: int, s: int, sz: int, Wn: int, c: int, K: int, nthreads: int = 0):
    """3D block matching over the planes of a volume [P,H,W] (channels of one image or frames of a
    video): d-plane patches, references at planes 0, sz, ... <= P - d, candidates
    at plane offsets [-floor(c/2), c-1-floor(c/2)] x the clipped spatial window. Returns (idx int32,
    dist int32 (uint8) / float64) [n_zref, n_refs, K], idx = (z * H + y) * W + x."""
    a = np.ascontiguousarray(vol)
    if a.ndim == 4:
        a = a.reshape((-1,) + a.shape[2:])
    P, H, W = a.shape
    ny, nx = grid(H, W, b, s)
    nz = (P - d) // sz + 1
    code = _dtype_code(a)
    idx = np.empty((nz, ny * nx, K), dtype=np.int32)
    dist = np.empty((nz, ny * nx, K), dtype=np.int32 if code == U8 else np.float64)
    rc = lib().sco_bm3d(a.ctypes.data, code, P, H, W, d, b, s, sz, Wn, c, K,
                        idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), dist.ctypes.data, nthreads)
    if rc != 0:
        raise ValueError("oracle.bm3d: invalid arguments")
    return idx, dist


def nlm_weights(img: np.ndarray, b: int, s: int, Wn: int, h: float, nthreads: int = 0) -> np.ndarray:
    """NLM weights (Eq. 2) over each reference's clipped window, one image [C,H,W]:
    [refs, Wn*Wn] float64, 0 in clipped slots, rows summing to 1."""
    a = np.ascontiguousarray(img)
    if a.ndim == 2:
        a = a[None]
    C, H, W = a.shape
    ny, nx = grid(H, W, b, s)
    out = np.empty((ny * nx, Wn * Wn), dtype=np.float64)
    rc = lib().sco_nlm_weights(a.ctypes.data, _dtype_code(a), C, H, W, b, s, Wn, float(h),
                               out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), nthreads)
    if rc != 0:
        raise ValueError("oracle.nlm_weights: invalid arguments")
    return out


def nlm_average(img: np.ndarray, b: int, s: int, Wn: int, h: float, *, refs=None) -> np.ndarray:
    """NL-means estimate of every reference patch: X_i ~ sum_j s_i(j) X_j (after
    Eq. 2), the weights s_i(j) of nlm_weights over the clipped window, X_j the raw input patches.
    One image [C,H,W] -> [refs, C, b, b] float64 (refs: optional list of reference numbers).
    Plain loops over the definition (small images or sampled references)."""
    a = np.asarray(img)
    if a.ndim == 2:
        a = a[None]
    C, H, W = a.shape
    ny, nx = grid(H, W, b, s)
    w = nlm_weights(a, b, s, Wn, h)
    lo = -(Wn // 2)
    sel = range(ny * nx) if refs is None else refs
    out = np.zeros((len(sel), C, b, b), dtype=np.float64)
    x = a.astype(np.float64)
    for o, r in enumerate(sel):
        ry, rx = (r // nx) * s, (r % nx) * s
        for slot in range(Wn * Wn):
            if w[r, slot] == 0.0:
                continue
            cy, cx = ry + lo + slot // Wn, rx + lo + slot % Wn
            out[o] += w[r, slot] * x[:, cy:cy + b, cx:cx + b]
    return out


def bm_dense(img: np.ndarray, b: int, s: int, Wn: int, nthreads: int = 0) -> np.ndarray:
    """Every window distance of one image [C,H,W]: [refs, Wn*Wn] float64, -1 where clipped."""
    a = np.ascontiguousarray(img)
    if a.ndim == 2:
        a = a[None]
    C, H, W = a.shape
    ny, nx = grid(H, W, b, s)
    out = np.empty((ny * nx, Wn * Wn), dtype=np.float64)
    rc = lib().sco_bm_dense(a.ctypes.data, _dtype_code(a), C, H, W, b, s, Wn,
                            out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), nthreads)
    if rc != 0:
        raise ValueError("oracle.bm_dense: invalid arguments")
    return out


def norm_map(img: np.ndarray, b: int) -> np.ndarray:
    """h_X (.) h_X over valid positions, channels summed: [(H-b+1), (W-b+1)] float64."""
    a = np.ascontiguousarray(img)
    if a.ndim == 2:
        a = a[None]
    C, H, W = a.shape
    out = np.empty((H - b + 1, W - b + 1), dtype=np.float64)
    rc = lib().sco_norm_map(a.ctypes.data, _dtype_code(a), C, H, W, b,
                            out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    if rc != 0:
        raise ValueError("oracle.norm_map: invalid arguments")
    return out


def selfconv(img: np.ndarray, b: int, ry: int, rx: int) -> np.ndarray:
    """Eq. 5 Self-Convolution map C_i for the reference at (ry, rx): [(H-b+1), (W-b+1)]."""
    a = np.ascontiguousarray(img)
    if a.ndim == 2:
        a = a[None]
    C, H, W = a.shape
    out = np.empty((H - b + 1, W - b + 1), dtype=np.float64)
    rc = lib().sco_selfconv(a.ctypes.data, _dtype_code(a), C, H, W, b, ry, rx,
                            out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    if rc != 0:
        raise ValueError("oracle.selfconv: invalid arguments")
    return out


def pair_ncc(img: np.ndarray, b: int, ry, rx, cy, cx) -> np.ndarray:
    """-NCC (Eq. 4) of explicit (ref, candidate) pairs of one image [C,H,W]."""
    a = np.ascontiguousarray(img)
    if a.ndim == 2:
        a = a[None]
    C, H, W = a.shape
    arrs = [np.ascontiguousarray(np.asarray(v, dtype=np.int32).ravel()) for v in (ry, rx, cy, cx)]
    n = arrs[0].size
    out = np.empty(n, dtype=np.float64)
    P = ctypes.POINTER(ctypes.c_int32)
    rc = lib().sco_pair_ncc(a.ctypes.data, _dtype_code(a), C, H, W, b, n,
                            *[x.ctypes.data_as(P) for x in arrs],
                            out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    if rc != 0:
        raise ValueError("oracle.pair_ncc: invalid arguments")
    return out


def pair_dist3d(vol: np.ndarray, d: int, b: int, zr, ry, rx, zc, cy, cx) -> np.ndarray:
    """Direct distances of explicit 3D pairs (d-plane patches) of a volume [P,H,W] (float64)."""
    a = np.ascontiguousarray(vol)
    P, H, W = a.shape
    arrs = [np.ascontiguousarray(np.asarray(v, dtype=np.int32).ravel()) for v in (zr, ry, rx, zc, cy, cx)]
    n = arrs[0].size
    out = np.empty(n, dtype=np.float64)
    Pt = ctypes.POINTER(ctypes.c_int32)
    rc = lib().sco_pair_dist3d(a.ctypes.data, _dtype_code(a), P, H, W, d, b, n, *[x.ctypes.data_as(Pt) for x in arrs],
                               out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    if rc != 0:
        raise ValueError("oracle.pair_dist3d: invalid arguments")
    return out


def pair_dist(img: np.ndarray, b: int, ry, rx, cy, cx) -> np.ndarray:
    """Direct distances for explicit (ref, candidate) pairs of one image [C,H,W] (float64)."""
    a = np.ascontiguousarray(img)
    if a.ndim == 2:
        a = a[None]
    C, H, W = a.shape
    arrs = [np.ascontiguousarray(np.asarray(v, dtype=np.int32).ravel()) for v in (ry, rx, cy, cx)]
    n = arrs[0].size
    out = np.empty(n, dtype=np.float64)
    P = ctypes.POINTER(ctypes.c_int32)
    rc = lib().sco_pair_dist(a.ctypes.data, _dtype_code(a), C, H, W, b, n,
                             *[x.ctypes.data_as(P) for x in arrs],
                             out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    if rc != 0:
        raise ValueError("oracle.pair_dist: invalid arguments")
    return out


def group(img: np.ndarray, idx: np.ndarray, b: int) -> np.ndarray:
    """Patch groups Y_i = [y_S(1), ..., y_S(K)] (footnote PAPER.md:548).

    img [N, C, H, W], idx [N, refs, K] (pixel-raster index of each match's top-left, -1 = none)
    -> [N, refs, K, C, b, b] in img's dtype: column k of Y_i is the full-depth b x b x C patch at
    idx (channel-major vectorisation, reading R13); -1 gives a zero column. Plain
    loops over the definition (use on small or sampled tables).
    """
    a = np.asarray(img)
    if a.ndim == 3:
        a = a[None]
    N, C, H, W = a.shape
    out = np.zeros(tuple(idx.shape) + (C, b, b), dtype=a.dtype)
    for n in range(idx.shape[0]):
        for r in range(idx.shape[1]):
            for k in range(idx.shape[2]):
                j = int(idx[n, r, k])
                if j < 0:
                    continue
                cy, cx = divmod(j, W)
                out[n, r, k] = a[n, :, cy:cy + b, cx:cx + b]
    return out


def num_threads() -> int:
    return int(lib().sco_num_threads())
