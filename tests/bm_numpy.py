"""An independent numpy brute force for pinning the oracle (tests only).

Written separately from oracle/oracle.c in a different style: it materialises every
patch with ``sliding_window_view``, computes distances to ALL positions of the image,
then applies the window as a boolean mask and selects with ``np.lexsort`` -- so a
wrong window bound, index, sign or tie-break in either implementation shows up as a
disagreement.
"""
import numpy as np
from numpy.lib.stride_tricks import sliding_window_view


def all_patches(img: np.ndarray, b: int) -> np.ndarray:
    """img [C,H,W] -> [My, Mx, C*b*b] (channels summed jointly in the distance)."""
    C, H, W = img.shape
    p = sliding_window_view(img, (b, b), axis=(1, 2))  # [C, My, Mx, b, b]
    return np.ascontiguousarray(p.transpose(1, 2, 0, 3, 4).reshape(H - b + 1, W - b + 1, C * b * b))


def bm_np(img: np.ndarray, b: int, s: int, Wn: int, K: int):
    """Returns idx [refs, K] int64, dist [refs, K] (int64 for integer input else float64)."""
    if img.ndim == 2:
        img = img[None]
    integer = np.issubdtype(img.dtype, np.integer)
    x = img.astype(np.int64 if integer else np.float64)
    C, H, W = x.shape
    P = all_patches(x, b)
    My, Mx = P.shape[:2]
    lo, hi = -(Wn // 2), Wn - 1 - Wn // 2
    ys = np.arange(0, H - b + 1, s)
    xs = np.arange(0, W - b + 1, s)
    cy = np.arange(My)[:, None]
    cx = np.arange(Mx)[None, :]
    pix_idx = (cy * W + cx).ravel()
    idx_out = np.full((len(ys) * len(xs), K), -1, dtype=np.int64)
    big = np.iinfo(np.int32).max if integer else np.inf
    dist_out = np.full((len(ys) * len(xs), K), big, dtype=np.int64 if integer else np.float64)
    r = 0
    for ry in ys:
        for rx in xs:
            D = ((P - P[ry, rx]) ** 2).sum(-1)
            mask = ((cy - ry >= lo) & (cy - ry <= hi) & (cx - rx >= lo) & (cx - rx <= hi)).ravel()
            d = D.ravel()[mask]
            ii = pix_idx[mask]
            order = np.lexsort((ii, d))[:K]
            idx_out[r, :len(order)] = ii[order]
            dist_out[r, :len(order)] = d[order]
            r += 1
    return idx_out, dist_out


def ncc_np(img: np.ndarray, b: int, s: int, Wn: int, K: int):
    """Independent NCC brute force (Eq. 4): sliding-window patches, all-position cross terms and
    norms, window mask, then an EXACT ordering -- Python Fractions of sign(C) C^2 / n_c for integer
    input (n_r is common to a reference), float64 NCC otherwise -- ties by pixel index.
    Returns idx [refs, K] int64 and d_NCC = -NCC [refs, K] float64."""
    from fractions import Fraction
    if img.ndim == 2:
        img = img[None]
    integer = np.issubdtype(img.dtype, np.integer)
    x = img.astype(np.int64 if integer else np.float64)
    C, H, W = x.shape
    P = all_patches(x, b)
    My, Mx = P.shape[:2]
    lo, hi = -(Wn // 2), Wn - 1 - Wn // 2
    ys, xs = np.arange(0, H - b + 1, s), np.arange(0, W - b + 1, s)
    idx_out = np.full((len(ys) * len(xs), K), -1, dtype=np.int64)
    d_out = np.full((len(ys) * len(xs), K), np.inf)
    r = 0
    for ry in ys:
        for rx in xs:
            pr = P[ry, rx]
            nr = (pr * pr).sum()
            cands = []
            for cy in range(max(0, ry + lo), min(My - 1, ry + hi) + 1):
                for cx in range(max(0, rx + lo), min(Mx - 1, rx + hi) + 1):
                    pc = P[cy, cx]
                    c, nc = (pr * pc).sum(), (pc * pc).sum()
                    f = float(c) / np.sqrt(float(nr) * float(nc)) if nr * nc > 0 else 0.0
                    if integer:
                        key = Fraction(int(c) * abs(int(c)), int(nc)) if nr * nc > 0 else Fraction(0)
                    else:
                        key = f
                    cands.append((-key, cy * W + cx, f))
            cands.sort()
            for k, (_, i, f) in enumerate(cands[:K]):
                idx_out[r, k] = i
                d_out[r, k] = -f
            r += 1
    return idx_out, d_out


def bm3d_np(vol: np.ndarray, d: int, b: int, s: int, sz: int, Wn: int, c: int, K: int):
    """Independent 3D brute force: every d-plane patch of the volume [P,H,W] materialised with
    sliding_window_view over (plane, y, x), distances to ALL patch positions, the (plane offset,
    row, column) window applied as a mask, lexsort by (distance, volume index)."""
    integer = np.issubdtype(vol.dtype, np.integer)
    x = vol.astype(np.int64 if integer else np.float64)
    P, H, W = x.shape
    pt = sliding_window_view(x, (d, b, b))  # [P-d+1, H-b+1, W-b+1, d, b, b]
    Z, My, Mx = pt.shape[:3]
    flat = pt.reshape(Z, My, Mx, d * b * b)
    lo, hi, loz, hiz = -(Wn // 2), Wn - 1 - Wn // 2, -(c // 2), c - 1 - c // 2
    zz, yy, xx = np.meshgrid(np.arange(Z), np.arange(My), np.arange(Mx), indexing="ij")
    vidx = ((zz * H + yy) * W + xx).ravel()
    out_i, out_d = [], []
    big = np.iinfo(np.int32).max if integer else np.inf
    for zr in range(0, P - d + 1, sz):
        for ry in range(0, H - b + 1, s):
            for rx in range(0, W - b + 1, s):
                D = ((flat - flat[zr, ry, rx]) ** 2).sum(-1).ravel()
                m = ((zz - zr >= loz) & (zz - zr <= hiz) & (yy - ry >= lo) & (yy - ry <= hi) &
                     (xx - rx >= lo) & (xx - rx <= hi)).ravel()
                o = np.lexsort((vidx[m], D[m]))[:K]
                ii = np.full(K, -1, np.int64)
                dd = np.full(K, big, np.int64 if integer else np.float64)
                ii[:len(o)] = vidx[m][o]
                dd[:len(o)] = D[m][o]
                out_i.append(ii)
                out_d.append(dd)
    nz = (P - d) // sz + 1
    return np.array(out_i).reshape(nz, -1, K), np.array(out_d).reshape(nz, -1, K)
