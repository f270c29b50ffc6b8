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
