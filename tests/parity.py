"""Parity rules, shared by the GPU tests and smoke().

* u8 : idx and dist equal the oracle element-wise, bit-exact, order included.
* f32: for every reference r, with D(r,c) the oracle's double distance, O_r its top-K set
  and d_K its K-th distance:
    1. the GPU's K indices are distinct valid candidates of r's clipped window;
    2. |dist - D(r, idx)| <= REL * D(r, idx); the self pair has dist == 0 exactly;
    3. each row is sorted ascending by (dist, idx);
    4. (GPU set) symmetric-difference O_r  is a subset of {c : |D(r,c) - d_K| <= REL * d_K}.
  REL = 1e-5 (BASELINE.json north_star).
"""
import numpy as np

import oracle

REL = 1e-5


def check_u8(gi, gd, oi, od, where=""):
    gi, gd, oi, od = (np.asarray(x) for x in (gi, gd, oi, od))
    assert gi.shape == oi.shape, (gi.shape, oi.shape)
    bad = np.argwhere((gi != oi) | (gd != od))
    assert bad.size == 0, f"{where}: {len(bad)} mismatches, first at {bad[:3].tolist()}: " \
        f"gpu {gi[tuple(bad[0][:-1])].tolist()} / {gd[tuple(bad[0][:-1])].tolist()} vs " \
        f"oracle {oi[tuple(bad[0][:-1])].tolist()} / {od[tuple(bad[0][:-1])].tolist()}"


def check_f32(img, b, s, Wn, K, gi, gd, oi, od, iy_range=None, rel=REL, where=""):
    """img [C,H,W] float32; gi/gd/oi/od [refs, K] for reference rows iy_range of one image."""
    C, H, W = img.shape
    ny, nx = oracle.grid(H, W, b, s)
    iy0, iy1 = iy_range if iy_range is not None else (0, ny)
    gi, gd, oi, od = (np.asarray(x) for x in (gi, gd, oi, od))
    refs = (iy1 - iy0) * nx
    assert gi.shape == (refs, K) and oi.shape == (refs, K)
    lo, hi = -(Wn // 2), Wn - 1 - Wn // 2
    t = np.arange(refs)
    ry = (iy0 + t // nx) * s
    rx = (t % nx) * s
    cy0, cy1 = np.maximum(0, ry + lo), np.minimum(H - b, ry + hi)
    cx0, cx1 = np.maximum(0, rx + lo), np.minimum(W - b, rx + hi)
    ncand = (cy1 - cy0 + 1) * (cx1 - cx0 + 1)
    valid_slot = np.arange(K)[None, :] < np.minimum(ncand, K)[:, None]
    # padding slots
    assert ((gi == -1) == ~valid_slot).all(), f"{where}: padding mismatch"
    assert np.isinf(gd[~valid_slot]).all()
    gcy, gcx = np.where(valid_slot, gi // W, 0), np.where(valid_slot, gi % W, 0)
    # 1. valid candidates of the window, distinct
    inwin = (gcy >= cy0[:, None]) & (gcy <= cy1[:, None]) & (gcx >= cx0[:, None]) & (gcx <= cx1[:, None])
    assert (inwin | ~valid_slot).all(), f"{where}: candidate outside its window"
    srt = np.sort(np.where(valid_slot, gi, -1 - np.arange(K)[None, :]), axis=1)
    assert (np.diff(srt, axis=1) != 0).all(), f"{where}: duplicate indices"
    # 2. distances within rel of the oracle's direct distance; self pair exact 0
    RY, RX = np.broadcast_to(ry[:, None], gi.shape), np.broadcast_to(rx[:, None], gi.shape)
    D = np.zeros(gi.shape)
    m = valid_slot
    D[m] = oracle.pair_dist(img, b, RY[m], RX[m], gcy[m], gcx[m])
    err = np.abs(gd.astype(np.float64) - D)
    assert (err[m] <= rel * D[m]).all(), f"{where}: max rel err {np.max(err[m] / np.maximum(D[m], 1e-300)):.3g}"
    is_self = m & (gcy == RY) & (gcx == RX)
    assert (gd[is_self] == 0).all(), f"{where}: self distance not exactly 0"
    # 3. sorted by (dist, idx)
    d64 = gd.astype(np.float64)
    ok_order = (d64[:, 1:] > d64[:, :-1]) | ((d64[:, 1:] == d64[:, :-1]) & (gi[:, 1:] > gi[:, :-1]))
    ok_order |= ~valid_slot[:, 1:]
    assert ok_order.all(), f"{where}: row not sorted by (dist, idx)"
    # 4. set difference only within tolerance of the K-th distance (rows whose sorted index
    #    sets already agree -- nearly all of them -- are settled without a Python loop)
    same = (np.sort(gi, axis=1) == np.sort(oi, axis=1)).all(axis=1)
    for r in np.flatnonzero(~same):
        k = int(min(ncand[r], K))
        gs = set(gi[r, :k].tolist())
        os_ = set(oi[r, :k].tolist())
        if gs == os_:
            continue
        dK = od[r, k - 1]
        dmap = dict(zip(oi[r, :k].tolist(), od[r, :k].tolist()))
        dmap.update(zip(gi[r, :k].tolist(), D[r, :k].tolist()))
        for c in gs ^ os_:
            assert abs(dmap[c] - dK) <= rel * dK, f"{where}: ref {r} set differs beyond tolerance"


NCC_ATOL = 1e-5  # d_NCC = -NCC lies in [-1, 1]: absolute tolerance


def pair_ncc(img, b, ry, rx, cy, cx):
    """-NCC of explicit (reference, candidate) pairs of one image [C,H,W], float64 (Eq. 4)."""
    x = np.asarray(img, dtype=np.float64)
    out = np.empty(len(ry))
    for k in range(len(ry)):
        pr = x[:, ry[k]:ry[k] + b, rx[k]:rx[k] + b]
        pc = x[:, cy[k]:cy[k] + b, cx[k]:cx[k] + b]
        den = np.sqrt((pr * pr).sum() * (pc * pc).sum())
        out[k] = -((pr * pc).sum() / den) if den > 0 else 0.0
    return out


def check_ncc(img, b, s, Wn, K, gi, gd, oi, od, exact, iy_range=None, where=""):
    """NCC parity. exact (uint8): idx equal to the oracle's (order included), d_NCC within
    float32 rounding. Float input: the f32 rule of check_f32 with an absolute tolerance."""
    gi, gd, oi, od = (np.asarray(x) for x in (gi, gd, oi, od))
    assert gi.shape == oi.shape, (gi.shape, oi.shape)
    if exact:
        bad = np.argwhere(gi != oi)
        assert bad.size == 0, f"{where}: {len(bad)} idx mismatches, first at {bad[:3].tolist()}: " \
            f"gpu {gi[tuple(bad[0][:-1])].tolist()} vs oracle {oi[tuple(bad[0][:-1])].tolist()}"
        fin = np.isfinite(od)
        assert (np.isfinite(gd) == fin).all(), f"{where}: padding mismatch"
        assert np.max(np.abs(gd[fin] - od[fin]), initial=0) <= 2e-6, f"{where}: d_NCC off"
        return
    C, H, W = img.shape
    ny, nx = oracle.grid(H, W, b, s)
    iy0, iy1 = iy_range if iy_range is not None else (0, ny)
    refs = (iy1 - iy0) * nx
    assert gi.shape == (refs, K)
    lo, hi = -(Wn // 2), Wn - 1 - Wn // 2
    t = np.arange(refs)
    ry, rx = (iy0 + t // nx) * s, (t % nx) * s
    ncand = (np.minimum(H - b, ry + hi) - np.maximum(0, ry + lo) + 1) * \
        (np.minimum(W - b, rx + hi) - np.maximum(0, rx + lo) + 1)
    kk = np.minimum(ncand, K)
    valid = np.arange(K)[None, :] < kk[:, None]
    assert ((gi == -1) == ~valid).all(), f"{where}: padding slots"
    gcy, gcx = np.where(valid, gi // W, 0), np.where(valid, gi % W, 0)
    RY, RX = np.broadcast_to(ry[:, None], gi.shape), np.broadcast_to(rx[:, None], gi.shape)
    inwin = (gcy - RY >= lo) & (gcy - RY <= hi) & (gcx - RX >= lo) & (gcx - RX <= hi)
    assert (inwin | ~valid).all(), f"{where}: candidate outside its window"
    srt = np.sort(np.where(valid, gi, -1 - np.arange(K)[None, :]), axis=1)
    assert (np.diff(srt, axis=1) != 0).all(), f"{where}: duplicate indices"
    D = np.zeros(gi.shape)
    D[valid] = oracle.pair_ncc(img, b, RY[valid], RX[valid], gcy[valid], gcx[valid])
    assert np.max(np.abs(gd[valid] - D[valid]), initial=0) <= NCC_ATOL, f"{where}: d_NCC off"
    d = gd.astype(np.float64)
    ok = (d[:, 1:] > d[:, :-1]) | ((d[:, 1:] == d[:, :-1]) & (gi[:, 1:] > gi[:, :-1])) | ~valid[:, 1:]
    assert ok.all(), f"{where}: row not sorted by (d_NCC, idx)"
    same = (np.sort(gi, axis=1) == np.sort(oi, axis=1)).all(axis=1)
    for r in np.flatnonzero(~same):
        k = int(kk[r])
        gs, os_ = set(gi[r, :k].tolist()), set(oi[r, :k].tolist())
        dK = od[r, k - 1]
        dmap = dict(zip(oi[r, :k].tolist(), od[r, :k].tolist()))
        dmap.update(zip(gi[r, :k].tolist(), D[r, :k].tolist()))
        for c in gs ^ os_:
            assert abs(dmap[c] - dK) <= NCC_ATOL, f"{where}: ref {r} set differs beyond tolerance"


def check_f32_3d(vol, d, b, s, sz, Wn, c, K, gi, gd, oi, od, where, rel=1e-5):
    """The f32 parity rule in 3D: distinct valid candidates of the (plane, y, x) window, distances
    within rel of the direct ones (self exactly 0), rows sorted by (dist, idx), set differences only
    at the K-th distance."""
    P, H, W = vol.shape
    nz, refs, _ = gi.shape
    ny, nx = oracle.grid(H, W, b, s)
    lo, hi, loz, hiz = -(Wn // 2), Wn - 1 - Wn // 2, -(c // 2), c - 1 - c // 2
    assert gi.shape == oi.shape
    for zi in range(nz):
        zr = zi * sz
        t = np.arange(refs)
        ry, rx = (t // nx) * s, (t % nx) * s
        nzc = min(P - d, zr + hiz) - max(0, zr + loz) + 1
        ncand = nzc * (np.minimum(H - b, ry + hi) - np.maximum(0, ry + lo) + 1) * \
            (np.minimum(W - b, rx + hi) - np.maximum(0, rx + lo) + 1)
        valid = np.arange(K)[None, :] < np.minimum(ncand, K)[:, None]
        g, dd = gi[zi], gd[zi]
        assert ((g == -1) == ~valid).all(), f"{where}: padding"
        zc, rem = g // (H * W), g % (H * W)
        cy, cx = rem // W, rem % W
        RY, RX = np.broadcast_to(ry[:, None], g.shape), np.broadcast_to(rx[:, None], g.shape)
        ok = (zc - zr >= loz) & (zc - zr <= hiz) & (zc >= 0) & (zc <= P - d) & (cy - RY >= lo) & \
            (cy - RY <= hi) & (cx - RX >= lo) & (cx - RX <= hi)
        assert (ok | ~valid).all(), f"{where}: candidate outside its window"
        srt = np.sort(np.where(valid, g, -1 - np.arange(K)[None, :]), axis=1)
        assert (np.diff(srt, axis=1) != 0).all(), f"{where}: duplicates"
        D = np.zeros(g.shape)
        D[valid] = oracle.pair_dist3d(vol, d, b, np.full(int(valid.sum()), zr), RY[valid], RX[valid], zc[valid],
                                      cy[valid], cx[valid])
        err = np.abs(dd.astype(np.float64) - D)
        assert (err[valid] <= rel * D[valid]).all(), f"{where}: distance off"
        self_ = valid & (zc == zr) & (cy == RY) & (cx == RX)
        assert (dd[self_] == 0).all()
        d64 = dd.astype(np.float64)
        order = (d64[:, 1:] > d64[:, :-1]) | ((d64[:, 1:] == d64[:, :-1]) & (g[:, 1:] > g[:, :-1])) | ~valid[:, 1:]
        assert order.all(), f"{where}: order"
        same = (np.sort(g, axis=1) == np.sort(oi[zi], axis=1)).all(axis=1)
        for r in np.flatnonzero(~same):
            k = int(min(ncand[r], K))
            dK = od[zi, r, k - 1]
            dmap = dict(zip(oi[zi, r, :k].tolist(), od[zi, r, :k].tolist()))
            dmap.update(zip(g[r, :k].tolist(), D[r, :k].tolist()))
            for cnd in set(g[r, :k].tolist()) ^ set(oi[zi, r, :k].tolist()):
                assert abs(dmap[cnd] - dK) <= rel * dK, f"{where}: set differs"
