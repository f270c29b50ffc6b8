"""T0: pin the CPU oracle to things other than itself (no GPU needed).

Pins:
* hand-worked 3x3 example (tests/golden/worked_3x3.json; Eq. 5, Lemma 2, Theorem 1);
* Lemma 2 identity: norm map + ||X_i||^2 - 2 C_i == direct-difference distances, exactly
  in integers (proof PAPER.md:426-439);
* closed forms: b=1, Wn=1, constant image, periodic tiling, duplicated channels;
* invariants: d >= 0, self-distance 0, symmetry, constant shift, scaling, channel permutation;
* exhaustive 8x8 sweep against an independent numpy brute force (tests/bm_numpy.py);
* library special case: torch conv2d correlation + numpy lexsort.
"""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2006_13714_b200 import synth
from tests.bm_numpy import all_patches as _all_patches, bm_np, ncc_np, bm3d_np

GOLD = os.path.join(os.path.dirname(__file__), "golden", "worked_3x3.json")


def _rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


# ---------------------------------------------------------------- worked example
def test_worked_example_maps():
    g = json.load(open(GOLD))
    img = np.array(g["image"], dtype=np.uint8)
    b = g["b"]
    np.testing.assert_array_equal(oracle.norm_map(img, b), np.array(g["norms"], float))
    np.testing.assert_array_equal(oracle.selfconv(img, b, *g["ref"]), np.array(g["C"], float))
    # objective of Theorem 1 item 2, b_i = C_i - 1/2 h.h, largest value = nearest
    bi = oracle.selfconv(img, b, *g["ref"]) - 0.5 * oracle.norm_map(img, b)
    np.testing.assert_array_equal(bi, np.array(g["b_i"], float))
    dense = oracle.bm_dense(img, b, 1, g["window"])  # ref (0,0) is row 0; offsets -1..1
    d00 = dense[0].reshape(3, 3)[1:, 1:]
    np.testing.assert_array_equal(d00, np.array(g["d"], float))


@pytest.mark.parametrize("K", [1, 2, 3, 4, 5])
def test_worked_example_topk(K):
    g = json.load(open(GOLD))
    img = np.array(g["image"], dtype=np.uint8)
    idx, dist = oracle.bm(img, g["b"], 2, g["window"], K)  # stride 2: only ref (0,0)
    assert idx.shape == (1, 1, K)
    np.testing.assert_array_equal(idx[0, 0], g["topk"][str(K)]["idx"])
    np.testing.assert_array_equal(dist[0, 0], g["topk"][str(K)]["dist"])


def test_value_not_magnitude_selection():
    # b_i = [23, 21, 5, -9]: the K=3 set is {0,1,3}; magnitude selection would pick 4.
    g = json.load(open(GOLD))
    img = np.array(g["image"], dtype=np.uint8)
    idx, _ = oracle.bm(img, 2, 2, 3, 3)
    assert 4 not in idx[0, 0].tolist()


# ---------------------------------------------------------------- Lemma 2 identity
@pytest.mark.parametrize("C,b,s,Wn", [(1, 8, 4, 21), (1, 7, 1, 9), (3, 5, 2, 11), (4, 8, 3, 13)])
def test_lemma2_identity_exact(C, b, s, Wn):
    rng = _rng(10 + C + b)
    H, W = 29, 35
    img = rng.integers(0, 256, size=(C, H, W), dtype=np.uint8)
    dense = oracle.bm_dense(img, b, s, Wn)
    nm = oracle.norm_map(img, b)
    lo = -(Wn // 2)
    ny, nx = oracle.grid(H, W, b, s)
    for t in range(0, ny * nx, max(1, (ny * nx) // 17)):
        ry, rx = (t // nx) * s, (t % nx) * s
        Ci = oracle.selfconv(img, b, ry, rx)
        for a in range(Wn):
            for c in range(Wn):
                cy, cx = ry + lo + a, rx + lo + c
                v = dense[t, a * Wn + c]
                if cy < 0 or cx < 0 or cy > H - b or cx > W - b:
                    assert v == -1.0
                    continue
                assert v == nm[cy, cx] + nm[ry, rx] - 2.0 * Ci[cy, cx]


def test_lemma2_identity_after_shift():
    # shifting u8 by -128 leaves every distance unchanged (d is a difference, Eq. 3)
    rng = _rng(3)
    img = rng.integers(0, 256, size=(1, 20, 24), dtype=np.uint8)
    a = oracle.bm_dense(img, 6, 2, 7)
    b = oracle.bm_dense(img.astype(np.float64) - 128.0, 6, 2, 7)
    np.testing.assert_array_equal(a, b)


# ---------------------------------------------------------------- closed forms
def test_b1_closed_form():
    rng = _rng(5)
    img = rng.integers(0, 256, size=(1, 12, 13), dtype=np.uint8)
    dense = oracle.bm_dense(img, 1, 1, 5)
    x = img[0].astype(np.int64)
    for t in range(12 * 13):
        ry, rx = divmod(t, 13)
        for a in range(5):
            for c in range(5):
                cy, cx = ry - 2 + a, rx - 2 + c
                v = dense[t, a * 5 + c]
                if 0 <= cy < 12 and 0 <= cx < 13:
                    assert v == (x[ry, rx] - x[cy, cx]) ** 2
                else:
                    assert v == -1


def test_window_one_is_self_only():
    rng = _rng(6)
    img = rng.random((2, 15, 17)).astype(np.float32)
    idx, dist = oracle.bm(img, 4, 3, 1, 3)
    ny, nx = oracle.grid(15, 17, 4, 3)
    for t in range(ny * nx):
        ry, rx = (t // nx) * 3, (t % nx) * 3
        assert idx[0, t].tolist() == [ry * 17 + rx, -1, -1]
        assert dist[0, t, 0] == 0.0 and np.isinf(dist[0, t, 1:]).all()


@pytest.mark.parametrize("H,W,b,s,Wn,K", [(20, 23, 4, 3, 7, 10), (16, 16, 8, 4, 21, 16), (9, 30, 3, 2, 6, 40)])
def test_constant_image(H, W, b, s, Wn, K):
    img = np.full((1, H, W), 77, dtype=np.uint8)
    idx, dist = oracle.bm(img, b, s, Wn, K)
    lo, hi = -(Wn // 2), Wn - 1 - Wn // 2
    ny, nx = oracle.grid(H, W, b, s)
    for t in range(ny * nx):
        ry, rx = (t // nx) * s, (t % nx) * s
        cands = sorted(cy * W + cx
                       for cy in range(max(0, ry + lo), min(H - b, ry + hi) + 1)
                       for cx in range(max(0, rx + lo), min(W - b, rx + hi) + 1))
        want = (cands + [-1] * K)[:K]
        assert idx[0, t].tolist() == want
        assert all(d == 0 for d, i in zip(dist[0, t], want) if i >= 0)


def test_periodic_tiling_zero_distances():
    P, b = 8, 6
    rng = _rng(8)
    motif = rng.integers(0, 256, size=(P, P), dtype=np.uint8)
    img = np.tile(motif, (5, 5))[None]  # 40x40
    dense = oracle.bm_dense(img, b, 2, 17)
    ny, nx = oracle.grid(40, 40, b, 2)
    for t in range(ny * nx):
        for a in range(17):
            for c in range(17):
                v = dense[t, a * 17 + c]
                if v < 0:
                    continue
                dy, dx = a - 8, c - 8
                if dy % P == 0 and dx % P == 0:
                    assert v == 0
                else:
                    assert v > 0  # random motif: no other exact repeats at these sizes


def test_duplicated_channels_scale_distance():
    rng = _rng(9)
    one = rng.integers(0, 256, size=(1, 22, 19), dtype=np.uint8)
    three = np.repeat(one, 3, axis=0)
    i1, d1 = oracle.bm(one, 5, 2, 9, 12)
    i3, d3 = oracle.bm(three, 5, 2, 9, 12)
    np.testing.assert_array_equal(i1, i3)
    np.testing.assert_array_equal(d3, 3 * d1)


# ---------------------------------------------------------------- invariants
def test_nonnegative_and_self_zero():
    rng = _rng(11)
    img = rng.random((2, 25, 21))
    dense = oracle.bm_dense(img, 5, 3, 9)
    assert (dense[dense != -1] >= 0).all()
    ny, nx = oracle.grid(25, 21, 5, 3)
    assert (dense[:, 4 * 9 + 4] == 0).all()  # centre slot = self


def test_symmetry_odd_window():
    rng = _rng(12)
    img = rng.integers(0, 256, size=(1, 18, 20), dtype=np.uint8)
    b, Wn = 4, 7
    dense = oracle.bm_dense(img, b, 1, Wn)
    nx = 20 - b + 1
    r = Wn // 2
    for t in range(dense.shape[0]):
        ry, rx = divmod(t, nx)
        for a in range(Wn):
            for c in range(Wn):
                v = dense[t, a * Wn + c]
                if v < 0:
                    continue
                cy, cx = ry + a - r, rx + c - r
                u = (cy * nx + cx)
                back = dense[u, (ry - cy + r) * Wn + (rx - cx + r)]
                assert back == v


def test_shift_and_scale_invariance():
    rng = _rng(13)
    x = rng.integers(0, 100, size=(1, 17, 19)).astype(np.float64)
    base = oracle.bm(x, 5, 2, 9, 10)
    shifted = oracle.bm(x + 37.0, 5, 2, 9, 10)
    scaled = oracle.bm(2.0 * x, 5, 2, 9, 10)
    np.testing.assert_array_equal(base[0], shifted[0])
    np.testing.assert_array_equal(base[1], shifted[1])
    np.testing.assert_array_equal(base[0], scaled[0])
    np.testing.assert_array_equal(4.0 * base[1], scaled[1])


def test_channel_permutation_invariance():
    rng = _rng(14)
    x = rng.random((4, 16, 18)).astype(np.float32)
    a = oracle.bm(x, 4, 2, 7, 9)
    b = oracle.bm(x[[2, 0, 3, 1]], 4, 2, 7, 9)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_allclose(a[1], b[1], rtol=1e-12)


def test_thread_count_independent():
    rng = _rng(15)
    x = rng.integers(0, 4, size=(2, 1, 24, 26), dtype=np.uint8)  # many ties
    a = oracle.bm(x, 4, 1, 9, 20, nthreads=1)
    b = oracle.bm(x, 4, 1, 9, 20, nthreads=4)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])


def test_rows_subset_matches_full():
    rng = _rng(16)
    x = rng.integers(0, 256, size=(3, 1, 30, 28), dtype=np.uint8)
    full = oracle.bm(x, 6, 3, 11, 8)
    ny, nx = oracle.grid(30, 28, 6, 3)
    part = oracle.bm(x, 6, 3, 11, 8, images=(1, 3), rows=(2, 5))
    np.testing.assert_array_equal(part[0], full[0][1:3, 2 * nx:5 * nx])
    np.testing.assert_array_equal(part[1], full[1][1:3, 2 * nx:5 * nx])


# ---------------------------------------------------------------- exhaustive 8x8
def test_exhaustive_8x8_u8():
    rng = _rng(17)
    img = rng.integers(0, 6, size=(1, 8, 8), dtype=np.uint8)  # small range -> ties exercised
    for b in range(1, 9):
        for s in range(1, 5):
            for Wn in range(1, 18):
                Kmax = min(Wn, 9 - b) ** 2
                for K in sorted({1, max(1, Kmax // 2), Kmax, Kmax + 2}):
                    i_o, d_o = oracle.bm(img, b, s, Wn, K)
                    i_n, d_n = bm_np(img[0], b, s, Wn, K)
                    np.testing.assert_array_equal(i_o[0], i_n, err_msg=f"b={b} s={s} Wn={Wn} K={K}")
                    np.testing.assert_array_equal(d_o[0], d_n, err_msg=f"b={b} s={s} Wn={Wn} K={K}")


def test_exhaustive_8x8_float_multichannel():
    rng = _rng(18)
    img = rng.random((3, 8, 8)).astype(np.float32)
    for b in range(1, 9):
        for s in (1, 3):
            for Wn in (1, 2, 5, 8, 17):
                K = min(Wn, 9 - b) ** 2
                i_o, d_o = oracle.bm(img, b, s, Wn, K)
                i_n, d_n = bm_np(img, b, s, Wn, K)
                np.testing.assert_array_equal(i_o[0], i_n)
                np.testing.assert_allclose(d_o[0], d_n, rtol=1e-12, atol=0)


# ---------------------------------------------------------------- library special case
def test_torch_conv2d_special_case():
    torch = pytest.importorskip("torch")
    import torch.nn.functional as F
    rng = _rng(19)
    C, H, W, b, s, Wn, K = 2, 33, 37, 6, 3, 13, 11
    img = rng.random((C, H, W))
    x = torch.from_numpy(img)[None]  # [1,C,H,W] float64
    norms = F.conv2d(x * x, torch.ones(1, C, b, b, dtype=torch.float64))[0, 0].numpy()
    i_o, d_o = oracle.bm(img, b, s, Wn, K)
    ny, nx = oracle.grid(H, W, b, s)
    lo, hi = -(Wn // 2), Wn - 1 - Wn // 2
    for t in range(ny * nx):
        ry, rx = (t // nx) * s, (t % nx) * s
        w = x[:, :, ry:ry + b, rx:rx + b]
        corr = F.conv2d(x, w)[0, 0].numpy()  # torch conv2d is correlation (footnote 1)
        d = norms + norms[ry, rx] - 2.0 * corr
        ys = np.arange(max(0, ry + lo), min(H - b, ry + hi) + 1)
        xs = np.arange(max(0, rx + lo), min(W - b, rx + hi) + 1)
        cy, cx = np.meshgrid(ys, xs, indexing="ij")
        dd = d[cy, cx].ravel()
        ii = (cy * W + cx).ravel()
        # direct identity in float64 has rounding; compare sets/order on well-separated keys
        order = np.lexsort((ii, np.round(dd, 9)))[:K]
        np.testing.assert_array_equal(i_o[0, t], ii[order])
        np.testing.assert_allclose(d_o[0, t], dd[order], rtol=1e-9, atol=1e-9)


def test_pair_dist_matches_dense():
    rng = _rng(20)
    img = rng.random((2, 21, 23))
    b, s, Wn = 5, 3, 7
    dense = oracle.bm_dense(img, b, s, Wn)
    ny, nx = oracle.grid(21, 23, b, s)
    R, Cc, V = [], [], []
    for t in range(ny * nx):
        ry, rx = (t // nx) * s, (t % nx) * s
        for a in range(Wn):
            for c in range(Wn):
                if dense[t, a * Wn + c] >= 0:
                    R.append((ry, rx)); Cc.append((ry + a - 3, rx + c - 3)); V.append(dense[t, a * Wn + c])
    R, Cc = np.array(R), np.array(Cc)
    out = oracle.pair_dist(img, b, R[:, 0], R[:, 1], Cc[:, 0], Cc[:, 1])
    np.testing.assert_array_equal(out, np.array(V))


# ---------------------------------------------------------------- patch grouping Y_i
def test_group_worked_example():
    """Y_i of the hand-worked 3x3 example: K = 3 matches of ref (0,0) are positions (0,0), (0,1),
    (1,0) (tests/golden/worked_3x3.json), so the group's columns are those 2x2 patches."""
    g = json.load(open(GOLD))
    img = np.array(g["image"], dtype=np.uint8)
    idx, _ = oracle.bm(img, 2, 2, 3, 3)
    Y = oracle.group(img[None, None], idx, 2)
    assert Y.shape == (1, 1, 3, 1, 2, 2)
    np.testing.assert_array_equal(Y[0, 0, :, 0], [[[1, 2], [4, 5]], [[2, 3], [5, 6]], [[4, 5], [7, 8]]])
    Y5 = oracle.group(img[None, None], oracle.bm(img, 2, 2, 3, 5)[0], 2)  # 4 candidates: last column 0
    assert (Y5[0, 0, 4] == 0).all() and (Y5[0, 0, 3, 0] == [[5, 6], [8, 9]]).all()


@pytest.mark.parametrize("dtype", ["u8", "f32"])
def test_group_column_norms_and_self_first(dtype):
    """column j's squared norm = the norm map at S(j); on data without exact
    duplicates the first column is the reference patch itself (footnote PAPER.md:548)."""
    rng = _rng(77)
    x = synth.random_image(rng, 1, 2, 26, 31, dtype)
    b, s, Wn, K = 5, 3, 9, 6
    idx, _ = oracle.bm(x, b, s, Wn, K)
    Y = oracle.group(x, idx, b).astype(np.float64)
    nm = oracle.norm_map(x[0], b)
    W = x.shape[3]
    np.testing.assert_allclose((Y ** 2).sum(axis=(3, 4, 5)), nm[idx // W, idx % W], rtol=1e-12)
    ny, nx = oracle.grid(26, 31, b, s)
    for r in range(ny * nx):
        ry, rx = (r // nx) * s, (r % nx) * s
        np.testing.assert_array_equal(Y[0, r, 0], x[0, :, ry:ry + b, rx:rx + b])


# ---------------------------------------------------------------- NCC block matching (Eq. 4)
def test_ncc_worked_example():
    """NCC = C_i / (||X_i|| ||X_j||) from the hand-worked C and norms (worked_3x3.json, Lemma 1
    P:294-297): 46/46, 58/sqrt(46*74), 82/sqrt(46*154), 94/sqrt(46*206) -> order 0, 1, 3, 4."""
    g = json.load(open(GOLD))
    img = np.array(g["image"], dtype=np.uint8)
    Cm, nm = np.array(g["C"], float), np.array(g["norms"], float)
    want = (Cm / np.sqrt(nm[0, 0] * nm)).ravel()
    idx, dist = oracle.ncc(img, 2, 2, 3, 4)
    np.testing.assert_array_equal(idx[0, 0], [0, 1, 3, 4])
    np.testing.assert_allclose(-dist[0, 0], want[[0, 1, 2, 3]], rtol=1e-15)


@pytest.mark.parametrize("dtype", ["u8", "f32"])
@pytest.mark.parametrize("C,b,s,Wn,K", [(1, 3, 1, 5, 4), (1, 4, 2, 7, 9), (2, 2, 1, 4, 6), (1, 8, 4, 9, 16), (3, 3, 2, 17, 30)])
def test_ncc_vs_numpy_bruteforce(dtype, C, b, s, Wn, K):
    rng = _rng(500 + b * 7 + Wn)
    x = synth.random_image(rng, 1, C, 12, 13, dtype)[0]
    if dtype == "u8":
        x[:, :3, :3] = 0  # zero-norm patches: NCC := 0 reading
    idx, dist = oracle.ncc(x, b, s, Wn, K)
    ni, nd = ncc_np(x, b, s, Wn, K)
    np.testing.assert_array_equal(idx[0], ni)
    np.testing.assert_allclose(dist[0], nd, rtol=0, atol=1e-12)


def test_ncc_closed_forms():
    # b = 1 on positive pixels: every NCC is 1 -> pure index order of the clipped window
    x = (_rng(3).integers(1, 256, size=(1, 9, 10))).astype(np.uint8)
    idx, dist = oracle.ncc(x, 1, 2, 5, 7)
    ny, nx = oracle.grid(9, 10, 1, 2)
    for r in range(ny * nx):
        ry, rx = (r // nx) * 2, (r % nx) * 2
        win = [cy * 10 + cx for cy in range(max(0, ry - 2), min(8, ry + 2) + 1)
               for cx in range(max(0, rx - 2), min(9, rx + 2) + 1)]
        np.testing.assert_array_equal(idx[0, r], win[:7])
    assert (dist == -1.0).all()
    # an all-zero reference: NCC := 0 for every candidate -> index order
    z = np.zeros((1, 12, 12), np.uint8)
    z[:, 6:, :] = 200
    idx, dist = oracle.ncc(z, 4, 4, 5, 3)
    assert (dist[0, 0] == 0).all() and idx[0, 0].tolist() == [0, 1, 2]


@pytest.mark.parametrize("dtype", ["u8", "f32"])
def test_ncc_invariants(dtype):
    """Self is the best (NCC = 1, Cauchy-Schwarz) on data without scaled copies; NCC is invariant
    to a positive scale of the image (Eq. 4), exactly in the integer ordering."""
    rng = _rng(41)
    x = synth.random_image(rng, 1, 2, 21, 23, dtype)[0]
    if dtype == "u8":
        x = np.maximum(x, 1).astype(np.uint8)
    idx, dist = oracle.ncc(x, 4, 3, 9, 10)
    ny, nx = oracle.grid(21, 23, 4, 3)
    t = np.arange(ny * nx)
    np.testing.assert_array_equal(idx[0, :, 0], (t // nx) * 3 * 23 + (t % nx) * 3)
    np.testing.assert_allclose(dist[0, :, 0], -1.0, atol=1e-12)
    assert (np.diff(dist[0], axis=1) >= 0).all()
    if dtype == "u8":
        y = (x // 2).astype(np.uint8) * 2  # even values: y/2 is an exact scale of y
        i1, d1 = oracle.ncc(y, 4, 3, 9, 10)
        i2, d2 = oracle.ncc((y // 2).astype(np.uint8), 4, 3, 9, 10)
    else:
        i1, d1 = oracle.ncc(x, 4, 3, 9, 10)
        i2, d2 = oracle.ncc((x * np.float32(4.0)), 4, 3, 9, 10)
    np.testing.assert_array_equal(i1, i2)
    np.testing.assert_allclose(d1, d2, atol=1e-12)


def test_pair_ncc_pins():
    """oracle.pair_ncc (explicit pairs, the full-size parity checks' D): the worked example's hand
    NCC values (Lemma 1), an independent numpy loop, and the d_NCC oracle.ncc reports
    for the pairs it selects."""
    from tests.parity import pair_ncc as pair_ncc_np
    g = json.load(open(GOLD))
    img = np.array(g["image"], dtype=np.uint8)
    Cm, nm = np.array(g["C"], float), np.array(g["norms"], float)
    want = -(Cm / np.sqrt(nm[0, 0] * nm)).ravel()
    got = oracle.pair_ncc(img[None], 2, [0] * 4, [0] * 4, [0, 0, 1, 1], [0, 1, 0, 1])
    np.testing.assert_allclose(got, want, rtol=1e-15)
    rng = _rng(77)
    for dtype in ("u8", "f32"):
        x = synth.random_image(rng, 1, 3, 19, 23, dtype)[0]
        b, s, Wn, K = 5, 2, 9, 12
        idx, dist = oracle.ncc(x, b, s, Wn, K)
        ny, nx = oracle.grid(19, 23, b, s)
        t = np.repeat(np.arange(ny * nx), K)
        ry, rx = (t // nx) * s, (t % nx) * s
        ii = idx[0].ravel()
        d = oracle.pair_ncc(x, b, ry, rx, ii // 23, ii % 23)
        np.testing.assert_allclose(d, dist[0].ravel(), atol=1e-14)
        np.testing.assert_allclose(d[:200], pair_ncc_np(x, b, ry[:200], rx[:200], ii[:200] // 23, ii[:200] % 23),
                                   atol=1e-12)


# ---------------------------------------------------------------- NLM weights (Eq. 2, Prop. 1)
def test_nlm_worked_example():
    """Eq. 2 on the hand-worked distances d = [0, 4, 36, 64] of ref (0,0) (worked_3x3.json) with
    h^2 = 16: s = exp(-d/16) / sum exp(-d/16); the 3x3 window's 5 clipped slots are 0."""
    g = json.load(open(GOLD))
    img = np.array(g["image"], dtype=np.uint8)
    w = oracle.nlm_weights(img, 2, 2, 3, 4.0)[0].reshape(3, 3)
    e = np.exp(-np.array(g["d"], float) / 16.0)
    np.testing.assert_allclose(w[1:, 1:], e / e.sum(), rtol=1e-14)
    assert (w[0, :] == 0).all() and (w[:, 0] == 0).all()


@pytest.mark.parametrize("dtype", ["u8", "f32"])
def test_nlm_limits_and_invariants(dtype):
    """Rows sum to 1; h -> inf gives uniform weights over the clipped window; h -> 0 puts all the
    weight on the nearest candidate (the BM top-1, the reference itself on duplicate-free data);
    the weights are the softmax of -d/h^2 over the window (checked against oracle.bm_dense)."""
    rng = _rng(61)
    x = synth.random_image(rng, 1, 2, 20, 23, dtype)[0]
    b, s, Wn = 4, 3, 7
    w = oracle.nlm_weights(x, b, s, Wn, 40.0 if dtype == "u8" else 0.4)
    np.testing.assert_allclose(w.sum(1), 1.0, rtol=1e-12)
    dense = oracle.bm_dense(x, b, s, Wn)
    valid = dense >= 0
    assert ((w > 0) == valid).all()
    wu = oracle.nlm_weights(x, b, s, Wn, 1e12)
    np.testing.assert_allclose(wu, valid / valid.sum(1, keepdims=True), rtol=1e-9)
    w0 = oracle.nlm_weights(x, b, s, Wn, 1e-3)
    top1, _ = oracle.bm(x, b, s, Wn, 1)
    ny, nx = oracle.grid(20, 23, b, s)
    lo = -(Wn // 2)
    for r in range(ny * nx):
        ry, rx = (r // nx) * s, (r % nx) * s
        cy, cx = divmod(int(top1[0, r, 0]), 23)
        assert w0[r, (cy - ry - lo) * Wn + (cx - rx - lo)] == pytest.approx(1.0)
        assert (cy, cx) == (ry, rx)
    h = 40.0 if dtype == "u8" else 0.4
    z = np.where(valid, -dense / h ** 2, -np.inf)
    sm = np.exp(z - z.max(1, keepdims=True))
    np.testing.assert_allclose(w, sm / sm.sum(1, keepdims=True), rtol=1e-12, atol=1e-300)


def test_nlm_average_pins():
    """The NL-means patch estimate: h -> inf gives the plain mean of the clipped
    window's patches (a numpy brute force with its own window clipping); h -> 0 returns the
    reference patch itself (duplicate-free data: the unique zero distance); a constant image is a
    fixed point; scaling the image scales the estimate (the weights of x*c at h*c equal x's)."""
    rng = _rng(63)
    x = synth.random_image(rng, 1, 2, 18, 21, "f32")[0]
    b, s, Wn = 4, 3, 7
    ny, nx = oracle.grid(18, 21, b, s)
    lo, hi = -(Wn // 2), Wn - 1 - Wn // 2
    mu = oracle.nlm_average(x, b, s, Wn, 1e12)
    for r in range(ny * nx):
        ry, rx = (r // nx) * s, (r % nx) * s
        ps = [x[:, cy:cy + b, cx:cx + b].astype(np.float64)
              for cy in range(max(0, ry + lo), min(18 - b, ry + hi) + 1)
              for cx in range(max(0, rx + lo), min(21 - b, rx + hi) + 1)]
        np.testing.assert_allclose(mu[r], np.mean(ps, 0), rtol=1e-9)
    z = oracle.nlm_average(x, b, s, Wn, 1e-3)
    for r in range(ny * nx):
        ry, rx = (r // nx) * s, (r % nx) * s
        np.testing.assert_allclose(z[r], x[:, ry:ry + b, rx:rx + b], rtol=1e-12)
    c = np.full((1, 12, 13), 37, dtype=np.uint8)
    np.testing.assert_allclose(oracle.nlm_average(c, 4, 2, 5, 10.0), 37.0, rtol=1e-12)
    y = (x * np.float32(2.0)).astype(np.float32)
    np.testing.assert_allclose(oracle.nlm_average(y, b, s, Wn, 0.8, refs=[0, 5, 11]),
                               2.0 * oracle.nlm_average(x, b, s, Wn, 0.4, refs=[0, 5, 11]), rtol=1e-9)


# ---------------------------------------------------------------- 3D / temporal search
def test_temporal_reduces_to_spatial_and_exhaustive():
    """T = 0 is per-frame BM (idx offset by frame * H * W); T = 1 on a tiny video equals an
    independent numpy brute force over the stacked candidate sets."""
    rng = _rng(71)
    x = rng.integers(0, 256, size=(3, 1, 12, 13), dtype=np.uint8)
    i0, d0 = oracle.bm_temporal(x, 4, 2, 5, 6, 0)
    i1, d1 = oracle.bm(x, 4, 2, 5, 6)
    np.testing.assert_array_equal(i0, i1 + (np.arange(3) * 12 * 13)[:, None, None])
    np.testing.assert_array_equal(d0, d1)
    it, dt = oracle.bm_temporal(x, 4, 2, 5, 7, 1)
    P = [_all_patches(x[f].astype(np.int64), 4) for f in range(3)]
    ny, nx = oracle.grid(12, 13, 4, 2)
    for f in range(3):
        for r in range(ny * nx):
            ry, rx = (r // nx) * 2, (r % nx) * 2
            cand = []
            for fr in range(max(0, f - 1), min(2, f + 1) + 1):
                for cy in range(max(0, ry - 2), min(8, ry + 2) + 1):
                    for cx in range(max(0, rx - 2), min(9, rx + 2) + 1):
                        d = int(((P[f][ry, rx] - P[fr][cy, cx]) ** 2).sum())
                        cand.append((d, fr * 156 + cy * 13 + cx))
            cand.sort()
            np.testing.assert_array_equal(it[f, r], [c[1] for c in cand[:7]])
            np.testing.assert_array_equal(dt[f, r], [c[0] for c in cand[:7]])


def test_temporal_translated_video():
    """A sequence of pure translations: the best match of a reference in frame f within frame f+1
    is the translated position, at distance 0 (the motion-compensated neighbour)."""
    base = _rng(72).integers(0, 256, size=(40, 44), dtype=np.uint8)
    x = np.stack([base[2 * f:2 * f + 30, f:f + 32] for f in range(3)])[:, None].copy()
    idx, dist = oracle.bm_temporal(x, 8, 4, 9, 3, 1)
    ny, nx = oracle.grid(30, 32, 8, 4)
    for r in range(ny * nx):
        ry, rx = (r // nx) * 4, (r % nx) * 4
        if ry + 2 > 30 - 8 or rx + 1 > 32 - 8:  # the motion-compensated position leaves frame 0
            continue
        # frame 1's content at (y, x) is frame 0's at (y + 2, x + 1): frame 1 ref -> frame 0 (ry+2, rx+1)
        want = 0 * 30 * 32 + (ry + 2) * 32 + rx + 1
        assert want in idx[1, r].tolist() and dist[1, r, 0] == 0


# ---------------------------------------------------------------- 3D search
@pytest.mark.parametrize("dtype", ["u8", "f32"])
@pytest.mark.parametrize("P,d,b,s,sz,Wn,c,K", [(4, 1, 3, 2, 1, 5, 3, 6), (6, 3, 3, 1, 1, 5, 2, 9),
                                                (5, 2, 4, 3, 2, 7, 4, 11), (3, 3, 2, 1, 1, 3, 1, 4),
                                                (7, 1, 2, 2, 3, 4, 9, 20)])
def test_bm3d_vs_numpy_bruteforce(dtype, P, d, b, s, sz, Wn, c, K):
    rng = _rng(800 + P * 11 + d + Wn)
    x = synth.random_image(rng, 1, P, 11, 12, dtype)[0]
    if dtype == "u8":
        x[1:, :4, :4] = x[0, :4, :4]  # repeated content across planes: exact ties
    gi, gd = oracle.bm3d(x, d, b, s, sz, Wn, c, K)
    ni, nd = bm3d_np(x, d, b, s, sz, Wn, c, K)
    np.testing.assert_array_equal(gi, ni)
    if dtype == "u8":
        np.testing.assert_array_equal(gd, nd)
    else:
        np.testing.assert_allclose(gd, nd, rtol=1e-12, atol=1e-12)


def test_bm3d_special_cases():
    """d = P, c = 1: multi-channel 2D BM (Eq. 12's channel sum); d = 1, c = 2T + 1: the temporal
    search over the frames; c = 1, d = 1: per-plane 2D BM with the plane offset in idx."""
    rng = _rng(901)
    x = synth.random_image(rng, 1, 4, 19, 21, "f32")[0]
    i3, d3 = oracle.bm3d(x, 4, 5, 2, 1, 7, 1, 9)
    i2, d2 = oracle.bm(x, 5, 2, 7, 9)
    np.testing.assert_array_equal(i3, i2)
    np.testing.assert_array_equal(d3, d2)
    it, dt = oracle.bm_temporal(x[:, None], 5, 2, 7, 9, 1)
    i3, d3 = oracle.bm3d(x, 1, 5, 2, 1, 7, 3, 9)
    np.testing.assert_array_equal(i3, it)
    np.testing.assert_array_equal(d3, dt)
    i3, d3 = oracle.bm3d(x, 1, 5, 2, 1, 7, 1, 9)
    for z in range(4):
        i2, d2 = oracle.bm(x[z], 5, 2, 7, 9)
        np.testing.assert_array_equal(i3[z], i2[0] + z * 19 * 21)
        np.testing.assert_array_equal(d3[z], d2[0])


def test_bm3d_translated_volume():
    """Planes that are one canvas shifted by (2, -3) per plane: every reference away from the
    borders has an exact d = 0 match in the next plane at offset (+2, -3) (and the previous at
    (-2, +3)); with c = 3 and a window covering the motion the K-th list holds both."""
    rng = _rng(902)
    canvas = synth.random_image(rng, 1, 1, 60, 60, "f32")[0, 0]
    P, H, W, b = 4, 24, 24, 4
    vol = np.stack([canvas[20 + 2 * z:20 + 2 * z + H, 20 - 3 * z:20 - 3 * z + W] for z in range(P)]).astype(np.float32)
    idx, dist = oracle.bm3d(vol, 1, b, 4, 1, 9, 3, 3)
    ny, nx = oracle.grid(H, W, b, 4)
    for z in range(1, P - 1):
        for r in range(ny * nx):
            ry, rx = (r // nx) * 4, (r % nx) * 4
            if not (2 <= ry <= H - b - 2 and 3 <= rx <= W - b - 3):
                continue
            want = {((z + 1) * H + ry - 2) * W + rx + 3, ((z - 1) * H + ry + 2) * W + rx - 3}
            assert want <= set(idx[z, r].tolist())
            assert (dist[z, r] == 0).all()  # self + the two motion-compensated matches


def test_pair_dist3d_matches_bm3d():
    """oracle.pair_dist3d (the 3D check's D) against the distances oracle.bm3d reports for its own
    selected pairs, and a numpy patch difference."""
    rng = _rng(903)
    x = synth.random_image(rng, 1, 5, 17, 19, "f32")[0]
    d, b, s, sz, Wn, c, K = 2, 4, 2, 1, 7, 3, 10
    idx, dist = oracle.bm3d(x, d, b, s, sz, Wn, c, K)
    ny, nx = oracle.grid(17, 19, b, s)
    nz = idx.shape[0]
    zr = np.repeat(np.arange(nz) * sz, ny * nx * K)
    t = np.tile(np.repeat(np.arange(ny * nx), K), nz)
    ii = idx.ravel()
    zc, rem = ii // (17 * 19), ii % (17 * 19)
    D = oracle.pair_dist3d(x, d, b, zr, (t // nx) * s, (t % nx) * s, zc, rem // 19, rem % 19)
    np.testing.assert_allclose(D, dist.ravel(), rtol=1e-12)
    k = 37
    pr = x[zr[k]:zr[k] + d, (t[k] // nx) * s:(t[k] // nx) * s + b, (t[k] % nx) * s:(t[k] % nx) * s + b].astype(np.float64)
    pc = x[zc[k]:zc[k] + d, rem[k] // 19:rem[k] // 19 + b, rem[k] % 19:rem[k] % 19 + b].astype(np.float64)
    assert abs(D[k] - ((pr - pc) ** 2).sum()) < 1e-12
