"""Packed tables (sc_bm_set_packed, include/sc_bm.h): one uint32 word per result,
w = (dist << rb) | window slot, rows that do not fit in an overflow area.

CPU tests pin the HOST decoder (sc_bm_unpack_host) against the oracle's tables encoded by this
file's own restatement of the documented format; GPU tests check that a packed run decodes
(on the device and on the host) to exactly the plain run's tables and to the oracle."""
import math

import numpy as np
import pytest

import oracle
from paper_2006_13714_b200 import bm

INT32_MAX = 0x7FFFFFFF


def _rb(Wn):
    return max(2, math.ceil(math.log2(Wn * Wn))) if Wn > 1 else 2


def encode(idx, dist, H, W, b, s, Wn, cap, escape=(), rng=None):
    """The header's format written out: rows of words, then count, cap, records (2 + 2K words)."""
    n, nref, K = idx.shape
    ny, nx = oracle.grid(H, W, b, s)
    assert nref == ny * nx
    rb = _rb(Wn)
    lo = -(Wn // 2)
    dsat = (1 << (32 - rb)) - 1
    words = np.empty((n * nref, K), dtype=np.uint64)
    recs = []
    I, D = idx.reshape(-1, K), dist.reshape(-1, K)
    for row in range(n * nref):
        j = row % nref
        ry, rx = (j // nx) * s, (j % nx) * s
        fits = row not in escape and bool(np.all(I[row] >= 0)) and bool(np.all(D[row] < dsat))
        if not fits:
            words[row] = 0xFFFFFFFF
            recs.append([row & 0xFFFFFFFF, row >> 32] + [int(v) & 0xFFFFFFFF for v in I[row]] +
                        [int(v) & 0xFFFFFFFF for v in D[row]])
            continue
        cy, cx = I[row] // W, I[row] % W
        slot = (cy - ry - lo) * Wn + (cx - rx - lo)
        assert np.all((slot >= 0) & (slot < Wn * Wn))
        words[row] = (D[row].astype(np.uint64) << np.uint64(rb)) | slot.astype(np.uint64)
    if rng is not None:
        rng.shuffle(recs)  # records arrive in any order (device atomics)
    tail = [len(recs), cap]
    for r in recs[:cap]:
        tail += r
    tail += [0] * ((2 + 2 * K) * max(0, cap - len(recs)))
    return np.concatenate([words.reshape(-1), np.array(tail, dtype=np.uint64)]).astype(np.uint32), len(recs)


def _img(rng, n, H, W):
    return rng.integers(0, 256, size=(n, 1, H, W), dtype=np.uint8)


@pytest.mark.parametrize("H,W,b,s,Wn,K", [(40, 52, 8, 4, 9, 5), (37, 45, 8, 4, 33, 16), (24, 30, 8, 4, 7, 12)])
def test_unpack_host_matches_oracle(H, W, b, s, Wn, K):
    rng = np.random.default_rng(H * 1000 + Wn)
    img = _img(rng, 2, H, W)
    idx, dist = oracle.bm(img, b, s, Wn, K)
    nrows = idx.shape[0] * idx.shape[1]
    escape = set(rng.choice(nrows, size=min(5, nrows), replace=False).tolist())
    buf, nrec = encode(idx, dist, H, W, b, s, Wn, cap=nrows, escape=escape, rng=rng)
    assert nrec >= len(escape)
    i2, d2 = bm.unpack_host(H, W, b, s, Wn, K, buf, 2)
    np.testing.assert_array_equal(i2, idx)
    np.testing.assert_array_equal(d2, dist)


def test_unpack_host_short_windows_go_through_records():
    H, W, b, s, Wn, K = 12, 14, 8, 4, 3, 8  # a 3 x 3 window clipped at the borders: < 8 candidates
    rng = np.random.default_rng(7)
    img = _img(rng, 1, H, W)
    idx, dist = oracle.bm(img, b, s, Wn, K)
    assert (idx == -1).any()
    buf, nrec = encode(idx, dist, H, W, b, s, Wn, cap=idx.shape[1])
    assert nrec == int((idx == -1).any(axis=2).sum())
    i2, d2 = bm.unpack_host(H, W, b, s, Wn, K, buf, 1)
    np.testing.assert_array_equal(i2, idx)
    np.testing.assert_array_equal(d2[idx >= 0], dist[idx >= 0])
    assert np.all(d2[idx < 0] == INT32_MAX)


def test_unpack_host_overflow_and_bad_slot():
    H, W, b, s, Wn, K = 40, 52, 8, 4, 9, 5
    rng = np.random.default_rng(3)
    img = _img(rng, 1, H, W)
    idx, dist = oracle.bm(img, b, s, Wn, K)
    buf, _ = encode(idx, dist, H, W, b, s, Wn, cap=1, escape={0, 1, 2})  # 3 records, room for 1
    with pytest.raises(bm.ScError) as e:
        bm.unpack_host(H, W, b, s, Wn, K, buf, 1)
    assert e.value.code == 6
    buf, _ = encode(idx, dist, H, W, b, s, Wn, cap=4)
    buf[0] = (buf[0] & ~np.uint32(0xFF)) | np.uint32(Wn * Wn)  # a slot past the window (rb = 7 here)
    with pytest.raises(bm.ScError) as e:
        bm.unpack_host(H, W, b, s, Wn, K, buf, 1)
    assert e.value.code == 1


# ---------------------------------------------------------------------------------------- GPU
def _plan(H, W, Wn, K):
    return bm.Plan(H=H, W=W, C=1, b=8, stride=4, window=Wn, K=K, dtype="u8")


@pytest.mark.gpu
@pytest.mark.parametrize("n,H,W,Wn,K", [(3, 1080, 1920, 33, 16), (2, 100, 130, 33, 16), (2, 77, 201, 21, 24),
                                         (1, 64, 64, 9, 4)])
def test_packed_run_equals_plain_run(n, H, W, Wn, K):
    import torch
    from paper_2006_13714_b200 import synth
    x = torch.from_numpy(np.ascontiguousarray(synth.video_frames(n, H, W, seed=11, walk_seed=12)
                                              .reshape(n, 1, H, W))).cuda()
    plan = _plan(H, W, Wn, K)
    plan.set_kernel(bm.SC_KERNEL_BOX)  # (small images default to other matchers)
    idx, dist = plan.run(x)
    plan.set_packed(4096)
    buf = plan.run_packed(x)
    words, rb = plan.packed_words(n)
    assert buf.numel() == words
    i2, d2 = plan.unpack(buf, n)
    torch.cuda.synchronize()
    assert torch.equal(i2, idx) and torch.equal(d2, dist)
    i3, d3 = bm.unpack_host(H, W, 8, 4, Wn, K, buf.cpu(), n)
    np.testing.assert_array_equal(i3, idx.cpu().numpy())
    np.testing.assert_array_equal(d3, dist.cpu().numpy())
    # the words of a fitting row are (dist << rb) | slot
    row = buf[: K].cpu().numpy().view(np.uint32)
    if row[0] != 0xFFFFFFFF:
        assert int(row[0]) >> rb == int(dist.reshape(-1)[0])
    # host path: the same tables
    hb = plan.run_host_packed(x.cpu())
    i4, d4 = bm.unpack_host(H, W, 8, 4, Wn, K, hb, n)
    np.testing.assert_array_equal(i4, idx.cpu().numpy())
    np.testing.assert_array_equal(d4, dist.cpu().numpy())
    plan.set_packed(0)
    i5, _ = plan.run(x)
    assert torch.equal(i5, idx)


@pytest.mark.gpu
@pytest.mark.parametrize("n,H,W,Wn,K", [(2, 16, 40, 5, 24), (2, 60, 96, 33, 16), (1, 20, 200, 45, 32)])
def test_packed_escape_rows_match_oracle(n, H, W, Wn, K):
    # clipped windows with fewer than K candidates (the corners at Wn = 5, K = 24) escape through
    # the fix-up's overflow records; binary 0/255 noise puts distances near the 2^21 word limit
    import torch
    rng = np.random.default_rng(H + W)
    x_np = (rng.integers(0, 2, size=(n, 1, H, W), dtype=np.uint8) * 255).astype(np.uint8)
    x = torch.from_numpy(x_np).cuda()
    plan = _plan(H, W, Wn, K)
    plan.set_kernel(bm.SC_KERNEL_BOX)
    plan.set_packed(plan.n_refs * n)
    buf = plan.run_packed(x)
    torch.cuda.synchronize()
    idx, dist = oracle.bm(x_np, 8, 4, Wn, K)
    body = n * plan.n_refs * K
    count = int(buf[body].item())
    n_short = int((idx == -1).any(axis=2).sum())
    assert count >= n_short
    if Wn == 5:
        assert n_short > 0 and count == n_short
    i2, d2 = plan.unpack(buf, n)
    np.testing.assert_array_equal(i2.cpu().numpy(), idx)
    np.testing.assert_array_equal(d2.cpu().numpy(), dist)
    hb = plan.run_host_packed(x_np)
    i3, d3 = bm.unpack_host(H, W, 8, 4, Wn, K, hb, n)
    np.testing.assert_array_equal(i3, idx)
    np.testing.assert_array_equal(d3, dist)
    if count > 1:  # too small an overflow area: the decoders refuse (no silent loss)
        plan.set_packed(1)
        buf = plan.run_packed(x)
        with pytest.raises(bm.ScError) as e:
            plan.unpack(buf, n)
        assert e.value.code == 6
        with pytest.raises(bm.ScError) as e:
            bm.unpack_host(H, W, 8, 4, Wn, K, plan.run_host_packed(x_np), n)
        assert e.value.code == 6


@pytest.mark.gpu
def test_packed_rejections():
    import ctypes
    import torch
    H, W = 64, 80
    x = torch.zeros((1, 1, H, W), dtype=torch.uint8, device="cuda")
    pf = bm.Plan(H=H, W=W, C=1, b=8, stride=3, window=15, K=8, dtype="f32")
    with pytest.raises(bm.ScError) as e:
        pf.set_packed(16)
    assert e.value.code == 2
    plan = _plan(H, W, 15, 8)
    plan.set_packed(16)
    with pytest.raises(bm.ScError) as e:  # plain run call with a dist table in packed mode
        plan.run(x)
    assert e.value.code == 1
    buf = torch.empty(plan.packed_words(1)[0], dtype=torch.int32, device="cuda")
    code = plan._lib.sc_bm_run_rows(plan._h, ctypes.c_void_p(x.data_ptr()), 1, 0, 1,  # a partial band
                                    ctypes.c_void_p(buf.data_ptr()), None, None)
    assert code == 2
    plan.set_kernel(bm.SC_KERNEL_SIMT)
    with pytest.raises(bm.ScError) as e:
        plan.run_packed(x)
    assert e.value.code == 2
    plan.set_kernel(bm.SC_KERNEL_BOX)
    plan.set_temporal(1)
    with pytest.raises(bm.ScError) as e:
        plan.run_packed(x)
    assert e.value.code == 2
