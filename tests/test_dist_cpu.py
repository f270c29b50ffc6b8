"""Multi-process partitioner logic on CPU (gloo, world_size 2 and 3): frame sharding, row-band
sharding and the table gather reassemble exactly the single-process result. The local compute
is the CPU oracle here (no GPU); on GPUs it is the plan's CUDA run."""
import os
import socket

import numpy as np
import pytest

from paper_2006_13714_b200 import dist as sdist


def test_balanced_ranges():
    assert sdist.balanced_ranges(64, 8) == [(8 * i, 8 * i + 8) for i in range(8)]
    r = sdist.balanced_ranges(10, 4)
    assert r == [(0, 3), (3, 6), (6, 8), (8, 10)]
    assert sdist.balanced_ranges(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    for n in range(0, 40):
        for w in range(1, 9):
            rr = sdist.balanced_ranges(n, w)
            assert rr[0][0] == 0 and rr[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rr, rr[1:]))
            sizes = [e - s for s, e in rr]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, q):
    import torch
    import torch.distributed as dist

    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.Generator(np.random.PCG64(3))
        b, s, Wn, K = 5, 2, 9, 7
        if mode == "frames":
            frames = rng.integers(0, 256, size=(5, 1, 20, 23), dtype=np.uint8)

            def run(local):
                i, d = oracle.bm(local, b, s, Wn, K)
                return torch.from_numpy(i), torch.from_numpy(d)

            gi, gd = sdist.run_frames_sharded(run, frames, rank, world)
            wi, wd = oracle.bm(frames, b, s, Wn, K)
        elif mode == "pipelined":
            frames = rng.integers(0, 256, size=(4 * world, 1, 20, 23), dtype=np.uint8)

            def run(local):
                i, d = oracle.bm(local, b, s, Wn, K)
                return torch.from_numpy(i), torch.from_numpy(d)

            gi, gd = sdist.run_frames_pipelined(run, frames, rank, world, chunk=2)
            wi, wd = oracle.bm(frames, b, s, Wn, K)
        else:
            img = rng.random((1, 2, 31, 22)).astype(np.float32)
            ny, nx = oracle.grid(31, 22, b, s)

            def run_rows(x, iy0, iy1):
                i, d = oracle.bm(x, b, s, Wn, K, rows=(iy0, iy1))
                return torch.from_numpy(i), torch.from_numpy(d)

            gi, gd = sdist.run_bands_sharded(run_rows, img, ny, nx, rank, world)
            wi, wd = oracle.bm(img, b, s, Wn, K)
        ok = np.array_equal(gi.numpy(), wi) and np.array_equal(gd.numpy(), wd)
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["frames", "bands", "pipelined"])
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gather_equals_single_process(mode, world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(world))
    assert all(ok for _, ok in res), res


def _temporal_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.Generator(np.random.PCG64(5))
        n, H, W, b, s, Wn, K, T = 7, 20, 23, 4, 2, 7, 6, 2
        video = rng.integers(0, 256, size=(n, 1, H, W), dtype=np.uint8)
        a, e = sdist.frame_shard(n, rank, world)

        def run_window(ext, f0, f1, foff):  # the oracle standing in for plan.run_temporal
            i, d = oracle.bm_temporal(ext.numpy(), b, s, Wn, K, T)
            i = i[f0:f1]
            i = np.where(i >= 0, i + foff * H * W, i)
            return i, d[f0:f1]

        gi, gd = sdist.run_temporal_sharded(run_window, torch.from_numpy(video[a:e]), rank, world, n, T)
        wi, wd = oracle.bm_temporal(video, b, s, Wn, K, T)
        q.put((rank, bool(np.array_equal(gi, wi[a:e]) and np.array_equal(gd, wd[a:e]))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_temporal_halo_equals_single_process(world):
    """Temporal search on frame shards with the T-frame halo exchange (point-to-point) reproduces
    the whole-video search for every rank's frames, global idx included."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_temporal_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(world))
    assert all(ok for _, ok in res), res


def _halo_reject_worker(rank, world, port, use_n, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n_frames, T = 5, 3  # shards 3 and 2: T fits rank 0's shard but not rank 1's
        a, e = sdist.frame_shard(n_frames, rank, world)
        local = torch.zeros((e - a, 1, 4, 4), dtype=torch.uint8)
        try:
            sdist.temporal_halo(local, rank, world, T, n_frames=n_frames if use_n else None)
            q.put((rank, "no error"))
        except ValueError:
            q.put((rank, "raised"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("use_n", [True, False])
def test_temporal_halo_rejects_on_every_rank(use_n):
    """A T larger than the smallest shard raises on EVERY rank before any point-to-point op
    (a rank-local check would let the larger shards block in batch_isend_irecv forever)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_reject_worker, args=(r, 2, port, use_n, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert res == [(0, "raised"), (1, "raised")], res


def _packed_worker(rank, world, port, overflow, q):
    """Each rank encodes its frame shard's oracle tables in the packed format (tests/test_packed.py's
    restatement of include/sc_bm.h), gather_packed merges them, the host decoder must give the whole
    batch's oracle tables (escape rows of several ranks included) -- or SC_ERR_OVERFLOW when a rank
    lost records."""
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2006_13714_b200 import bm
    from tests.test_packed import encode
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.Generator(np.random.PCG64(11))
        H, W, b, s, Wn, K = 37, 45, 8, 4, 9, 5
        n = 5
        frames = rng.integers(0, 256, size=(n, 1, H, W), dtype=np.uint8)
        frames[1, 0, :20] = 0  # constant areas: tie-heavy rows
        a, e = sdist.frame_shard(n, rank, world)
        li, ld = oracle.bm(frames[a:e], b, s, Wn, K)
        nrefs = li.shape[1]
        esc = {(3 * rank + 2 * j) % (li.shape[0] * nrefs) for j in range(3)} if e > a else set()
        cap = 1 if (overflow and rank == world - 1) else 8
        buf, _ = encode(li, ld, H, W, b, s, Wn, cap=cap, escape=esc, rng=rng)
        counts = [f1 - f0 for f0, f1 in sdist.balanced_ranges(n, world)]
        full = sdist.gather_packed(torch.from_numpy(buf.view(np.int32)), counts, nrefs, K)
        wi, wd = oracle.bm(frames, b, s, Wn, K)
        if overflow:
            try:
                bm.unpack_host(H, W, b, s, Wn, K, full, n)
                ok = False
            except bm.ScError as err:
                ok = err.code == 6
        else:
            gi, gd = bm.unpack_host(H, W, b, s, Wn, K, full, n)
            ok = np.array_equal(gi, wi) and np.array_equal(gd, wd) and full.numel() * 2 < 2 * wi.size + 8 * wi.size // K
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("overflow", [False, True])
@pytest.mark.parametrize("world", [2, 3])
def test_packed_gather_equals_single_process(world, overflow):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_packed_worker, args=(r, world, port, overflow, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(world))
    assert all(ok for _, ok in res), res
