"""The fused peer-store gather (dist.PeerTables): every rank's matcher writes its frames' rows
straight into the root rank's tables through CUDA IPC mappings. On a multi-GPU node those are
NVLink peer stores; here (one GPU per gpurun box) the ranks are processes sharing cuda:0, which
exercises the same handle exchange, mapping and out-of-process stores -- the ranks never wait on
each other inside a kernel, only at the host barrier."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dtype, q):
    import torch
    import torch.distributed as dist

    from paper_2006_13714_b200 import dist as sdist
    from paper_2006_13714_b200 import synth
    from paper_2006_13714_b200.bm import Plan
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.Generator(np.random.PCG64(7))
        n, H, W = 5, 70, 150
        frames = synth.random_image(rng, n, 1, H, W, dtype)
        plan = Plan(H, W, 1, 8, 4, 21, 16, dtype)
        pt = sdist.PeerTables(plan, n, rank, world)
        a, b = pt.range
        pt.run(torch.from_numpy(frames[a:b]).cuda())
        res = pt.finish()
        ok = True
        if rank == 0:
            wi, wd = plan.run(torch.from_numpy(frames).cuda())  # the same kernels, one process
            torch.cuda.synchronize()
            ok = torch.equal(res[0], wi) and torch.equal(res[1], wd)
        dist.barrier()  # the root's tables stay alive until every rank is done with the mapping
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dtype", [(2, "u8"), (3, "f32")])
def test_peer_tables_equal_single_process(world, dtype):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dtype, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(world))
    assert all(ok for _, ok in res), res
