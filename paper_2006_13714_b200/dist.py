"""Multi-GPU partitioner (one process per GPU, torch.distributed for the plumbing).

Block matching shards with no data-path exchange: every reference is independent given read
access to its search window (Eq. 3 with footnote 2). Two splits:

* frames: rank g of G owns a contiguous, balanced range of the batch's images (config c5);
* row bands: rank g owns a contiguous, balanced range of reference-grid rows of one image;
  the image is replicated (1-13 MB), each rank calls ``sc_bm_run_rows`` for its band.

The only exchange the method has is collecting the result tables. ``gather_tables`` does it
with ``all_gather_into_tensor`` (NCCL over NVLink on GPUs; gloo in the CPU tests) after
padding every shard to the largest shard, then strips the padding.
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple


def balanced_ranges(n: int, world: int) -> List[Tuple[int, int]]:
    """Split range(n) into `world` contiguous ranges whose sizes differ by at most one."""
    if world < 1 or n < 0:
        raise ValueError("balanced_ranges: world >= 1 and n >= 0 required")
    base, extra = divmod(n, world)
    out, start = [], 0
    for r in range(world):
        size = base + (1 if r < extra else 0)
        out.append((start, start + size))
        start += size
    return out


def frame_shard(n_frames: int, rank: int, world: int) -> Tuple[int, int]:
    return balanced_ranges(n_frames, world)[rank]


def band_shard(n_ref_rows: int, rank: int, world: int) -> Tuple[int, int]:
    return balanced_ranges(n_ref_rows, world)[rank]


def gather_tables(tables: Sequence, counts: Sequence[int], group=None):
    """All-gather per-rank tables along dim 0 (uneven shards padded to the largest).

    tables: tensors [count_r, ...] of this rank (same trailing shape / dtype on every rank);
    counts: the leading size of every rank's shard. Returns full tensors [sum(counts), ...].
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    mx = max(counts)
    out = []
    for t in tables:
        if t.shape[0] != counts[dist.get_rank(group)]:
            raise ValueError("gather_tables: local shard size does not match counts")
        pad = t
        if t.shape[0] < mx:
            pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
            pad[: t.shape[0]] = t
        full = torch.empty((world * mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(full, pad.contiguous(), group=group)
        parts = [full[r * mx: r * mx + counts[r]] for r in range(world)]
        out.append(torch.cat(parts, 0))
    return out


def gather_packed(buf, counts: Sequence[int], n_refs: int, K: int, group=None):
    """All-gather PACKED tables of frame shards (sc_bm_set_packed, include/sc_bm.h):
    one uint32 word per result instead of an (idx, dist) pair, so half the bytes cross NVLink.

    buf: this rank's packed buffer (int32 tensor in the header's layout: its counts[rank] * n_refs
    rows of K words, the escape-row count, cap_rows, then the records); counts: frames per rank.
    Returns ONE packed buffer of the whole batch in the same layout: the rows of every rank in
    frame order (the words are position-relative -- the window slot -- so they need no rewrite),
    then count = the sum of the ranks' counts, cap = the records kept, and the records of every
    rank with their row numbers rebased by the rank's first frame. A rank that lost records
    (count > cap) makes the merged count exceed the merged cap, so the decoders (Plan.unpack,
    unpack_host) report SC_ERR_OVERFLOW instead of returning a wrong table.
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if len(counts) != world:
        raise ValueError("gather_packed: one frame count per rank required")
    rw = n_refs * K
    nrow = counts[rank] * rw
    if buf.dtype != torch.int32 or buf.dim() != 1 or buf.numel() < nrow + 2:
        raise ValueError("gather_packed: buf must be a 1-D int32 packed buffer of this rank's frames")
    rows = buf[:nrow].view(-1, K)
    (rows_all,) = gather_tables([rows], [c * n_refs for c in counts], group)
    head = buf[nrow:nrow + 2].to(torch.int64)
    heads = torch.empty(world * 2, dtype=torch.int64, device=buf.device)
    dist.all_gather_into_tensor(heads, head.contiguous(), group=group)
    heads = heads.view(world, 2).cpu()
    rec_words = 2 + 2 * K
    kept = [min(int(heads[r, 0]), int(heads[r, 1])) for r in range(world)]
    recs = buf[nrow + 2:nrow + 2 + kept[rank] * rec_words].view(-1, rec_words)
    parts = []
    if max(kept) > 0:
        (recs_all,) = gather_tables([recs], kept, group)
        first = 0
        off = 0
        for r in range(world):
            part = recs_all[off:off + kept[r]].clone()
            off += kept[r]
            if kept[r]:
                lo = part[:, 0].to(torch.int64) & 0xFFFFFFFF
                hi = part[:, 1].to(torch.int64) & 0xFFFFFFFF
                row = (lo | (hi << 32)) + first * n_refs
                part[:, 0] = (row & 0xFFFFFFFF).to(torch.int32)  # (wraps into int32 bits)
                part[:, 1] = (row >> 32).to(torch.int32)
                parts.append(part.view(-1))
            first += counts[r]
    tail = torch.tensor([int(heads[:, 0].sum()), sum(kept)], dtype=torch.int64)
    tail = ((tail + 2**31) % 2**32 - 2**31).to(torch.int32).to(buf.device)
    return torch.cat([rows_all.reshape(-1), tail] + parts)


def run_frames_sharded(run: Callable, frames, rank: int, world: int, gather: bool = True, group=None):
    """Frame-parallel BM. `run(local_frames) -> (idx, dist)` is the local plan's run (the CUDA
    path on GPUs). `frames` is the full batch (each rank slices its range). Returns the local
    tables, or the full gathered tables when `gather`."""
    n = frames.shape[0]
    a, b = frame_shard(n, rank, world)
    idx, dist_ = run(frames[a:b])
    if not gather or world == 1:
        return idx, dist_
    counts = [e - s for s, e in balanced_ranges(n, world)]
    return tuple(gather_tables([idx, dist_], counts, group))


def run_bands_sharded(run_rows: Callable, img, n_ref_rows: int, n_ref_x: int, rank: int, world: int,
                      gather: bool = True, group=None):
    """Row-band BM of one image. `run_rows(img, iy0, iy1) -> (idx, dist)` shaped [1, refs_band, K].
    Returns local or gathered tables ([1, n_refs, K] in reference raster order)."""
    iy0, iy1 = band_shard(n_ref_rows, rank, world)
    idx, dist_ = run_rows(img, iy0, iy1)
    if not gather or world == 1:
        return idx, dist_
    counts = [(e - s) * n_ref_x for s, e in balanced_ranges(n_ref_rows, world)]
    gi, gd = gather_tables([idx[0], dist_[0]], counts, group)
    return gi[None], gd[None]


def run_frames_pipelined(run: Callable, frames, rank: int, world: int, chunk: int, group=None,
                         local: bool = False):
    """Frame-parallel BM with the table gather pipelined behind the compute.

    Each rank owns frames [rank * per, (rank + 1) * per) (per = n / world, n divisible by
    world * chunk) and processes them in chunks of `chunk` frames; right after chunk c is
    enqueued, its tables are all-gathered ASYNCHRONOUSLY (NCCL runs on its own stream and waits
    for the chunk's kernels only), so the gather of chunk c overlaps the compute of chunk c+1.
    Returns the full tables [n, ...] in global frame order. local=True: `frames` already is this
    rank's shard (n = world * len(frames)).
    """
    import torch
    import torch.distributed as dist
    n = frames.shape[0] * (world if local else 1)
    if n % (world * chunk) != 0:
        raise ValueError("run_frames_pipelined: n_frames must be a multiple of world * chunk")
    per = n // world
    a = 0 if local else rank * per
    pending = []
    for c0 in range(0, per, chunk):
        idx, dist_ = run(frames[a + c0:a + c0 + chunk])
        outs = []
        works = []
        for t in (idx, dist_):
            full = torch.empty((world * chunk,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
            works.append(dist.all_gather_into_tensor(full, t.contiguous(), group=group, async_op=True))
            outs.append(full)
        pending.append((c0, outs, works))
    res = [None, None]
    parts = [[None] * n, [None] * n]
    for c0, outs, works in pending:
        for w in works:
            w.wait()
        for k in range(2):
            for r in range(world):
                for j in range(chunk):
                    parts[k][r * per + c0 + j] = outs[k][r * chunk + j]
    for k in range(2):
        res[k] = torch.stack(parts[k], 0)
    return res[0], res[1]


class PeerTables:
    """The gather fused into the matcher's epilogue ("fused peer-store epilogue").

    The root rank allocates the FULL result tables [n, n_refs, K]; their CUDA IPC handles are
    broadcast over the process group and every other rank maps them into its own address space
    (NVLink peer memory on an NVSwitch node). Each rank then runs the matcher on its frames with
    the output pointers aimed at its rows of the root's tables: the kernels' coalesced (idx, dist)
    row stores -- and the fix-up's -- go straight over NVLink, overlapped with the matching itself;
    there is no separate collective pass. ``finish()`` (device sync + barrier) makes the root's
    tables complete. NCCL's ``all_gather_into_tensor`` (``gather_tables``) stays the reference path.

    Only the product plumbing lives here: handles travel as pickled torch IPC records
    (``torch.multiprocessing.reductions``), the writes are the CUDA kernels' own stores.
    """

    def __init__(self, plan, n_frames: int, rank: int, world: int, root: int = 0, group=None):
        import torch
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor
        self.plan, self.n, self.rank, self.world, self.root, self.group = plan, n_frames, rank, world, root, group
        self.range = frame_shard(n_frames, rank, world)
        if rank == root:
            self.idx, self.dist = plan.alloc_out(n_frames)
            recs = [reduce_tensor(self.idx), reduce_tensor(self.dist)] if world > 1 else None
        else:
            recs = None
        box = [recs]
        if world > 1:
            dist.broadcast_object_list(box, src=root, group=group)
        if rank != root:
            (f_i, a_i), (f_d, a_d) = box[0]
            self.idx, self.dist = f_i(*a_i), f_d(*a_d)  # the root's tables, mapped (cudaIpcOpenMemHandle)
        if self.idx.shape != (n_frames, plan.n_refs, plan.K):
            raise RuntimeError("PeerTables: mapped tables have an unexpected shape")

    def run(self, local_frames, stream=None):
        """Match this rank's frames [a, b) straight into rows [a, b) of the root's tables."""
        a, b = self.range
        if local_frames.shape[0] != b - a:
            raise ValueError("PeerTables.run: expected this rank's frame shard")
        if b > a:
            self.plan.run(local_frames, out=(self.idx[a:b], self.dist[a:b]), stream=stream)

    def finish(self):
        """Every rank's stores have landed: on return the root's tables are complete."""
        import torch
        import torch.distributed as dist
        torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier(group=self.group)
        return (self.idx, self.dist) if self.rank == self.root else None


def temporal_halo(local, rank: int, world: int, T: int, group=None, n_frames=None):
    """The one real data exchange of the method: 3D / temporal search on
    frame shards needs, for the references of a rank's first and last frames, the T neighbouring
    frames held by the adjacent ranks. Every rank sends its first T frames to rank-1 and its last
    T to rank+1 (point-to-point NCCL over NVLink on GPUs; gloo in the CPU tests) and returns the
    extended buffer [left halo | own frames | right halo] plus the halo sizes (0 at the ends).
    T must not exceed the SMALLEST shard (each halo comes from one neighbour); the check uses a
    value every rank shares -- n_frames // world when n_frames is given, else the all-reduced
    minimum shard size -- so all ranks raise together before any point-to-point op starts."""
    import torch
    import torch.distributed as dist
    n = local.shape[0]
    if world > 1 and T > 0:
        if n_frames is not None:
            min_shard = n_frames // world
        else:
            t = torch.tensor([n], dtype=torch.int64, device=local.device)
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
            min_shard = int(t.item())
        if T > min_shard:
            raise ValueError(f"temporal_halo: T = {T} larger than the smallest frame shard ({min_shard})")
    left = T if rank > 0 else 0
    right = T if rank < world - 1 else 0
    if world == 1 or T == 0:
        return local, 0, 0
    shape = tuple(local.shape[1:])
    rl = torch.empty((left,) + shape, dtype=local.dtype, device=local.device)
    rr = torch.empty((right,) + shape, dtype=local.dtype, device=local.device)
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, local[:T].contiguous(), rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, rl, rank - 1, group))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, local[n - T:].contiguous(), rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, rr, rank + 1, group))
    for w in dist.batch_isend_irecv(ops):
        w.wait()
    return torch.cat([rl, local, rr], 0).contiguous(), left, right


def run_temporal_sharded(run_window: Callable, local, rank: int, world: int, n_frames: int, T: int, group=None):
    """Frame-sharded temporal search with the halo exchange. `run_window(ext, f_begin, f_end,
    frame_offset) -> (idx, dist)` is the plan's ``run_temporal`` (references from ext frames
    [f_begin, f_end), candidates from all of ext, idx offset to global frames) on GPUs. Returns this
    rank's tables for its own frames, with global (whole-video) idx."""
    a, b = frame_shard(n_frames, rank, world)
    if local.shape[0] != b - a:
        raise ValueError("run_temporal_sharded: expected this rank's frame shard")
    ext, left, _ = temporal_halo(local, rank, world, T, group, n_frames=n_frames)
    return run_window(ext, left, left + (b - a), a - left)
