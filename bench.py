"""Benchmark: Self-Convolution block matching on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

A "step" is one pass of the whole hot path (norm map -> cross term -> distance assembly ->
top-K -> output tables) over the config's batch, inputs resident in HBM.
Default workload: config c5 (64 uint8 1080x1920 frames, b=8, s=4, Wn=33, K=16), the
config the metric's 1/2/4/8-GPU scaling is quoted on; its frames are sharded across ranks
(strong scaling: the 64-frame batch is fixed). Under torchrun each rank runs its shard;
the timed region is bracketed by barrier + synchronize, per-step CUDA events on the run
stream, and the max over ranks is reported. ``--impl reference`` times the CPU oracle
(the brute-force definition, oracle/) on the host cores on a bounded sample instead.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidate patch distances/sec"
UNIT = "candidate distances/s"


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0, "_fallback": True}


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: an NVML thread (every ~2 ms,
    so even a 100 ms region gets dozens of samples); `nvidia-smi -lms` if NVML is unavailable."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int, period_s: float = 0.002):
        self.gpu, self.period = gpu_index, period_s
        self.proc = None
        self.nvml = None
        self.rows = []  # (sm_mhz, max_mhz, set of active reason names)
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            self.nvml = (pynvml, h, bits)
            self._sample_nvml()  # one sample as the region starts
            self._t = threading.Thread(target=self._loop_nvml, daemon=True)
            self._t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read_smi, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        return self

    def _sample_nvml(self):
        pynvml, h, bits = self.nvml
        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        self.rows.append((float(sm), float(mx), {n for n, b in bits.items() if r & b}))

    def _loop_nvml(self):
        while not self._stop.wait(self.period):
            try:
                self._sample_nvml()
            except Exception:
                return

    def _read_smi(self):
        for line in self.proc.stdout:
            r = [v.strip() for v in line.split(",")]
            if len(r) >= 9 and r[1].replace(".", "").isdigit():
                self.rows.append((float(r[1]), float(r[2]),
                                  {n for i, n in enumerate(self.NAMES) if r[5 + i].lower() == "active"}))

    def __exit__(self, *exc):
        self._stop.set()
        if self.nvml is not None:
            self._t.join(timeout=1)
            try:
                self._sample_nvml()  # one sample as the region ends
            except Exception:
                pass
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        reasons = set().union(*[r[2] for r in self.rows])
        return {"sm_mhz": float(np.median([r[0] for r in self.rows])), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted(reasons), "samples": len(self.rows),
                "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def _free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _launch_ranks(args) -> None:
    """One process per GPU. Under torchrun (WORLD_SIZE set) the world must equal --gpus.
    Without it, ``--gpus N > 1`` re-executes this script under torch.distributed.run with N
    local ranks (127.0.0.1 rendezvous), refusing with a non-zero exit when fewer than N GPUs
    are visible -- never a silent single-rank run reported as N GPUs."""
    env_ws = os.environ.get("WORLD_SIZE")
    if env_ws is not None:
        if args.impl == "ours" and int(env_ws) != args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_ws}\n")
            sys.exit(2)
        return
    if args.gpus <= 1 or args.impl == "reference":  # the reference arm runs on rank 0 only
        return
    if not args.selftest_cpu:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} requested but only {have} GPU(s) visible\n")
            sys.exit(3)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def selftest_cpu(args, cfg):
    """CPU plumbing check of the multi-rank bench (tests/test_bench_cpu.py): the launcher, the
    frame shards, barrier-bracketed timing with the max over ranks and the line's fields, on
    gloo with a stand-in step (a numpy pass over a buffer sized by the shard). NOT a measurement."""
    import torch
    import torch.distributed as tdist

    from paper_2006_13714_b200.dist import balanced_ranges
    ws, rank, _ = _dist_env()
    if ws > 1:
        import datetime
        tdist.init_process_group("gloo", timeout=datetime.timedelta(seconds=120))
    shards = balanced_ranges(cfg.N, ws)
    f0, f1 = shards[rank]
    buf = np.random.default_rng(rank).random((max(1, f1 - f0), 1 << 16))

    def step():
        return float(np.sort(buf, axis=1)[:, 0].sum())

    for _ in range(args.warmup):
        step()
    if ws > 1:
        tdist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    local_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    t = torch.tensor([local_ms, float(f1 - f0)], dtype=torch.float64)
    if ws > 1:
        tdist.barrier()
        tm = t.clone()
        tdist.all_reduce(tm, op=tdist.ReduceOp.MAX)
        tn = t.clone()
        tdist.all_reduce(tn, op=tdist.ReduceOp.SUM)
        ms, frames = tm[0].item(), tn[1].item()
    else:
        ms, frames = local_ms, float(f1 - f0)
    if rank == 0:
        line = {"selftest": "cpu plumbing only (launcher, shards, max over ranks); not a measurement",
                "metric": METRIC, "value": frames / (ms / 1e3), "unit": "frames/s (stand-in step)",
                "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong" if cfg.N > 1 else "weak",
                "config": dict(_config_obj(cfg, args), shards=shards), "frames_timed": frames}
        print(json.dumps(line), flush=True)
    if ws > 1:
        tdist.barrier()
        tdist.destroy_process_group()


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _cpu_sample(cfg, x, target_s=8.0, images=(0, 1), metric="l2", want_tables=False):
    """Time the oracle on a bounded sample of the workload: reference rows of image 0."""
    import oracle
    run = oracle.ncc if metric == "ncc" else oracle.bm
    from paper_2006_13714_b200 import synth  # noqa: F401
    ny = (cfg.H - cfg.b) // cfg.s + 1
    nx = (cfg.W - cfg.b) // cfg.s + 1
    lo, hi = -(cfg.Wn // 2), cfg.Wn - 1 - cfg.Wn // 2

    def pairs(r0, r1):
        ys = [min(cfg.H - cfg.b, iy * cfg.s + hi) - max(0, iy * cfg.s + lo) + 1 for iy in range(r0, r1)]
        xs = [min(cfg.W - cfg.b, ix * cfg.s + hi) - max(0, ix * cfg.s + lo) + 1 for ix in range(nx)]
        return sum(ys) * sum(xs)

    # calibrate on one row, then size the sample (starting at the top rows) to ~target_s seconds
    mid = 0
    t0 = time.perf_counter()
    run(x, cfg.b, cfg.s, cfg.Wn, cfg.K, images=images, rows=(ny // 2, ny // 2 + 1))
    dt = max(time.perf_counter() - t0, 1e-3)
    rows = int(max(1, min(ny, target_s / dt)))
    n_img = 1
    if rows == ny and x.shape[0] > 1:  # more than one frame's worth of CPU time: whole frames
        n_img = int(max(1, min(x.shape[0], -(-target_s // (dt * ny)))))  # ceil
    t0 = time.perf_counter()
    imgs = (0, n_img) if n_img > 1 else images
    out = run(x, cfg.b, cfg.s, cfg.Wn, cfg.K, images=imgs, rows=(mid, mid + rows))
    dt = time.perf_counter() - t0
    p = pairs(mid, mid + rows) * n_img
    what = (f"{cfg.name} images 0:{n_img} (all {ny} reference rows)" if n_img > 1 else
            f"{cfg.name} image 0, reference rows {mid}:{mid + rows} of {ny}")
    res = {"value": p / dt, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
           "sample": f"{what} ({rows * nx * n_img} refs, {p} candidate pairs), {dt:.2f} s"}
    if want_tables:
        return res, p, dt, (imgs, (mid, mid + rows), out)
    return res, p, dt


def _parity_of_sample(cfg, x_host, idx, dst, sample, metric):
    """The bench checks what it times: the GPU tables of the frames / reference rows the
    cpu_baseline leg just computed with the oracle, compared element by element (u8 bit-exact,
    f32 by the 1e-5 rule of tests/parity.py)."""
    from tests.parity import check_f32, check_ncc, check_u8
    (i0, i1), (r0, r1), (oi, od) = sample
    nx = (cfg.W - cfg.b) // cfg.s + 1
    sl = slice(r0 * nx, r1 * nx)
    gi = idx[i0:i1, sl].cpu().numpy()
    gd = dst[i0:i1, sl].cpu().numpy()
    what = f"images {i0}:{i1}, reference rows {r0}:{r1} ({(i1 - i0) * (r1 - r0) * nx} references)"
    try:
        if metric == "ncc":
            for n in range(i1 - i0):
                check_ncc(x_host[i0 + n], cfg.b, cfg.s, cfg.Wn, cfg.K, gi[n], gd[n], oi[n], od[n],
                          exact=cfg.dtype == "u8", iy_range=(r0, r1), where="bench")
            rule = "idx bit-exact, d_NCC within 2e-6" if cfg.dtype == "u8" else "NCC tolerance rule"
        elif cfg.dtype == "u8":
            check_u8(gi, gd, oi, od, "bench")
            rule = "idx and dist bit-exact"
        else:
            for n in range(i1 - i0):
                check_f32(x_host[i0 + n], cfg.b, cfg.s, cfg.Wn, cfg.K, gi[n], gd[n], oi[n], od[n],
                          iy_range=(r0, r1), where="bench")
            rule = "f32 rule: rel 1e-5, set differences only at the K-th distance"
        return {"checked": what, "rule": rule, "result": "pass"}
    except AssertionError as e:
        return {"checked": what, "result": "FAIL", "detail": str(e)[:300]}


def run_reference(args, cfg):
    ws, rank, _ = _dist_env()
    if rank != 0:
        return
    import oracle
    from paper_2006_13714_b200 import synth
    x = synth.make_input(cfg, n_frames=1)
    oracle.build()
    for _ in range(args.warmup):
        _cpu_sample(cfg, x, target_s=1.0)
    vals, tot_p, tot_t = [], 0, 0.0
    last = None
    for _ in range(args.steps):
        last, p, dt = _cpu_sample(cfg, x, target_s=args.ref_step_s)
        vals.append(last["value"])
        tot_p += p
        tot_t += dt
    value = tot_p / tot_t
    cpu = dict(last)
    cpu["value"] = value
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": _dtype_name(cfg),
            "data": "synthetic", "config": _config_obj(cfg, args), "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _pairs_3d(cfg, info, n_planes):
    """Candidate pairs of one 3D step: per reference plane, the valid plane offsets x the 2D pairs."""
    nz = (n_planes - cfg.d) // cfg.sz + 1
    zlo, zhi = -(cfg.zwin // 2), cfg.zwin - 1 - cfg.zwin // 2
    zc = [min(n_planes - cfg.d, z * cfg.sz + zhi) - max(0, z * cfg.sz + zlo) + 1 for z in range(nz)]
    return nz, sum(zc) * info["total_candidates"]


def _oracle_3d_sample(cfg, vol, n_sub):
    """The oracle on the first n_sub planes (reference planes whose plane window lies inside them
    see exactly the full volume's candidates)."""
    import oracle
    zhi = cfg.zwin - 1 - cfg.zwin // 2
    t0 = time.perf_counter()
    oi, od = oracle.bm3d(vol[:n_sub], cfg.d, cfg.b, cfg.s, cfg.sz, cfg.Wn, cfg.zwin, cfg.K)
    dt = time.perf_counter() - t0
    n_exact = max(0, (n_sub - cfg.d - zhi) // cfg.sz + 1)  # reference planes unaffected by the crop
    return oi, od, dt, n_exact


def bench_3d(args, cfg):
    """3D search: one volume per step through sc_bm_run3d on the float box-sum
    kernel with a plane loop; metric candidate distances/s; parity of the sampled reference planes."""
    import torch
    from paper_2006_13714_b200.bm import Plan3D
    ws, rank, local = _dist_env()
    torch.cuda.set_device(local)
    vol_h = synth_input = None
    from paper_2006_13714_b200 import synth
    vol_h = np.ascontiguousarray(synth.make_input(cfg)[0])
    vol = torch.from_numpy(vol_h).cuda()
    plan = Plan3D(cfg.H, cfg.W, cfg.d, cfg.b, cfg.s, cfg.Wn, cfg.sz, cfg.zwin, cfg.K)
    info = plan.info()
    P = vol_h.shape[0]
    nz, pairs = _pairs_3d(cfg, info, P)
    idx, dst = plan.alloc_out(nz)
    for _ in range(args.warmup):
        plan.run(vol, out=(idx, dst))
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = plan.info()["launches"]
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            starts[k].record(stream)
            plan.run(vol, out=(idx, dst))
            ends[k].record(stream)
        torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in zip(starts, ends)]
    ms = float(np.mean(step_ms))
    peaks = _peaks()
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    macs = pairs * cfg.b * cfg.b * cfg.d
    ffma = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12
    achieved = 2.0 * macs / (ms / 1e3) / 1e12
    line = {"metric": METRIC, "value": pairs / (ms / 1e3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "ms_per_step_min": float(np.min(step_ms)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg.name, "planes": P, "H": cfg.H, "W": cfg.W, "patch": [cfg.b, cfg.b, cfg.d],
                       "stride": cfg.s, "window": [cfg.Wn, cfg.Wn, cfg.zwin], "plane_stride": cfg.sz, "K": cfg.K,
                       "l2": "flushed between timed steps (256 MiB write)"},
            "candidate_pairs_per_step": pairs, "ref_patches_per_s": nz * info["n_refs"] / (ms / 1e3),
            "roofline": {"bound": "alu", "kernel": "bm_boxf_kernel (Z3)", "achieved": achieved, "peak": ffma,
                         "unit": "TFLOP/s", "frac": achieved / ffma, "traffic": None,
                         "algorithmic_flops_per_step": 2.0 * macs, "macs_per_pair": cfg.b * cfg.b * cfg.d,
                         "peak_source": "FFMA: 148 SM x 128 lanes x 2 x sm_max_mhz"},
            "gpu_launches": int(plan.info()["launches"] - launches0), "clocks": clk.summary()}
    if not args.no_cpu:
        import oracle
        n_sub = min(P, cfg.d + (cfg.zwin - 1 - cfg.zwin // 2) + 2 * cfg.sz)
        oi, od, dt, n_exact = _oracle_3d_sample(cfg, vol_h, n_sub)
        sub = Plan3D(cfg.H, cfg.W, cfg.d, cfg.b, cfg.s, cfg.Wn, cfg.sz, cfg.zwin, cfg.K)
        _, p_sub = _pairs_3d(cfg, info, n_sub)
        line["cpu_baseline"] = {"value": p_sub / dt, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                                "sample": f"{cfg.name} planes 0:{n_sub} ({p_sub} candidate pairs), {dt:.2f} s"}
        del sub
        from tests.parity import check_f32_3d
        gi, gd = idx[:n_exact].cpu().numpy(), dst[:n_exact].cpu().numpy()
        what = f"reference planes 0:{n_exact} ({n_exact * info['n_refs']} references)"
        try:
            check_f32_3d(vol_h, cfg.d, cfg.b, cfg.s, cfg.sz, cfg.Wn, cfg.zwin, cfg.K, gi, gd, oi[:n_exact],
                         od[:n_exact], "bench")
            line["parity"] = {"checked": what, "rule": "f32 rule in 3D (tests/parity.py check_f32_3d)", "result": "pass"}
        except AssertionError as e:
            line["parity"] = {"checked": what, "result": "FAIL", "detail": str(e)[:300]}
    print(json.dumps(line), flush=True)


def run_reference_3d(args, cfg):
    ws, rank, _ = _dist_env()
    if rank != 0:
        return
    import oracle
    from paper_2006_13714_b200 import synth
    vol = np.ascontiguousarray(synth.make_input(cfg)[0])
    oracle.build()
    n_sub = min(vol.shape[0], cfg.d + (cfg.zwin - 1 - cfg.zwin // 2) + 1)
    for _ in range(args.warmup):
        _oracle_3d_sample(cfg, vol[:, :64, :64].copy(), n_sub)
    tot_p, tot_t = 0, 0.0
    from types import SimpleNamespace
    H, W = cfg.H, cfg.W
    ny, nx = (H - cfg.b) // cfg.s + 1, (W - cfg.b) // cfg.s + 1
    lo, hi = -(cfg.Wn // 2), cfg.Wn - 1 - cfg.Wn // 2
    tc = sum(min(H - cfg.b, iy * cfg.s + hi) - max(0, iy * cfg.s + lo) + 1 for iy in range(ny)) * \
        sum(min(W - cfg.b, ix * cfg.s + hi) - max(0, ix * cfg.s + lo) + 1 for ix in range(nx))
    info = {"total_candidates": tc}
    for _ in range(args.steps):
        _, _, dt, _ = _oracle_3d_sample(cfg, vol, n_sub)
        tot_p += _pairs_3d(cfg, info, n_sub)[1]
        tot_t += dt
    value = tot_p / tot_t
    print(json.dumps({"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
                      "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
                      "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                      "data": "synthetic", "config": {"workload": cfg.name},
                      "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                                       "sample": f"{cfg.name} planes 0:{n_sub}"},
                      "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
          flush=True)


def _dtype_name(cfg):
    return "int32" if cfg.dtype == "u8" else "f32"


def _config_obj(cfg, args):
    return {"workload": cfg.name, "images": cfg.N, "channels": cfg.C, "H": cfg.H, "W": cfg.W,
            "input_dtype": "u8" if cfg.dtype == "u8" else "f32", "patch": cfg.b, "stride": cfg.s,
            "window": cfg.Wn, "K": cfg.K, "sharding": "frames" if cfg.N > 1 else "replicas",
            "similarity": getattr(args, "metric", "l2"), "temporal_radius": getattr(args, "temporal", 0),
            "l2": "flushed between timed steps (256 MiB write); working set > L2"}


def bench_nlm(args, cfg, plan, x, ws, rank, local, dist):
    """NLM weights (Eq. 2 via Prop. 1) of one image per rank: weights/s, dense-table bytes vs HBM."""
    import torch
    info = plan.info()
    h = args.nlm_h or (np.sqrt(cfg.b * cfg.b * cfg.C) * (25.0 if cfg.dtype == "u8" else 0.1))
    img = x[:1]
    avg = args.op == "nlm_avg"  # the fused NL-means estimate instead of the weight table
    if avg:
        out = torch.empty((info["n_refs"], cfg.C, cfg.b, cfg.b), dtype=torch.float32, device=x.device)
        call = plan.nlm_average
    else:
        out = torch.empty((info["n_refs"], cfg.Wn * cfg.Wn), dtype=torch.float32, device=x.device)
        call = plan.nlm_weights
    for _ in range(args.warmup):
        call(img, h, out=out)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = plan.info()["launches"]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            starts[k].record(stream)
            call(img, h, out=out)
            ends[k].record(stream)
        torch.cuda.synchronize()
    ms = float(np.mean([s.elapsed_time(e) for s, e in zip(starts, ends)]))
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    pairs = info["total_candidates"]
    table = out.numel() * 4
    peaks = _peaks()
    gbs = 3 * table / (ms / 1e3) / 1e9  # distances written, re-read, weights written
    if rank == 0 and avg:
        # per candidate pair: b^2 C MACs of the cross term (Eq. 5) + b^2 C of the weighted sum
        flops = 2.0 * pairs * 2 * cfg.b * cfg.b * cfg.C
        peak = 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        tf = flops / (ms / 1e3) / 1e12
        line = {"metric": "NL-means weighted candidate patches/sec", "op": "nlm_avg", "value": pairs * ws / (ms / 1e3),
                "unit": "candidate patches/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "config": dict(_config_obj(cfg, args), nlm_h=h, images=1),
                "ref_patches_per_s": info["n_refs"] * ws / (ms / 1e3),
                "roofline": {"bound": "alu", "kernel": "bm_simt_kernel (AVG: fused weights + weighted sum)",
                             "achieved": tf, "peak": peak, "unit": "TFLOP/s", "frac": tf / peak, "traffic": None,
                             "algorithmic_flops_per_step": flops,
                             "peak_source": "FFMA: 148 SM x 128 lanes x 2 x sm_max_mhz"},
                "gpu_launches": int(plan.info()["launches"] - launches0), "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    elif rank == 0:
        line = {"metric": "NLM weights/sec", "op": "nlm", "value": pairs * ws / (ms / 1e3), "unit": "weights/s",
                "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "config": dict(_config_obj(cfg, args), nlm_h=h, images=1),
                "roofline": {"bound": "hbm", "kernel": "bm_simt_kernel dense + fused normalisation", "achieved": gbs,
                             "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": gbs / peaks["hbm_gbs"],
                             "traffic": None, "algorithmic_bytes_per_step": 3 * table},
                "gpu_launches": int(plan.info()["launches"] - launches0), "clocks": clk.summary()}
        print(json.dumps(line), flush=True)


def bench_group(args, cfg, plan, x, idx, ws, rank, local, dist):
    """Patch grouping Y_i of the run's idx table: gathered bytes/s vs HBM."""
    import torch
    info = plan.info()
    n = x.shape[0]
    Y = torch.empty((n, info["n_refs"], cfg.K, cfg.C, cfg.b, cfg.b), dtype=x.dtype, device=x.device)
    for _ in range(args.warmup):
        plan.group(x, idx, out=Y)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = plan.info()["launches"]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            starts[k].record(stream)
            plan.group(x, idx, out=Y)
            ends[k].record(stream)
        torch.cuda.synchronize()
    ms = float(np.mean([s.elapsed_time(e) for s, e in zip(starts, ends)]))
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    out_bytes = Y.numel() * Y.element_size()
    in_bytes = x.numel() * x.element_size() + idx.numel() * 4
    alg = out_bytes + in_bytes  # algorithmic bytes: every group byte written once, inputs read once
    peaks = _peaks()
    gbs = alg / (ms / 1e3) / 1e9
    if rank == 0:
        line = {"metric": "patch-group bytes/sec", "op": "group", "value": alg * ws / (ms / 1e3), "unit": "B/s",
                "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype,
                "data": "synthetic", "config": _config_obj(cfg, args),
                "groups_per_s": n * ws * info["n_refs"] / (ms / 1e3),
                "roofline": {"bound": "hbm", "kernel": "group_kernel", "achieved": gbs, "peak": peaks["hbm_gbs"],
                             "unit": "GB/s", "frac": gbs / peaks["hbm_gbs"], "traffic": None,
                             "algorithmic_bytes_per_launch": alg},
                "gpu_launches": int(plan.info()["launches"] - launches0), "clocks": clk.summary()}
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", help="c1..c5 (BASELINE.json configs), v1 / m1 (3D search)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--gather", action="store_true", help="also time an NCCL all-gather of the tables")
    ap.add_argument("--graph", action="store_true", help="also time the step replayed from a CUDA graph")
    ap.add_argument("--ref-step-s", type=float, default=4.0)
    ap.add_argument("--metric", default="l2", choices=["l2", "ncc"],
                    help="l2: Euclidean BM, Eq. 3 (the headline); ncc: normalised cross-correlation, Eq. 4")
    ap.add_argument("--op", default="bm", choices=["bm", "group", "nlm", "nlm_avg"],
                    help="bm: the block-matching hot path (default); group: patch grouping Y_i of its "
                         "output; nlm: NLM weights (Eq. 2) of the config's first image")
    ap.add_argument("--temporal", type=int, default=0,
                    help="3D / temporal search radius T: candidates in frames f-T..f+T of the batch")
    ap.add_argument("--nlm-h", type=float, default=0.0, help="NLM bandwidth (default: 1.0 * sqrt(b^2 C) * value scale)")
    ap.add_argument("--kernel", default="auto", choices=["auto", "simt", "warp", "tc", "box", "boxf", "tcf"],
                    help="force the matching kernel (default: the plan's choice)")
    ap.add_argument("--selftest-cpu", action="store_true",
                    help="CPU check of the multi-rank plumbing (gloo, stand-in step); prints no measurement")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    _launch_ranks(args)

    from paper_2006_13714_b200 import synth
    cfg = synth.config_by_name(args.config)
    if args.impl == "reference" and cfg.d > 0:
        return run_reference_3d(args, cfg)
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.selftest_cpu:
        return selftest_cpu(args, cfg)
    if cfg.d > 0:
        return bench_3d(args, cfg)

    import torch
    from paper_2006_13714_b200 import bm
    from paper_2006_13714_b200.bm import Plan

    ws, rank, local = _dist_env()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1 or args.gather:  # (--gather at N = 1: a one-rank NCCL group, so the gather paths run too)
        import torch.distributed as dist
        if ws == 1 and "MASTER_ADDR" not in os.environ:
            import socket
            with socket.socket() as so:
                so.bind(("127.0.0.1", 0))
                os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(so.getsockname()[1]),
                                  RANK="0", WORLD_SIZE="1")
        # a bounded collective timeout: a hung peer fails the run instead of blocking it forever
        # (TORCH_NCCL_ASYNC_ERROR_HANDLING is on by default for NCCL in this torch)
        import datetime
        dist.init_process_group("nccl", device_id=torch.device("cuda", local),
                                timeout=datetime.timedelta(seconds=int(os.environ.get("SCBM_NCCL_TIMEOUT_S", "300"))))

    # shard frames (strong scaling); single-image configs run as replicas
    if cfg.N > 1:
        per = [cfg.N // ws + (1 if r < cfg.N % ws else 0) for r in range(ws)]
        f0 = sum(per[:rank])
        nloc = per[rank]
    else:
        f0, nloc = 0, 1
    x_all = synth.make_input(cfg)
    x_host = np.ascontiguousarray(x_all[f0:f0 + nloc])
    del x_all
    x = torch.from_numpy(x_host).cuda()
    plan = Plan(cfg.H, cfg.W, cfg.C, cfg.b, cfg.s, cfg.Wn, cfg.K, cfg.dtype, metric=args.metric)
    if args.temporal > 0:
        plan.set_temporal(args.temporal)
    if args.kernel != "auto":
        plan.set_kernel({"simt": 0, "tc": 1, "warp": 2, "box": 3, "boxf": 4, "tcf": 5}[args.kernel])
    info = plan.info()
    idx, dst = plan.alloc_out(nloc)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    halo = args.temporal > 0 and ws > 1 and cfg.N > 1  # temporal search across frame shards

    def step():
        if halo:  # the T-frame halo exchange (NCCL point-to-point) + the window run, both timed
            from paper_2006_13714_b200.dist import run_temporal_sharded
            run_temporal_sharded(lambda ext, a0, a1, off: plan.run_temporal(ext, a0, a1, off, out=(idx, dst)),
                                 x, rank, ws, cfg.N, args.temporal)
        else:
            plan.run(x, out=(idx, dst))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if args.op == "group":
        return bench_group(args, cfg, plan, x, idx, ws, rank, local, dist)
    if args.op in ("nlm", "nlm_avg"):
        return bench_nlm(args, cfg, plan, x, ws, rank, local, dist)

    plan.set_timing(True)
    plan.get_timing()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = plan.info()["launches"]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.fill_(k & 0xFF)  # L2 flush outside the step's events
            torch.cuda.nvtx.range_push(f"bm_step_{k}")  # (NVTX: step boundaries in an nsys / ncu timeline)
            starts[k].record(stream)
            step()
            ends[k].record(stream)
            torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches = plan.info()["launches"] - launches0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    tm = plan.get_timing()
    plan.set_timing(False)
    ms_local = float(np.mean(step_ms))
    match_ms_local = tm["match_ms"] / max(1, args.steps)
    norm_ms_local = tm["norm_ms"] / max(1, args.steps)
    t = torch.tensor([ms_local, match_ms_local, norm_ms_local, float(np.median(step_ms)), float(np.min(step_ms))],
                     dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, match_ms, norm_ms, ms_median, ms_min = t.tolist()

    # the same step captured once into a CUDA graph and replayed (launch-bound small configs)
    graph = None
    if args.graph:
        gs = torch.cuda.Stream()
        gs.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=gs):
            plan.run(x, out=(idx, dst), stream=gs)
        torch.cuda.synchronize()
        gst = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        gen = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            gst[k].record(stream)
            g.replay()
            gen[k].record(stream)
        torch.cuda.synchronize()
        gms = torch.tensor([float(np.mean([a.elapsed_time(b) for a, b in zip(gst, gen)]))], dtype=torch.float64,
                           device="cuda")
        if dist:
            dist.all_reduce(gms, op=dist.ReduceOp.MAX)
        graph = {"ms_per_step": gms.item(), "note": "one captured plan.run replayed per step (torch.cuda.CUDAGraph)"}

    pairs_per_image = info["total_candidates"]
    n_images_total = cfg.N if cfg.N > 1 else ws
    pairs_step = pairs_per_image * n_images_total
    if args.temporal > 0:  # every reference also searches the frames f-T..f+T of the video
        nvid = cfg.N if cfg.N > 1 else 1
        T_ = args.temporal
        fs = [min(nvid - 1, f + T_) - max(0, f - T_) + 1 for f in range(nvid)]
        pairs_step = pairs_per_image * sum(fs) * (1 if cfg.N > 1 else ws)
        pairs_rank_t = pairs_per_image * (sum(fs[f0:f0 + nloc]) if cfg.N > 1 else fs[0])
    refs_step = info["n_refs"] * n_images_total
    value = pairs_step / (ms / 1e3)
    if graph:
        graph["value"] = pairs_step / (graph["ms_per_step"] / 1e3)

    # roofline of the dominant kernel (the fused cross-term / top-K kernel)
    peaks = _peaks()
    # algorithmic MACs per candidate pair = SURVEY.md 8d's per-unit figure MAC_alg: the cross term
    # of Eq. 5 is b^2 C multiply-adds per (reference, candidate) pair. The
    # kernels EXECUTE fewer: the box-sum kernel forms each product of the shifted product image
    # once, s^2 C per pair (its 4x4 block sums are shared by 2 x 2 references, c5); the float box
    # kernel correlates one s-column strip per reference and offset, b s C per pair. Both are
    # reported (frac_executed = the executed MACs at the same peak).
    mac_pair = cfg.b * cfg.b * cfg.C
    mac_exec = {3: cfg.s * cfg.s * cfg.C, 4: cfg.b * cfg.s * cfg.C,
                5: 3 * cfg.C * cfg.b * 8}.get(info["kernel"], mac_pair)  # 3xTF32: 3 MMAs of K = 8 b
    pairs_rank = pairs_rank_t if args.temporal > 0 else pairs_per_image * nloc
    macs_launch = pairs_rank * mac_pair  # algorithmic MACs per rank-step
    macs_direct = pairs_rank * cfg.b * cfg.b * cfg.C
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    tf32x3_peak = 0.5 * peaks["bf16_tflops"] / 3.0  # tf32 = 1/2 bf16 (guide ratio, tools/tc_peaks.cu), 3 MMAs per MAC
    if info["kernel"] == 1:
        peak = 2.0 * peaks["bf16_tflops"]  # int8 tcgen05 = 2x the measured bf16 (guide's nominal ratio)
        bound, unit, peak_note = "tensor", "TOP/s", "int8 dense = 2 x measured bf16 burst (MEASURED_PEAKS.json x guide ratio)"
    elif info["kernel"] == 5:
        peak = tf32x3_peak
        bound, unit, peak_note = "tensor", "TFLOP/s", ("3xTF32: tf32 dense = 1/2 x measured bf16 burst (MEASURED_PEAKS.json x "
                                                       "guide ratio, confirmed by tools/tc_peaks.cu) / 3 MMAs per product")
    elif cfg.dtype == "u8":
        # dp4a: 64 lanes/SM/clk (half rate, measured by tools/peaks.cu) x 4 MACs x 2 ops
        peak = 148 * 64 * 4 * 2 * sm_mhz * 1e6 / 1e12
        bound, unit, peak_note = "alu", "TOP/s", "dp4a: 148 SM x 64 lanes x 4 MAC x 2 x sm_max_mhz (DESIGN.md section 7)"
    else:
        peak = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12  # FP32 FFMA lanes x 2 ops x max clock
        bound, unit, peak_note = "alu", "TFLOP/s", "FFMA: 148 SM x 128 lanes x 2 x sm_max_mhz (DESIGN.md section 7)"
    achieved = 2.0 * macs_launch / (match_ms / 1e3) / 1e12 if match_ms > 0 else None
    traffic, traffic_src = None, None
    kname = {0: "bm_lanes_kernel", 1: "bm_tc_i8_kernel", 2: "bm_simt_kernel", 3: "bm_box_kernel",
             4: "bm_boxf_kernel", 5: "bm_tcf_kernel"}[info["kernel"]]
    # the ncu capture of THIS kernel, config, metric and temporal mode (newest round first)
    tag = f"{kname.replace('_kernel', '')}{'_ncc' if args.metric == 'ncc' else ''}_{cfg.name}" + \
        (f"_t{args.temporal}" if args.temporal else "")
    prof = next((c for c in (os.path.join(ROOT, "profiles", r, f"ncu_full_{tag}_metrics.json")
                             for r in ("r02", "r01", os.path.join("r01", "next"))) if os.path.exists(c)), "")
    if prof:
        m = json.load(open(prof))
        mb = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
        traffic = sum(float(m[k]["value"]) * mb.get(m[k]["unit"], 1.0) for k in
                      ("dram__bytes_read.sum", "dram__bytes_write.sum")) * 1e6
        traffic_src = (f"{os.path.relpath(prof, ROOT)}: dram read+write bytes of one launch "
                       f"({min(info['frames_per_chunk'], cfg.N)} frames), ncu --set full")
    roof = {"bound": bound, "kernel": kname,
            "achieved": achieved, "peak": peak, "unit": unit,
            "frac": (achieved / peak) if achieved else None, "traffic": traffic, "traffic_source": traffic_src,
            "peak_source": peak_note, "kernel_ms_per_step": match_ms, "norm_ms_per_step": norm_ms,
            "kernel_share_of_step": match_ms / ms if ms > 0 else None,
            "algorithmic_ops_per_launch": 2.0 * macs_launch, "macs_per_pair": mac_pair,
            "executed_macs_per_pair": mac_exec,
            "frac_executed": (achieved * mac_exec / mac_pair / peak) if achieved else None}
    # the north_star's roofline: direct b^2 C MACs per pair at the int8 / fp32 peak vs image +
    # output bytes at HBM bandwidth (whichever is slower), against the measured step time
    if cfg.dtype == "u8":
        mac_peak, mac_unit = 2.0 * peaks["bf16_tflops"] * 1e12 / 2.0, "int8 tcgen05 (2 x measured bf16)"
    else:
        mac_peak, mac_unit = 148 * 128 * sm_mhz * 1e6, "fp32 FFMA"
    io_bytes = nloc * (cfg.C * cfg.H * cfg.W * (1 if cfg.dtype == "u8" else 4) + info["n_refs"] * cfg.K * 8)
    t_mac, t_hbm = macs_direct / mac_peak, io_bytes / (peaks["hbm_gbs"] * 1e9)
    roof["north_star"] = {"t_roof_ms": 1e3 * max(t_mac, t_hbm), "t_mac_ms": 1e3 * t_mac, "t_hbm_ms": 1e3 * t_hbm,
                          "mac_unit": mac_unit, "frac": (1e3 * max(t_mac, t_hbm)) / ms if ms > 0 else None}
    if cfg.dtype != "u8":  # the best-available float unit too, so the unit choice cannot inflate the number
        t_best = max(macs_direct / (tf32x3_peak * 1e12 / 2.0), t_hbm)
        roof["north_star"]["best_unit"] = {"unit": "3xTF32 tcgen05 (tf32 = 1/2 measured bf16, / 3)",
                                           "t_roof_ms": 1e3 * t_best, "frac": 1e3 * t_best / ms if ms > 0 else None}

    # end-to-end through the public API with host buffers (pinned), copies inside the timing
    e2e = None
    if not args.no_e2e and args.temporal == 0:  # the host path has no temporal mode
        xh = torch.from_numpy(x_host).pin_memory()
        hi = torch.empty((nloc, info["n_refs"], cfg.K), dtype=torch.int32).pin_memory()
        hd = torch.empty((nloc, info["n_refs"], cfg.K),
                         dtype=torch.int32 if (cfg.dtype == "u8" and args.metric == "l2") else torch.float32).pin_memory()
        plan.run_host(xh, out=(hi, hd))
        e_steps = max(3, min(args.steps, 5))
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            plan.run_host(xh, out=(hi, hd))
        e_ms = (time.perf_counter() - t0) * 1e3 / e_steps
        te = torch.tensor([e_ms], dtype=torch.float64, device="cuda")
        if dist:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e_ms = te.item()
        e2e = {"value": pairs_step / (e_ms / 1e3), "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(xh.numel() * xh.element_size()) * (ws if cfg.N > 1 else 1),
               "d2h_bytes_per_step": int(2 * hi.numel() * 4) * (ws if cfg.N > 1 else 1),
               "steps": e_steps, "timing": "wall clock around sc_bm_run_host (synchronous), max over ranks"}
        # the same through the packed tables (sc_bm_set_packed: one lossless uint32 word per result,
        # SURVEY 8e), which halve the PCIe-bound device->host copy; decoded and compared once
        if cfg.dtype == "u8" and args.metric == "l2" and info["kernel"] == 3:
            plan.set_packed(max(4096, info["n_refs"] // 4))
            words, _ = plan.packed_words(nloc)
            hp = torch.empty(words, dtype=torch.int32).pin_memory()
            plan.run_host_packed(xh, out=hp)
            if dist:
                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(e_steps):
                plan.run_host_packed(xh, out=hp)
            p_ms = (time.perf_counter() - t0) * 1e3 / e_steps
            tp = torch.tensor([p_ms], dtype=torch.float64, device="cuda")
            if dist:
                dist.all_reduce(tp, op=dist.ReduceOp.MAX)
            p_ms = tp.item()
            body = nloc * info["n_refs"] * cfg.K
            n_esc = int(hp[body].item())
            pi, pd = bm.unpack_host(cfg.H, cfg.W, cfg.b, cfg.s, cfg.Wn, cfg.K, hp, nloc)
            same = bool(np.array_equal(pi, hi.numpy()) and np.array_equal(pd, hd.numpy()))
            plan.set_packed(0)
            e2e["packed"] = {"value": pairs_step / (p_ms / 1e3), "unit": UNIT, "ms_per_step": p_ms,
                             "h2d_bytes_per_step": e2e["h2d_bytes_per_step"],
                             "d2h_bytes_per_step": int((body + 2 + n_esc * (2 + 2 * cfg.K)) * 4) * (ws if cfg.N > 1 else 1),
                             "escape_rows": n_esc, "decoded_equals_plain": same,
                             "what": "sc_bm_run_host with packed tables (uint32 (dist << rb) | window slot, "
                                     "lossless); host decode sc_bm_unpack_host outside the timed region"}

    gather = None
    if dist and (args.gather or (cfg.N > 1 and args.temporal == 0)):  # default at N > 1
        gi = torch.empty((ws * idx.shape[0],) + tuple(idx.shape[1:]), dtype=idx.dtype, device="cuda")
        gd = torch.empty_like(gi, dtype=dst.dtype)
        dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        dist.all_gather_into_tensor(gi, idx)
        dist.all_gather_into_tensor(gd, dst)
        g1.record()
        torch.cuda.synchronize()
        tg = torch.tensor([g0.elapsed_time(g1)], dtype=torch.float64, device="cuda")
        dist.all_reduce(tg, op=dist.ReduceOp.MAX)
        gather = {"ms": tg.item(), "bytes_per_rank": int(2 * gi.numel() * 4), "backend": "nccl",
                  "equal_shards": bool(cfg.N % ws == 0)}
        # end to end with the NCCL gather: pinned host frames -> HBM, the matcher, the all-gather
        # of both tables (every rank ends with the whole batch's tables), device-timed per step,
        # max over ranks
        xp = torch.from_numpy(x_host).pin_memory()
        e_steps = max(3, min(args.steps, 5))
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(e_steps)]
        dist.barrier()
        torch.cuda.synchronize()
        for a_, b_ in ev:
            a_.record()
            x.copy_(xp, non_blocking=True)
            plan.run(x, out=(idx, dst))
            dist.all_gather_into_tensor(gi, idx)
            dist.all_gather_into_tensor(gd, dst)
            b_.record()
        torch.cuda.synchronize()
        te = torch.tensor([float(np.mean([a_.elapsed_time(b_) for a_, b_ in ev]))], dtype=torch.float64, device="cuda")
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        gather["h2d_compute_gather_ms"] = te.item()
        gather["h2d_compute_gather_value"] = pairs_step / (te.item() / 1e3)
        if e2e is not None:
            e2e["nccl_gather"] = {"value": pairs_step / (te.item() / 1e3), "ms_per_step": te.item(),
                                  "what": "pinned H2D of the rank's frames + matcher + NCCL all-gather of "
                                          "idx and dist to every rank (device events, max over ranks)"}
        # compute + gather pipelined per frame chunk (the gather of chunk c overlaps chunk c+1)
        from paper_2006_13714_b200.dist import run_frames_pipelined
        chunk = max(1, nloc // 4)
        if nloc % chunk == 0:
            run_frames_pipelined(lambda fr: plan.run(fr), x, rank, ws, chunk, local=True)  # warm (async NCCL setup)
            torch.cuda.synchronize()
            dist.barrier()
            p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            p0.record()
            run_frames_pipelined(lambda fr: plan.run(fr), x, rank, ws, chunk, local=True)
            p1.record()
            torch.cuda.synchronize()
            tp = torch.tensor([p0.elapsed_time(p1)], dtype=torch.float64, device="cuda")
            dist.all_reduce(tp, op=dist.ReduceOp.MAX)
            gather["compute_plus_gather_pipelined_ms"] = tp.item()
            gather["chunk_frames"] = chunk
        # the gather fused into the matcher's epilogue: every rank's kernels store their rows
        # straight into rank 0's tables through CUDA IPC / NVLink peer mappings (dist.PeerTables)
        if args.temporal == 0:
            from paper_2006_13714_b200.dist import PeerTables
            pt = PeerTables(plan, nloc * ws, rank, ws)
            for _ in range(2):  # warm the mapping
                pt.run(x)
            pt.finish()
            q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            q0.record()
            pt.run(x)
            q1.record()
            torch.cuda.synchronize()
            tq = torch.tensor([q0.elapsed_time(q1)], dtype=torch.float64, device="cuda")
            dist.all_reduce(tq, op=dist.ReduceOp.MAX)
            pt.finish()
            gather["compute_plus_peer_store_ms"] = tq.item()
            del pt
        # packed tables through the gather (dist.gather_packed: one uint32 word per result, half the
        # NVLink bytes of the (idx, dist) all-gather): matcher in packed mode + packed all-gather
        if cfg.dtype == "u8" and args.metric == "l2" and args.temporal == 0 and info["kernel"] == 3:
            from paper_2006_13714_b200.dist import balanced_ranges, gather_packed
            counts = [e_ - s_ for s_, e_ in balanced_ranges(cfg.N, ws)]
            plan.set_packed(max(4096, info["n_refs"] // 4))
            words, _ = plan.packed_words(nloc)
            pbuf = torch.empty(words, dtype=torch.int32, device="cuda")
            for _ in range(2):
                plan.run_packed(x, out=pbuf)
                full = gather_packed(pbuf, counts, info["n_refs"], cfg.K)
            dist.barrier()
            torch.cuda.synchronize()
            k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k0.record()
            plan.run_packed(x, out=pbuf)
            full = gather_packed(pbuf, counts, info["n_refs"], cfg.K)
            k1.record()
            torch.cuda.synchronize()
            tk = torch.tensor([k0.elapsed_time(k1)], dtype=torch.float64, device="cuda")
            dist.all_reduce(tk, op=dist.ReduceOp.MAX)
            wN, _ = plan.packed_words(cfg.N)  # (the device decoder takes a buffer of the plan's layout)
            same = False
            if full.numel() <= wN:
                padded = torch.zeros(wN, dtype=torch.int32, device="cuda")
                padded[:full.numel()] = full
                pi, pd = plan.unpack(padded, cfg.N)
                same = bool(torch.equal(pi[f0:f0 + nloc], idx) and torch.equal(pd[f0:f0 + nloc], dst))
                del padded, pi, pd
            plan.set_packed(0)
            gather["compute_plus_packed_gather_ms"] = tk.item()
            gather["packed_gather_bytes_per_rank"] = int(full.numel() * 4)
            gather["packed_decoded_equals_plain"] = same
            del pbuf, full

    cpu, parity = None, None
    if rank == 0 and ws == 1 and not args.no_cpu:
        # the oracle on ~10-30 s of the same workload (whole frames where one frame takes less;
        # the middle-row calibration overestimates a frame, whose border rows have clipped windows)
        cpu, _, _, sample = _cpu_sample(cfg, x_host, target_s=20.0, metric=args.metric, want_tables=True)
        if args.temporal == 0:
            parity = _parity_of_sample(cfg, x_host, idx, dst, sample, args.metric)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "ms_per_step_median": ms_median, "ms_per_step_min": ms_min,
                "higher_is_better": True,
                "scaling": "strong" if cfg.N > 1 else "weak", "vs_baseline": None,
                "dtype": _dtype_name(cfg), "data": "synthetic", "config": _config_obj(cfg, args),
                "ref_patches_per_s": refs_step / (ms / 1e3), "candidate_pairs_per_step": pairs_step,
                "roofline": roof, "cpu_baseline": cpu, "parity": parity, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clk.summary(), "gather": gather, "graph": graph,
                "kernel": info["kernel"], "frames_per_chunk": info["frames_per_chunk"], "metric_kind": args.metric}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
