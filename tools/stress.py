"""Randomised parity stress run (GPU): many random geometries / images per matcher and metric
against the CPU oracle, beyond the fixed pytest sweeps. Prints one line per failure and a summary.

    python tools/stress.py [seconds_budget] [seed]
"""
import os
import sys
import time
import traceback

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from paper_2006_13714_b200 import synth  # noqa: E402
from paper_2006_13714_b200.bm import (SC_KERNEL_BOX, SC_KERNEL_BOXF, SC_KERNEL_SIMT,  # noqa: E402
                                      SC_KERNEL_SIMT_WARP, SC_KERNEL_TC_F32, Plan, Plan3D, ScError)
from parity import check_f32, check_f32_3d, check_ncc, check_u8  # noqa: E402


def image(rng, kind, N, C, H, W, dtype):
    if kind == "random":
        return synth.random_image(rng, N, C, H, W, dtype)
    if kind == "binary":
        x = rng.integers(0, 2, size=(N, C, H, W)) * (255 if dtype == "u8" else 1.0)
    elif kind == "smooth":
        yy, xx = np.mgrid[0:H, 0:W]
        x = np.stack([np.stack([np.sin(0.05 * (c + 1) * yy + 0.07 * xx + n) for c in range(C)]) for n in range(N)])
        x = (x + 1) * (127.5 if dtype == "u8" else 0.5)
    else:  # "quantised": few levels, many exact ties
        x = rng.integers(0, 4, size=(N, C, H, W)) * (60 if dtype == "u8" else 0.25)
    return np.round(x).astype(np.uint8) if dtype == "u8" else x.astype(np.float32)


FOCUS = os.environ.get("STRESS_FOCUS", "")  # "", "ncc", "box" (u8 b=8 s=4: the dp4a kernels), "3d"


def one3d(rng):
    """The 3D search (sc_bm_plan3d) against oracle.bm3d on a random volume."""
    kind = rng.choice(["random", "binary", "smooth", "quantised"])
    s, b = [(3, 8), (1, 7), (4, 8), (2, 8), (1, 6)][rng.integers(0, 5)]
    P = int(rng.integers(1, 8))
    d = int(rng.integers(1, min(P, 3) + 1))
    H, W = int(rng.integers(b, 60)), int(rng.integers(b, 80))
    Wn, c, sz = int(rng.integers(1, 24)), int(rng.integers(1, 6)), int(rng.integers(1, 3))
    K = int(rng.integers(1, 40))
    vol = image(rng, kind, 1, P, H, W, "f32")[0]
    desc = f"3d {kind} P{P} d{d} {H}x{W} b{b} s{s} sz{sz} Wn{Wn} c{c} K{K}"
    try:
        p = Plan3D(H, W, d, b, s, Wn, sz, c, K)
    except ScError:
        return "skip", desc
    gi, gd = p.run(torch.from_numpy(vol).cuda())
    torch.cuda.synchronize()
    oi, od = oracle.bm3d(vol, d, b, s, sz, Wn, c, K)
    check_f32_3d(vol, d, b, s, sz, Wn, c, K, gi.cpu().numpy(), gd.cpu().numpy(), oi, od, desc)
    return "ok", desc


def one(rng):
    if FOCUS == "3d" or (FOCUS == "" and rng.random() < 0.15):
        return one3d(rng)
    metric = "ncc" if FOCUS == "ncc" else rng.choice(["l2", "l2", "l2", "ncc"])
    dtype = "u8" if FOCUS == "box" else rng.choice(["u8", "f32"])
    kind = rng.choice(["random", "binary", "smooth", "quantised"])
    if FOCUS == "box" or (dtype == "u8" and rng.random() < 0.6):  # the dp4a box kernel's geometry
        b, s, C = 8, 4, 1
    elif rng.random() < 0.5:  # the float box kernel's shapes
        s, b = [(3, 8), (1, 7), (4, 8), (2, 8), (1, 6)][rng.integers(0, 5)]
        C = int(rng.choice([1, 1, 2, 4]))
    else:
        b, s, C = int(rng.integers(1, 13)), int(rng.integers(1, 6)), int(rng.integers(1, 4))
    H, W = int(rng.integers(b, 90)), int(rng.integers(b, 130))
    Wn = int(rng.integers(1, 40))
    K = int(rng.integers(1, (25 if dtype == "u8" else 77) if metric == "ncc" else 72))
    N = int(rng.integers(1, 4))
    kernel = "box" if FOCUS == "box" and rng.random() < 0.7 else \
        rng.choice(["default", "box", "boxf", "warp", "lanes", "tcf"])
    T = int(rng.integers(1, 3)) if (metric == "l2" and dtype == "u8" and b == 8 and s == 4 and C == 1
                                    and rng.random() < 0.25) else 0
    x = image(rng, kind, N, C, H, W, dtype)
    desc = f"{metric} {dtype} {kind} N{N} C{C} {H}x{W} b{b} s{s} Wn{Wn} K{K} {kernel} T{T}"
    try:
        p = Plan(H, W, C, b, s, Wn, K, dtype, metric=metric)
        if T:
            p.set_temporal(T)
        elif kernel != "default":
            p.set_kernel({"box": SC_KERNEL_BOX, "boxf": SC_KERNEL_BOXF, "warp": SC_KERNEL_SIMT_WARP,
                          "lanes": SC_KERNEL_SIMT, "tcf": SC_KERNEL_TC_F32}[kernel])
    except ScError:
        return "skip", desc
    t = torch.from_numpy(x).cuda()
    if rng.random() < 0.2 and not T:  # the pipelined host path instead of the device call
        hi, hd = p.run_host(torch.from_numpy(x).pin_memory())
        gi, gd = hi.numpy(), hd.numpy()
    else:
        gi, gd = p.run(t)
        torch.cuda.synchronize()
        gi, gd = gi.cpu().numpy(), gd.cpu().numpy()
    if rng.random() < 0.3:  # the next rows on the same plan: groups of this run, NLM weights / estimate
        Y = p.group(t, torch.from_numpy(gi).cuda()).cpu().numpy()
        if T:  # batch-global idx: the frames stacked vertically (C = 1)
            want = oracle.group(x.reshape(1, 1, N * H, W), gi.reshape(1, -1, K), b).reshape(Y.shape)
        else:
            want = oracle.group(x, gi, b)
        assert np.array_equal(Y, want), f"group mismatch: {desc}"
        if metric == "l2" and not T and b * b * C <= 256:
            h = float(rng.choice([0.3, 3.0, 1e6])) * (255.0 if dtype == "u8" else 1.0) * b
            scale = 255.0 if dtype == "u8" else 1.0
            w = p.nlm_weights(t[0], h).cpu().numpy().astype(np.float64)
            ww = oracle.nlm_weights(x[0], b, s, Wn, h)
            m = ww > 1e-6
            assert np.allclose(w[m], ww[m], rtol=1e-4, atol=1e-9), f"nlm weights mismatch: {desc} h={h}"
            a = p.nlm_average(t[0], h).cpu().numpy().astype(np.float64)
            aa = oracle.nlm_average(x[0], b, s, Wn, h)
            assert np.allclose(a, aa, rtol=0, atol=1e-4 * scale), f"nlm average mismatch: {desc} h={h}"

    if T:
        oi, od = oracle.bm_temporal(x, b, s, Wn, K, T)
        check_u8(gi, gd, oi, od, desc)
    elif metric == "ncc":
        oi, od = oracle.ncc(x, b, s, Wn, K)
        for n in range(N):
            check_ncc(x[n], b, s, Wn, K, gi[n], gd[n], oi[n], od[n], exact=dtype == "u8", where=desc)
    else:
        oi, od = oracle.bm(x, b, s, Wn, K)
        for n in range(N):
            if dtype == "u8":
                check_u8(gi[n], gd[n], oi[n], od[n], desc)
            else:
                check_f32(x[n], b, s, Wn, K, gi[n], gd[n], oi[n], od[n], where=desc)
    return "ok", desc


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 2026
    rng = np.random.Generator(np.random.PCG64(seed))
    t0, counts, fails = time.time(), {"ok": 0, "skip": 0, "fail": 0}, []
    while time.time() - t0 < budget:
        try:
            st, desc = one(rng)
            counts[st] += 1
        except AssertionError as e:
            counts["fail"] += 1
            fails.append(str(e).splitlines()[0][:300])
            print("FAIL", fails[-1], flush=True)
        except Exception:
            counts["fail"] += 1
            fails.append(traceback.format_exc().splitlines()[-1][:300])
            print("ERROR", fails[-1], flush=True)
    print("stress summary:", counts, f"{time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
