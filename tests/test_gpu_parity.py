"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs. u8 bit-exact; f32 per the tolerance rule in tests/parity.py."""
import numpy as np
import pytest

import oracle
from paper_2006_13714_b200 import synth
from tests.parity import check_f32, check_u8

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _plan(cfg_or_args, dtype=None):
    from paper_2006_13714_b200.bm import Plan
    if isinstance(cfg_or_args, synth.BMConfig):
        c = cfg_or_args
        return Plan(c.H, c.W, c.C, c.b, c.s, c.Wn, c.K, c.dtype)
    return Plan(*cfg_or_args, dtype)


def _run(plan, x):
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    idx, dist = plan.run(t)
    torch.cuda.synchronize()
    return idx.cpu().numpy(), dist.cpu().numpy()


def _compare(x, b, s, Wn, K, dtype, where="", kernel=None):
    N, C, H, W = x.shape
    p = _plan((H, W, C, b, s, Wn, K), dtype)
    if kernel is not None:
        p.set_kernel(kernel)
    gi, gd = _run(p, x)
    oi, od = oracle.bm(x, b, s, Wn, K)
    if dtype == "u8":
        check_u8(gi, gd, oi, od, where)
    else:
        for n in range(N):
            check_f32(x[n], b, s, Wn, K, gi[n], gd[n], oi[n], od[n], where=f"{where} img{n}")


# ------------------------------------------------------------------ steps a1 and a2+a3
@pytest.mark.parametrize("dtype", ["u8", "f32"])
@pytest.mark.parametrize("C,H,W,b", [(1, 64, 64, 8), (1, 37, 53, 7), (4, 40, 33, 8), (3, 19, 100, 1), (2, 30, 30, 16)])
def test_norm_map(dtype, C, H, W, b):
    rng = np.random.Generator(np.random.PCG64(H * W + C))
    x = synth.random_image(rng, 1, C, H, W, dtype)[0]
    p = _plan((H, W, C, b, 1, 3, 1), dtype)
    got = p.norm_map(torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64)
    if dtype == "u8":
        want = oracle.norm_map(x.astype(np.float64) - 128.0, b)
        np.testing.assert_array_equal(got, want)
    else:
        xc = (x - np.float32(0.5)).astype(np.float32).astype(np.float64)
        want = oracle.norm_map(xc, b)
        np.testing.assert_allclose(got, want, rtol=2e-7, atol=0)


@pytest.mark.parametrize("dtype", ["u8", "f32"])
@pytest.mark.parametrize("C,H,W,b,s,Wn", [(1, 64, 64, 8, 4, 21), (1, 40, 45, 7, 1, 13), (4, 36, 41, 8, 3, 17),
                                          (1, 20, 20, 3, 2, 30), (2, 33, 29, 12, 5, 9)])
@pytest.mark.parametrize("kernel", ["default", "lanes", "warp"])
def test_dense_cross_term(dtype, C, H, W, b, s, Wn, kernel):
    from paper_2006_13714_b200.bm import SC_KERNEL_SIMT, SC_KERNEL_SIMT_WARP
    rng = np.random.Generator(np.random.PCG64(7 * H + W))
    x = synth.random_image(rng, 1, C, H, W, dtype)[0]
    p = _plan((H, W, C, b, s, Wn, 1), dtype)
    if kernel != "default":  # the lanes matcher's dense mode (heap layout even where u8 b = 8 uses registers)
        p.set_kernel(SC_KERNEL_SIMT if kernel == "lanes" else SC_KERNEL_SIMT_WARP)
    got = p.dense_debug(torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64)
    want = oracle.bm_dense(x, b, s, Wn)
    np.testing.assert_array_equal(got == -1, want == -1)
    if dtype == "u8":
        np.testing.assert_array_equal(got, want)
    else:
        # identity in fp32 on centred data: error relative to the norms, not to d
        scale = b * b * C * 0.25
        m = want >= 0
        assert np.max(np.abs(got[m] - want[m])) <= 4e-6 * scale + 1e-5 * np.max(want[m])


# ------------------------------------------------------------------ configs
def test_c1_full_bitexact():
    cfg = synth.CONFIGS["c1"]
    x = synth.make_input(cfg)
    p = _plan(cfg)
    gi, gd = _run(p, x)
    oi, od = oracle.bm(x, cfg.b, cfg.s, cfg.Wn, cfg.K)
    check_u8(gi, gd, oi, od, "c1")
    assert (gd[..., 0] == 0).all()


def test_c5_full_batch_all_frames():
    """The bench launch configuration (all 64 frames in one call): EVERY reference of every
    frame, idx and dist bit-exact against the oracle (Eq. 3; the paper's
    "identical results"). ~1 min of oracle time on 16 host cores."""
    cfg = synth.CONFIGS["c5"]
    x = synth.make_input(cfg)
    p = _plan(cfg)
    gi, gd = _run(p, x)
    for f0 in range(0, cfg.N, 16):  # 16 frames per oracle call bounds host memory
        oi, od = oracle.bm(x, cfg.b, cfg.s, cfg.Wn, cfg.K, images=(f0, f0 + 16))
        check_u8(gi[f0:f0 + 16], gd[f0:f0 + 16], oi, od, f"c5 frames {f0}:{f0 + 16}")


def test_c2_full():
    cfg = synth.CONFIGS["c2"]
    x = synth.make_input(cfg)
    p = _plan(cfg)
    gi, gd = _run(p, x)
    oi, od = oracle.bm(x, cfg.b, cfg.s, cfg.Wn, cfg.K)
    check_f32(x[0], cfg.b, cfg.s, cfg.Wn, cfg.K, gi[0], gd[0], oi[0], od[0], where="c2")


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_c3_c4_full(name):
    """Every reference of c3 (WNNM-shaped, K = 70) and c4 (4-channel, K = 32) under the f32 rule."""
    cfg = synth.CONFIGS[name]
    x = synth.make_input(cfg)
    p = _plan(cfg)
    gi, gd = _run(p, x)
    oi, od = oracle.bm(x, cfg.b, cfg.s, cfg.Wn, cfg.K)
    check_f32(x[0], cfg.b, cfg.s, cfg.Wn, cfg.K, gi[0], gd[0], oi[0], od[0], where=f"{name} full")


# ------------------------------------------------------------------ random sweeps
def _sweep_cases(n, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    while len(out) < n:
        b = int(rng.integers(1, 17))
        C = int(rng.choice([1, 1, 1, 2, 3, 4, 8]))
        H = int(rng.integers(b, b + 60))
        W = int(rng.integers(b, b + 70))
        s = int(rng.integers(1, 6))
        Wn = int(rng.integers(1, 42))
        K = int(rng.integers(1, 129))
        pairs = ((H - b) // s + 1) * ((W - b) // s + 1) * Wn * Wn * b * b * C
        if pairs > 3e8:
            continue
        out.append((C, H, W, b, s, Wn, K))
    return out


@pytest.mark.parametrize("case", _sweep_cases(24, 101))
@pytest.mark.parametrize("dtype", ["u8", "f32"])
def test_random_sweep(case, dtype):
    C, H, W, b, s, Wn, K = case
    rng = np.random.Generator(np.random.PCG64(hash(case) % (1 << 32)))
    x = synth.random_image(rng, 2, C, H, W, dtype)
    _compare(x, b, s, Wn, K, dtype, where=f"{dtype} {case}")


@pytest.mark.parametrize("case", _sweep_cases(10, 202))
@pytest.mark.parametrize("dtype", ["u8", "f32"])
def test_random_sweep_warp_kernel(case, dtype):
    """The one-warp-per-reference SIMT kernel (SC_KERNEL_SIMT_WARP) on its own sweep."""
    from paper_2006_13714_b200.bm import SC_KERNEL_SIMT_WARP
    C, H, W, b, s, Wn, K = case
    rng = np.random.Generator(np.random.PCG64(hash(case) % (1 << 32)))
    x = synth.random_image(rng, 2, C, H, W, dtype)
    _compare(x, b, s, Wn, K, dtype, where=f"warp {dtype} {case}", kernel=SC_KERNEL_SIMT_WARP)


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_configs_warp_kernel(name):
    from paper_2006_13714_b200.bm import SC_KERNEL_SIMT_WARP
    cfg = synth.CONFIGS[name]
    x = synth.make_input(cfg)
    _compare(x, cfg.b, cfg.s, cfg.Wn, cfg.K, cfg.dtype, where=f"warp {name}", kernel=SC_KERNEL_SIMT_WARP)


# ------------------------------------------------------------------ edge cases
@pytest.mark.parametrize("dtype", ["u8", "f32"])
def test_constant_image_ties(dtype):
    x = np.full((1, 1, 41, 37), 200 if dtype == "u8" else 0.75, dtype=np.uint8 if dtype == "u8" else np.float32)
    N, C, H, W = x.shape
    p = _plan((H, W, C, 6, 3, 15, 40), dtype)
    gi, gd = _run(p, x)
    oi, od = oracle.bm(x, 6, 3, 15, 40)
    np.testing.assert_array_equal(gi, oi)  # all ties: the (distance, idx) order decides
    assert (gd[gi >= 0] == 0).all()


def test_periodic_tiling_duplicates_u8():
    rng = np.random.Generator(np.random.PCG64(5))
    motif = rng.integers(0, 256, size=(8, 8), dtype=np.uint8)
    x = np.tile(motif, (9, 11))[None, None].copy()
    _compare(x, 8, 4, 33, 16, "u8", where="periodic")


@pytest.mark.parametrize("dtype", ["u8", "f32"])
@pytest.mark.parametrize("H,W,b,s,Wn,K", [
    (30, 31, 5, 2, 1, 3),        # Wn = 1: self only, padding
    (12, 14, 4, 1, 41, 128),     # window covers the image; K > candidates
    (16, 16, 16, 1, 5, 2),       # single position
    (17, 40, 16, 3, 9, 20),      # max patch side
    (50, 9, 3, 4, 6, 7),         # even window
    (64, 64, 8, 64, 21, 16),     # stride larger than the image: one ref row/col
])
def test_edge_geometry(dtype, H, W, b, s, Wn, K):
    rng = np.random.Generator(np.random.PCG64(H + W + b))
    x = synth.random_image(rng, 1, 1, H, W, dtype)
    _compare(x, b, s, Wn, K, dtype, where=f"edge {H}x{W} b{b} s{s} Wn{Wn} K{K}")


@pytest.mark.parametrize("dtype", ["u8", "f32"])
def test_eight_channels(dtype):
    rng = np.random.Generator(np.random.PCG64(88))
    x = synth.random_image(rng, 1, 8, 30, 34, dtype)
    _compare(x, 5, 2, 11, 9, dtype, where="C=8")


def test_saturated_u8_extremes():
    rng = np.random.Generator(np.random.PCG64(9))
    x = (rng.integers(0, 2, size=(1, 1, 48, 48)) * 255).astype(np.uint8)  # max |x-128|
    _compare(x, 16, 2, 13, 32, "u8", where="saturated")


# ------------------------------------------------------------------ API behaviour
def test_rows_band_matches_full():
    cfg = synth.CONFIGS["c1"]
    x = torch.from_numpy(synth.make_input(cfg)).cuda()
    p = _plan(cfg)
    fi, fd = p.run(x)
    bi, bd = p.run_rows(x, 4, 9)
    torch.cuda.synchronize()
    sl = slice(4 * p.nx, 9 * p.nx)
    assert torch.equal(bi[0], fi[0, sl]) and torch.equal(bd[0], fd[0, sl])


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c5"])
def test_host_path_matches_device(name):
    """The pipelined host path (H2D / match / D2H stages: several frames per stage, one frame,
    or reference-row bands of one frame when its table is large -- c3) equals the device run."""
    cfg = synth.CONFIGS[name]
    xn = synth.make_input(cfg, n_frames=5) if name == "c5" else synth.make_input(cfg)
    if name in ("c1", "c2"):
        xn = np.concatenate([xn] * 3)  # several chunks
    p = _plan(cfg)
    di, dd = p.run(torch.from_numpy(xn).cuda())
    hi, hd = p.run_host(torch.from_numpy(xn).pin_memory())
    torch.cuda.synchronize()
    assert torch.equal(hi, di.cpu()) and torch.equal(hd, dd.cpu())


def test_misaligned_pointer_rejected():
    from paper_2006_13714_b200.bm import ScError
    p = _plan((32, 32, 1, 8, 4, 9, 4), "u8")
    buf = torch.zeros(32 * 32 + 16, dtype=torch.uint8, device="cuda")
    x = buf[1:1 + 32 * 32].view(1, 1, 32, 32)
    with pytest.raises(ScError) as e:
        p.run(x)
    assert e.value.code == 1


def test_launch_counter_and_info():
    cfg = synth.CONFIGS["c5"]
    p = _plan(cfg)
    inf = p.info()
    assert inf["n_refs"] == 269 * 479
    assert inf["total_candidates"] * 64 == 8_854_426_816
    assert inf["min_candidates"] == 289 and inf["max_candidates"] == 1089


# ------------------------------------------------------------------ tensor-core kernel
def _tc_cases(n, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    while len(out) < n:
        H = int(rng.integers(8, 90))
        W = int(rng.integers(8, 130))
        s = int(rng.integers(1, 6))
        Wn = int(rng.integers(1, 46))  # TC: Wn^2 <= 2048 (32-bit keys keep >= 21 distance bits)
        K = int(rng.integers(1, 17))  # the TC kernel keeps a 16-key register list per reference
        out.append((H, W, s, Wn, K))
    return out


def _tc_compare(x, s, Wn, K, where):
    from paper_2006_13714_b200.bm import SC_KERNEL_TC_I8
    _compare(x, 8, s, Wn, K, "u8", where=where, kernel=SC_KERNEL_TC_I8)


@pytest.mark.parametrize("case", _tc_cases(20, 303))
def test_tc_random_sweep(case):
    H, W, s, Wn, K = case
    rng = np.random.Generator(np.random.PCG64(hash(case) % (1 << 32)))
    x = synth.random_image(rng, 2, 1, H, W, "u8")
    _tc_compare(x, s, Wn, K, f"tc {case}")


def test_tc_c1_full():
    cfg = synth.CONFIGS["c1"]
    _tc_compare(synth.make_input(cfg), cfg.s, cfg.Wn, cfg.K, "tc c1")


def test_tc_c5_sampled():
    from paper_2006_13714_b200.bm import SC_KERNEL_TC_I8
    cfg = synth.CONFIGS["c5"]
    x = synth.make_input(cfg, n_frames=4)
    p = _plan((cfg.H, cfg.W, 1, 8, cfg.s, cfg.Wn, cfg.K), "u8")
    p.set_kernel(SC_KERNEL_TC_I8)
    gi, gd = _run(p, x)
    ny = p.ny
    for f in (0, 3):
        for r0, r1 in [(0, 3), (ny // 2, ny // 2 + 2), (ny - 3, ny)]:
            oi, od = oracle.bm(x, cfg.b, cfg.s, cfg.Wn, cfg.K, images=(f, f + 1), rows=(r0, r1))
            sl = slice(r0 * p.nx, r1 * p.nx)
            check_u8(gi[f:f + 1, sl], gd[f:f + 1, sl], oi, od, f"tc c5 frame {f} rows {r0}:{r1}")


@pytest.mark.parametrize("kind", ["constant", "periodic", "saturated"])
def test_tc_ties_and_extremes(kind):
    rng = np.random.Generator(np.random.PCG64(11))
    if kind == "constant":
        x = np.full((1, 1, 50, 70), 93, dtype=np.uint8)
    elif kind == "periodic":
        x = np.tile(rng.integers(0, 256, size=(8, 8), dtype=np.uint8), (7, 9))[None, None].copy()
    else:
        x = (rng.integers(0, 2, size=(1, 1, 48, 64)) * 255).astype(np.uint8)
    _tc_compare(x, 3, 21, 16, f"tc {kind}")


def test_tc_rejects_unsupported():
    from paper_2006_13714_b200.bm import SC_KERNEL_TC_I8, ScError
    for args, dt in [((64, 64, 1, 8, 4, 21, 32), "u8"), ((64, 64, 1, 7, 4, 21, 16), "u8"),
                     ((64, 64, 2, 8, 4, 21, 16), "u8"), ((64, 64, 1, 8, 4, 21, 16), "f32")]:
        p = _plan(args, dt)
        with pytest.raises(ScError) as e:
            p.set_kernel(SC_KERNEL_TC_I8)
        assert e.value.code == 2


# ------------------------------------------------------------------ 32-bit register top-K + fix-up
@pytest.mark.parametrize("kernel", ["box", "lanes"])
@pytest.mark.parametrize("kind,Wn,K", [("saturated", 35, 16), ("short", 3, 16), ("short", 5, 30),
                                        ("random", 33, 16), ("random", 41, 32), ("constant", 33, 16)])
def test_r32_keys_and_fixup(kind, Wn, K, kernel):
    """u8, b=8, s=4: the box and lanes kernels keep 32-bit keys (distance field saturating at
    2^21-1 for Wn >= 33) and recompute saturated / short references exactly (fixup.cu)."""
    from paper_2006_13714_b200.bm import SC_KERNEL_BOX, SC_KERNEL_SIMT
    rng = np.random.Generator(np.random.PCG64(31))
    if kind == "saturated":
        x = (rng.integers(0, 2, size=(2, 1, 72, 200)) * 255).astype(np.uint8)
    elif kind == "constant":
        x = np.full((1, 1, 60, 150), 17, dtype=np.uint8)
    else:
        x = rng.integers(0, 256, size=(2, 1, 70, 260), dtype=np.uint8)
    kern = SC_KERNEL_BOX if kernel == "box" else SC_KERNEL_SIMT
    _compare(x, 8, 4, Wn, K, "u8", where=f"r32 {kernel} {kind} Wn{Wn} K{K}", kernel=kern)


# ------------------------------------------------------------------ box-sum kernel (u8, b=8, s=4)
def _box_cases(n, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    while len(out) < n:
        H = int(rng.integers(8, 150))
        W = int(rng.integers(8, 300))  # odd widths: unaligned rows take the byte-load staging path
        Wn = int(rng.integers(1, 46))  # Wn^2 <= 2048: 32-bit keys keep >= 21 distance bits
        K = int(rng.integers(1, 33))
        out.append((H, W, Wn, K))
    return out


def _box(x, Wn, K, where, rows=None):
    from paper_2006_13714_b200.bm import SC_KERNEL_BOX
    _compare(x, 8, 4, Wn, K, "u8", where=where, kernel=SC_KERNEL_BOX)


@pytest.mark.parametrize("case", _box_cases(24, 404))
def test_box_random_sweep(case):
    H, W, Wn, K = case
    rng = np.random.Generator(np.random.PCG64(hash(case) % (1 << 32)))
    x = synth.random_image(rng, 3, 1, H, W, "u8")
    _box(x, Wn, K, f"box {case}")


@pytest.mark.parametrize("kind", ["constant", "periodic", "saturated", "ramp"])
def test_box_ties_and_extremes(kind):
    rng = np.random.Generator(np.random.PCG64(12))
    if kind == "constant":
        x = np.full((1, 1, 70, 150), 93, dtype=np.uint8)
    elif kind == "periodic":
        x = np.tile(rng.integers(0, 256, size=(8, 8), dtype=np.uint8), (9, 19))[None, None].copy()
    elif kind == "saturated":
        x = (rng.integers(0, 2, size=(1, 1, 64, 140)) * 255).astype(np.uint8)
    else:
        x = np.add.outer(np.arange(66), np.arange(170)).astype(np.uint8)[None, None].copy()
    _box(x, 21, 16, f"box {kind}")


def test_box_c1_and_c5_frames():
    from paper_2006_13714_b200.bm import SC_KERNEL_BOX
    _box(synth.make_input(synth.CONFIGS["c1"]), 21, 16, "box c1")
    cfg = synth.CONFIGS["c5"]
    x = synth.make_input(cfg, n_frames=3)
    p = _plan(cfg)
    p.set_kernel(SC_KERNEL_BOX)
    gi, gd = _run(p, x)
    ny = p.ny
    for f in (0, 2):
        for r0, r1 in [(0, 4), (ny // 2 - 1, ny // 2 + 2), (ny - 4, ny)]:
            oi, od = oracle.bm(x, cfg.b, cfg.s, cfg.Wn, cfg.K, images=(f, f + 1), rows=(r0, r1))
            sl = slice(r0 * p.nx, r1 * p.nx)
            check_u8(gi[f:f + 1, sl], gd[f:f + 1, sl], oi, od, f"box c5 frame {f} rows {r0}:{r1}")


def test_box_row_bands():
    from paper_2006_13714_b200.bm import SC_KERNEL_BOX
    rng = np.random.Generator(np.random.PCG64(13))
    x = torch.from_numpy(synth.random_image(rng, 2, 1, 140, 210, "u8")).cuda()
    p = _plan((140, 210, 1, 8, 4, 33, 16), "u8")
    p.set_kernel(SC_KERNEL_BOX)
    fi, fd = p.run(x)
    for r0, r1 in [(0, 1), (3, 20), (17, 34), (30, p.ny)]:
        bi, bd = p.run_rows(x, r0, r1)
        torch.cuda.synchronize()
        sl = slice(r0 * p.nx, r1 * p.nx)
        assert torch.equal(bi, fi[:, sl]) and torch.equal(bd, fd[:, sl]), (r0, r1)


def test_lanes_kernel_c1_c5():
    """The lanes = references kernel stays covered now that the box kernel is the u8 default."""
    from paper_2006_13714_b200.bm import SC_KERNEL_SIMT
    cfg = synth.CONFIGS["c1"]
    _compare(synth.make_input(cfg), 8, 4, 21, 16, "u8", where="lanes c1", kernel=SC_KERNEL_SIMT)
    cfg = synth.CONFIGS["c5"]
    x = synth.make_input(cfg, n_frames=2)
    p = _plan(cfg)
    p.set_kernel(SC_KERNEL_SIMT)
    gi, gd = _run(p, x)
    ny = p.ny
    for r0, r1 in [(0, 2), (ny - 2, ny)]:
        oi, od = oracle.bm(x, cfg.b, cfg.s, cfg.Wn, cfg.K, images=(1, 2), rows=(r0, r1))
        sl = slice(r0 * p.nx, r1 * p.nx)
        check_u8(gi[1:2, sl], gd[1:2, sl], oi, od, f"lanes c5 rows {r0}:{r1}")


def test_box_default_and_rejects_unsupported():
    from paper_2006_13714_b200.bm import SC_KERNEL_BOX, ScError
    assert _plan(synth.CONFIGS["c5"]).info()["kernel"] == SC_KERNEL_BOX
    for args, dt in [((64, 64, 1, 8, 3, 21, 16), "u8"), ((64, 64, 1, 7, 4, 21, 16), "u8"),
                     ((64, 64, 2, 8, 4, 21, 16), "u8"), ((64, 64, 1, 8, 4, 21, 33), "u8"),
                     ((64, 64, 1, 8, 4, 47, 16), "u8"), ((64, 64, 1, 8, 4, 21, 16), "f32")]:
        p = _plan(args, dt)
        with pytest.raises(ScError) as e:
            p.set_kernel(SC_KERNEL_BOX)
        assert e.value.code == 2


# ------------------------------------------------------------------ float box-sum kernel
def _boxf_fits(s, b, Wn, K, C=1):
    """Mirror of boxf_supported's shared-memory / key-width rule (bm_boxf.cu)."""
    ns = -(-b // s)
    kp = K + (8 if K > 48 else 4)  # plan.cpp's re-rank margin
    kr = next((r for r in (24, 32, 40, 48, 80) if kp <= r), 0)
    rb = max(1, (Wn * Wn).bit_length())
    if kr == 0 or rb > 12:
        return False
    nblk = -(-Wn // 8)
    pl = (7 * s + nblk * 8 + b) * (32 * s + Wn)
    hp = ((kp + 3) & ~3) + 2
    scr = 512 + (33 - ns) * hp if kr == 80 else max(512, (33 - ns) * (kr + 1))
    return (((C * pl + 1) & ~1) + 8 * scr) * 4 <= 227 * 1024


def _boxf_cases(n, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    shapes = [(3, 8), (1, 7), (4, 8), (2, 8)]
    out = []
    while len(out) < n:
        s, b = shapes[len(out) % len(shapes)]
        H = int(rng.integers(b, 110))
        W = int(rng.integers(b, 160))
        Wn = int(rng.integers(1, 64))
        K = int(rng.integers(1, 73))
        C = int(rng.choice([1, 1, 2, 4]))
        if ((H - b) // s + 1) * ((W - b) // s + 1) * Wn * Wn * C > 4e7 or not _boxf_fits(s, b, Wn, K, C):
            continue
        out.append((s, b, C, H, W, Wn, K))
    return out


def _boxf(x, b, s, Wn, K, where):
    from paper_2006_13714_b200.bm import SC_KERNEL_BOXF
    _compare(x, b, s, Wn, K, "f32", where=where, kernel=SC_KERNEL_BOXF)


@pytest.mark.parametrize("case", _boxf_cases(24, 505))
def test_boxf_random_sweep(case):
    s, b, C, H, W, Wn, K = case
    rng = np.random.Generator(np.random.PCG64(hash(case) % (1 << 32)))
    x = synth.random_image(rng, 2, C, H, W, "f32")
    _boxf(x, b, s, Wn, K, f"boxf {case}")


@pytest.mark.parametrize("kind", ["constant", "periodic", "binary", "smooth"])
@pytest.mark.parametrize("s,b", [(3, 8), (1, 7)])
def test_boxf_ties_and_extremes(kind, s, b):
    rng = np.random.Generator(np.random.PCG64(14))
    if kind == "constant":
        x = np.full((1, 1, 60, 90), 0.3, dtype=np.float32)
    elif kind == "periodic":
        x = np.tile(rng.random((8, 8), dtype=np.float32), (8, 12))[None, None].copy()
    elif kind == "binary":
        x = rng.integers(0, 2, size=(1, 1, 60, 90)).astype(np.float32)
    else:
        yy, xx = np.mgrid[0:64, 0:96]
        x = (0.5 + 0.4 * np.sin(yy / 7.0) * np.cos(xx / 9.0)).astype(np.float32)[None, None].copy()
    _boxf(x, b, s, 21, 30, f"boxf {kind} s{s} b{b}")


def test_boxf_default_and_rejects_unsupported():
    from paper_2006_13714_b200.bm import SC_KERNEL_BOXF, ScError
    from paper_2006_13714_b200.bm import SC_KERNEL_TC_F32
    for name in ("c2", "c4"):
        assert _plan(synth.CONFIGS[name]).info()["kernel"] == SC_KERNEL_BOXF
    assert _plan(synth.CONFIGS["c3"]).info()["kernel"] == SC_KERNEL_TC_F32  # stride 1: tensor cores
    for args, dt in [((64, 64, 1, 8, 5, 21, 16), "f32"), ((64, 64, 8, 8, 3, 41, 32), "f32"),
                     ((64, 64, 1, 8, 3, 21, 80), "f32"), ((64, 64, 1, 8, 3, 21, 16), "u8")]:
        p = _plan(args, dt)
        with pytest.raises(ScError) as e:
            p.set_kernel(SC_KERNEL_BOXF)
        assert e.value.code == 2


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_warp_kernel_sampled_rows(name):
    """The warp kernel stays covered on c3/c4 now that the float box kernel is their default."""
    from paper_2006_13714_b200.bm import SC_KERNEL_SIMT_WARP
    cfg = synth.CONFIGS[name]
    x = synth.make_input(cfg)
    p = _plan(cfg)
    p.set_kernel(SC_KERNEL_SIMT_WARP)
    gi, gd = _run(p, x)
    for r0, r1 in [(0, 2), (p.ny - 2, p.ny)]:
        oi, od = oracle.bm(x, cfg.b, cfg.s, cfg.Wn, cfg.K, rows=(r0, r1))
        sl = slice(r0 * p.nx, r1 * p.nx)
        check_f32(x[0], cfg.b, cfg.s, cfg.Wn, cfg.K, gi[0, sl], gd[0, sl], oi[0], od[0],
                  iy_range=(r0, r1), where=f"warp {name} rows {r0}:{r1}")


# ------------------------------------------------------------------ patch grouping Y_i
@pytest.mark.parametrize("dtype,C,H,W,b,s,Wn,K", [("u8", 1, 64, 64, 8, 4, 21, 16), ("f32", 2, 37, 45, 7, 2, 11, 9),
                                                   ("u8", 3, 30, 41, 5, 3, 9, 12), ("f32", 1, 40, 40, 8, 3, 39, 30)])
def test_group_matches_oracle(dtype, C, H, W, b, s, Wn, K):
    rng = np.random.Generator(np.random.PCG64(H * W + K))
    x = synth.random_image(rng, 2, C, H, W, dtype)
    p = _plan((H, W, C, b, s, Wn, K), dtype)
    t = torch.from_numpy(x).cuda()
    idx, _ = p.run(t)
    if Wn * Wn < K:  # exercise the -1 padding path explicitly
        assert (idx == -1).any()
    Y = p.group(t, idx)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(Y.cpu().numpy(), oracle.group(x, idx.cpu().numpy(), b))


@pytest.mark.parametrize("dtype,b", [("u8", 8), ("f32", 8), ("f32", 7), ("u8", 5)])
def test_group_arbitrary_idx(dtype, b):
    # idx not produced by a search (any patch of the image, -1 holes): the staged gather must fall
    # back to global reads for candidates outside a tile's windows; ragged tiles in both directions
    # (f32 b = 7: the element-pair stores; u8 b = 5: single elements)
    H, W, C, s, Wn, K = 150, 203, 2, 4, 9, 8
    rng = np.random.Generator(np.random.PCG64(11))
    x = synth.random_image(rng, 3, C, H, W, dtype)
    p = _plan((H, W, C, b, s, Wn, K), dtype)
    cy = rng.integers(0, H - b + 1, (3, p.n_refs, K))
    cx = rng.integers(0, W - b + 1, (3, p.n_refs, K))
    ii = (cy * W + cx).astype(np.int32)
    ii[rng.random(ii.shape) < 0.1] = -1
    t = torch.from_numpy(x).cuda()
    Y = p.group(t, torch.from_numpy(ii).cuda())
    np.testing.assert_array_equal(Y.cpu().numpy(), oracle.group(x, ii, b))


def test_group_padding_and_c5_sample():
    # K > window candidates: -1 entries -> zero columns
    rng = np.random.Generator(np.random.PCG64(3))
    x = synth.random_image(rng, 1, 1, 20, 24, "u8")
    p = _plan((20, 24, 1, 4, 2, 3, 12), "u8")
    t = torch.from_numpy(x).cuda()
    idx, _ = p.run(t)
    assert (idx == -1).any()
    np.testing.assert_array_equal(p.group(t, idx).cpu().numpy(), oracle.group(x, idx.cpu().numpy(), 4))
    # c5 (bench configuration, 64 frames in one call): sampled references of frames 0 and 63
    cfg = synth.CONFIGS["c5"]
    xs = synth.make_input(cfg)
    p = _plan(cfg)
    t = torch.from_numpy(xs).cuda()
    idx, _ = p.run(t)
    Y = p.group(t, idx)
    sel = np.random.Generator(np.random.PCG64(5)).choice(p.n_refs, 300, replace=False)
    for f in (0, 63):
        ii = idx[f:f + 1, sel].cpu().numpy()
        np.testing.assert_array_equal(Y[f:f + 1, sel].cpu().numpy(), oracle.group(xs[f:f + 1], ii, cfg.b))


# ------------------------------------------------------------------ NCC metric (Eq. 4)
def _ncc_run(x, b, s, Wn, K, dtype):
    from paper_2006_13714_b200.bm import Plan
    N, C, H, W = x.shape
    p = Plan(H, W, C, b, s, Wn, K, dtype, metric="ncc")
    gi, gd = _run(p, x)
    return p, gi, gd


def _ncc_cases(n, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    shapes = [(4, 8), (3, 8), (1, 7), (2, 8)]
    out = []
    while len(out) < n:
        s, b = shapes[len(out) % 4]
        H, W = int(rng.integers(b, 90)), int(rng.integers(b, 130))
        Wn, K = int(rng.integers(1, 46)), int(rng.integers(1, 25))
        C = int(rng.choice([1, 1, 3]))
        dtype = ["u8", "f32"][len(out) % 2]
        if ((H - b) // s + 1) * ((W - b) // s + 1) * Wn * Wn * C > 2e7:
            continue
        out.append((dtype, s, b, C, H, W, Wn, K))
    return out


@pytest.mark.parametrize("case", _ncc_cases(16, 606))
def test_ncc_random_sweep(case):
    from tests.parity import check_ncc
    dtype, s, b, C, H, W, Wn, K = case
    rng = np.random.Generator(np.random.PCG64(hash(case) % (1 << 32)))
    x = synth.random_image(rng, 2, C, H, W, dtype)
    p, gi, gd = _ncc_run(x, b, s, Wn, K, dtype)
    oi, od = oracle.ncc(x, b, s, Wn, K)
    for n in range(2):
        check_ncc(x[n], b, s, Wn, K, gi[n], gd[n], oi[n], od[n], exact=dtype == "u8", where=f"ncc {case} img{n}")


@pytest.mark.parametrize("kind", ["zeros", "constant", "periodic", "scaled", "near_scaled"])
def test_ncc_ties_and_degenerate(kind):
    """Zero-norm patches (NCC := 0), all-ties images, periodic tilings, exact scaled copies and
    rounded near-scaled copies (NCC within rounding of 1): the exact uint8 ordering must reproduce
    the oracle's tie-breaks; references whose quantised keys cannot decide go to the fix-up."""
    from tests.parity import check_ncc
    rng = np.random.Generator(np.random.PCG64(15))
    if kind == "zeros":
        x = rng.integers(0, 256, size=(1, 1, 48, 70), dtype=np.uint8)
        x[:, :, 10:30, 20:50] = 0
    elif kind == "constant":
        x = np.full((1, 1, 48, 70), 77, dtype=np.uint8)
    elif kind == "periodic":
        x = np.tile(rng.integers(0, 256, size=(8, 8), dtype=np.uint8), (6, 9))[None, None].copy()
    elif kind == "scaled":
        base = rng.integers(1, 64, size=(48, 35), dtype=np.uint8)
        x = np.concatenate([base, base * 2], axis=1)[None, None].copy()
    else:
        tile = rng.integers(60, 200, size=(8, 8)).astype(np.float64)
        gains = rng.uniform(0.9, 1.1, size=(6, 9))
        x = np.clip(np.round(np.kron(gains, np.ones((8, 8))) * np.tile(tile, (6, 9))), 0, 255)
        x = x.astype(np.uint8)[None, None].copy()
    p, gi, gd = _ncc_run(x, 8, 4, 21, 16, "u8")
    oi, od = oracle.ncc(x, 8, 4, 21, 16)
    check_ncc(x[0], 8, 4, 21, 16, gi[0], gd[0], oi[0], od[0], exact=True, where=f"ncc {kind}")
    from paper_2006_13714_b200.bm import SC_KERNEL_BOX
    p.set_kernel(SC_KERNEL_BOX)  # the dp4a kernel and its fix-up (small images default to the float kernel)
    gi, gd = _run(p, x)
    check_ncc(x[0], 8, 4, 21, 16, gi[0], gd[0], oi[0], od[0], exact=True, where=f"ncc {kind} box")
    if kind == "constant":  # every candidate ties at NCC = 1: the float keys cannot order them
        assert p.debug_fix_count() > 0


@pytest.mark.parametrize("metric", ["l2", "ncc"])
def test_boxf_quantised_key_fixup(metric):
    """The float box kernel's 32-bit keys quantise the score (~1e-4 relative): on a constant image
    every candidate ties, the worst kept key cannot separate the K-th candidate from dropped ones,
    so every reference goes to the exact fix-up -- whose output must still satisfy the parity rule;
    a tiny-noise image mixes flagged and unflagged references."""
    from paper_2006_13714_b200.bm import SC_KERNEL_BOXF, Plan
    from tests.parity import check_ncc
    H, W, b, s, Wn, K = 40, 56, 8, 3, 15, 12
    rng = np.random.Generator(np.random.PCG64(21))
    for kind in ("constant", "tiny_noise"):
        x = np.full((1, 1, H, W), 0.5 if metric == "l2" else 0.7, dtype=np.float32)
        if kind == "tiny_noise":
            x += (rng.standard_normal(x.shape) * 1e-3).astype(np.float32)
        p = Plan(H, W, 1, b, s, Wn, K, "f32", metric=metric)
        p.set_kernel(SC_KERNEL_BOXF)
        gi, gd = _run(p, x)
        if kind == "constant":
            assert p.debug_fix_count() == p.n_refs
        if metric == "l2":
            oi, od = oracle.bm(x, b, s, Wn, K)
            check_f32(x[0], b, s, Wn, K, gi[0], gd[0], oi[0], od[0], where=f"boxf fixup {kind}")
        else:
            oi, od = oracle.ncc(x, b, s, Wn, K)
            check_ncc(x[0], b, s, Wn, K, gi[0], gd[0], oi[0], od[0], exact=False, where=f"boxf ncc fixup {kind}")


def test_ncc_configs_and_rejects():
    """c5 frames (u8, exact) and c2 (f32) with the NCC metric; unsupported geometry is refused."""
    from paper_2006_13714_b200.bm import Plan, ScError
    from tests.parity import check_ncc
    from paper_2006_13714_b200.bm import SC_KERNEL_BOX
    cfg = synth.CONFIGS["c5"]
    x = synth.make_input(cfg, n_frames=2)
    p, gi, gd = _ncc_run(x, cfg.b, cfg.s, cfg.Wn, cfg.K, "u8")
    assert p.info()["kernel"] == SC_KERNEL_BOX
    for r0, r1 in [(0, 2), (p.ny - 2, p.ny)]:
        oi, od = oracle.ncc(x, cfg.b, cfg.s, cfg.Wn, cfg.K, images=(1, 2), rows=(r0, r1))
        sl = slice(r0 * p.nx, r1 * p.nx)
        check_ncc(x[1], cfg.b, cfg.s, cfg.Wn, cfg.K, gi[1, sl], gd[1, sl], oi[0], od[0], exact=True,
                  where=f"ncc c5 rows {r0}:{r1}")
    cfg = synth.CONFIGS["c2"]
    x = synth.make_input(cfg)
    p, gi, gd = _ncc_run(x, cfg.b, cfg.s, cfg.Wn, cfg.K, "f32")
    oi, od = oracle.ncc(x, cfg.b, cfg.s, cfg.Wn, cfg.K, rows=(80, 83))
    sl = slice(80 * p.nx, 83 * p.nx)
    check_ncc(x[0], cfg.b, cfg.s, cfg.Wn, cfg.K, gi[0, sl], gd[0, sl], oi[0], od[0], exact=False,
              iy_range=(80, 83), where="ncc c2")
    for args in [(64, 64, 1, 8, 5, 21, 16), (64, 64, 1, 8, 4, 21, 31)]:
        with pytest.raises(ScError) as e:
            Plan(*args, "u8", metric="ncc")
        assert e.value.code == 2


@pytest.mark.parametrize("kernel", ["box", "boxf"])
def test_ncc_u8_both_kernels(kernel):
    """uint8 stride-4 NCC on the dp4a box kernel (default) and on the float box kernel."""
    from paper_2006_13714_b200.bm import SC_KERNEL_BOX, SC_KERNEL_BOXF, Plan
    from tests.parity import check_ncc
    rng = np.random.Generator(np.random.PCG64(16))
    x = synth.random_image(rng, 2, 1, 90, 160, "u8")
    p = Plan(90, 160, 1, 8, 4, 25, 20, "u8", metric="ncc")
    p.set_kernel(SC_KERNEL_BOX if kernel == "box" else SC_KERNEL_BOXF)
    gi, gd = _run(p, x)
    oi, od = oracle.ncc(x, 8, 4, 25, 20)
    for n in range(2):
        check_ncc(x[n], 8, 4, 25, 20, gi[n], gd[n], oi[n], od[n], exact=True, where=f"ncc {kernel} img{n}")


@pytest.mark.parametrize("Wn,K", [(14, 4), (15, 2), (21, 8), (12, 12), (33, 28)])
def test_ncc_box_small_lists(Wn, K):
    """The dp4a NCC kernel's list sizes for every window-block geometry (VY 7 / 8 / 11): the
    shared-memory layout must match the instantiated list length (found by tools/stress.py)."""
    from paper_2006_13714_b200.bm import SC_KERNEL_BOX, Plan
    from tests.parity import check_ncc
    rng = np.random.Generator(np.random.PCG64(Wn * 100 + K))
    x = synth.random_image(rng, 2, 1, 55, 120, "u8")
    p = Plan(55, 120, 1, 8, 4, Wn, K, "u8", metric="ncc")
    p.set_kernel(SC_KERNEL_BOX)
    gi, gd = _run(p, x)
    oi, od = oracle.ncc(x, 8, 4, Wn, K)
    for n in range(2):
        check_ncc(x[n], 8, 4, Wn, K, gi[n], gd[n], oi[n], od[n], exact=True, where=f"ncc box Wn{Wn} K{K} img{n}")


# ------------------------------------------------------------------ NLM weights (Eq. 2 / Prop. 1)
@pytest.mark.parametrize("dtype,C,H,W,b,s,Wn,h", [("u8", 1, 64, 64, 8, 4, 21, 300.0), ("u8", 1, 50, 77, 5, 2, 13, 120.0),
                                                   ("f32", 1, 48, 52, 7, 2, 15, 0.6), ("f32", 3, 30, 41, 4, 3, 9, 0.5),
                                                   ("u8", 2, 40, 40, 8, 3, 17, 1e6)])
@pytest.mark.parametrize("kernel", ["default", "lanes"])
def test_nlm_weights_match_oracle(dtype, C, H, W, b, s, Wn, h, kernel):
    """default: the one-warp-per-reference dense matcher with the fused normalisation epilogue;
    lanes: the lanes dense matcher followed by the stand-alone nlm_normalize kernel."""
    from paper_2006_13714_b200.bm import SC_KERNEL_SIMT
    rng = np.random.Generator(np.random.PCG64(H + W + b + C))
    x = synth.random_image(rng, 1, C, H, W, dtype)[0]
    p = _plan((H, W, C, b, s, Wn, 1), dtype)
    if kernel == "lanes":
        p.set_kernel(SC_KERNEL_SIMT)
    got = p.nlm_weights(torch.from_numpy(x).cuda(), h).cpu().numpy().astype(np.float64)
    want = oracle.nlm_weights(x, b, s, Wn, h)
    np.testing.assert_allclose(got.sum(1), 1.0, rtol=2e-5)
    assert (got[want == 0] == 0).all()  # clipped slots (float32 may also underflow tiny weights to 0)
    # float32 weights of the identity distances: relative 1e-4 on weights above 1e-6 of the row
    m = want > 1e-6
    np.testing.assert_allclose(got[m], want[m], rtol=1e-4, atol=1e-9)


def test_nlm_c2_full_image():
    cfg = synth.CONFIGS["c2"]
    x = synth.make_input(cfg)[0]
    p = _plan(cfg)
    h = 25.0 / 255.0 * 8  # a sigma-scaled bandwidth for the 8x8 noisy patches
    got = p.nlm_weights(torch.from_numpy(x).cuda(), h).cpu().numpy().astype(np.float64)
    want = oracle.nlm_weights(x, cfg.b, cfg.s, cfg.Wn, h)
    m = want > 1e-6
    np.testing.assert_allclose(got[m], want[m], rtol=1e-4, atol=1e-9)


@pytest.mark.parametrize("dtype,C,H,W,b,s,Wn,h", [("u8", 1, 64, 64, 8, 4, 21, 300.0), ("f32", 1, 48, 52, 7, 2, 15, 0.6),
                                                   ("f32", 3, 30, 41, 4, 3, 9, 0.5), ("u8", 2, 40, 40, 8, 3, 17, 1e6),
                                                   ("u8", 1, 33, 47, 5, 1, 11, 60.0), ("f32", 4, 36, 36, 8, 3, 13, 0.3)])
def test_nlm_average_matches_oracle(dtype, C, H, W, b, s, Wn, h):
    """The fused NL-means estimate (no weight table): float32 identity distances and weights,
    so relative 1e-4 of the image's value range; h -> inf gives the window mean, h -> 0 the
    reference patch."""
    rng = np.random.Generator(np.random.PCG64(H * W + C))
    x = synth.random_image(rng, 1, C, H, W, dtype)[0]
    p = _plan((H, W, C, b, s, Wn, 1), dtype)
    t = torch.from_numpy(x).cuda()
    scale = 255.0 if dtype == "u8" else 1.0
    for hh in (h, 1e12, 1e-3 * scale):
        got = p.nlm_average(t, hh).cpu().numpy().astype(np.float64)
        want = oracle.nlm_average(x, b, s, Wn, hh)
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-4 * scale, err_msg=f"h={hh}")


def test_nlm_average_c2_sampled_and_rejects():
    from paper_2006_13714_b200.bm import Plan, ScError
    cfg = synth.CONFIGS["c2"]
    x = synth.make_input(cfg)[0]
    p = _plan(cfg)
    h = 25.0 / 255.0 * 8
    got = p.nlm_average(torch.from_numpy(x).cuda(), h).cpu().numpy().astype(np.float64)
    sel = list(np.random.Generator(np.random.PCG64(9)).choice(p.n_refs, 40, replace=False))
    want = oracle.nlm_average(x, cfg.b, cfg.s, cfg.Wn, h, refs=sel)
    np.testing.assert_allclose(got[sel], want, rtol=0, atol=1e-4)
    with pytest.raises(ScError):  # b^2 C > 256
        Plan(40, 40, 8, 8, 4, 9, 4, "f32").nlm_average(torch.zeros((8, 40, 40), device="cuda"), 1.0)
    with pytest.raises(ScError):  # NCC plans
        Plan(40, 40, 1, 8, 4, 9, 4, "u8", metric="ncc").nlm_average(
            torch.zeros((1, 40, 40), dtype=torch.uint8, device="cuda"), 1.0)


# ------------------------------------------------------------------ 3D / temporal search
@pytest.mark.parametrize("N,H,W,Wn,K,T", [(4, 70, 150, 21, 16, 1), (5, 60, 97, 15, 12, 2), (3, 90, 130, 33, 16, 1),
                                          (2, 40, 64, 9, 32, 1), (6, 48, 80, 13, 8, 3)])
def test_temporal_matches_oracle(N, H, W, Wn, K, T):
    rng = np.random.Generator(np.random.PCG64(N * H + W + T))
    x = synth.random_image(rng, N, 1, H, W, "u8")
    p = _plan((H, W, 1, 8, 4, Wn, K), "u8")
    p.set_temporal(T)
    gi, gd = _run(p, x)
    oi, od = oracle.bm_temporal(x, 8, 4, Wn, K, T)
    check_u8(gi, gd, oi, od, f"temporal N{N} {H}x{W} Wn{Wn} K{K} T{T}")


def test_group_temporal_idx():
    # a 3D / temporal run's idx is batch-global (frame * H * W + pixel); for C = 1 that is the pixel
    # index of the frames stacked vertically, so the oracle groups the stacked image
    N, H, W = 4, 52, 75
    rng = np.random.Generator(np.random.PCG64(17))
    x = synth.random_image(rng, N, 1, H, W, "u8")
    p = _plan((H, W, 1, 8, 4, 15, 12), "u8")
    p.set_temporal(1)
    t = torch.from_numpy(x).cuda()
    idx, _ = p.run(t)
    ii = idx.cpu().numpy()
    assert (ii // (H * W) != np.arange(N)[:, None, None]).any()  # some matches in neighbouring frames
    Y = p.group(t, idx).cpu().numpy()
    ref = oracle.group(x.reshape(1, 1, N * H, W), ii.reshape(1, -1, 12), 8)
    np.testing.assert_array_equal(Y.reshape(ref.shape), ref)


def test_run_temporal_frame_ranges():
    """sc_bm_run_temporal: references of frames [f_begin, f_end) of a batch, candidates from all of
    it, idx offset by frame_offset -- the per-rank call of the sharded temporal search on its
    halo-extended buffer (emulated here by slicing the video: the exchange itself is tested with
    gloo in test_dist_cpu.py); a saturated video exercises the offset in the fix-up."""
    from paper_2006_13714_b200 import dist as sdist
    from paper_2006_13714_b200.bm import ScError
    rng = np.random.Generator(np.random.PCG64(29))
    N, H, W, Wn, K, T = 7, 60, 97, 15, 12, 2
    for kind in ("random", "saturated"):
        if kind == "random":
            x = synth.random_image(rng, N, 1, H, W, "u8")
        else:
            x = (rng.integers(0, 2, size=(N, 1, H, W)) * 255).astype(np.uint8)
        oi, od = oracle.bm_temporal(x, 8, 4, Wn, K, T)
        p = _plan((H, W, 1, 8, 4, Wn, K), "u8")
        p.set_temporal(T)
        t = torch.from_numpy(x).cuda()
        for world in (2, 3):
            for r in range(world):
                a, b = sdist.frame_shard(N, r, world)
                lo_, hi_ = max(0, a - T), min(N, b + T)  # what the halo exchange assembles
                gi, gd = p.run_temporal(t[lo_:hi_].clone(), a - lo_, b - lo_, lo_)  # a fresh (aligned) buffer
                torch.cuda.synchronize()
                np.testing.assert_array_equal(gi.cpu().numpy(), oi[a:b], err_msg=f"{kind} world {world} rank {r}")
                np.testing.assert_array_equal(gd.cpu().numpy(), od[a:b])
    with pytest.raises(ScError):
        _plan((H, W, 1, 8, 4, Wn, K), "u8").run_temporal(t, 0, 2)  # T = 0


def test_temporal_c5_frames_and_saturation():
    """The c5 video (random-walk crops): every reference's K best over frames f-1..f+1, bit-exact
    on sampled rows; a saturated video exercises the temporal fix-up."""
    cfg = synth.CONFIGS["c5"]
    x = synth.make_input(cfg, n_frames=3)
    p = _plan(cfg)
    p.set_temporal(1)
    gi, gd = _run(p, x)
    oi, od = oracle.bm_temporal(x[:, :, :64, :], cfg.b, cfg.s, cfg.Wn, cfg.K, 1)  # rows whose windows stay in 64 rows
    nx = p.nx
    for f in range(3):
        for r in range(3):  # reference rows 0..2 of the crop see the same candidates as in the full frame
            sl = slice(r * nx, (r + 1) * nx)
            go = gi[f, sl].copy()
            fr, pix = go // (cfg.H * cfg.W), go % (cfg.H * cfg.W)
            remap = fr * (64 * cfg.W) + pix  # batch-global idx of the 64-row crop
            np.testing.assert_array_equal(remap, oi[f, sl])
            np.testing.assert_array_equal(gd[f, sl], od[f, sl])
    rng = np.random.Generator(np.random.PCG64(3))
    xs = (rng.integers(0, 2, size=(3, 1, 48, 96)) * 255).astype(np.uint8)
    p = _plan((48, 96, 1, 8, 4, 21, 16), "u8")
    p.set_temporal(1)
    gi, gd = _run(p, xs)
    oi, od = oracle.bm_temporal(xs, 8, 4, 21, 16, 1)
    check_u8(gi, gd, oi, od, "temporal saturated")


def test_temporal_rejects():
    from paper_2006_13714_b200.bm import ScError
    for args, dt, T in [((64, 64, 1, 8, 3, 21, 16), "u8", 1), ((64, 64, 1, 8, 4, 33, 16), "u8", 2),
                        ((64, 64, 1, 8, 4, 21, 16), "f32", 1)]:
        p = _plan(args, dt)
        with pytest.raises(ScError) as e:
            p.set_temporal(T)
        assert e.value.code == 2


def test_temporal_row_bands_match_full_run():
    """Row bands (the multi-GPU spatial split) with temporal search = the matching rows of the full run."""
    rng = np.random.Generator(np.random.PCG64(17))
    x = torch.from_numpy(synth.random_image(rng, 3, 1, 96, 150, "u8")).cuda()
    p = _plan((96, 150, 1, 8, 4, 21, 16), "u8")
    p.set_temporal(1)
    fi, fd = p.run(x)
    for r0, r1 in [(0, 3), (5, 17), (20, p.ny)]:
        bi, bd = p.run_rows(x, r0, r1)
        torch.cuda.synchronize()
        sl = slice(r0 * p.nx, r1 * p.nx)
        assert torch.equal(bi, fi[:, sl]) and torch.equal(bd, fd[:, sl]), (r0, r1)


# ------------------------------------------------------------------ CUDA-graph capture
@pytest.mark.parametrize("cfg_name", ["c1", "c2", "c5"])
def test_run_is_graph_capturable(cfg_name):
    """sc_bm_run* never allocates or synchronises: one step captured into a CUDA graph and
    replayed on new input equals the eager run (box / float box / warp matchers + fix-up)."""
    cfg = synth.CONFIGS[cfg_name]
    n = 2 if cfg_name == "c5" else cfg.N
    x = torch.from_numpy(synth.make_input(cfg, n_frames=n) if cfg_name == "c5" else synth.make_input(cfg)).cuda()
    p = _plan(cfg)
    idx, dist = p.alloc_out(x.shape[0])
    xin = torch.empty_like(x)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        p.run(xin.copy_(x), out=(idx, dist), stream=s)  # warm-up outside the capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        p.run(xin, out=(idx, dist), stream=s)
    y = torch.flip(x, dims=[-1]).contiguous()  # a different input for the replay
    xin.copy_(y)
    g.replay()
    torch.cuda.synchronize()
    wi, wd = p.run(y)
    torch.cuda.synchronize()
    assert torch.equal(idx, wi) and torch.equal(dist, wd)


def test_batch_larger_than_one_launch():
    """More frames than one box-kernel launch takes (FB = 64): the chunked run (64 + 3 frames, the
    second chunk's fix-up list and output offsets) equals per-frame runs."""
    rng = np.random.Generator(np.random.PCG64(41))
    N, H, W = 67, 96, 160
    x = synth.random_image(rng, N, 1, H, W, "u8")
    x[N - 1] = (rng.integers(0, 2, size=(1, H, W)) * 255).astype(np.uint8)  # saturating: fix-up in chunk 2
    p = _plan((H, W, 1, 8, 4, 33, 16), "u8")
    t = torch.from_numpy(x).cuda()
    gi, gd = p.run(t)
    for f in (0, 63, 64, 65, 66):
        fi, fd = p.run(t[f:f + 1].clone())
        assert torch.equal(gi[f], fi[0]) and torch.equal(gd[f], fd[0]), f
    oi, od = oracle.bm(x, 8, 4, 33, 16, images=(N - 1, N))
    check_u8(gi[N - 1:].cpu().numpy(), gd[N - 1:].cpu().numpy(), oi, od, "saturated frame in the second chunk")


def test_next_rows_argument_validation():
    """Synchronous argument checks of the next rows' entry points (SC_ERR_INVALID_ARGUMENT = 1,
    SC_ERR_UNSUPPORTED = 2): nothing is launched for a rejected call."""
    from paper_2006_13714_b200.bm import Plan, ScError
    p = Plan(64, 96, 1, 8, 4, 15, 8, "u8")
    x = torch.zeros((3, 1, 64, 96), dtype=torch.uint8, device="cuda")
    with pytest.raises(ScError) as e:
        p.run_temporal(x, 0, 2)  # T = 0
    assert e.value.code == 2
    p.set_temporal(1)
    for args, kw in [((x, 2, 4), {}), ((x, 2, 1), {}), ((x, -1, 2), {}), ((x, 0, 2), {"frame_offset": -1})]:
        with pytest.raises(ScError) as e:
            p.run_temporal(*args, **kw)
        assert e.value.code == 1, (args, kw)
    with pytest.raises(ScError) as e:
        p.nlm_weights(x[0], 0.0)
    assert e.value.code == 1
    with pytest.raises(ScError) as e:
        p.nlm_average(x[0], -1.0)
    assert e.value.code == 1
    q = Plan(64, 96, 1, 8, 4, 15, 8, "u8", metric="ncc")
    with pytest.raises(ScError) as e:
        q.set_temporal(1)  # temporal search is L2-only
    assert e.value.code == 2
    idx, _ = Plan(64, 96, 1, 8, 4, 15, 8, "u8").run(x)
    buf = torch.empty(idx.numel() * 64 + 16, dtype=torch.uint8, device="cuda")
    with pytest.raises(ScError) as e:  # misaligned groups_out
        Plan(64, 96, 1, 8, 4, 15, 8, "u8").group(x, idx, out=buf[1:1 + idx.numel() * 64].view(3, -1, 8, 1, 8, 8))
    assert e.value.code == 1


# ------------------------------------------------------------------ round-2 API fixes
@pytest.mark.parametrize("kernel", ["default", "lanes"])
def test_nlm_weights_unnormalised_scale(kernel):
    """Float images on the 0..255 scale: fp32 identity distances of real candidates can round
    below -0.5; clipped slots are decided from the window geometry, so every real candidate
    (the reference itself included) keeps its weight."""
    from paper_2006_13714_b200.bm import SC_KERNEL_SIMT
    rng = np.random.Generator(np.random.PCG64(2024))
    x = (rng.random((1, 40, 44)) * 255.0).astype(np.float32)
    b, s, Wn = 8, 3, 13
    h = 8.0 * 255.0 * 0.3
    p = _plan((40, 44, 1, b, s, Wn, 1), "f32")
    if kernel == "lanes":
        p.set_kernel(SC_KERNEL_SIMT)
    got = p.nlm_weights(torch.from_numpy(x).cuda(), h).cpu().numpy().astype(np.float64)
    want = oracle.nlm_weights(x, b, s, Wn, h)
    np.testing.assert_allclose(got.sum(1), 1.0, rtol=2e-5)
    np.testing.assert_array_equal(got == 0, want == 0)
    m = want > 1e-6
    np.testing.assert_allclose(got[m], want[m], rtol=2e-3, atol=1e-9)


def test_set_temporal_zero_restores_kernel():
    from paper_2006_13714_b200.bm import SC_KERNEL_BOX, SC_KERNEL_SIMT_WARP
    p = _plan((72, 160, 1, 8, 4, 33, 16), "u8")
    p.set_kernel(SC_KERNEL_SIMT_WARP)
    p.set_temporal(1)
    assert p.info()["kernel"] == SC_KERNEL_BOX
    p.set_temporal(0)
    assert p.info()["kernel"] == SC_KERNEL_SIMT_WARP
    q = _plan((72, 160, 1, 8, 4, 33, 16), "u8")
    k0 = q.info()["kernel"]
    q.set_temporal(1)
    q.set_temporal(0)
    assert q.info()["kernel"] == k0


def test_run_host_validates_buffers():
    p = _plan((40, 48, 1, 8, 4, 9, 4), "f32")
    xu = np.zeros((1, 1, 40, 48), dtype=np.uint8)
    with pytest.raises(ValueError):
        p.run_host(xu)  # wrong dtype: would read 4x past the buffer
    with pytest.raises(ValueError):
        p.run_host(np.zeros((1, 1, 40, 47), dtype=np.float32))  # wrong shape
    x = np.zeros((2, 1, 40, 48), dtype=np.float32)
    bad = (torch.empty((1, p.n_refs, 4), dtype=torch.int32), torch.empty((1, p.n_refs, 4), dtype=torch.float32))
    with pytest.raises(ValueError):
        p.run_host(x, out=bad)  # output tables for one image, two given
    with pytest.raises(ValueError):
        p.run(torch.from_numpy(x).cuda(), out=tuple(t.cuda() for t in bad))


def test_temporal_batch_idx_range_checked():
    """Batch-global temporal idx (frame * H * W + pixel) must stay int32: the C ABI refuses a
    sc_bm_run_batch / sc_bm_run_rows batch that would overflow it (SC_ERR_INVALID_ARGUMENT)."""
    from paper_2006_13714_b200.bm import ScError
    p = _plan((1080, 1920, 1, 8, 4, 33, 16), "u8")
    p.set_temporal(1)
    n = (1 << 31) // (1080 * 1920) + 1
    x = torch.empty((n, 1, 1080, 1920), dtype=torch.uint8, device="cuda")  # 2.1 GB, never read
    out = p.alloc_out(n, rows=(0, 1))
    with pytest.raises(ScError):
        p.run_rows(x, 0, 1, out=out)
    with pytest.raises(ScError):
        p.run(x)


# ------------------------------------------------------------------ tensor-core float matcher (3xTF32)
def _tcf(x, b, s, Wn, K, where):
    from paper_2006_13714_b200.bm import SC_KERNEL_TC_F32
    N, C, H, W = x.shape
    p = _plan((H, W, C, b, s, Wn, K), "f32")
    p.set_kernel(SC_KERNEL_TC_F32)
    gi, gd = _run(p, x)
    oi, od = oracle.bm(x, b, s, Wn, K)
    for n in range(N):
        check_f32(x[n], b, s, Wn, K, gi[n], gd[n], oi[n], od[n], where=f"{where} img{n}")
    return p


@pytest.mark.parametrize("H,W,b,s,Wn", [(40, 52, 8, 3, 17), (37, 45, 7, 1, 13), (33, 61, 5, 2, 21), (50, 40, 8, 4, 9)])
def test_tcf_dense_cross_term(H, W, b, s, Wn):
    """Steps a2 + a3 on the tensor cores (3xTF32, MN-major shift-expanded B): every window
    distance of the identity against the oracle's direct differences."""
    from paper_2006_13714_b200.bm import SC_KERNEL_TC_F32
    rng = np.random.Generator(np.random.PCG64(H * W + b))
    x = synth.random_image(rng, 1, 1, H, W, "f32")[0]
    p = _plan((H, W, 1, b, s, Wn, 1), "f32")
    p.set_kernel(SC_KERNEL_TC_F32)
    got = p.dense_debug(torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64)
    want = oracle.bm_dense(x, b, s, Wn)
    np.testing.assert_array_equal(got == -1, want == -1)
    m = want >= 0
    scale = b * b * 0.25
    assert np.max(np.abs(got[m] - want[m])) <= 4e-6 * scale + 1e-5 * np.max(want[m])


def _tcf_cases(n, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    while len(out) < n:
        b = int(rng.integers(1, 9))
        s = int(rng.integers(1, 5))
        H = int(rng.integers(b + 4, b + 70))
        W = int(rng.integers(max(b + 4, 24), b + 90))
        Wn = int(rng.integers(1, 46))
        K = int(rng.choice([1, 5, 16, 30, 45, 70]))
        out.append((b, s, H, W, Wn, K))
    return out


@pytest.mark.parametrize("case", _tcf_cases(24, 77))
def test_tcf_random_sweep(case):
    b, s, H, W, Wn, K = case
    rng = np.random.Generator(np.random.PCG64(hash(case) % (1 << 32)))
    x = synth.random_image(rng, 2, 1, H, W, "f32")
    _tcf(x, b, s, Wn, K, f"tcf {case}")


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_tcf_configs_full(name):
    cfg = synth.CONFIGS[name]
    x = synth.make_input(cfg)
    _tcf(x, cfg.b, cfg.s, cfg.Wn, cfg.K, f"tcf {name}")


@pytest.mark.parametrize("kind", ["constant", "periodic", "binary", "smooth"])
def test_tcf_ties_and_extremes(kind):
    rng = np.random.Generator(np.random.PCG64(15))
    if kind == "constant":
        x = np.full((1, 1, 60, 90), 0.3, dtype=np.float32)
    elif kind == "periodic":
        x = np.tile(rng.random((8, 8), dtype=np.float32), (8, 12))[None, None].copy()
    elif kind == "binary":
        x = rng.integers(0, 2, size=(1, 1, 60, 90)).astype(np.float32)
    else:
        yy, xx = np.mgrid[0:64, 0:96]
        x = (0.5 + 0.4 * np.sin(yy / 7.0) * np.cos(xx / 9.0)).astype(np.float32)[None, None].copy()
    for (s, b, K) in [(3, 8, 30), (1, 7, 70)]:
        p = _tcf(x, b, s, 21, K, f"tcf {kind} s{s} b{b}")
        if kind == "constant":
            assert p.debug_fix_count() == p.n_refs  # every reference ties: exact fix-up


# ------------------------------------------------------------------ NCC with wide lists (round 2)
def _ncc_wide_cases(n, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    shapes = [(3, 8), (1, 7), (4, 8), (2, 8)]
    out = []
    while len(out) < n:
        s, b = shapes[len(out) % 4]
        H, W = int(rng.integers(b + 8, 80)), int(rng.integers(b + 8, 110))
        Wn, K = int(rng.integers(9, 46)), int(rng.integers(29, 77))
        C = int(rng.choice([1, 1, 2, 4]))
        if ((H - b) // s + 1) * ((W - b) // s + 1) * Wn * Wn * C > 2e7:
            continue
        out.append((s, b, C, H, W, Wn, K))
    return out


@pytest.mark.parametrize("case", _ncc_wide_cases(12, 909))
def test_ncc_f32_wide_lists(case):
    """NCC (Eq. 4) with K + m > 32 on float input: register lists of 40 / 48 keys or shared heaps
    (K up to 76), channels summed, against oracle.ncc under the float NCC rule."""
    from tests.parity import check_ncc
    s, b, C, H, W, Wn, K = case
    rng = np.random.Generator(np.random.PCG64(hash(case) % (1 << 32)))
    x = synth.random_image(rng, 2, C, H, W, "f32")
    p, gi, gd = _ncc_run(x, b, s, Wn, K, "f32")
    oi, od = oracle.ncc(x, b, s, Wn, K)
    for n in range(2):
        check_ncc(x[n], b, s, Wn, K, gi[n], gd[n], oi[n], od[n], exact=False, where=f"ncc wide {case} img{n}")


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_ncc_c3_c4_full(name):
    """The NCC metric on the WNNM-shaped c3 (K = 70) and the 4-channel c4 (K = 32): every reference."""
    from tests.parity import check_ncc
    cfg = synth.CONFIGS[name]
    x = synth.make_input(cfg)
    p, gi, gd = _ncc_run(x, cfg.b, cfg.s, cfg.Wn, cfg.K, "f32")
    oi, od = oracle.ncc(x, cfg.b, cfg.s, cfg.Wn, cfg.K)
    check_ncc(x[0], cfg.b, cfg.s, cfg.Wn, cfg.K, gi[0], gd[0], oi[0], od[0], exact=False, where=f"ncc {name} full")


@pytest.mark.parametrize("K", [40, 70])
def test_ncc_wide_lists_fixup(K):
    """A constant / tiny-noise image ties every NCC: the wide-list references go to the exact fix-up,
    whose float path ranks (float32 d_NCC, idx) 64-bit keys for K > 32."""
    from tests.parity import check_ncc
    H, W, b, s, Wn = 40, 56, 8, 3, 15
    rng = np.random.Generator(np.random.PCG64(31))
    for kind in ("constant", "tiny_noise"):
        x = np.full((1, 1, H, W), 0.7, dtype=np.float32)
        if kind == "tiny_noise":
            x += (rng.standard_normal(x.shape) * 1e-3).astype(np.float32)
        p, gi, gd = _ncc_run(x, b, s, Wn, K, "f32")
        if kind == "constant":  # (references whose window holds fewer than K + m candidates keep all)
            assert p.debug_fix_count() >= p.n_refs * 9 // 10
        oi, od = oracle.ncc(x, b, s, Wn, K)
        check_ncc(x[0], b, s, Wn, K, gi[0], gd[0], oi[0], od[0], exact=False, where=f"ncc wide fixup {kind} K{K}")


# ------------------------------------------------------------------ 3D search
def _bm3d_check(vol, d, b, s, sz, Wn, c, K, where):
    from paper_2006_13714_b200.bm import Plan3D
    P, H, W = vol.shape
    p = Plan3D(H, W, d, b, s, Wn, sz, c, K)
    gi, gd = p.run(torch.from_numpy(vol).cuda())
    torch.cuda.synchronize()
    gi, gd = gi.cpu().numpy(), gd.cpu().numpy()
    oi, od = oracle.bm3d(vol, d, b, s, sz, Wn, c, K)
    from tests.parity import check_f32_3d
    check_f32_3d(vol, d, b, s, sz, Wn, c, K, gi, gd, oi, od, where)
    return p


@pytest.mark.parametrize("P,d,s,b,sz,Wn,c,K", [(5, 1, 1, 6, 1, 13, 3, 16), (6, 3, 1, 6, 1, 11, 2, 12),
                                                (4, 2, 3, 8, 1, 17, 3, 20), (7, 1, 2, 8, 2, 9, 5, 30),
                                                (3, 1, 1, 7, 1, 15, 1, 16), (6, 1, 4, 8, 3, 21, 4, 8)])
def test_bm3d_matches_oracle(P, d, s, b, sz, Wn, c, K):
    rng = np.random.Generator(np.random.PCG64(P * 100 + Wn * 3 + c))
    vol = synth.random_image(rng, 1, P, 41, 53, "f32")[0]
    _bm3d_check(vol, d, b, s, sz, Wn, c, K, f"bm3d {(P, d, s, b, sz, Wn, c, K)}")


def test_bm3d_translated_video_and_fixup():
    """A translated video (exact d = 0 motion-compensated matches across planes) and a constant
    volume (every candidate ties: every reference goes to the exact 3D fix-up)."""
    rng = np.random.Generator(np.random.PCG64(5))
    canvas = synth.random_image(rng, 1, 1, 90, 90, "f32")[0, 0]
    vol = np.stack([canvas[20 + 2 * z:20 + 2 * z + 40, 30 - 3 * z:30 - 3 * z + 44] for z in range(5)]).astype(np.float32)
    _bm3d_check(vol, 1, 6, 1, 1, 15, 3, 16, "bm3d translated")
    p = _bm3d_check(np.full((4, 30, 40), 0.25, np.float32), 1, 6, 1, 1, 9, 3, 16, "bm3d constant")
    assert p.debug_fix_count() > 0


def test_bm3d_rejects():
    from paper_2006_13714_b200.bm import Plan, Plan3D, ScError
    with pytest.raises(ScError):
        Plan3D(40, 40, 1, 5, 1, 13, 1, 3, 16)  # (s, b) not a box-kernel shape
    with pytest.raises(ScError):
        Plan3D(40, 40, 1, 6, 1, 31, 1, 9, 16)  # 9 * 31^2 window slots > 2^13
    p = Plan3D(40, 40, 1, 6, 1, 13, 1, 3, 16)
    with pytest.raises(ScError):
        p.run(torch.zeros((0, 40, 40), dtype=torch.float32, device="cuda"))
    x = torch.zeros((1, 1, 40, 40), dtype=torch.float32, device="cuda")
    with pytest.raises(ScError):
        Plan.run(p, x)  # a 3D plan refuses 2D runs


def test_bm3d_partial_reference_rows_and_guard():
    """Reference rows that do not fill the last 8-row CTA (ny % 8 != 0) over several planes: every
    plane's table matches the oracle and nothing is written past the output tables (the idle
    warps of the last CTA row join the plane restaging but must not reach the output stage)."""
    from paper_2006_13714_b200.bm import Plan3D
    from tests.parity import check_f32_3d
    rng = np.random.Generator(np.random.PCG64(808))
    for (P, d, H, W, b, s, sz, Wn, c, K) in [(3, 2, 50, 49, 8, 2, 2, 1, 1, 4), (5, 1, 44, 76, 7, 1, 1, 12, 4, 9),
                                             (6, 2, 25, 32, 8, 3, 1, 13, 2, 30)]:
        vol = synth.random_image(rng, 1, P, H, W, "f32")[0]
        p = Plan3D(H, W, d, b, s, Wn, sz, c, K)
        nz = p.n_zref(P)
        gi_full = torch.full((nz + 2, p.n_refs, K), -7, dtype=torch.int32, device="cuda")
        gd_full = torch.full((nz + 2, p.n_refs, K), -7.0, dtype=torch.float32, device="cuda")
        p.run(torch.from_numpy(vol).cuda(), out=(gi_full[:nz], gd_full[:nz]))
        torch.cuda.synchronize()
        assert (gi_full[nz:] == -7).all() and (gd_full[nz:] == -7.0).all(), "write past the tables"
        oi, od = oracle.bm3d(vol, d, b, s, sz, Wn, c, K)
        check_f32_3d(vol, d, b, s, sz, Wn, c, K, gi_full[:nz].cpu().numpy(), gd_full[:nz].cpu().numpy(), oi, od,
                     f"bm3d guard {(P, d, H, W)}")


# ------------------------------------------------------------------ float box kernel tile heights
@pytest.mark.parametrize("rows", [3, 7])
def test_boxf_forced_tile_heights(rows):
    """The float box kernel's tile height (reference rows per CTA, chosen per launch to fill the
    last wave: bm_boxf.cu boxf_rows) forced to `rows` through SC_BM_BOXF_ROWS: the boxf parity
    cases (random sweep, ties, c2 whole image, NCC sweep, 3D search) rerun in a child process
    (the library reads the variable once)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SC_BM_BOXF_ROWS=str(rows))
    sel = ("boxf_random_sweep or boxf_ties or c2_full or ncc_random_sweep or bm3d_matches_oracle "
           "or bm3d_translated")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", sel,
                        os.path.join(root, "tests", "test_gpu_parity.py")],
                       cwd=root, env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
