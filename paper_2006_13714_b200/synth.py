"""Seeded synthetic inputs for the five BM workloads (BASELINE.json ``configs``).

This module holds NO block-matching arithmetic: it only draws images. It is the one
module shared by the oracle tests and the CUDA path.

The paper measures on unnamed 512x512 / 256x256 gray images (Table III
protocol) and on the IVRG RGB-NIR dataset. Neither is available, so
these generators stand in with the paper's workload *shapes* (SURVEY.md section 8d):

* ``G(H, W, seed)``: 6 random-orientation sinusoids + 10 random added rectangles + one
  repeated 16x16 random texture tile, min-max normalised to [0, 255], rounded
  half-to-even, uint8.
* c1: G(64, 64) u8.
* c2/c3: G(512, 512)/255 + N(0, sigma^2) i.i.d. noise, float32, not clipped
  (sigma = 25/255, 50/255), mirroring the paper's additive Gaussian noise protocol.
* c4: planar [R, G, B, NIR] float32 768x1024 (RGB gains, NIR = 0.6 luma + sinusoid),
  noise on RGB only.
* c5: 64 u8 frames 1080x1920, crops of one large canvas along a seeded random walk
  (integer translation of up to 8 px per frame).

3D search workloads (the next row SURVEY.md 8f rank 4; PAPER.md:696-697's multi-channel task,
256 x 256 x q data, patch stride 1, 6 x 6 x d patches, 30 x 30 x c windows):
* v1 (SALT video): 20 float32 frames 256x256 = crops of one canvas along a seeded random walk,
  /255 + N(0, (25/255)^2); d = 1, c = 9 frames.
* m1 (Self-MM multi-modality): a 6-plane 256x256 float32 image (gains x luma + independent
  sinusoids per plane, noise sigma 25/255); d = 3, c = 2.
"""
from __future__ import annotations

import dataclasses

import numpy as np

__all__ = ["BMConfig", "CONFIGS", "CONFIGS3D", "G", "make_input", "config_by_name"]


@dataclasses.dataclass(frozen=True)
class BMConfig:
    name: str
    dtype: str  # "u8" or "f32"
    N: int      # images / frames
    C: int      # channels
    H: int
    W: int
    b: int      # patch side
    s: int      # reference stride
    Wn: int     # search-window side (candidate top-left offsets)
    K: int      # matches per reference
    seed: int
    noise_seed: int = 0
    sigma: float = 0.0
    d: int = 0        # 3D search: patch depth in planes (0 = 2D block matching)
    sz: int = 1       # 3D search: reference plane stride
    zwin: int = 1     # 3D search: plane offsets per reference (window depth c)

    @property
    def shape(self):
        return (self.N, self.C, self.H, self.W)


CONFIGS = {
    "c1": BMConfig("c1", "u8", 1, 1, 64, 64, 8, 4, 21, 16, seed=1),
    "c2": BMConfig("c2", "f32", 1, 1, 512, 512, 8, 3, 39, 16, seed=2, noise_seed=1002, sigma=25 / 255),
    "c3": BMConfig("c3", "f32", 1, 1, 512, 512, 7, 1, 61, 70, seed=3, noise_seed=1003, sigma=50 / 255),
    "c4": BMConfig("c4", "f32", 1, 4, 768, 1024, 8, 3, 41, 32, seed=4, noise_seed=1004, sigma=25 / 255),
    "c5": BMConfig("c5", "u8", 64, 1, 1080, 1920, 8, 4, 33, 16, seed=5, noise_seed=3005),
}

# 3D search (volumes of P planes [1, P, H, W]); K = 16 (the paper does not state it)
CONFIGS3D = {
    "v1": BMConfig("v1", "f32", 1, 20, 256, 256, 6, 1, 30, 16, seed=6, noise_seed=1006, sigma=25 / 255,
                   d=1, sz=1, zwin=9),
    "m1": BMConfig("m1", "f32", 1, 6, 256, 256, 6, 1, 30, 16, seed=7, noise_seed=1007, sigma=25 / 255,
                   d=3, sz=1, zwin=2),
}


def config_by_name(name: str) -> BMConfig:
    return CONFIGS[name] if name in CONFIGS else CONFIGS3D[name]


def _sinusoid(rng, H, W, amp_lo, amp_hi, f_lo, f_hi):
    A = rng.uniform(amp_lo, amp_hi)
    f = rng.uniform(f_lo, f_hi)
    th = rng.uniform(0.0, np.pi)
    ph = rng.uniform(0.0, 2.0 * np.pi)
    y = np.arange(H, dtype=np.float64)[:, None]
    x = np.arange(W, dtype=np.float64)[None, :]
    return A * np.sin(2.0 * np.pi * f * (x * np.cos(th) + y * np.sin(th)) + ph)


def G(H: int, W: int, seed: int) -> np.ndarray:
    """Base generator: uint8 [H, W]."""
    rng = np.random.Generator(np.random.PCG64(seed))
    img = np.zeros((H, W), dtype=np.float64)
    for _ in range(6):
        img += _sinusoid(rng, H, W, 10.0, 40.0, 0.01, 0.15)
    for _ in range(10):
        y0 = int(rng.integers(0, H))
        x0 = int(rng.integers(0, W))
        h = int(rng.integers(4, max(5, H // 3) + 1))
        w = int(rng.integers(4, max(5, W // 3) + 1))
        a = rng.uniform(-60.0, 60.0)
        img[y0:y0 + h, x0:x0 + w] += a
    tile = rng.uniform(-25.0, 25.0, size=(16, 16))
    reps = (-(-H // 16), -(-W // 16))
    img += np.tile(tile, reps)[:H, :W]
    lo, hi = img.min(), img.max()
    img = (img - lo) * (255.0 / (hi - lo))
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def _noisy_gray(cfg: BMConfig) -> np.ndarray:
    base = G(cfg.H, cfg.W, cfg.seed).astype(np.float64) / 255.0
    rng = np.random.Generator(np.random.PCG64(cfg.noise_seed))
    noisy = base + rng.normal(0.0, cfg.sigma, size=base.shape)
    return noisy.astype(np.float32).reshape(1, 1, cfg.H, cfg.W)


def _rgbnir(cfg: BMConfig) -> np.ndarray:
    H, W = cfg.H, cfg.W
    L = G(H, W, cfg.seed).astype(np.float64) / 255.0
    rng = np.random.Generator(np.random.PCG64(2000 + cfg.seed))
    gains = rng.uniform(0.6, 1.0, size=3)
    R, Gc, B = (np.clip(L * g, 0.0, 1.0) for g in gains)
    nir = 0.6 * (0.299 * R + 0.587 * Gc + 0.114 * B) + _sinusoid(rng, H, W, 0.2, 0.2, 0.01, 0.1)
    nrng = np.random.Generator(np.random.PCG64(cfg.noise_seed))
    chans = [c + nrng.normal(0.0, cfg.sigma, size=c.shape) for c in (R, Gc, B)] + [nir]
    return np.stack(chans).astype(np.float32).reshape(1, 4, H, W)


def video_frames(N: int, H: int, W: int, seed: int, walk_seed: int, margin: int = 512,
                 max_step: int = 8) -> np.ndarray:
    """N uint8 frames [N,1,H,W]: crops of one canvas along a seeded integer random walk."""
    canvas = G(H + 2 * margin, W + 2 * margin, seed)
    rng = np.random.Generator(np.random.PCG64(walk_seed))
    oy = ox = margin
    out = np.empty((N, 1, H, W), dtype=np.uint8)
    for f in range(N):
        out[f, 0] = canvas[oy:oy + H, ox:ox + W]
        dy, dx = rng.integers(-max_step, max_step + 1, size=2)
        oy = int(np.clip(oy + dy, 0, 2 * margin))
        ox = int(np.clip(ox + dx, 0, 2 * margin))
    return out


def _video_f32(cfg: BMConfig) -> np.ndarray:
    frames = video_frames(cfg.C, cfg.H, cfg.W, cfg.seed, 3000 + cfg.seed, margin=64, max_step=4)
    rng = np.random.Generator(np.random.PCG64(cfg.noise_seed))
    v = frames[:, 0].astype(np.float64) / 255.0 + rng.normal(0.0, cfg.sigma, size=(cfg.C, cfg.H, cfg.W))
    return v.astype(np.float32).reshape(1, cfg.C, cfg.H, cfg.W)


def _multimodal(cfg: BMConfig) -> np.ndarray:
    H, W = cfg.H, cfg.W
    L = G(H, W, cfg.seed).astype(np.float64) / 255.0
    rng = np.random.Generator(np.random.PCG64(2000 + cfg.seed))
    planes = [np.clip(L * rng.uniform(0.6, 1.0), 0.0, 1.0) + _sinusoid(rng, H, W, 0.05, 0.2, 0.01, 0.1)
              for _ in range(cfg.C)]
    nrng = np.random.Generator(np.random.PCG64(cfg.noise_seed))
    v = np.stack(planes) + nrng.normal(0.0, cfg.sigma, size=(cfg.C, H, W))
    return v.astype(np.float32).reshape(1, cfg.C, H, W)


def make_input(cfg: BMConfig, n_frames: int | None = None) -> np.ndarray:
    """The config's input as a contiguous numpy array [N, C, H, W] (uint8 or float32); the 3D
    configs return one volume [1, P, H, W]."""
    if cfg.d > 0:
        return _video_f32(cfg) if cfg.name == "v1" else _multimodal(cfg)
    if cfg.name == "c5" or (cfg.dtype == "u8" and cfg.N > 1):
        n = cfg.N if n_frames is None else n_frames
        return video_frames(n, cfg.H, cfg.W, cfg.seed, cfg.noise_seed)
    if cfg.dtype == "u8":
        return G(cfg.H, cfg.W, cfg.seed).reshape(1, 1, cfg.H, cfg.W)
    if cfg.C == 4:
        return _rgbnir(cfg)
    return _noisy_gray(cfg)


def random_image(rng: np.random.Generator, N: int, C: int, H: int, W: int, dtype: str) -> np.ndarray:
    """Plain i.i.d. random test image (used by small random parity sweeps)."""
    if dtype == "u8":
        return rng.integers(0, 256, size=(N, C, H, W), dtype=np.uint8)
    return rng.random(size=(N, C, H, W), dtype=np.float64).astype(np.float32)
