"""Seeded synthetic inputs: shapes, dtypes, determinism, value ranges (no GPU)."""
import numpy as np
import pytest

from paper_2006_13714_b200 import synth


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_shapes_and_determinism(name):
    cfg = synth.CONFIGS[name]
    a = synth.make_input(cfg)
    b = synth.make_input(cfg)
    assert a.shape == cfg.shape
    assert a.dtype == (np.uint8 if cfg.dtype == "u8" else np.float32)
    assert a.flags.c_contiguous
    np.testing.assert_array_equal(a, b)
    assert np.isfinite(a.astype(np.float64)).all()


def test_video_frames_are_translated_crops():
    f = synth.video_frames(4, 64, 96, seed=5, walk_seed=3005, margin=16, max_step=3)
    assert f.shape == (4, 1, 64, 96) and f.dtype == np.uint8
    canvas = synth.G(64 + 32, 96 + 32, 5)
    # frame 0 is the centre crop
    np.testing.assert_array_equal(f[0, 0], canvas[16:80, 16:112])
    # every frame is a crop of the same canvas
    for k in range(4):
        found = any((canvas[y:y + 64, x:x + 96] == f[k, 0]).all()
                    for y in range(33) for x in range(33))
        assert found


def test_c5_subset_frames():
    cfg = synth.CONFIGS["c5"]
    f = synth.make_input(cfg, n_frames=2)
    assert f.shape == (2, 1, 1080, 1920)
    assert 0 < f.mean() < 255
