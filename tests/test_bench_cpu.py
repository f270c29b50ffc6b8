"""bench.py's multi-rank plumbing on CPU: ``--gpus N`` without torchrun re-launches itself with
N ranks (gloo here, via --selftest-cpu), every rank takes its frame shard, the max over ranks
is reported and n_gpus equals N; without N visible GPUs a real run refuses (non-zero exit)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=240):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                          text=True, timeout=timeout, env=env, cwd=ROOT)


@pytest.mark.parametrize("n", [1, 2])
def test_selftest_launcher(n):
    r = _run("--gpus", str(n), "--selftest-cpu", "--steps", "3", "--warmup", "3")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == n and line["steps"] == 3 and line["warmup"] == 3
    assert line["scaling"] == "strong" and line["config"]["workload"] == "c5"
    shards = line["config"]["shards"]
    assert len(shards) == n and shards[0][0] == 0 and shards[-1][1] == 64
    assert line["frames_timed"] == 64  # every rank's shard is counted exactly once
    assert line["ms_per_step"] > 0


def test_refuses_without_gpus():
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("GPUs visible")
    r = _run("--gpus", "2", "--steps", "3", "--warmup", "3")
    assert r.returncode != 0 and "GPU" in r.stderr


def test_world_size_mismatch_refused():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3"],
                       capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert r.returncode == 2 and "WORLD_SIZE" in r.stderr
