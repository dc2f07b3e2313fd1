"""bench.py's multi-rank path on this box's GPU: `--gpus 2` spawns the second rank itself
(no torchrun, no NCCL: a gloo group only for the barrier and the timing max), each rank
runs its contiguous batch x head shard, and every unit's O, L, dQ, dK, dV are bit-identical
to the same unit of a single-rank run of the same global problem (per-unit input seeds)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _bench(tmp_path, tag, gpus, batch):
    out = tmp_path / f"h{tag}.json"
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--batch", str(batch), "--heads", "3",
           "--seq", "640", "--steps", "2", "--warmup", "3", "--no-e2e", "--no-cpu-baseline", "--dump-hashes",
           str(out)]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    return json.loads(lines[0]), json.loads(out.read_text())


def test_two_ranks_match_one(cuda_dev, tmp_path):
    line2, h2 = _bench(tmp_path, "2", gpus=2, batch=1)
    line1, h1 = _bench(tmp_path, "1", gpus=1, batch=2)
    assert line2["n_gpus"] == 2 and line2["config"]["global_batch"] == 2
    assert line2["value"] > 0 and line2["gpu_launches"] > 0
    assert len(h1) == 6 and h2 == h1
