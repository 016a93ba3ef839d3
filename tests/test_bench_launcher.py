"""bench.py's multi-rank launcher and sharding host logic on CPU (gloo, host-only plans).

`python bench.py --gpus N` without a torch.distributed environment re-launches itself under
torch.distributed.run with N ranks; `--plan-only` runs that path without a GPU:
every rank builds the workload's plans host-only, takes its whole-image shard of the fixed
256-image conv batch, and the ranks compare plan digests over gloo."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*argv, timeout=240):
    env = dict(os.environ, OMP_NUM_THREADS="2")
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *argv], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=timeout)
    return p


@pytest.mark.parametrize("world", [2, 4])
def test_plan_only_self_launch_shards_conv_batch(world):
    p = _run("--plan-only", "--gpus", str(world), "--workload", "conv")
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_ranks"] == world and d["scaling"] == "strong"
    assert d["replica_digests_equal"] is True
    ranges = [r[0]["images"] for r in d["ranks"]]
    # whole images, contiguous, covering the fixed batch of 256 exactly once, balanced
    assert ranges[0][0] == 0 and ranges[-1][1] == 256
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 1
    assert all(r[0]["N"] == (b - a) * 196 for r, (a, b) in zip(d["ranks"], ranges))


def test_plan_only_weak_scaling_layers():
    p = _run("--plan-only", "--gpus", "2", "--workload", "rn50_b8")
    assert p.returncode == 0, p.stderr[-2000:]
    d = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][0])
    assert d["scaling"] == "weak" and d["replica_digests_equal"] is True
    assert [x["N"] for x in d["ranks"][0]] == [x["N"] for x in d["ranks"][1]]


def test_gpu_arm_refuses_more_gpus_than_visible():
    # no GPU here: --gpus 2 must fail loudly instead of silently running one rank
    p = _run("--gpus", "2", "--quick", timeout=120)
    assert p.returncode != 0
    assert "GPU" in p.stderr


def test_world_size_mismatch_is_an_error():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--plan-only", "--gpus", "2"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=120)
    assert p.returncode != 0 and "WORLD_SIZE" in p.stderr
