"""bench.py's multi-rank launch path on CPU (gloo): `--gpus N` outside torchrun launches N
ranks itself, a WORLD_SIZE that disagrees with --gpus is refused, and a box with fewer
GPUs than requested errors instead of timing fewer."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _run(args, env=None, timeout=180):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, BENCH] + args, capture_output=True, text=True, env=e,
                          timeout=timeout, cwd=ROOT)


def test_self_launch_two_ranks_dry_run():
    r = _run(["--gpus", "2", "--dry-run", "--steps", "2", "--warmup", "3"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1                       # rank 0 alone prints
    assert lines[0]["n_gpus"] == 2 and lines[0]["ranks_seen"] == 2 and lines[0]["steps"] == 2


def test_more_gpus_than_visible_is_an_error():
    torch = pytest.importorskip("torch")
    if torch.cuda.device_count() >= 2:
        pytest.skip("a multi-GPU box: the real run would start")
    r = _run(["--gpus", "2", "--steps", "1", "--warmup", "3"])
    assert r.returncode != 0
    assert "requested" in r.stderr and not any(l.startswith("{") for l in r.stdout.splitlines())


def test_world_size_mismatch_is_refused():
    r = _run(["--gpus", "1", "--dry-run"], env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE=2" in r.stderr
