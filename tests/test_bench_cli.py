"""bench.py's launcher contract on CPU: `--gpus N` without a torchrun environment re-launches
itself as N ranks (torch.distributed.run, 127.0.0.1) -- checked with --dry-run (gloo, no GPU
work) -- and refuses (exit 2, no JSON line) when the rank count cannot match --gpus."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _run(args, env=None):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True, env=e,
                          timeout=300, cwd=str(ROOT))


def test_bench_spawns_n_ranks():
    r = _run(["--gpus", "2", "--dry-run"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert lines == [{"dry_run": True, "n_gpus": 2, "rank_sum": 1}]


def test_bench_refuses_mismatched_world():
    r = _run(["--gpus", "2", "--steps", "1"], env={"WORLD_SIZE": "1", "RANK": "0"})
    assert r.returncode == 2 and not r.stdout.strip()


def test_bench_refuses_more_gpus_than_visible():
    r = _run(["--gpus", "64", "--steps", "1"], env={"CUDA_VISIBLE_DEVICES": ""})
    assert r.returncode == 2 and not r.stdout.strip()
