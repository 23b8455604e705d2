"""bench.py's multi-rank launch on CPU: ``--gpus N`` outside torchrun spawns N
ranks itself (gloo here), and rank 0 prints the max over ranks with n_gpus = N."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("n", [2, 3])
def test_bench_gpus_flag_spawns_ranks(n):
    r = subprocess.run([sys.executable, str(REPO / "bench.py"), "--gpus", str(n), "--dry-run", "--steps", "3",
                        "--warmup", "3"], capture_output=True, text=True, timeout=300,
                       env={**__import__("os").environ, "LSDF_BENCH_BACKEND": "gloo"})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    out = json.loads(lines[0])
    assert out["n_gpus"] == n and out["backend"] == "gloo"
    assert out["ms_per_step"] == float(n)  # max over ranks: rank r reports 1 + r


def test_bench_single_rank_dry_run():
    r = subprocess.run([sys.executable, str(REPO / "bench.py"), "--dry-run"], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["n_gpus"] == 1
