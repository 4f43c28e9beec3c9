"""bench.py's JSON contract on CPU: the reference arm (the unmodified
reference package on a tiny ring pair) prints one line with every key the
driver reads; our arm refuses to run without a GPU instead of falling back."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent


def _run(*args, timeout=300):
    return subprocess.run([sys.executable, str(REPO / "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, cwd=REPO)


def test_reference_arm_line(reference):
    r = _run("--impl", "reference", "--nu", "40", "--nv", "20", "--steps", "1", "--warmup", "0")
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["higher_is_better"] is False and line["value"] > 0
    assert set(line["cpu_baseline"]) >= {"value", "unit", "cores", "kind", "sample"}
    assert line["cpu_baseline"]["kind"] in ("reference", "port") and line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert "workload" in line["config"]


def test_gpu_arm_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    r = _run("--steps", "1", "--warmup", "3", "--nu", "40", "--nv", "20", timeout=120)
    assert r.returncode != 0 and "no CUDA device" in r.stderr


def test_self_launch_two_ranks_dry_run():
    """`bench.py --gpus 2` outside torchrun starts the 2 ranks itself
    (torch.distributed.run on 127.0.0.1, gloo without GPUs): one line from
    rank 0 with n_gpus 2, the max-over-ranks reduction and the frame
    all-gather done."""
    r = _run("--gpus", "2", "--dry-run", timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["dry_run"] and line["gather_ok"] and line["max_over_ranks"] == 2.0
