"""bench.py end to end: one GPU, and the N > 1 launch path (torchrun, 2 ranks sharing
cuda:0 over gloo) — one JSON line from rank 0 with the contract's keys."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks"}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(cmd, env=None):
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


SMALL = ["--steps", "3", "--warmup", "3", "--num-vertices", "200000", "--no-cpu-baseline", "--train-epochs", "0"]


def test_bench_single_gpu_contract():
    d = _run([sys.executable, "bench.py", *SMALL])
    assert KEYS <= set(d) and d["n_gpus"] == 1 and d["value"] > 0
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1.5
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0


def test_bench_two_ranks_weak_scaling():
    env = dict(os.environ, GC_DIST_BACKEND="gloo")
    d = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
              "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
              *SMALL, "--no-e2e"], env=env)
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    assert d["config"]["dist_backend"] == "gloo"


def test_bench_reference_arm():
    d = _run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
              "--num-vertices", "200000"])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0
