"""bench.py end to end: one GPU, and the N > 1 launch path (torchrun, 2 ranks sharing
cuda:0 over gloo) — one JSON line from rank 0 with the contract's keys."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
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


SMALL = ["--steps", "3", "--warmup", "3", "--num-vertices", "200000", "--no-cpu-baseline", "--train-epochs", "0",
         "--c3-scale", "0.002", "--c3-steps", "2", "--c3-warmup", "1"]


def _check_c3(d, world):
    c3 = d["c3_three_tier"]
    assert c3["n_gpus"] == world and c3["value"] > 0
    assert c3["pcie"]["measured_gb_per_batch"] > 0 and c3["pcie"]["measured_over_predicted"] > 0
    assert 0 < c3["tier_roofline"]["frac_min_over_ranks"] <= c3["tier_roofline"]["frac_clique"] * world + 1e-9
    tiers = c3["tiers_per_batch_rank0"]
    assert tiers["rows_local"] > 0 and tiers["rows_host"] > 0
    if world > 1:  # the partitioned cache: peers' slabs are read through CUDA IPC
        assert tiers["rows_peer"] > 0 and tiers["reads_peer"] > 0
    else:
        assert tiers["rows_peer"] == 0


def test_bench_single_gpu_contract():
    d = _run([sys.executable, "bench.py", *SMALL])
    assert KEYS <= set(d) and d["n_gpus"] == 1 and d["value"] > 0
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1.5
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["scaling"] == "strong"
    _check_c3(d, 1)


def test_bench_two_ranks_partitioned_clique():
    env = dict(os.environ, GC_DIST_BACKEND="gloo")
    d = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
              "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
              *SMALL, "--no-e2e", "--train-epochs", "1"], env=env)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["dist_backend"] == "gloo"
    ge = d["graphsage_epoch"]  # DDP: the gradient all-reduce every step across the two ranks
    assert ge["ddp_ranks"] == 2 and ge["seconds"] > 0 and np.isfinite(ge["bf16"]["last_loss"])
    _check_c3(d, 2)


def test_bench_c3_self_check_against_reference():
    """The C3 section's CPU leg runs the unmodified reference and the bench compares its
    batches with the device's (distinct vertices + rows through all three tiers)."""
    d = _run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--num-vertices", "200000",
              "--train-epochs", "0", "--no-e2e", "--cpu-seconds", "3", "--c3-scale", "0.01", "--c3-steps", "2",
              "--c3-warmup", "1"])
    assert d["verified"]["bit_exact"] and d["c3_three_tier"]["verified"]["bit_exact"]
    assert d["c3_three_tier"]["cpu_baseline"]["kind"] == "reference"


def test_bench_reference_arm():
    d = _run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
              "--num-vertices", "200000"])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_bench_c3_full_shape_self_check():
    """C3 at its full ogbn-papers100M shape (111M vertices, 1.55B edges, 57 GB host tier):
    the bench's three-tier section samples and gathers through TopologyStore and
    FeatureStore built from the reference plan and compares 4 batches of epoch 0 — every
    hop's offsets and neighbours, the distinct vertices and their rows — with the
    unmodified reference, bit for bit."""
    d = _run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--num-vertices", "200000",
              "--train-epochs", "0", "--no-e2e", "--cpu-seconds", "2", "--c3-scale", "1.0", "--c3-steps", "1",
              "--c3-warmup", "1"])
    c3 = d["c3_three_tier"]
    assert c3["config"]["num_vertices"] == 111_000_000 and c3["config"]["num_edges"] == 1_554_000_000
    assert c3["verified"]["bit_exact"] and c3["verified"]["batches"] == 4
    assert c3["cpu_baseline"]["kind"] == "reference"
    assert c3["tiers_per_batch_rank0"]["rows_host"] > 0 and c3["tiers_per_batch_rank0"]["reads_host"] > 0
