"""Probe: reuse of host-tier feature rows across the batches of a window at C3.

Builds the C3 three-tier setup like bench_tiers.py (scale, budget), runs one epoch and
for each window counts the host-tier row reads (sum over batches of the batch's distinct
host-tier vertices) against the window's distinct host-tier vertices: the PCIe rows a
window-level host-row staging would save.

    python tools/host_reuse_probe.py [scale] [window]
"""
import math
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2305_16588_b200 as P  # noqa: E402
from paper_2305_16588_b200 import planner as PL  # noqa: E402
from paper_2305_16588_b200.cache import FeatureStore, TopologyStore  # noqa: E402
from paper_2305_16588_b200.graph import synthetic_features_device  # noqa: E402
from paper_2305_16588_b200.partition import single_clique_partitioning  # noqa: E402
from paper_2305_16588_b200.pipeline import SampleGatherPipeline  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
window = int(sys.argv[2]) if len(sys.argv) > 2 else 256
torch.cuda.set_device(0)
n = int(round(111_000_000 * scale))
deg, dim, fanouts, bs = 14, 128, (25, 10), 1024
g = P.generate_synthetic_device(n, deg, 1.2, seed=P.derive_seed(7, 1))
train = P.select_training_set(g, 0.1, seed=P.derive_seed(7, 2))
layout = P.block_layout(1, 1)
pools = P.assign_tablets(P.split_intra_clique(train, single_clique_partitioning(g), layout), layout)
feat = P.FeatureSpec(dim)
budget = int(0.1 * (g.num_edges * 4 + 8 * n + n * feat.row_bytes))
spec = P.HardwareSpec(layout, clique_budget_bytes=budget)
cfg = P.SamplingConfig(fanouts=fanouts, batch_size=bs, presample_epochs=4, seed=P.derive_seed(7, 4))
hot = P.run_presampling(g, pools, layout, cfg, spec)[0]
orders = PL.build_candidate_orders(hot)
plan, est = PL.search_optimal_plan(orders, budget, 0.01, g, feat, spec, hot.sampling_txn_total)
asg = PL.materialize_assignment([orders], [plan], layout, g, feat, spec)
host_table = torch.empty((n, dim), dtype=torch.float32, pin_memory=True)
for r0 in range(0, n, 1 << 24):
    rows = min(1 << 24, n - r0)
    host_table[r0 : r0 + rows].copy_(synthetic_features_device(r0, rows, dim))
topo = TopologyStore(g, asg.topo_vertices, 0, host_full=True)
fstore = FeatureStore.from_assignment(host_table, asg.feat_vertices, 0)
pool = pools[0]
nb = math.ceil(len(pool) / bs)
pipe = SampleGatherPipeline(g, cfg, fstore, len(pool), window=min(window, nb), feat_rows_cap=60_000, topology=topo)
loc = fstore.location
stats = {"reads": 0, "distinct": 0, "windows": 0, "rows": 0}


def on_window(p, w0, nbw):
    sp = p.sampler
    cnt = sp.ucount[:nbw].long()
    cap = sp.unique.shape[1]
    mask = torch.arange(cap, device="cuda").unsqueeze(0) < cnt.unsqueeze(1)
    ids = sp.unique[:nbw][mask].long()
    host = ids[loc[ids] == -1]
    stats["reads"] += host.numel()
    stats["distinct"] += torch.unique(host).numel()
    stats["rows"] += ids.numel()
    stats["windows"] += 1


pipe.run_epoch(pipe.plan_epoch(pool, P.KeyedRng(P.derive_seed(7, 5)).derive(0, 0, 0)), on_window=on_window)
torch.cuda.synchronize()
r, d = stats["reads"], stats["distinct"]
print(f"C3 x{scale}: window {pipe.window} batches, {stats['windows']} windows, {nb} batches")
print(f"rows gathered {stats['rows']}, host-tier reads {r} ({r / nb:.0f}/batch), distinct per window {d} "
      f"({d / nb:.0f}/batch): a window-level host-row staging reads {d / max(r, 1):.3f} of the host rows")
