"""Three-tier bench: Legion's full flow on a papers100M-shaped graph with a host tier.

BASELINE configs[2] shape (ogbn-papers100M: 111M vertices, degree ~14, 128-d fp32,
fanouts [25,10], batch 1024, 10% training set), scaled by --scale (default 0.1 so the
host tables fit a desk-size box; --scale 1 is the full shape). On the device:

  1. presampling epoch (K1/K2/K3/K5)         -> HotnessMatrices, N_TSUM
  2. CSLP ranking + alpha search (K6/K7)      -> plan, predicted PCIe transactions
  3. materialize + cache fill (K8)            -> topology slab + feature slab in HBM;
                                                 everything else stays in pinned host
                                                 memory, read over PCIe through UVA
  4. validation epochs through the three tiers (K2 tiered topology, K4 gather)

Reports batches/s through the tiers and measured PCIe bytes per batch next to the
reference cost model's prediction N_total x CLS / batches (planner.py:142-169).

    python bench_tiers.py [--scale 0.1] [--budget-frac 0.1] [--steps 3]
"""

from __future__ import annotations

import argparse
import json
import math
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=0.1)
    ap.add_argument("--budget-frac", type=float, default=0.1,
                    help="per-GPU cache budget / (topology + feature bytes); the clique budget is K times it")
    ap.add_argument("--clique", type=int, default=1,
                    help="emulate GPU 0 of a K-GPU NVSwitch clique on this one GPU: K tablets, the K-way "
                         "partitioned cache with every peer slab in local HBM (peer rows then move at HBM "
                         "speed; the tier roofline still charges them to NVLink)")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--window", type=int, default=256)
    ap.add_argument("--lanes", type=int, default=2, help="concurrent window lanes (inter-batch pipeline)")
    ap.add_argument("--presample-epochs", type=int, default=32,
                    help="presampling epochs behind the plan (more: less optimistic estimate, better cache)")
    ap.add_argument("--graph", type=int, default=1, help="1: each timed epoch is one CUDA-graph launch")
    ap.add_argument("--sweep-lanes", default="", help="extra schedules to time after the main run, e.g. 1,3,2d,2du,2w64 (d: host rows deferred, read in address order; du: deferred, list order; wN: window)")
    ap.add_argument("--alpha-sweep", type=int, default=0,
                    help="validate the cost model: time one epoch at this many alpha points (+ both objectives' picks)")
    ap.add_argument("--pcie-gbs", type=float, default=64.0, help="nominal PCIe Gen5 x16 GB/s for the tier roofline")
    ap.add_argument("--nvlink-gbs", type=float, default=900.0, help="NVLink 5 GB/s per direction")
    a = ap.parse_args()

    import torch

    import paper_2305_16588_b200 as P
    from paper_2305_16588_b200 import planner as PL
    from paper_2305_16588_b200.cache import FeatureStore, TopologyStore
    from paper_2305_16588_b200.graph import synthetic_features_device
    from paper_2305_16588_b200.partition import single_clique_partitioning
    from paper_2305_16588_b200.pipeline import SampleGatherPipeline, StageTimer

    torch.cuda.set_device(0)
    t_setup = time.perf_counter()
    n = int(round(111_000_000 * a.scale))
    deg, dim, fanouts, bs = 14, 128, (25, 10), 1024
    g = P.generate_synthetic_device(n, deg, 1.2, seed=P.derive_seed(7, 1))
    train = P.select_training_set(g, 0.1, seed=P.derive_seed(7, 2))
    K = a.clique
    layout = P.block_layout(K, K)
    pools = P.assign_tablets(P.split_intra_clique(train, single_clique_partitioning(g), layout), layout)
    feat = P.FeatureSpec(dim)
    total_bytes = g.num_edges * 4 + 8 * n + n * feat.row_bytes
    budget = int(a.budget_frac * total_bytes) * K
    spec = P.HardwareSpec(layout, clique_budget_bytes=budget)
    cfg = P.SamplingConfig(fanouts=fanouts, batch_size=bs, presample_epochs=a.presample_epochs,
                           seed=P.derive_seed(7, 4))

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hot = P.run_presampling(g, pools, layout, cfg, spec)[0]
    t_pre = time.perf_counter() - t0
    t0 = time.perf_counter()
    orders = PL.build_candidate_orders(hot)
    plan, est = PL.search_optimal_plan(orders, budget, 0.01, g, feat, spec, hot.sampling_txn_total)
    asg = PL.materialize_assignment([orders], [plan], layout, g, feat, spec)
    torch.cuda.synchronize()
    t_plan = time.perf_counter() - t0

    # host tier: the whole fp32 table in pinned, mapped memory (filled from the device)
    host_table = torch.empty((n, dim), dtype=torch.float32, pin_memory=True)
    step = 1 << 24
    for r0 in range(0, n, step):
        rows = min(step, n - r0)
        host_table[r0 : r0 + rows].copy_(synthetic_features_device(r0, rows, dim))
    t0 = time.perf_counter()
    topo = TopologyStore(g, asg.topo_vertices, 0, host_full=True)
    fstore = FeatureStore.from_assignment(host_table, asg.feat_vertices, 0)
    torch.cuda.synchronize()
    t_fill = time.perf_counter() - t0
    pool = pools[0]
    nb = math.ceil(len(pool) / bs)
    pipe = SampleGatherPipeline(g, cfg, fstore, len(pool), window=min(a.window, nb), feat_rows_cap=60_000,
                                topology=topo, lanes=a.lanes)
    root = P.KeyedRng(P.derive_seed(7, 5))
    plans = [pipe.plan_epoch(pool, root.derive(e, 0, 0)) for e in range(a.warmup + a.steps)]
    setup_s = time.perf_counter() - t_setup
    for e in range(a.warmup):
        (pipe.run_epoch_graph if a.graph else pipe.run_epoch)(plans[e])
    torch.cuda.synchronize()
    topo.reset_counters()
    fstore.reset_counters()
    ms = []
    for s in range(a.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        (pipe.run_epoch_graph if a.graph else pipe.run_epoch)(plans[a.warmup + s])
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    # stage durations and algorithmic bytes: the same epochs once more on one lane
    # (kernels timed alone); tier counters are read before this pass
    t, f = topo.tier_counts(), fstore.tier_counts()
    sweep = {}
    for tag in [x for x in a.sweep_lanes.split(",") if x]:
        # "2": two lanes; "2d": host rows deferred; "2w64": windows of 64 batches;
        # "2g2": gather grid of 2 CTAs per SM
        from paper_2305_16588_b200 import _lib

        head, _, gsm = tag.partition("g")
        head, _, win = head.partition("w")
        # "2du": deferred host rows read in list order instead of address order
        lanes, defer = int(head.rstrip("du")), "d" in head
        wsize = int(win) if win else a.window
        _lib.check(_lib.lib().gc_set_option(_lib.GC_OPT_GATHER_CTAS_PER_SM, int(gsm) if gsm else 16))
        _lib.check(_lib.lib().gc_set_option(_lib.GC_OPT_DEFER_ORDER, 0 if "u" in head else 1))
        del pipe
        torch.cuda.empty_cache()
        pipe = SampleGatherPipeline(g, cfg, fstore, len(pool), window=min(wsize, nb), feat_rows_cap=60_000,
                                    topology=topo, lanes=lanes, defer_host=defer)
        (pipe.run_epoch_graph if a.graph else pipe.run_epoch)(plans[0])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in range(a.steps):
            (pipe.run_epoch_graph if a.graph else pipe.run_epoch)(plans[a.warmup + s])
        e1.record()
        torch.cuda.synchronize()
        sweep[tag] = nb * a.steps / (e0.elapsed_time(e1) / 1000.0)
        _lib.check(_lib.lib().gc_set_option(_lib.GC_OPT_GATHER_CTAS_PER_SM, 16))
        _lib.check(_lib.lib().gc_set_option(_lib.GC_OPT_DEFER_ORDER, 1))
    seq = pipe
    if a.lanes > 1 or sweep:
        del pipe
        torch.cuda.empty_cache()
        seq = SampleGatherPipeline(g, cfg, fstore, len(pool), window=min(a.window, nb), feat_rows_cap=60_000,
                                   topology=topo, lanes=1)
    timer = StageTimer()
    seq.timer = timer
    acc = {"sampling": 0, "dedup": 0, "gather": 0}

    def account(p, w0, nbw):
        wb = p.window_bytes(nbw)
        for k in acc:
            acc[k] += wb[k]

    for s in range(a.steps):
        StageTimer.hold()  # the host runs ahead: stage events see device time only
        seq.run_epoch(plans[a.warmup + s])
    seq.timer = None
    for s in range(a.steps):
        seq.run_epoch(plans[a.warmup + s], on_window=account)
    torch.cuda.synchronize()
    batches = nb * a.steps
    # the presampling epochs' batches: the plan's N_total counts all of them
    clique_batches = a.presample_epochs * sum(math.ceil(len(pl) / bs) for pl in pools)
    row_txns = PL.feature_row_transactions(feat, spec)
    cls = spec.cache_line_bytes
    measured_txn = t["host_txn"] + f["host"] * row_txns
    pred_txn = est.total_txns
    stages = {k: v[1] / a.steps for k, v in timer.summary().items()}
    # tier roofline (north star): per batch, max over tiers of bytes / bandwidth
    row = feat.row_bytes
    pcie_b = t["reads_host"] * 16 + t["edges_host"] * 4 + f["host"] * row
    nvl_b = t["reads_peer"] * 16 + t["edges_peer"] * 4 + f["peer"] * row
    hbm_b = acc["sampling"] + acc["dedup"] + acc["gather"] - pcie_b - nvl_b
    hbm_gbs = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    t_tier = {"hbm": hbm_b / batches / (hbm_gbs * 1e9), "nvlink": nvl_b / batches / (a.nvlink_gbs * 1e9),
              "pcie": pcie_b / batches / (a.pcie_gbs * 1e9)}
    t_roof = max(t_tier.values())
    t_meas = sum(ms) / 1000.0 / batches
    out = {
        "metric": "three-tier sampled+gathered batches/s; PCIe GB/batch vs plan prediction",
        "value": batches / (sum(ms) / 1000.0),
        "unit": "batches/s",
        "n_gpus": 1,
        "steps": a.steps,
        "config": {"workload": f"C3 ogbn-papers100M-shaped synthetic x{a.scale}", "num_vertices": n,
                   "num_edges": g.num_edges, "feature_dim": dim, "fanouts": list(fanouts), "batch_size": bs,
                   "budget_bytes": budget, "budget_frac_per_gpu": a.budget_frac, "batches_per_epoch": nb,
                   "clique": K, "peers": "emulated in local HBM" if K > 1 else None},
        "plan": {"presample_epochs": a.presample_epochs, "alpha": plan.alpha, "topo_prefix_len": est.topo_prefix_len, "feat_prefix_len": est.feat_prefix_len,
                 "predicted_txn_per_epoch": pred_txn, "presample_txn_total": hot.sampling_txn_total},
        "pcie": {
            "measured_gb_per_batch": measured_txn * cls / batches / 1e9,
            "predicted_gb_per_batch": pred_txn * cls / clique_batches / 1e9,
            "measured_over_predicted": (measured_txn / batches) / (pred_txn / clique_batches) if pred_txn else None,
            "payload_gb_per_batch": (t["reads_host"] * 16 + t["edges_host"] * 4 + f["host"] * feat.row_bytes)
            / batches / 1e9,
            "unit_note": "transactions x 64 B cache lines, the reference's PCIe unit (SPEC.md:403)",
        },
        "tier_roofline": {
            "bytes_per_batch": {"hbm": hbm_b / batches, "nvlink": nvl_b / batches, "pcie": pcie_b / batches},
            "gbs": {"hbm": hbm_gbs, "nvlink": a.nvlink_gbs, "pcie": a.pcie_gbs},
            "t_us_per_batch": {k: v * 1e6 for k, v in t_tier.items()},
            "bound": max(t_tier, key=t_tier.get), "t_roof_us_per_batch": t_roof * 1e6,
            "measured_us_per_batch": t_meas * 1e6, "frac": t_roof / t_meas,
        },
        "lanes": a.lanes,
        "cuda_graph": bool(a.graph),
        "lane_sweep_batches_per_s": sweep,
        "tiers_per_batch": {**{k: v / batches for k, v in t.items()}, **{f"rows_{k}": v / batches for k, v in f.items()}},
        "stages_ms_per_epoch": stages,
        "setup_s": {"total": setup_s, "presampling": t_pre, "plan": t_plan, "cache_fill": t_fill},
    }
    if a.alpha_sweep:
        out["alpha_sweep"] = alpha_sweep(a, g, cfg, hot, orders, budget, feat, spec, layout, host_table, topo, pool, nb,
                                          plans[a.warmup], t_pre)
    print(json.dumps(out), flush=True)


def alpha_sweep(a, g, cfg, hot, orders, budget, feat, spec, layout, host_table, topo, pool, nb, plan_e, t_pre):
    """Cost-model validation on the device (the B200 counterpart of the reference's
    sweep-alpha, cli.py:276-340, judged as SPEC.md:542 does by rank correlation): the
    host tier's two access shapes are measured on this box, then one epoch is timed
    through a cache materialised at each alpha; predicted transactions (reference
    objective) and predicted seconds (measured-bandwidth objective) are rank-correlated
    with measured host transactions and measured epoch time."""
    import torch

    from paper_2305_16588_b200 import bandwidth as BW
    from paper_2305_16588_b200 import planner as PL
    from paper_2305_16588_b200.cache import FeatureStore, TopologyStore
    from paper_2305_16588_b200.pipeline import SampleGatherPipeline

    full = g.device("host")
    hbm = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else None
    probe = BW.measure_host_tier(full.c_struct.col_indices, g.num_edges * 4, host_table.data_ptr(),
                                 host_table.numel() * 4, feat, spec, hbm_gbs=hbm)
    bw = BW.calibrate_host_tier(g, np.asarray(pool)[: 64 * cfg.batch_size], cfg.fanouts, cfg.batch_size,
                                host_table.data_ptr(), host_table.numel() * 4, feat, spec, hbm_gbs=hbm)
    pts = PL.sweep_alpha(orders, budget, 0.01, g, feat, spec, hot.sampling_txn_total, bw)
    pts_probe = PL.sweep_alpha(orders, budget, 0.01, g, feat, spec, hot.sampling_txn_total, probe)
    p_probe, _ = PL.search_optimal_plan(orders, budget, 0.01, g, feat, spec, hot.sampling_txn_total, bandwidths=probe)
    p_txn, _ = PL.search_optimal_plan(orders, budget, 0.01, g, feat, spec, hot.sampling_txn_total)
    p_time, _ = PL.search_optimal_plan(orders, budget, 0.01, g, feat, spec, hot.sampling_txn_total, bandwidths=bw)
    step = max(1, (len(pts) - 1) // max(1, a.alpha_sweep - 1))
    idx = sorted(set(list(range(0, len(pts), step)) + [len(pts) - 1] +
                     [i for i, p in enumerate(pts) if p[0] in (p_txn.alpha, p_time.alpha, p_probe.alpha)]))
    rows = []
    row_txns = PL.feature_row_transactions(feat, spec)
    for i in idx:
        alpha, est, secs = pts[i]
        asg = PL.materialize_assignment([orders], [PL.CachePlan.from_alpha(budget, alpha)], layout, g, feat, spec)
        ts = TopologyStore(g, asg.topo_vertices, 0, host_full=True)
        fs = FeatureStore.from_assignment(host_table, asg.feat_vertices, 0)
        pipe = SampleGatherPipeline(g, cfg, fs, len(pool), window=min(a.window, nb), feat_rows_cap=60_000,
                                    topology=ts, lanes=a.lanes)
        pipe.run_epoch(plan_e)  # warm-up
        torch.cuda.synchronize()
        ts.reset_counters()
        fs.reset_counters()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pipe.run_epoch(plan_e)
        e1.record()
        torch.cuda.synchronize()
        tc, fc = ts.tier_counts(), fs.tier_counts()
        rows.append({"alpha": alpha, "predicted_txn": est.total_txns, "predicted_s": secs,
                     "predicted_s_probe": pts_probe[i][2],
                     "measured_host_txn": tc["host_txn"] + fc["host"] * row_txns,
                     "measured_ms": e0.elapsed_time(e1)})
        del pipe, ts, fs, asg
        torch.cuda.empty_cache()
    col = lambda k: [r[k] for r in rows]  # noqa: E731
    best = min(rows, key=lambda r: r["measured_ms"])
    pick = lambda al: next(r for r in rows if r["alpha"] == al)  # noqa: E731
    return {
        "bandwidths": json.loads(bw.to_json()),
        "bandwidths_random_probe": json.loads(probe.to_json()),
        "points": rows,
        "spearman_txn_vs_measured_txn": BW.spearman(col("predicted_txn"), col("measured_host_txn")),
        "spearman_txn_vs_time": BW.spearman(col("predicted_txn"), col("measured_ms")),
        "spearman_seconds_vs_time": BW.spearman(col("predicted_s"), col("measured_ms")),
        "spearman_probe_seconds_vs_time": BW.spearman(col("predicted_s_probe"), col("measured_ms")),
        "alpha_probe_objective": p_probe.alpha,
        "alpha_txn_objective": p_txn.alpha, "alpha_time_objective": p_time.alpha,
        "measured_ms_txn_pick": pick(p_txn.alpha)["measured_ms"],
        "measured_ms_time_pick": pick(p_time.alpha)["measured_ms"],
        "measured_ms_probe_pick": pick(p_probe.alpha)["measured_ms"],
        "best_measured": {"alpha": best["alpha"], "ms": best["measured_ms"]},
        "note": "predicted seconds are host-tier (PCIe) time only; measured_ms is the whole epoch",
    }


if __name__ == "__main__":
    main()
