"""Generate the golden vectors of tests/golden/ from the reference itself.

Imports the unmodified reference (`gnncache` 0.1.0) read-only from
/root/reference/pkg/src (and its test helpers from /root/reference/pkg/tests) and
records its outputs on small seeded inputs. Run once in the build container:

    python tests/golden/make_golden.py

The .npz files are committed; nothing at test or bench time reads /root/reference.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("GNNCACHE_REF", "/root/reference/pkg"))
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
sys.dont_write_bytecode = True

from gnncache.graph import FeatureSpec, generate_synthetic, select_training_set  # noqa: E402
from gnncache.hardware import HardwareSpec, block_layout  # noqa: E402
from gnncache.partition import Partitioning, assign_tablets, split_intra_clique  # noqa: E402
from gnncache.planner import build_candidate_orders, materialize_assignment, search_optimal_plan  # noqa: E402
from gnncache.rng import KeyedRng, derive_seed, mix64  # noqa: E402
from gnncache.sampling import SamplingConfig, run_presampling, run_sampling_epoch, sample_batch  # noqa: E402
from gnncache.simulator import account_assignment  # noqa: E402
from helpers import random_graph  # noqa: E402

OUT = Path(__file__).resolve().parent


def rng_vectors():
    vals = np.array([0, 1, 17, 2**63, 2**64 - 1, 0xDEADBEEF, 0x9E3779B97F4A7C15, 2 * 0x9E3779B97F4A7C15 % 2**64],
                    dtype=np.uint64)
    d = {"mix64_in": vals, "mix64_out": np.array([mix64(int(v)) for v in vals], dtype=np.uint64)}
    paths = [(3, (0, 0, 0)), (3, (0, 0, 0, 2, 0, 0)), (7, (1, 2, 3)), (42, (1, 2)), (0, (1,)), (2**64 - 1, (5, 9))]
    d["derive_seed"] = np.array([p[0] for p in paths], dtype=np.uint64)
    d["derive_path"] = np.array([list(p[1]) + [-1] * (6 - len(p[1])) for p in paths], dtype=np.int64)
    d["derive_out"] = np.array([KeyedRng(s).derive(*c).key for s, c in paths], dtype=np.uint64)
    key = KeyedRng(3).derive(0, 0, 0).derive(2, 0).derive(0).key
    a = np.arange(0, 64, dtype=np.int64).repeat(3)
    b = np.tile(np.array([0, 5, 31], dtype=np.int64), 64)
    d["pairs_key"] = np.array([key], dtype=np.uint64)
    d["pairs_a"], d["pairs_b"] = a, b
    d["pairs_out"] = KeyedRng(key).hash_pairs(a, b)
    d["counters_out"] = KeyedRng(key).hash_counters(np.arange(100))
    for n in (0, 1, 2, 17, 257, 5000):
        d[f"perm_{n}"] = KeyedRng(11).derive(4).permutation(n)
    d["perm_key"] = np.array([KeyedRng(11).derive(4).key], dtype=np.uint64)
    np.savez_compressed(OUT / "rng.npz", **d)


GRAPHS = [
    # name, builder
    ("syn_d10", lambda: generate_synthetic(2000, 10, 1.2, seed=3)),
    ("syn_d26", lambda: generate_synthetic(3000, 26, 1.2, seed=5)),
    ("syn_d40", lambda: generate_synthetic(1500, 40, 1.0, seed=7)),
    ("syn_d70", lambda: generate_synthetic(1200, 70, 0.8, seed=9)),
    ("syn_d150", lambda: generate_synthetic(900, 150, 1.1, seed=13)),
    ("rand_d9", lambda: random_graph(np.random.default_rng(11), 80, 9)),
    ("rand_d40", lambda: random_graph(np.random.default_rng(12), 300, 40)),
]

CASES = [
    # graph, fanouts, nseeds, seed-key path
    ("syn_d10", (25, 10), 64, (1, 0, 0, 0)),
    ("syn_d26", (15, 10, 5), 48, (2, 1, 0, 1)),
    ("syn_d26", (40,), 100, (3, 0, 1, 2)),
    ("syn_d40", (25, 10), 32, (4, 0, 0, 0)),
    ("syn_d40", (33, 3), 40, (5, 0, 0, 7)),
    ("syn_d70", (25, 10), 24, (6, 2, 0, 3)),
    ("syn_d70", (64, 2), 20, (6, 2, 0, 4)),
    ("syn_d150", (25, 10), 16, (7, 0, 0, 0)),
    ("syn_d150", (140, 1), 8, (7, 1, 0, 0)),
    ("rand_d9", (3, 2), 12, (8, 0, 0, 0)),
    ("rand_d9", (1, 1, 1, 1), 5, (8, 0, 0, 1)),
    ("rand_d40", (25, 10), 30, (9, 0, 0, 0)),
    ("rand_d40", (5, 5, 5), 10, (9, 0, 1, 0)),
]


def sampling_vectors():
    graphs = {name: build() for name, build in GRAPHS}
    d = {}
    for name, g in graphs.items():
        d[f"g_{name}_ro"] = g.row_offsets
        d[f"g_{name}_ci"] = g.col_indices
    for i, (gname, fanouts, nseeds, path) in enumerate(CASES):
        g = graphs[gname]
        rs = np.random.default_rng(100 + i)
        seeds = rs.integers(0, g.num_vertices, size=nseeds).astype(np.int64)
        stream = KeyedRng(path[0]).derive(*path[1:])
        cfg = SamplingConfig(fanouts=fanouts, batch_size=nseeds)
        batch = sample_batch(g, seeds, cfg, stream)
        d[f"c{i}_graph"] = np.array(gname)
        d[f"c{i}_fanouts"] = np.array(fanouts, dtype=np.int64)
        d[f"c{i}_key"] = np.array([stream.key], dtype=np.uint64)
        d[f"c{i}_seeds"] = seeds
        for h, hop in enumerate(batch.hops):
            d[f"c{i}_h{h}_src"] = np.asarray(hop.sources, dtype=np.int64)
            d[f"c{i}_h{h}_off"] = np.asarray(hop.offsets, dtype=np.int64)
            d[f"c{i}_h{h}_nbr"] = np.asarray(hop.neighbors, dtype=np.int64)
        d[f"c{i}_distinct"] = batch.distinct_vertices()
    d["num_cases"] = np.array(len(CASES))
    np.savez_compressed(OUT / "sampling.npz", **d)


def presampling_vectors():
    d = {}
    configs = [
        # (n, deg, skew, gseed, gpus, clique, fanouts, batch, epochs, seed)
        (400, 10, 1.0, 2, 4, 2, (5, 3), 16, 1, 21),
        (600, 26, 1.2, 4, 2, 2, (15, 10, 5), 32, 2, 3),
        (500, 40, 1.1, 6, 1, 1, (25, 10), 50, 1, 9),
    ]
    for i, (n, deg, skew, gseed, gpus, clique, fanouts, bs, epochs, seed) in enumerate(configs):
        g = generate_synthetic(n, deg, skew, seed=gseed)
        layout = block_layout(gpus, clique)
        spec = HardwareSpec(layout, clique_budget_bytes=1 << 20)
        pools = [np.arange(j, n, gpus + 3, dtype=np.int64) for j in range(gpus)]
        cfg = SamplingConfig(fanouts=fanouts, batch_size=bs, presample_epochs=epochs, seed=seed)
        hot = run_presampling(g, pools, layout, cfg, spec)
        d[f"p{i}_cfg"] = np.array([n, deg, gseed, gpus, clique, bs, epochs, seed], dtype=np.int64)
        d[f"p{i}_skew"] = np.array([skew])
        d[f"p{i}_fanouts"] = np.array(fanouts, dtype=np.int64)
        for ci, h in enumerate(hot):
            d[f"p{i}_c{ci}_HT"] = h.topo_hotness
            d[f"p{i}_c{ci}_HF"] = h.feat_hotness
            d[f"p{i}_c{ci}_txn"] = np.array([h.sampling_txn_total], dtype=np.int64)
        traces = run_sampling_epoch(g, pools, layout, cfg, seed, 0)
        for gi, tr in enumerate(traces):
            d[f"p{i}_t{gi}_reads"] = tr.topo_reads
            d[f"p{i}_t{gi}_looks"] = tr.feat_lookups
            d[f"p{i}_t{gi}_trav"] = tr.edge_traversals
            d[f"p{i}_t{gi}_nb"] = np.array([tr.num_batches])
    d["num_configs"] = np.array(len(configs))
    np.savez_compressed(OUT / "presampling.npz", **d)


def planner_vectors():
    d = {}
    g = generate_synthetic(3000, 12, 1.2, seed=31)
    layout = block_layout(4, 4)
    feat = FeatureSpec(100)
    train = select_training_set(g, 0.1, seed=derive_seed(7, 2))
    tablets = split_intra_clique(train, Partitioning(np.zeros(g.num_vertices, dtype=np.int32), 1), layout)
    pools = assign_tablets(tablets, layout)
    d["train_ids"] = train.vertex_ids
    for gi, p in enumerate(pools):
        d[f"pool{gi}"] = p
    budget = 200_000
    spec = HardwareSpec(layout, clique_budget_bytes=budget)
    cfg = SamplingConfig(fanouts=(10, 5), batch_size=64, presample_epochs=1, seed=derive_seed(7, 4))
    hot = run_presampling(g, pools, layout, cfg, spec)[0]
    orders = build_candidate_orders(hot)
    plan, est = search_optimal_plan(orders, budget, 0.01, g, feat, spec, hot.sampling_txn_total)
    asg = materialize_assignment([orders], [plan], layout, g, feat, spec)
    d["HT"], d["HF"], d["txn"] = hot.topo_hotness, hot.feat_hotness, np.array([hot.sampling_txn_total])
    for k in ("topo_totals", "feat_totals", "topo_order", "feat_order", "topo_owner", "feat_owner"):
        d[k] = getattr(orders, k)
    d["alpha"] = np.array([plan.alpha])
    d["est"] = np.array([est.sampling_txns, est.feature_txns, est.total_txns, est.topo_prefix_len, est.feat_prefix_len],
                        dtype=np.float64)
    for gi in range(layout.num_gpus):
        d[f"asg_topo{gi}"] = asg.topo_vertices[gi]
        d[f"asg_feat{gi}"] = asg.feat_vertices[gi]
        d[f"asg_bytes{gi}"] = np.array([asg.topo_bytes[gi], asg.feat_bytes[gi]])
    traces = run_sampling_epoch(g, pools, layout, cfg, derive_seed(7, 5), 0)
    rep = account_assignment(traces, asg, layout, g, spec, feat)
    for k in ("sampling_cpu_txn", "sampling_peer_txn", "feature_cpu_txn", "feature_peer_txn", "topo_reads",
              "topo_local_hits", "topo_peer_hits", "feat_lookups", "feat_local_hits", "feat_peer_hits",
              "traffic_matrix"):
        d[f"rep_{k}"] = getattr(rep, k)
    d["graph_ro"], d["graph_ci"] = g.row_offsets, g.col_indices
    d["budget"] = np.array([budget])
    np.savez_compressed(OUT / "planner.npz", **d)


def policy_vectors():
    """run_policy_pipeline for every cache policy (simulator.py:259-402) on two layouts;
    the LDG partitions the reference computes (partition.py:85-130) are recorded too,
    so the device side can be fed the same partitioning."""
    from gnncache.partition import partition_inter_clique
    from gnncache.simulator import POLICY_VARIANTS, CachePolicy, run_policy_pipeline

    d = {}
    g = generate_synthetic(2500, 10, 1.2, seed=41)
    train = select_training_set(g, 0.1, seed=derive_seed(5, 2))
    feat = FeatureSpec(64)
    cfg = SamplingConfig(fanouts=(8, 4), batch_size=32, presample_epochs=1, seed=derive_seed(5, 4))
    d["graph_ro"], d["graph_ci"], d["train_ids"] = g.row_offsets, g.col_indices, train.vertex_ids
    cases = []
    for li, (ngpu, csize) in enumerate([(4, 2), (4, 4)]):
        layout = block_layout(ngpu, csize)
        spec = HardwareSpec(layout, clique_budget_bytes=60_000 * csize)
        for n_parts in {layout.clique_count, layout.num_gpus}:
            part = partition_inter_clique(g, n_parts, 0.05, derive_seed(5, 0x52))
            d[f"L{li}_part{n_parts}"] = part.assignments
        for vi, variant in enumerate(POLICY_VARIANTS):
            for ri, kw in enumerate([{"cache_ratio": 0.05}, {"budget_bytes": 40_000}]):
                policy = CachePolicy(variant, **kw)
                run = run_policy_pipeline(policy, g, train, layout, cfg, spec, feat, master_seed=5, epsilon=0.05)
                key = f"L{li}_v{vi}_r{ri}"
                cases.append((li, vi, ri))
                for gi in range(run.layout.num_gpus):
                    d[f"{key}_pool{gi}"] = run.pools[gi]
                    d[f"{key}_topo{gi}"] = run.assignment.topo_vertices[gi]
                    d[f"{key}_feat{gi}"] = run.assignment.feat_vertices[gi]
                d[f"{key}_cpu_txn"] = np.array([run.report.total_cpu_txn])
                d[f"{key}_matrix"] = run.report.traffic_matrix
                d[f"{key}_csize"] = np.array([run.layout.clique_size])
    d["cases"] = np.array(cases, dtype=np.int64)
    d["variants"] = np.array(POLICY_VARIANTS)
    np.savez_compressed(OUT / "policies.npz", **d)


def partition_vectors():
    """partition_inter_clique (partition.py:85-130) over graphs with self loops,
    duplicate edges, isolated vertices and several components, for a grid of part
    counts, imbalance and refinement passes; edge_cut_ratio of each result."""
    from gnncache.graph import CsrGraph
    from gnncache.partition import edge_cut_ratio, partition_inter_clique

    d = {}
    rng = np.random.default_rng(77)
    graphs = [generate_synthetic(3000, 8, 1.2, seed=3), random_graph(rng, 700, 6)]
    # self loops + duplicates + isolated tail + a second component
    src = np.array([0, 0, 1, 2, 2, 3, 5, 6, 6, 9, 9, 10, 11], dtype=np.int64)
    dst = np.array([0, 1, 1, 3, 3, 2, 6, 5, 7, 10, 9, 11, 9], dtype=np.int64)
    graphs.append(CsrGraph.from_edges(16, src, dst))
    cases = []
    for gi, g in enumerate(graphs):
        d[f"g{gi}_ro"], d[f"g{gi}_ci"] = g.row_offsets, g.col_indices
        for parts in (2, 3, 5, 8):
            for eps in (0.0, 0.05, 0.3):
                for passes in (0, 1, 2, 5):
                    for seed in (0, 1234):
                        if parts > g.num_vertices:
                            continue
                        part = partition_inter_clique(g, parts, eps, seed, passes)
                        k = len(cases)
                        d[f"c{k}"] = part.assignments
                        d[f"c{k}_cut"] = np.array([edge_cut_ratio(g, part)])
                        cases.append((gi, parts, int(eps * 100), passes, seed))
    d["cases"] = np.array(cases, dtype=np.int64)
    np.savez_compressed(OUT / "partition.npz", **d)


def hardware_vectors():
    """detect_cliques (hardware.py:109-139) on random symmetric NVLink matrices (some
    decompose into unequal cliques and raise) and block matrices; save/load text."""
    import tempfile

    from gnncache.hardware import HeterogeneousTopologyError, NvlinkMatrix, detect_cliques, save_hardware_config

    rng = np.random.default_rng(5)
    d = {}
    mats = []
    for n in (1, 2, 3, 4, 6, 8, 8, 10, 12):
        for p in (0.3, 0.6, 0.9):
            a = rng.random((n, n)) < p
            a = np.triu(a, 1)
            mats.append(a | a.T | np.eye(n, dtype=bool))
    for n, c in ((8, 2), (8, 4), (8, 8), (12, 3)):
        blk = np.arange(n) // c
        mats.append(blk[:, None] == blk[None, :])
    # equal-size cliques with ties between several maximum cliques
    ring = np.eye(6, dtype=bool)
    for i in range(6):
        ring[i, (i + 1) % 6] = ring[(i + 1) % 6, i] = True
    mats.append(ring)
    for k, a in enumerate(mats):
        d[f"m{k}"] = a
        try:
            lay = detect_cliques(NvlinkMatrix(a))
            d[f"m{k}_cliques"] = np.array([g for c in lay.cliques for g in c], dtype=np.int64)
            d[f"m{k}_size"] = np.array([lay.clique_size])
        except HeterogeneousTopologyError:
            d[f"m{k}_size"] = np.array([-1])
    d["count"] = np.array([len(mats)])
    from gnncache.hardware import HardwareSpec, block_layout

    with tempfile.TemporaryDirectory() as tmp:
        path = Path(tmp) / "hw.txt"
        save_hardware_config(HardwareSpec(block_layout(8, 4), 123456, 128), path)
        d["saved_text"] = np.array([path.read_text()])
    np.savez_compressed(OUT / "hardware.npz", **d)


def sweep_vectors():
    """sweep_gpus (simulator.py:412-441) for two policies over 1/2/4 GPUs."""
    from gnncache.simulator import CachePolicy, sweep_gpus

    g = generate_synthetic(2000, 8, 1.2, seed=43)
    train = select_training_set(g, 0.1, seed=derive_seed(6, 2))
    cfg = SamplingConfig(fanouts=(6, 3), batch_size=32, presample_epochs=1, seed=derive_seed(6, 4))
    d = {"graph_ro": g.row_offsets, "graph_ci": g.col_indices, "train_ids": train.vertex_ids}
    for name, policy in (("hier", CachePolicy("legion-hierarchical", cache_ratio=0.05)),
                         ("pagraph", CachePolicy("pagraph-plus", budget_bytes=30_000))):
        pts = sweep_gpus(policy, [4, 1, 2], g, train, cfg, FeatureSpec(32), clique_size=2, seed=9)
        d[f"{name}_counts"] = np.array([p.gpu_count for p in pts])
        d[f"{name}_txn"] = np.array([p.total_cpu_txn for p in pts])
        d[f"{name}_norm"] = np.array([p.normalized for p in pts])
    np.savez_compressed(OUT / "sweep.npz", **d)


def report_vectors():
    """write_report_csv / write_traffic_matrix_csv (simulator.py:444-470) of one policy
    run, and plan_report (planner.py:322-351) of the hierarchical plan."""
    import json
    import tempfile

    from gnncache.planner import plan_report
    from gnncache.simulator import CachePolicy, run_policy_pipeline, write_report_csv, write_traffic_matrix_csv

    g = generate_synthetic(2000, 8, 1.2, seed=43)
    train = select_training_set(g, 0.1, seed=derive_seed(6, 2))
    cfg = SamplingConfig(fanouts=(6, 3), batch_size=32, presample_epochs=1, seed=derive_seed(6, 4))
    layout = block_layout(4, 2)
    spec = HardwareSpec(layout, clique_budget_bytes=50_000)
    feat = FeatureSpec(32)
    run = run_policy_pipeline(CachePolicy("legion-hierarchical"), g, train, layout, cfg, spec, feat, master_seed=3)
    d = {"graph_ro": g.row_offsets, "graph_ci": g.col_indices, "train_ids": train.vertex_ids}
    with tempfile.TemporaryDirectory() as tmp:
        write_report_csv(run.report, Path(tmp) / "r.csv", provenance="seed 3")
        write_traffic_matrix_csv(run.report, Path(tmp) / "m.csv")
        d["report_csv"] = np.array([(Path(tmp) / "r.csv").read_text()])
        d["matrix_csv"] = np.array([(Path(tmp) / "m.csv").read_text()])
    orders = [build_candidate_orders(h) for h in run.hotness]
    plans, ests = zip(*[search_optimal_plan(o, spec.clique_budget_bytes, 0.05, g, feat, spec, h.sampling_txn_total)
                        for o, h in zip(orders, run.hotness)])
    d["plan_report"] = np.array([json.dumps(plan_report(layout, list(plans), list(ests), 0.05, [[3, 4], [5, 6]]),
                                            sort_keys=True)])
    np.savez_compressed(OUT / "reports.npz", **d)


def format_vectors():
    """Files the reference itself writes: an LGCSR1 graph (save_csr, graph.py:112-117)
    and the u32 hotness dump of a 2-clique presampling (write_hotness,
    sampling.py:292-303), stored byte for byte, plus what load_csr/read_hotness return."""
    import tempfile

    from gnncache.graph import load_csr, save_csr
    from gnncache.sampling import read_hotness, write_hotness

    g = generate_synthetic(600, 7, 1.1, seed=21)
    train = select_training_set(g, 0.2, seed=5)
    layout = block_layout(4, 2)
    spec = HardwareSpec(layout, clique_budget_bytes=10_000)
    tablets = split_intra_clique(train, Partitioning(np.array([v % 2 for v in range(600)]), 2), layout)
    cfg = SamplingConfig(fanouts=(5, 3), batch_size=16, presample_epochs=2, seed=17)
    hot = run_presampling(g, tablets, layout, cfg, spec)
    d = {"graph_ro": g.row_offsets, "graph_ci": g.col_indices}
    with tempfile.TemporaryDirectory() as tmp:
        save_csr(g, Path(tmp) / "g.lgcsr")
        write_hotness(Path(tmp) / "h.bin", hot)
        d["lgcsr1_bytes"] = np.frombuffer((Path(tmp) / "g.lgcsr").read_bytes(), dtype=np.uint8)
        d["hotness_bytes"] = np.frombuffer((Path(tmp) / "h.bin").read_bytes(), dtype=np.uint8)
        back = read_hotness(Path(tmp) / "h.bin")
        assert np.array_equal(load_csr(Path(tmp) / "g.lgcsr").col_indices, g.col_indices)
    for ci, h in enumerate(back):
        d[f"hot{ci}_topo"] = h.topo_hotness
        d[f"hot{ci}_feat"] = h.feat_hotness
        d[f"hot{ci}_txn"] = np.array([h.sampling_txn_total], dtype=np.int64)
        d[f"hot{ci}_id"] = np.array([h.clique_id], dtype=np.int64)
    d["num_cliques"] = np.array([len(back)])
    np.savez_compressed(OUT / "formats.npz", **d)


if __name__ == "__main__":
    if "--formats" in sys.argv:
        format_vectors()
        raise SystemExit(0)
    if "--reports" in sys.argv:
        report_vectors()
        raise SystemExit(0)
    if "--sweep" in sys.argv:
        sweep_vectors()
        raise SystemExit(0)
    if "--hardware" in sys.argv:
        hardware_vectors()
        raise SystemExit(0)
    if "--policies" in sys.argv:
        policy_vectors()
        raise SystemExit(0)
    if "--partition" in sys.argv:
        partition_vectors()
        raise SystemExit(0)
    rng_vectors()
    sampling_vectors()
    presampling_vectors()
    planner_vectors()
    policy_vectors()
    partition_vectors()
    hardware_vectors()
    sweep_vectors()
    report_vectors()
    format_vectors()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
