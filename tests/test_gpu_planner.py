"""Cost-model kernels (K6/K7) vs the reference's golden plan and the CPU oracle."""

import numpy as np
import pytest

import gnncache_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _device():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    torch.cuda.set_device(0)


def _golden_setup(golden):
    import paper_2305_16588_b200 as P

    g = golden("planner")
    graph = P.CsrGraph(len(g["graph_ro"]) - 1, len(g["graph_ci"]), g["graph_ro"], g["graph_ci"])
    layout = P.block_layout(4, 4)
    spec = P.HardwareSpec(layout, clique_budget_bytes=int(g["budget"][0]))
    hot = P.HotnessMatrices(0, g["HT"].copy(), g["HF"].copy(), int(g["txn"][0]))
    return P, g, graph, layout, spec, hot


def test_candidate_orders_plan_and_assignment_match_reference(golden):
    P, g, graph, layout, spec, hot = _golden_setup(golden)
    from paper_2305_16588_b200 import planner as PL

    orders = PL.build_candidate_orders(hot)
    for k in ("topo_totals", "feat_totals", "topo_order", "feat_order", "topo_owner", "feat_owner"):
        assert np.array_equal(getattr(orders, k), g[k]), k
    for gi in range(4):
        assert np.array_equal(orders.gpu_topo_queues[gi], g["topo_order"][g["topo_owner"][g["topo_order"]] == gi])
        assert np.array_equal(orders.gpu_feat_queues[gi], g["feat_order"][g["feat_owner"][g["feat_order"]] == gi])
    feat = P.FeatureSpec(100)
    plan, est = PL.search_optimal_plan(orders, int(g["budget"][0]), 0.01, graph, feat, spec, hot.sampling_txn_total)
    assert plan.alpha == g["alpha"][0]
    assert [est.sampling_txns, est.feature_txns, est.total_txns, est.topo_prefix_len, est.feat_prefix_len] == \
        [float(x) for x in g["est"]]
    again = PL.estimate_traffic(orders, plan, graph, feat, spec, hot.sampling_txn_total)
    assert again == est
    asg = PL.materialize_assignment([orders], [plan], layout, graph, feat, spec)
    for gi in range(4):
        assert np.array_equal(asg.topo_vertices[gi], g[f"asg_topo{gi}"])
        assert np.array_equal(asg.feat_vertices[gi], g[f"asg_feat{gi}"])
        assert [asg.topo_bytes[gi], asg.feat_bytes[gi]] == list(g[f"asg_bytes{gi}"])


def test_boundaries_match_linear_scan(golden):
    P, g, graph, layout, spec, hot = _golden_setup(golden)
    from paper_2305_16588_b200 import planner as PL

    orders = PL.build_candidate_orders(hot)
    deg = graph.out_degrees[orders.topo_order]
    costs = deg * 4 + 8
    feat = P.FeatureSpec(100)
    for budget in (0.0, 7.5, 8.0, 1000.0, 12345.6, float(costs.sum()), float(costs.sum()) + 1):
        total, want = 0, len(costs)
        for i, c in enumerate(costs):
            total += int(c)
            if total > budget:
                want = i
                break
        assert PL.boundary_topology(orders, budget, graph, spec) == want
        assert PL.boundary_feature(orders, budget, feat) == min(len(orders.feat_order), int(budget // 400))
    with pytest.raises(ValueError):
        PL.boundary_topology(orders, -1.0, graph, spec)


@pytest.mark.parametrize("n,k,hi", [(2_000_003, 8, 5), (300_000, 3, 1000), (100_000, 1, 2**40), (50_000, 2, 1),
                                    (70_001, 2, 2**61)])
def test_ranking_with_heavy_ties_matches_lexsort(n, k, hi):
    """Stable descending sort: ties (many, with small hi) must stay in ascending-id order.
    The radix sort runs only the digit passes below the largest total's top bit: all
    totals zero (hi=1) runs none, totals near 2^62 (hi=2^61, k=2) run all eight."""
    from paper_2305_16588_b200 import planner as PL

    rng = np.random.default_rng(n)
    rows = rng.integers(0, hi, size=(k, n)).astype(np.int64)
    hot = PL.HotnessMatrices(0, rows, rows[::-1].copy(), 0)
    orders = PL.build_candidate_orders(hot)
    want = O.candidate_orders(rows, rows[::-1].copy())
    for key in ("topo_totals", "topo_order", "topo_owner", "feat_order", "feat_owner"):
        assert np.array_equal(getattr(orders, key), want[key]), key


def test_plan_search_matches_oracle_on_generated_hotness():
    import paper_2305_16588_b200 as P
    from paper_2305_16588_b200 import planner as PL

    g = P.generate_synthetic(50_000, 14, 1.1, seed=5)
    layout = P.block_layout(2, 2)
    rng = np.random.default_rng(2)
    ht = rng.zipf(1.5, size=(2, g.num_vertices)).astype(np.int64) % 1000
    hf = rng.zipf(1.3, size=(2, g.num_vertices)).astype(np.int64) % 1000
    hot = P.HotnessMatrices(0, ht, hf, 123_456_789)
    feat = P.FeatureSpec(128)
    for budget in (1_000_000, 20_000_000, 10**12):
        spec = P.HardwareSpec(layout, clique_budget_bytes=budget)
        orders = PL.build_candidate_orders(hot)
        plan, est = PL.search_optimal_plan(orders, budget, 0.01, g, feat, spec, hot.sampling_txn_total)
        o = O.candidate_orders(ht, hf)
        alpha, total, bt, bf, samp, fe = O.plan_search(o, g.row_offsets, budget, 0.01, 512, hot.sampling_txn_total)
        assert (plan.alpha, est.total_txns, est.topo_prefix_len, est.feat_prefix_len) == (alpha, total, bt, bf)


def test_account_assignment_matches_reference_report(golden):
    """Device tier accounting of the reference's golden epoch equals its TrafficReport."""
    P, g, graph, layout, spec, hot = _golden_setup(golden)
    from paper_2305_16588_b200 import planner as PL
    from paper_2305_16588_b200.simulator import account_assignment, hit_rate_summary, simulate_epoch

    feat = P.FeatureSpec(100)
    asg = PL.CacheAssignment(
        4, [g[f"asg_topo{i}"] for i in range(4)], [g[f"asg_feat{i}"] for i in range(4)],
        [int(g[f"asg_bytes{i}"][0]) for i in range(4)], [int(g[f"asg_bytes{i}"][1]) for i in range(4)])
    pools = [g[f"pool{i}"] for i in range(4)]
    cfg = P.SamplingConfig(fanouts=(10, 5), batch_size=64, presample_epochs=1, seed=P.derive_seed(7, 4))
    rep = simulate_epoch(graph, pools, cfg, asg, layout, spec, feat, seed=P.derive_seed(7, 5))
    for k in ("sampling_cpu_txn", "sampling_peer_txn", "feature_cpu_txn", "feature_peer_txn", "topo_reads",
              "topo_local_hits", "topo_peer_hits", "feat_lookups", "feat_local_hits", "feat_peer_hits",
              "traffic_matrix"):
        assert np.array_equal(getattr(rep, k), g[f"rep_{k}"]), k
    s = hit_rate_summary(rep)
    assert 0.0 <= s.aggregate_feat <= 1.0 and 0.0 <= s.aggregate_topo <= 1.0
    traces = P.run_sampling_epoch(graph, pools, layout, cfg, P.derive_seed(7, 5), 0)
    assert np.array_equal(account_assignment(traces, asg, layout, graph, spec, feat).traffic_matrix,
                          g["rep_traffic_matrix"])


def test_time_objective_with_uniform_bandwidth_picks_the_transaction_optimum(golden):
    """With one GB/s for both access shapes the predicted seconds are the reference's
    N_total x 64 B / bandwidth (feature rows cost ceil(row/CLS) lines; here 100-d rows
    are 400 B = 6.25 lines, so the seconds use 400 B, not 7 x 64): the picks agree
    whenever the row is a whole number of lines, and every grid point's estimate is the
    reference's."""
    P, g, graph, layout, spec, hot = _golden_setup(golden)
    from paper_2305_16588_b200 import planner as PL
    from paper_2305_16588_b200.bandwidth import MeasuredBandwidths, estimate_seconds

    orders = PL.build_candidate_orders(hot)
    feat = P.FeatureSpec(128)  # 512 B = 8 whole lines
    bw = MeasuredBandwidths(10.0, 10.0)
    plan_t, est_t = PL.search_optimal_plan(orders, spec.clique_budget_bytes, 0.01, graph, feat, spec,
                                           hot.sampling_txn_total)
    plan_s, est_s = PL.search_optimal_plan(orders, spec.clique_budget_bytes, 0.01, graph, feat, spec,
                                           hot.sampling_txn_total, bandwidths=bw)
    assert plan_s.alpha == plan_t.alpha and est_s == est_t
    pts = PL.sweep_alpha(orders, spec.clique_budget_bytes, 0.01, graph, feat, spec, hot.sampling_txn_total, bw)
    assert [p[0] for p in pts] == PL.alpha_grid(0.01)
    for alpha, est, secs in pts:
        want = PL.estimate_traffic(orders, PL.CachePlan.from_alpha(spec.clique_budget_bytes, alpha), graph, feat,
                                   spec, hot.sampling_txn_total)
        assert est == want
        assert secs == pytest.approx(est.total_txns * 64 / 10e9, rel=1e-12)
        assert secs == estimate_seconds(est, feat, spec, bw)


def test_time_objective_prefers_the_slower_access_shape(golden):
    """Making topology reads 20x slower per byte can only move the pick toward caching
    more topology (alpha up), never less."""
    P, g, graph, layout, spec, hot = _golden_setup(golden)
    from paper_2305_16588_b200 import planner as PL
    from paper_2305_16588_b200.bandwidth import MeasuredBandwidths

    orders = PL.build_candidate_orders(hot)
    feat = P.FeatureSpec(128)
    base, _ = PL.search_optimal_plan(orders, spec.clique_budget_bytes, 0.01, graph, feat, spec,
                                     hot.sampling_txn_total, bandwidths=MeasuredBandwidths(10.0, 10.0))
    slow, _ = PL.search_optimal_plan(orders, spec.clique_budget_bytes, 0.01, graph, feat, spec,
                                     hot.sampling_txn_total, bandwidths=MeasuredBandwidths(0.5, 10.0))
    fast, _ = PL.search_optimal_plan(orders, spec.clique_budget_bytes, 0.01, graph, feat, spec,
                                     hot.sampling_txn_total, bandwidths=MeasuredBandwidths(200.0, 10.0))
    assert fast.alpha <= base.alpha <= slow.alpha


@pytest.mark.parametrize("supplied", [True, False])
def test_cache_policies_match_reference(golden, supplied):
    """run_policy_pipeline for all four policies (simulator.py:259-402) on 4 GPUs as two
    cliques of 2 and one clique of 4, two size parameters each: seed pools, cache
    contents and the epoch's CPU transactions / traffic matrix equal the reference's
    (supplied: the reference's own LDG partitions from the golden file; else the
    pipeline partitions the graph itself, device permutation + gc_partition_ldg)."""
    import warnings

    import paper_2305_16588_b200 as P
    from paper_2305_16588_b200 import simulator as S

    g = golden("policies")
    graph = P.CsrGraph(len(g["graph_ro"]) - 1, len(g["graph_ci"]), g["graph_ro"], g["graph_ci"])
    train = P.TrainingSet(g["train_ids"], 0.1)
    feat = P.FeatureSpec(64)
    cfg = P.SamplingConfig(fanouts=(8, 4), batch_size=32, presample_epochs=1, seed=P.derive_seed(5, 4))
    for li, vi, ri in g["cases"]:
        ngpu, csize = [(4, 2), (4, 4)][li]
        layout = P.block_layout(ngpu, csize)
        spec = P.HardwareSpec(layout, clique_budget_bytes=60_000 * csize)
        variant = str(g["variants"][vi])
        policy = S.CachePolicy(variant, **[{"cache_ratio": 0.05}, {"budget_bytes": 40_000}][ri])
        parts_needed = ngpu if variant == S.POLICY_PAGRAPH else layout.clique_count
        part = P.Partitioning(g[f"L{li}_part{parts_needed}"], parts_needed)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            run = S.run_policy_pipeline(policy, graph, train, layout, cfg, spec, feat, master_seed=5, epsilon=0.05,
                                        partitioning=part if supplied else None)
        key = f"L{li}_v{vi}_r{ri}"
        assert run.layout.clique_size == int(g[f"{key}_csize"][0])
        for gi in range(ngpu):
            assert np.array_equal(run.pools[gi], g[f"{key}_pool{gi}"]), (key, gi)
            assert np.array_equal(run.assignment.topo_vertices[gi], g[f"{key}_topo{gi}"]), (key, gi)
            assert np.array_equal(run.assignment.feat_vertices[gi], g[f"{key}_feat{gi}"]), (key, gi)
        assert run.report.total_cpu_txn == int(g[f"{key}_cpu_txn"][0]), key
        assert np.array_equal(run.report.traffic_matrix, g[f"{key}_matrix"]), key


def test_partition_inter_clique_matches_reference(golden):
    """partition_inter_clique on the device box (BFS roots by gc_permutation, LDG by
    gc_partition_ldg) gives the reference's partitions; a partition with the wrong
    part count is rejected by the policy pipeline."""
    import paper_2305_16588_b200 as P
    from paper_2305_16588_b200 import simulator as S

    g = golden("partition")
    for k, (gi, parts, eps100, passes, seed) in enumerate(g["cases"]):
        if k % 7:  # every 7th case here; all of them run on CPU in test_partition_cpu.py
            continue
        graph = P.CsrGraph(len(g[f"g{gi}_ro"]) - 1, len(g[f"g{gi}_ci"]), g[f"g{gi}_ro"], g[f"g{gi}_ci"])
        part = P.partition_inter_clique(graph, int(parts), eps100 / 100.0, int(seed), int(passes))
        assert np.array_equal(part.assignments, g[f"c{k}"]), k
        assert P.edge_cut_ratio(graph, part) == float(g[f"c{k}_cut"][0])
    graph = P.generate_synthetic(500, 6, 1.2, seed=1)
    train = P.select_training_set(graph, 0.2, seed=3)
    with pytest.raises(ValueError):
        S.policy_seed_pools(S.CachePolicy(S.POLICY_PAGRAPH, cache_ratio=0.1), graph, train, P.block_layout(4, 2), 5,
                            partitioning=P.Partitioning(np.zeros(500, dtype=np.int32), 2))
    with pytest.raises(ValueError):
        P.partition_inter_clique(graph, 0)
    with pytest.raises(ValueError):
        P.partition_inter_clique(graph, 501)
    with pytest.raises(ValueError):
        P.partition_inter_clique(graph, 2, epsilon=-0.1)
    pools = S.policy_seed_pools(S.CachePolicy(S.POLICY_HIERARCHICAL, cache_ratio=0.1), graph, train,
                                P.block_layout(4, 4), 5)
    assert sorted(np.concatenate(pools).tolist()) == sorted(train.vertex_ids.tolist())


def test_sweep_gpus_matches_reference(golden):
    """sweep_gpus (simulator.py:412-441): per-GPU-count host transactions and their
    normalisation equal the reference's, for the hierarchical policy and pagraph-plus
    (which partitions the graph itself at every count)."""
    import paper_2305_16588_b200 as P

    g = golden("sweep")
    graph = P.CsrGraph(len(g["graph_ro"]) - 1, len(g["graph_ci"]), g["graph_ro"], g["graph_ci"])
    train = P.TrainingSet(g["train_ids"], 0.1)
    cfg = P.SamplingConfig(fanouts=(6, 3), batch_size=32, presample_epochs=1, seed=P.derive_seed(6, 4))
    for name, policy in (("hier", P.CachePolicy("legion-hierarchical", cache_ratio=0.05)),
                         ("pagraph", P.CachePolicy("pagraph-plus", budget_bytes=30_000))):
        pts = P.sweep_gpus(policy, [4, 1, 2], graph, train, cfg, P.FeatureSpec(32), clique_size=2, seed=9)
        assert [p.gpu_count for p in pts] == list(g[f"{name}_counts"])
        assert [p.total_cpu_txn for p in pts] == list(g[f"{name}_txn"]), name
        assert [p.normalized for p in pts] == list(g[f"{name}_norm"])


def test_probe_nvlink_matrix_layout():
    """The visible GPUs' peer table gives a valid clique layout (one clique per box)."""
    import torch

    import paper_2305_16588_b200 as P

    m = P.probe_nvlink_matrix()
    assert m.size == torch.cuda.device_count()
    lay = P.detect_cliques(m)
    assert lay.num_gpus == m.size


def test_reports_match_reference(golden, tmp_path):
    """write_report_csv / write_traffic_matrix_csv / plan_report produce the reference's
    text for the same policy run and plans (simulator.py:444-470, planner.py:322-351)."""
    import json

    import paper_2305_16588_b200 as P
    from paper_2305_16588_b200 import simulator as S
    from paper_2305_16588_b200.planner import plan_report

    g = golden("reports")
    graph = P.CsrGraph(len(g["graph_ro"]) - 1, len(g["graph_ci"]), g["graph_ro"], g["graph_ci"])
    train = P.TrainingSet(g["train_ids"], 0.1)
    cfg = P.SamplingConfig(fanouts=(6, 3), batch_size=32, presample_epochs=1, seed=P.derive_seed(6, 4))
    layout = P.block_layout(4, 2)
    spec = P.HardwareSpec(layout, clique_budget_bytes=50_000)
    feat = P.FeatureSpec(32)
    run = S.run_policy_pipeline(P.CachePolicy("legion-hierarchical"), graph, train, layout, cfg, spec, feat,
                                master_seed=3)
    S.write_report_csv(run.report, tmp_path / "r.csv", provenance="seed 3")
    S.write_traffic_matrix_csv(run.report, tmp_path / "m.csv")
    assert (tmp_path / "r.csv").read_text() == str(g["report_csv"][0])
    assert (tmp_path / "m.csv").read_text() == str(g["matrix_csv"][0])
    orders = [P.build_candidate_orders(h) for h in run.hotness]
    plans, ests = zip(*[P.search_optimal_plan(o, spec.clique_budget_bytes, 0.05, graph, feat, spec,
                                              h.sampling_txn_total) for o, h in zip(orders, run.hotness)])
    got = json.dumps(plan_report(layout, list(plans), list(ests), 0.05, [[3, 4], [5, 6]]), sort_keys=True)
    assert got == str(g["plan_report"][0])
