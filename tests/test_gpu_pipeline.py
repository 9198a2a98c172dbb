"""Windowed epoch pipeline (shuffle -> sample -> dedup -> relabel -> gather) vs the oracle."""

import math

import numpy as np
import pytest

import gnncache_oracle as O

pytestmark = pytest.mark.gpu


def local_ids(t):
    """Relabelled ids as int64 (the sampler stores u16 in int16 when a window's batches fit)."""
    from paper_2305_16588_b200.sampling import local_ids as decode

    return decode(t)
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _device():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    torch.cuda.set_device(0)


@pytest.fixture(params=[False, True], ids=["tile_passes", "cta_per_batch"])
def unique_batch_path(request):
    """Dense compaction through the per-tile passes, or forced onto the CTA-per-batch
    kernel (taken by windows of >= SM-count batches, e.g. C2's 235) for every window."""
    from paper_2305_16588_b200 import _lib

    lib = _lib.lib()
    _lib.check(lib.gc_set_option(_lib.GC_OPT_UNIQUE_BATCH_CTAS, 1 if request.param else 0))
    yield request.param
    _lib.check(lib.gc_set_option(_lib.GC_OPT_UNIQUE_BATCH_CTAS, 0))


@pytest.mark.parametrize("sparse", [False, True])
@pytest.mark.parametrize("window,batch,fanouts,deg", [(0, 256, (15, 10, 5), 26), (3, 100, (25, 10), 14),
                                                       (2, 77, (4, 4), 40), (5, 64, (3,), 200)])
def test_epoch_windows_match_oracle(window, batch, fanouts, deg, sparse, unique_batch_path):
    if sparse and unique_batch_path:
        pytest.skip("the CTA-per-batch kernel is a dense-bitmap path")
    import paper_2305_16588_b200 as P
    from paper_2305_16588_b200.cache import FeatureStore
    from paper_2305_16588_b200.graph import synthetic_features_device
    from paper_2305_16588_b200.pipeline import SampleGatherPipeline

    n, dim = 40_000, 100
    g = P.generate_synthetic(n, deg, 1.2, seed=3)
    pool = np.sort(np.random.default_rng(1).choice(n, 1500, replace=False)).astype(np.int64)
    cfg = P.SamplingConfig(fanouts=fanouts, batch_size=batch)
    store = FeatureStore.resident(synthetic_features_device(0, n, dim))
    pipe = SampleGatherPipeline(g, cfg, store, len(pool), window=window or None, sparse_visited=sparse)
    gs = P.KeyedRng(9).derive(2, 0, 0)
    plan = pipe.plan_epoch(pool, gs)
    table = O.synthetic_features(np.arange(n), dim)
    shuffled = pool[O.permutation(gs.derive(1).key, len(pool))]
    seen = []

    def check(p, w0, nbw):
        sp = p.sampler
        torch.cuda.synchronize()
        counts = sp.counts[:, :nbw].cpu().numpy()
        for bi in range(nbw):
            b = w0 + bi
            seeds = shuffled[b * batch : (b + 1) * batch]
            hops = O.sample_batch(g.row_offsets, g.col_indices, n, seeds, fanouts, gs.derive(2, b).key)
            got_seeds = sp.seeds[bi, : counts[0, bi]].cpu().numpy().view(np.uint32)
            assert np.array_equal(got_seeds, seeds)
            uniq = O.distinct_vertices(seeds, hops)
            u = int(sp.ucount[bi])
            assert np.array_equal(sp.unique[bi, :u].cpu().numpy().view(np.uint32), uniq)
            assert np.array_equal(local_ids(sp.local_seeds[bi, : len(seeds)]).cpu().numpy(), O.relabel(uniq, seeds))
            for h, (_, off, nbr) in enumerate(hops):
                t = int(counts[h + 1, bi])
                assert t == len(nbr)
                assert np.array_equal(sp.nbrs[h][bi, :t].cpu().numpy().view(np.uint32), nbr)
                assert np.array_equal(sp.offsets[h][bi, : len(off)].cpu().numpy(), off)
                assert np.array_equal(local_ids(sp.local_nbrs[h][bi, :t]).cpu().numpy(), O.relabel(uniq, nbr))
            assert np.array_equal(p.features[bi, :u].cpu().numpy(), table[uniq])
            seen.append(b)

    pipe.run_epoch(plan, on_window=check)
    assert seen == list(range(math.ceil(len(pool) / batch)))


@pytest.mark.parametrize("sparse", [False, True])
def test_epoch_presampling_counters_match_reference_semantics(sparse, unique_batch_path):
    """Hotness fused into the window pipeline equals the oracle epoch trace."""
    if sparse and unique_batch_path:
        pytest.skip("the CTA-per-batch kernel is a dense-bitmap path")
    import paper_2305_16588_b200 as P
    from paper_2305_16588_b200.pipeline import SampleGatherPipeline
    from paper_2305_16588_b200.sampling import DeviceHotness

    n = 20_000
    g = P.generate_synthetic(n, 12, 1.2, seed=8)
    pool = np.arange(0, n, 13, dtype=np.int64)
    cfg = P.SamplingConfig(fanouts=(10, 5), batch_size=128)
    pipe = SampleGatherPipeline(g, cfg, None, len(pool), window=4, sparse_visited=sparse)
    hot = DeviceHotness(n)
    seed = 77
    plan = pipe.plan_epoch(pool, P.KeyedRng(seed).derive(0, 0, 0))
    pipe.run_epoch(plan, hot=hot)
    reads, looks, trav, nb = O.sampling_epoch(g.row_offsets, g.col_indices, n, [pool], [(0,)], [10, 5], 128, seed, 0)[0]
    assert np.array_equal(hot.topo_reads.cpu().numpy(), reads)
    assert np.array_equal(hot.feat_lookups.cpu().numpy(), looks)
    assert np.array_equal(hot.edge_traversals.cpu().numpy(), trav)
    t = O.transaction_cost_table(g.row_offsets)
    assert int(hot.txn_total.item()) == int((reads * t).sum())


@pytest.mark.parametrize("host_full", [True, False])
def test_tiered_topology_sampling_matches_oracle(host_full):
    """Neighbour lists read from local slab / peer slabs / host CSR give the reference
    sample, and the per-tier read counters match the tier rule (simulator.py:161-202)."""
    import paper_2305_16588_b200 as P
    from paper_2305_16588_b200.cache import TopologyStore
    from paper_2305_16588_b200.sampling import WindowSampler

    n = 60_000
    g = P.generate_synthetic(n, 26, 1.2, seed=21)
    rng = np.random.default_rng(4)
    perm = rng.permutation(n)
    parts = [np.sort(perm[i * 9000 : (i + 1) * 9000]) for i in range(4)]  # 60% cached across 4 GPUs, 40% host
    store = TopologyStore(g, parts, self_rank=1, host_full=host_full)
    fanouts = (15, 10, 5)
    sp = WindowSampler(g, fanouts, 512, 2, topology=store)
    seeds = rng.integers(0, n, (2, 512))
    keys = np.array([[P.KeyedRng(5).derive(b).derive(h).key for h in range(3)] for b in range(2)], dtype=np.uint64)
    sp.load(torch.from_numpy(seeds.astype(np.int32).reshape(-1)).cuda(), np.array([512, 512]), keys)
    sp.run()
    tier, _ = O.tier_of(parts, n, 1)
    reads, edges = np.zeros(3, np.int64), np.zeros(3, np.int64)
    for b in range(2):
        got = sp.batch_to_host(b)
        want = O.sample_batch(g.row_offsets, g.col_indices, n, seeds[b], fanouts, P.KeyedRng(5).derive(b).key)
        for hop, (src, off, nbr) in zip(got.hops, want):
            assert np.array_equal(hop.neighbors, nbr) and np.array_equal(hop.offsets, off)
            np.add.at(reads, tier[src], 1)
            np.add.at(edges, tier[src], np.diff(off))
    c = store.tier_counts()
    assert [c["reads_local"], c["reads_peer"], c["reads_host"]] == list(reads)
    assert [c["edges_local"], c["edges_peer"], c["edges_host"]] == list(edges)
    assert store.host_bytes() == 16 * reads[2] + 4 * edges[2]


def test_plan_built_cache_traffic_equals_reference_report():
    """Presample -> CSLP plan -> materialize -> three-tier cache -> one validation epoch:
    the device's measured local/peer/host traffic equals the reference simulator's
    TrafficReport for the same epoch and plan (simulator.py:132-228)."""
    import paper_2305_16588_b200 as P
    from paper_2305_16588_b200 import planner as PL
    from paper_2305_16588_b200.cache import FeatureStore, TopologyStore
    from paper_2305_16588_b200.graph import synthetic_features_device
    from paper_2305_16588_b200.partition import single_clique_partitioning
    from paper_2305_16588_b200.pipeline import SampleGatherPipeline
    from paper_2305_16588_b200.simulator import simulate_epoch

    n, dim, k = 150_000, 128, 4
    g = P.generate_synthetic(n, 14, 1.2, seed=P.derive_seed(3, 1))
    train = P.select_training_set(g, 0.1, seed=P.derive_seed(3, 2))
    layout = P.block_layout(k, k)
    pools = P.assign_tablets(P.split_intra_clique(train, single_clique_partitioning(g), layout), layout)
    feat = P.FeatureSpec(dim)
    budget = int(0.15 * (g.num_edges * 4 + 8 * n + n * feat.row_bytes))
    spec = P.HardwareSpec(layout, clique_budget_bytes=budget)
    cfg = P.SamplingConfig(fanouts=(25, 10), batch_size=1024, presample_epochs=1, seed=P.derive_seed(3, 4))
    hot = P.run_presampling(g, pools, layout, cfg, spec)[0]
    orders = PL.build_candidate_orders(hot)
    plan, est = PL.search_optimal_plan(orders, budget, 0.01, g, feat, spec, hot.sampling_txn_total)
    asg = PL.materialize_assignment([orders], [plan], layout, g, feat, spec)
    assert 0 < sum(map(len, asg.feat_vertices)) < n and sum(map(len, asg.topo_vertices)) > 0
    val_seed = P.derive_seed(3, 5)
    rep = simulate_epoch(g, pools, cfg, asg, layout, spec, feat, seed=val_seed)
    host_table = synthetic_features_device(0, n, dim).cpu()
    row_txns = PL.feature_row_transactions(feat, spec)
    for gpu in (0, 2):
        topo = TopologyStore(g, asg.topo_vertices, gpu)
        fstore = FeatureStore.from_assignment(host_table, asg.feat_vertices, gpu)
        pipe = SampleGatherPipeline(g, cfg, fstore, len(pools[gpu]), window=8, topology=topo)
        pipe.run_epoch(pipe.plan_epoch(pools[gpu], P.KeyedRng(val_seed).derive(0, 0, gpu)))
        t, f = topo.tier_counts(), fstore.tier_counts()
        assert t["reads_local"] == rep.topo_local_hits[gpu]
        assert t["reads_peer"] == rep.topo_peer_hits[gpu]
        assert t["reads_local"] + t["reads_peer"] + t["reads_host"] == rep.topo_reads[gpu]
        assert t["host_txn"] == rep.sampling_cpu_txn[gpu]
        assert f["local"] == rep.feat_local_hits[gpu] and f["peer"] == rep.feat_peer_hits[gpu]
        assert f["host"] * row_txns == rep.feature_cpu_txn[gpu]


def test_sparse_visited_reuse_across_windows_and_large_ids():
    """Sparse compaction over a 20M-vertex id space: ids near the top block, windows
    reusing cleared bitmaps/summaries, and the flat path agree with np.unique."""
    import paper_2305_16588_b200 as P
    from paper_2305_16588_b200.sampling import WindowSampler

    n = 20_000_000
    rng = np.random.default_rng(5)
    src = np.repeat(np.arange(n - 3000, n, dtype=np.int64), 8)
    dst = np.concatenate([rng.integers(0, n, len(src) // 2), rng.integers(n - 70_000, n, len(src) - len(src) // 2)])
    g = P.CsrGraph.from_edges(n, src, dst)
    all_seeds = [rng.integers(n - 3000, n, (3, 256)), rng.integers(n - 3000, n, (3, 256)), np.full((3, 256), n - 1)]
    results = {}
    for sparse in (False, True):
        sp = WindowSampler(g, (5, 3), 256, 3, sparse_visited=sparse)
        outs = []
        for rep in range(3):  # the same buffers are cleared and reused
            seeds = all_seeds[rep]
            keys = np.array([[P.KeyedRng(rep).derive(b).derive(h).key for h in range(2)] for b in range(3)],
                            dtype=np.uint64)
            sp.load(torch.from_numpy(seeds.astype(np.int64).astype(np.uint32).view(np.int32).reshape(-1)).cuda(),
                    np.array([256, 256, 256]), keys)
            sp.run()
            for b in range(3):
                bs = sp.batch_to_host(b)
                want = np.unique(np.concatenate([bs.seeds] + [h.neighbors for h in bs.hops]))
                got = bs.distinct_vertices()
                assert np.array_equal(got, want)
                outs.append(got)
        results[sparse] = outs
    for a, b in zip(results[False], results[True]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("lanes", [2, 3])
def test_lanes_overlap_matches_sequential(lanes):
    """Inter-batch pipelining (windows alternating over concurrent streams) gives the
    same per-window results as one stream; captures are device clones on the window's
    stream, so nothing synchronises the lanes while they overlap."""
    import paper_2305_16588_b200 as P
    from paper_2305_16588_b200.cache import FeatureStore
    from paper_2305_16588_b200.graph import synthetic_features_device
    from paper_2305_16588_b200.pipeline import SampleGatherPipeline

    n, dim, batch, fanouts = 60_000, 64, 128, (10, 5)
    g = P.generate_synthetic(n, 16, 1.2, seed=5)
    pool = np.sort(np.random.default_rng(2).choice(n, 3000, replace=False)).astype(np.int64)
    cfg = P.SamplingConfig(fanouts=fanouts, batch_size=batch)
    store = FeatureStore.resident(synthetic_features_device(0, n, dim))
    gs = P.KeyedRng(11).derive(3, 0, 0)

    def run(k):
        pipe = SampleGatherPipeline(g, cfg, store, len(pool), window=4, sparse_visited=True, lanes=k)
        plan = pipe.plan_epoch(pool, gs)
        got = []

        def grab(p, w0, nbw):
            sp = p.sampler
            got.append((w0, sp.ucount[:nbw].clone(), sp.unique[:nbw].clone(), p.features[:nbw].clone(),
                        [t[:nbw].clone() for t in sp.local_nbrs], sp.counts[:, :nbw].clone()))

        pipe.run_epoch(plan, on_window=grab)
        torch.cuda.synchronize()
        return got

    ref, par = run(1), run(lanes)
    assert [w[0] for w in ref] == [w[0] for w in par]
    for a, b in zip(ref, par):
        assert torch.equal(a[1], b[1]) and torch.equal(a[5], b[5])
        for bi in range(a[1].numel()):
            u = int(a[1][bi])
            assert torch.equal(a[2][bi, :u], b[2][bi, :u])
            assert torch.equal(a[3][bi, :u], b[3][bi, :u])
            for h in range(len(fanouts)):
                t = int(a[5][h + 1, bi])
                assert torch.equal(a[4][h][bi, :t], b[4][h][bi, :t])


@pytest.mark.parametrize("lanes", [1, 2])
def test_epoch_graph_replay_matches_eager(lanes):
    """run_epoch_graph (one CUDA-graph launch per epoch, inputs copied into the captured
    buffers) gives run_epoch's results for several epochs with different shuffle and
    hop keys."""
    import paper_2305_16588_b200 as P
    from paper_2305_16588_b200.cache import FeatureStore
    from paper_2305_16588_b200.graph import synthetic_features_device
    from paper_2305_16588_b200.pipeline import SampleGatherPipeline

    n, dim, batch, fanouts = 30_000, 32, 128, (8, 4)
    g = P.generate_synthetic(n, 12, 1.2, seed=6)
    pool = np.sort(np.random.default_rng(5).choice(n, 2000, replace=False)).astype(np.int64)
    cfg = P.SamplingConfig(fanouts=fanouts, batch_size=batch)
    store = FeatureStore.resident(synthetic_features_device(0, n, dim))
    eager = SampleGatherPipeline(g, cfg, store, len(pool), window=8 if lanes > 1 else None, lanes=lanes)
    graph = SampleGatherPipeline(g, cfg, store, len(pool), window=8 if lanes > 1 else None, lanes=lanes)
    root = P.KeyedRng(77)

    def snapshot(p):
        out = []
        for sp, feats in zip(p.lane_samplers, p.lane_features):
            out.append([t.clone() for t in (sp.counts, sp.ucount, sp.unique, feats, *sp.local_nbrs)])
        return out

    for e in range(3):
        gs = root.derive(e, 0, 0)
        eager.run_epoch(eager.plan_epoch(pool, gs))
        graph.run_epoch_graph(graph.plan_epoch(pool, gs))
        torch.cuda.synchronize()
        a, b = snapshot(eager), snapshot(graph)
        for la, lb in zip(a, b):
            cnt = la[1].cpu().numpy()
            assert torch.equal(la[0], lb[0]) and torch.equal(la[1], lb[1])
            for bi, u in enumerate(cnt):
                assert torch.equal(la[2][bi, :u], lb[2][bi, :u])
                assert torch.equal(la[3][bi, :u], lb[3][bi, :u])


@pytest.mark.parametrize("lanes", [1, 2])
def test_epoch_graph_replay_tiered_matches_eager(lanes):
    """Graph replay through the tiered path (neighbour lists from local slab / peer
    slabs / host CSR, features from HBM / peers / pinned host rows over UVA): same
    results and same per-tier counters as eager run_epoch, epoch after epoch."""
    import paper_2305_16588_b200 as P
    from paper_2305_16588_b200.cache import FeatureStore, TopologyStore
    from paper_2305_16588_b200.graph import synthetic_features_device
    from paper_2305_16588_b200.pipeline import SampleGatherPipeline

    n, dim, batch, fanouts = 40_000, 32, 128, (10, 5)
    g = P.generate_synthetic(n, 14, 1.2, seed=8)
    rng = np.random.default_rng(9)
    pool = np.sort(rng.choice(n, 2000, replace=False)).astype(np.int64)
    perm = rng.permutation(n)
    topo_parts = [np.sort(perm[i * 6000 : (i + 1) * 6000]) for i in range(4)]
    feat_parts = [np.sort(perm[24_000 + i * 3000 : 24_000 + (i + 1) * 3000]) for i in range(4)]
    host_table = synthetic_features_device(0, n, dim).cpu()
    cfg = P.SamplingConfig(fanouts=fanouts, batch_size=batch)

    def make():
        topo = TopologyStore(g, topo_parts, self_rank=1, host_full=True)
        fs = FeatureStore.from_assignment(host_table, feat_parts, 1)
        pipe = SampleGatherPipeline(g, cfg, fs, len(pool), window=8 if lanes > 1 else None, topology=topo,
                                    lanes=lanes)
        return pipe, topo, fs

    (eager, te, fe), (graph, tg, fg) = make(), make()
    root = P.KeyedRng(31)
    for e in range(3):
        for s in (te, fe, tg, fg):
            s.reset_counters()
        gs = root.derive(e, 0, 0)
        eager.run_epoch(eager.plan_epoch(pool, gs))
        graph.run_epoch_graph(graph.plan_epoch(pool, gs))
        torch.cuda.synchronize()
        # replayed kernels keep counting; the first call also ran one uncaptured warm-up epoch
        mult = 2 if e == 0 else 1
        ct, cg = te.tier_counts(), tg.tier_counts()
        assert all(cg[k] == mult * ct[k] for k in ct), (e, ct, cg)
        assert all(fg.tier_counts()[k] == mult * fe.tier_counts()[k] for k in ("local", "peer", "host"))
        assert min(fe.tier_counts()[k] for k in ("local", "peer", "host")) > 0
        assert min(ct[f"reads_{k}"] for k in ("local", "peer", "host")) > 0
        for pa, pb in zip(zip(eager.lane_samplers, eager.lane_features), zip(graph.lane_samplers, graph.lane_features)):
            (sa, xa), (sb, xb) = pa, pb
            assert torch.equal(sa.counts, sb.counts) and torch.equal(sa.ucount, sb.ucount)
            for bi, u in enumerate(sa.ucount.cpu().numpy()):
                assert torch.equal(sa.unique[bi, :u], sb.unique[bi, :u])
                assert torch.equal(xa[bi, :u], xb[bi, :u])
                assert torch.equal(xa[bi, :u].cpu(), host_table[sa.unique[bi, :u].cpu().long() & 0xFFFFFFFF])


@pytest.mark.parametrize("relabel,lanes,compact,big", [(True, 1, False, False), (False, 1, False, False),
                                                        (True, 2, False, False), (True, 1, True, False),
                                                        (False, 1, True, False), (True, 1, True, True),
                                                        (True, 1, False, True)])
def test_window_to_host_packs_every_batch(relabel, lanes, compact, big):
    """window_to_host: one packed pinned copy per array equals the per-batch slices of
    the padded device buffers, batch boundaries included; staging is reused. compact:
    relabelled ids travel as 16-bit values (global ids never do); wait=False returns an
    event the host waits on before reading. big: the unique capacity exceeds 65536, so
    the sampler keeps u32 local ids (narrowed by the packing when compact), else u16
    (widened by the packing when not compact) — every gc_pack_segments mode; compact
    offsets travel as u8 counts and offsets_from_counts rebuilds them."""
    import paper_2305_16588_b200 as P
    from paper_2305_16588_b200.cache import FeatureStore
    from paper_2305_16588_b200.graph import synthetic_features_device
    from paper_2305_16588_b200.pipeline import SampleGatherPipeline, offsets_from_counts

    n, dim, batch, fanouts = (100_000, 32, 1024, (15, 10)) if big else (30_000, 100, 96, (7, 3))
    g = P.generate_synthetic(n, 12, 1.2, seed=12)
    npool = 3000 if big else 1000
    pool = np.sort(np.random.default_rng(13).choice(n, npool, replace=False)).astype(np.int64)  # last batch partial
    store = FeatureStore.resident(synthetic_features_device(0, n, dim))
    pipe = SampleGatherPipeline(g, P.SamplingConfig(fanouts=fanouts, batch_size=batch), store, len(pool),
                                window=2 if big else 4, relabel=relabel, lanes=lanes)
    if relabel:
        assert pipe.sampler.local_bits == (32 if big else 16)
    staging, seen = {}, []

    def check(p, w0, nbw):
        out = p.window_to_host(nbw, staging, compact_ids=compact, wait=not compact)
        if compact:
            out["ready"].synchronize()
        assert out["local_bits"] == (16 if compact and relabel else 32)
        sp = p.sampler
        if compact:  # offsets travel as u8 per-position counts
            assert "offsets" not in out and all(c.dtype == torch.uint8 for c in out["counts"])
            offsets = []
            for h in range(len(fanouts)):
                o, optr = offsets_from_counts(out["counts"][h], out["counts_ptr"][h])
                assert np.array_equal(optr, out["offsets_ptr"][h])
                offsets.append(o)
        else:
            offsets = out["offsets"]
        for b in range(nbw):
            u0, u1 = out["unique_ptr"][b : b + 2]
            u = int(sp.ucount[b])
            assert u1 - u0 == u
            assert torch.equal(out["unique"][u0:u1], sp.unique[b, :u].cpu())
            assert torch.equal(out["features"][u0:u1], p.features[b, :u].cpu())
            for h in range(len(fanouts)):
                f, t = int(sp.counts[h, b]), int(sp.counts[h + 1, b])
                o0, o1 = out["offsets_ptr"][h][b : b + 2]
                l0, l1 = out["local_ptr"][h][b : b + 2]
                assert o1 - o0 == f + 1 and l1 - l0 == t
                assert torch.equal(offsets[h][o0:o1], sp.offsets[h][b, : f + 1].cpu())
                want = local_ids(sp.local_nbrs[h][b, :t]) if relabel else sp.nbrs[h][b, :t].long()
                got = out["local"][h][l0:l1]
                if out["local_bits"] == 16:
                    assert got.dtype == torch.int16
                assert torch.equal(local_ids(got), want.cpu())
        seen.append(nbw)

    pipe.run_epoch(pipe.plan_epoch(pool, P.KeyedRng(3).derive(0, 0, 0)), on_window=check)
    assert sum(seen) == -(-len(pool) // batch) and len(seen) == (2 if big else 3)
    assert staging["features"].is_pinned()


@pytest.mark.parametrize("sparse,window", [(False, 3), (True, 3), (False, 0)])
def test_launch_accounting_matches_profiler(sparse, window, unique_batch_path):
    """pipe.launches (the bench's gpu_launches) equals the number of this library's
    kernels the CUDA profiler sees for an eager epoch."""
    if sparse and unique_batch_path:
        pytest.skip("the CTA-per-batch kernel is a dense-bitmap path")
    from torch.profiler import ProfilerActivity, profile

    import paper_2305_16588_b200 as P
    from paper_2305_16588_b200.cache import FeatureStore
    from paper_2305_16588_b200.graph import synthetic_features_device
    from paper_2305_16588_b200.pipeline import SampleGatherPipeline

    n = 30_000
    g = P.generate_synthetic(n, 12, 1.2, seed=5)
    pool = np.arange(0, n, 7, dtype=np.int64)
    store = FeatureStore.resident(synthetic_features_device(0, n, 64))
    pipe = SampleGatherPipeline(g, P.SamplingConfig(fanouts=(10, 5), batch_size=256), store, len(pool),
                                window=window or None, sparse_visited=sparse)
    plan = pipe.plan_epoch(pool, P.KeyedRng(4).derive(0, 0, 0))
    pipe.run_epoch(plan)  # warm-up (lazy allocations)
    torch.cuda.synchronize()
    before = pipe.launches
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        pipe.run_epoch(plan)
        torch.cuda.synchronize()
    seen = sum(e.count for e in prof.key_averages() if "gc::" in e.key)
    if seen == 0:
        pytest.skip("the CUDA profiler saw no kernels (CUPTI unavailable, e.g. under compute-sanitizer)")
    assert seen == pipe.launches - before > 0
