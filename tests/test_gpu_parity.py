"""Device path vs the reference's golden vectors and the CPU oracle (needs a B200)."""

import numpy as np
import pytest

import gnncache_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _device():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2305_16588_b200 import _lib

    _lib.load_library()
    torch.cuda.set_device(0)


def _pkg():
    import paper_2305_16588_b200 as P

    return P


# ------------------------------------------------------------------ K0 rng / K1 shuffle
def test_rng_device_matches_reference(golden):
    P = _pkg()
    g = golden("rng")
    assert np.array_equal(P.mix64_array(g["mix64_in"]), g["mix64_out"])
    key = int(g["pairs_key"][0])
    assert np.array_equal(P.KeyedRng(key).hash_pairs(g["pairs_a"], g["pairs_b"]), g["pairs_out"])
    assert np.array_equal(P.KeyedRng(key).hash_counters(np.arange(100)), g["counters_out"])
    pk = int(g["perm_key"][0])
    for n in (0, 1, 2, 17, 257, 5000):
        assert np.array_equal(P.KeyedRng(pk).permutation(n), g[f"perm_{n}"]), n


@pytest.mark.parametrize("n", [1_390_000, 4_000_000])
def test_permutation_large_matches_oracle(n):
    """1.39M = one C3 tablet at 8 GPUs; 4M keys hold ~1.9K pairs of equal high words,
    which the 32-bit radix sort leaves to the tie fix-up."""
    P = _pkg()
    key = P.KeyedRng(99).derive(1).key
    want = O.permutation(key, n)
    hi = (O.hash_counters(key, np.arange(n)) >> np.uint64(32))[want]
    assert (hi[1:] == hi[:-1]).sum() > 100  # the fix-up path is exercised
    assert np.array_equal(P.KeyedRng(key).permutation(n), want)


def test_shuffle_fused_gather():
    P = _pkg()
    pool = np.random.default_rng(1).integers(0, 10**9, 100_003)
    s = P.KeyedRng(5).derive(0, 0, 0).derive(1)
    got = s.permutation_device(len(pool), torch.from_numpy(pool).cuda()).cpu().numpy()
    assert np.array_equal(got, pool[O.permutation(s.key, len(pool))])


# ------------------------------------------------------------------ K2/K3 sampling
def test_sample_batch_matches_reference_golden(golden):
    P = _pkg()
    g = golden("sampling")
    graphs = {}
    for i in range(int(g["num_cases"])):
        name = str(g[f"c{i}_graph"])
        if name not in graphs:
            ro, ci = g[f"g_{name}_ro"], g[f"g_{name}_ci"]
            graphs[name] = P.CsrGraph(len(ro) - 1, len(ci), ro, ci)
        gr = graphs[name]
        fan = tuple(int(f) for f in g[f"c{i}_fanouts"])
        cfg = P.SamplingConfig(fanouts=fan, batch_size=len(g[f"c{i}_seeds"]))
        batch = P.sample_batch(gr, g[f"c{i}_seeds"], cfg, P.KeyedRng(int(g[f"c{i}_key"][0])))
        for h, hop in enumerate(batch.hops):
            assert np.array_equal(hop.sources, g[f"c{i}_h{h}_src"]), (i, h)
            assert np.array_equal(hop.offsets, g[f"c{i}_h{h}_off"]), (i, h)
            assert np.array_equal(hop.neighbors, g[f"c{i}_h{h}_nbr"]), (i, h)
        assert np.array_equal(batch.distinct_vertices(), g[f"c{i}_distinct"]), i


@pytest.mark.parametrize(
    "n,deg,skew,fanouts,nseeds",
    [
        (100_000, 10, 1.2, (25, 10), 1024),  # BASELINE config 1: copy path only
        (200_000, 26, 1.2, (15, 10, 5), 1024),  # config 2 shape (choice path every hop)
        (100_000, 14, 1.2, (25, 10), 1024),  # config 3 shape
        (50_000, 35, 1.0, (25, 10), 512),  # config 4 shape (deg > 32: two keys per lane)
        (40_000, 55, 1.0, (25, 10), 512),  # config 5 shape
        (20_000, 200, 0.9, (25, 10), 128),  # streaming path (deg > 128)
        (20_000, 40, 1.0, (60, 2), 256),  # fanout > 32, multi-round staging
    ],
)
def test_sample_batch_matches_oracle_at_config_shapes(n, deg, skew, fanouts, nseeds):
    P = _pkg()
    gr = P.generate_synthetic(n, deg, skew, seed=17)
    seeds = np.random.default_rng(n).integers(0, n, nseeds)
    stream = P.KeyedRng(3).derive(0, 0, 1).derive(2, 5)
    cfg = P.SamplingConfig(fanouts=fanouts, batch_size=nseeds)
    got = P.sample_batch(gr, seeds, cfg, stream)
    want = O.sample_batch(gr.row_offsets, gr.col_indices, n, seeds, fanouts, stream.key)
    for hop, (src, off, nbr) in zip(got.hops, want):
        assert np.array_equal(hop.sources, src)
        assert np.array_equal(hop.offsets, off)
        assert np.array_equal(hop.neighbors, nbr)
    assert np.array_equal(got.distinct_vertices(), O.distinct_vertices(seeds, want))


def test_edge_cases_empty_and_zero_degree():
    P = _pkg()
    # 0 -> 1 -> 2 chain; vertex 3 isolated (sampling.py:138-142 empty-frontier padding)
    g = P.CsrGraph.from_edges(4, np.array([0, 1]), np.array([1, 2]))
    cfg = P.SamplingConfig(fanouts=(3, 3, 3), batch_size=2)
    b = P.sample_batch(g, np.array([3]), cfg, P.KeyedRng(2).derive(0))
    assert [len(h.neighbors) for h in b.hops] == [0, 0, 0]
    assert list(b.hops[0].offsets) == [0, 0] and list(b.hops[1].offsets) == [0]
    assert list(b.distinct_vertices()) == [3]
    b = P.sample_batch(g, np.array([0, 0]), cfg, P.KeyedRng(2).derive(0))
    assert [list(h.neighbors) for h in b.hops] == [[1, 1], [2, 2], []]
    with pytest.raises(ValueError):
        P.sample_batch(g, np.array([], dtype=np.int64), cfg, P.KeyedRng(0))
    with pytest.raises(ValueError):
        P.sample_batch(g, np.array([4]), cfg, P.KeyedRng(0))


# ------------------------------------------------------------------ K5 presampling
def test_presampling_matches_reference_golden(golden):
    P = _pkg()
    g = golden("presampling")
    for i in range(int(g["num_configs"])):
        n, deg, gseed, gpus, clique, bs, epochs, seed = [int(x) for x in g[f"p{i}_cfg"]]
        gr = P.generate_synthetic(n, deg, float(g[f"p{i}_skew"][0]), seed=gseed)
        layout = P.block_layout(gpus, clique)
        spec = P.HardwareSpec(layout, clique_budget_bytes=1 << 20)
        pools = [np.arange(j, n, gpus + 3, dtype=np.int64) for j in range(gpus)]
        fan = tuple(int(f) for f in g[f"p{i}_fanouts"])
        cfg = P.SamplingConfig(fanouts=fan, batch_size=bs, presample_epochs=epochs, seed=seed)
        hot = P.run_presampling(gr, pools, layout, cfg, spec)
        for ci, h in enumerate(hot):
            assert np.array_equal(h.topo_hotness, g[f"p{i}_c{ci}_HT"])
            assert np.array_equal(h.feat_hotness, g[f"p{i}_c{ci}_HF"])
            assert h.sampling_txn_total == int(g[f"p{i}_c{ci}_txn"][0])
        traces = P.run_sampling_epoch(gr, pools, layout, cfg, seed, 0)
        for gi, tr in enumerate(traces):
            assert np.array_equal(tr.topo_reads, g[f"p{i}_t{gi}_reads"])
            assert np.array_equal(tr.feat_lookups, g[f"p{i}_t{gi}_looks"])
            assert np.array_equal(tr.edge_traversals, g[f"p{i}_t{gi}_trav"])
            assert tr.num_batches == int(g[f"p{i}_t{gi}_nb"][0])


def test_presampling_c1_full_epoch_matches_oracle():
    """BASELINE config 1 end to end: 100K vertices, degree 10, 10% training, batch 1024."""
    P = _pkg()
    gr = P.generate_synthetic(100_000, 10, 1.2, seed=P.derive_seed(7, 1))
    train = P.select_training_set(gr, 0.1, seed=P.derive_seed(7, 2))
    layout = P.block_layout(1, 1)
    cfg = P.SamplingConfig(fanouts=(25, 10), batch_size=1024, presample_epochs=1, seed=P.derive_seed(7, 4))
    hot = P.run_presampling(gr, [train.vertex_ids], layout, cfg, P.HardwareSpec(layout, 1 << 30))[0]
    ht, hf, txn = O.presampling(gr.row_offsets, gr.col_indices, gr.num_vertices, [train.vertex_ids], [(0,)],
                                [25, 10], 1024, cfg.seed, 1)[0]
    assert np.array_equal(hot.topo_hotness, ht)
    assert np.array_equal(hot.feat_hotness, hf)
    assert hot.sampling_txn_total == txn


def test_accumulate_hotness_matches_oracle():
    P = _pkg()
    gr = P.generate_synthetic(3000, 12, 1.2, seed=4)
    seeds = np.arange(0, 3000, 37)
    b = P.sample_batch(gr, seeds, P.SamplingConfig(fanouts=(5, 5), batch_size=len(seeds)), P.KeyedRng(9))
    hot = P.HotnessMatrices(0, np.zeros((2, 3000), np.int64), np.zeros((2, 3000), np.int64))
    P.accumulate_hotness(b, 1, hot)
    want_t = np.zeros(3000, np.int64)
    for h in b.hops:
        np.add.at(want_t, h.sources, np.diff(h.offsets))
    want_f = np.zeros(3000, np.int64)
    want_f[O.distinct_vertices(b.seeds, [(h.sources, h.offsets, h.neighbors) for h in b.hops])] = 1
    assert np.array_equal(hot.topo_hotness[1], want_t) and np.array_equal(hot.feat_hotness[1], want_f)
    assert hot.topo_hotness[0].sum() == 0


# ------------------------------------------------------------------ K4 gather
@pytest.mark.parametrize("dim", [33, 100, 128, 256, 512, 600])
def test_gather_three_tiers_bit_exact(dim):
    """Every row width path: 4-byte vectors (D=33), warp per row with 1/2/4 16-byte
    vectors per lane (D <= 128 / C5's D=256 / 512), thread per vector (D=600)."""
    from paper_2305_16588_b200.cache import FeatureStore, gather_rows

    n = 50_000
    table = O.synthetic_features(np.arange(n), dim)
    rng = np.random.default_rng(0)
    perm = rng.permutation(n)
    # GPU 0 of a 4-GPU clique holds 10%, peers 1..3 hold 10% each, the rest is host-only
    parts = [perm[i * 5000 : (i + 1) * 5000] for i in range(4)]
    store = FeatureStore.from_assignment(table, parts, self_rank=0)
    ids = np.sort(rng.choice(n, 20_000, replace=False))
    got = gather_rows(store, ids)
    assert np.array_equal(got, table[ids])
    tiers = store.tier_counts()
    want_local = np.isin(ids, parts[0]).sum()
    want_peer = np.isin(ids, np.concatenate(parts[1:])).sum()
    assert tiers == {"local": want_local, "peer": want_peer, "host": len(ids) - want_local - want_peer}


@pytest.mark.parametrize("dim", [64, 100, 128, 256])
def test_gather_deferred_host_rows_bit_exact(dim):
    """gc_gather_deferred (host rows by a second small-grid kernel) == gc_gather, over a
    window of batches with ragged counts and a capacity clamp: list order, address order,
    a few fat CTAs (32 x 256 rows for 512-byte rows, as the C3 bench runs it) and a tiny
    grid (3 CTAs x 5 rows: many rounds per CTA, a partial last round)."""
    from paper_2305_16588_b200.cache import FeatureStore

    n, W, cap = 30_000, 5, 3000
    table = O.synthetic_features(np.arange(n), dim)
    rng = np.random.default_rng(1)
    perm = rng.permutation(n)
    parts = [perm[i * 4000 : (i + 1) * 4000] for i in range(2)]
    store = FeatureStore.from_assignment(table, parts, self_rank=0)
    counts = np.array([3000, 0, 1, 2999, 5000])  # the last one is clamped to cap
    ids = np.zeros((W, cap), dtype=np.int64)
    for b in range(W):
        ids[b, : min(counts[b], cap)] = np.sort(rng.choice(n, min(counts[b], cap), replace=False))
    d_ids = torch.from_numpy(ids.astype(np.uint32).view(np.int32)).cuda()
    d_cnt = torch.from_numpy(counts.astype(np.int32)).cuda()
    from paper_2305_16588_b200 import _lib

    outs = []
    # (deferred, address order, host-row CTAs, rows in flight per CTA; 0 = defaults)
    for deferred, order, ctas, rows in ((False, 1, 0, 0), (True, 0, 0, 0), (True, 1, 0, 0), (True, 1, 32, 131072 // (4 * dim)),
                                        (True, 1, 3, 5)):
        _lib.check(_lib.lib().gc_set_option(_lib.GC_OPT_DEFER_ORDER, order))
        _lib.check(_lib.lib().gc_set_option(_lib.GC_OPT_DEFER_CTAS, ctas or 296))
        _lib.check(_lib.lib().gc_set_option(_lib.GC_OPT_DEFER_ROWS, rows))
        out = torch.full((W, cap, dim), float("nan"), dtype=torch.float32, device="cuda")
        store.reset_counters()
        store.gather(d_ids, d_cnt, out, deferred=deferred)
        outs.append((out.cpu().numpy(), store.tier_counts()))
    _lib.check(_lib.lib().gc_set_option(_lib.GC_OPT_DEFER_ORDER, 1))
    _lib.check(_lib.lib().gc_set_option(_lib.GC_OPT_DEFER_CTAS, 296))
    _lib.check(_lib.lib().gc_set_option(_lib.GC_OPT_DEFER_ROWS, 0))
    a, ta = outs[0]
    assert ta["host"] > 0
    for b_, tb in outs[1:]:
        assert ta == tb
        for b in range(W):
            k = min(counts[b], cap)
            assert np.array_equal(b_[b, :k], table[ids[b, :k]])
            assert np.array_equal(a[b, :k], b_[b, :k])


def test_gather_deferred_address_order_wide_ids():
    """The address-ordered deferred read (bucket sort on the id's top 16 significant
    bits) over 2^22 host rows of 16 bytes, unsorted ids with duplicates across batches:
    bit-exact against the table."""
    from paper_2305_16588_b200 import _lib
    from paper_2305_16588_b200.cache import FeatureStore

    n, dim, W, cap = 1 << 22, 4, 7, 9000
    table = O.synthetic_features(np.arange(n), dim)
    rng = np.random.default_rng(5)
    parts = [rng.choice(n, 100_000, replace=False)]
    store = FeatureStore.from_assignment(table, parts, self_rank=0)
    ids = rng.integers(0, n, size=(W, cap))
    counts = rng.integers(0, cap + 1, size=W)
    d_ids = torch.from_numpy(ids.astype(np.uint32).view(np.int32)).cuda()
    d_cnt = torch.from_numpy(counts.astype(np.int32)).cuda()
    _lib.check(_lib.lib().gc_set_option(_lib.GC_OPT_DEFER_ORDER, 1))
    out = torch.full((W, cap, dim), float("nan"), dtype=torch.float32, device="cuda")
    store.gather(d_ids, d_cnt, out, deferred=True)
    got = out.cpu().numpy()
    for b in range(W):
        k = counts[b]
        assert np.array_equal(got[b, :k], table[ids[b, :k]])


def test_synthetic_features_device_matches_oracle():
    from paper_2305_16588_b200.graph import synthetic_features_device

    for dim in (1, 100, 128, 256):
        x = synthetic_features_device(1000, 500, dim).cpu().numpy()
        assert np.array_equal(x, O.synthetic_features(np.arange(1000, 1500), dim))


def test_gather_unaligned_row_width():
    from paper_2305_16588_b200.cache import FeatureStore, gather_rows
    from paper_2305_16588_b200.graph import synthetic_features_device

    table = synthetic_features_device(0, 1000, 7)  # 28-byte rows: 4-byte vector path
    ids = np.array([5, 999, 0, 5, 321])
    got = gather_rows(FeatureStore.resident(table), ids)
    assert np.array_equal(got, O.synthetic_features(ids, 7))


@pytest.mark.parametrize("deg,fanouts", [(26, (15, 10, 5)), (55, (25, 10)), (100, (40, 3))])
def test_packed_and_exact_selection_agree(deg, fanouts):
    """The packed 32-bit REDUX extraction and the 64-bit path give identical samples."""
    P = _pkg()
    from paper_2305_16588_b200 import _lib

    lib = _lib.load_library()
    gr = P.generate_synthetic(30_000, deg, 1.1, seed=deg)
    seeds = np.random.default_rng(deg).integers(0, 30_000, 512)
    cfg = P.SamplingConfig(fanouts=fanouts, batch_size=512)
    stream = P.KeyedRng(11).derive(deg)
    fast = P.sample_batch(gr, seeds, cfg, stream)
    _lib.check(lib.gc_set_option(_lib.GC_OPT_EXACT_SELECTION, 1))
    try:
        exact = P.sample_batch(gr, seeds, cfg, stream)
    finally:
        _lib.check(lib.gc_set_option(_lib.GC_OPT_EXACT_SELECTION, 0))
    for a, b in zip(fast.hops, exact.hops):
        assert np.array_equal(a.neighbors, b.neighbors) and np.array_equal(a.offsets, b.offsets)
    want = O.sample_batch(gr.row_offsets, gr.col_indices, gr.num_vertices, seeds, fanouts, stream.key)
    for a, (_, off, nbr) in zip(exact.hops, want):
        assert np.array_equal(a.neighbors, nbr)


@pytest.mark.parametrize("fanouts", [(10, 5), (3, 300), (64, 1)])
def test_heavy_tailed_out_degrees_match_oracle(fanouts):
    """Power-law out-degrees (the reference generator's are constant): most lists are
    short, a few hubs hold 1K-3K edges, some vertices have none — every selection path
    (thread network, packed/exact warp extraction, streaming extraction, copy) and
    multi-round staging (fanout 300) in one batch."""
    P = _pkg()
    rng = np.random.default_rng(sum(fanouts))
    n = 30_000
    deg = np.minimum((rng.pareto(1.1, n) * 3).astype(np.int64), 3000)
    deg[rng.choice(n, 20, replace=False)] = rng.integers(1000, 3001, 20)
    src = np.repeat(np.arange(n), deg)
    dst = rng.integers(0, n, len(src))
    g = P.CsrGraph.from_edges(n, src, dst)
    seeds = rng.integers(0, n, 400)
    seeds[:20] = np.flatnonzero(deg >= 1000)[:20]  # hubs among the seeds
    stream = P.KeyedRng(12).derive(0, 0, 2).derive(2, 9)
    cfg = P.SamplingConfig(fanouts=fanouts, batch_size=len(seeds))
    got = P.sample_batch(g, seeds, cfg, stream)
    want = O.sample_batch(g.row_offsets, g.col_indices, n, seeds, fanouts, stream.key)
    for hop, (s, off, nbr) in zip(got.hops, want):
        assert np.array_equal(hop.sources, s)
        assert np.array_equal(hop.offsets, off)
        assert np.array_equal(hop.neighbors, nbr)
    assert np.array_equal(got.distinct_vertices(), O.distinct_vertices(seeds, want))


_RAND_CASES = [
    (int(n), int(d), tuple(int(f) for f in fs), int(s))
    for n, d, fs, s in [
        (np.random.default_rng(i).integers(500, 30_000), np.random.default_rng(i + 100).integers(1, 70),
         np.random.default_rng(i + 200).integers(1, 40, np.random.default_rng(i + 300).integers(1, 4)),
         np.random.default_rng(i + 400).integers(1, 2**62))
        for i in range(8)
    ]
]


@pytest.mark.parametrize("n,deg,fanouts,seed", _RAND_CASES)
def test_randomized_shapes_match_oracle(n, deg, fanouts, seed):
    """Seeded random (graph size, degree, 1-3 hop fanouts, stream key) — every network
    size S, copy and choice paths mixed within a hop."""
    P = _pkg()
    g = P.generate_synthetic(n, deg, 1.1, seed=seed % 1000)
    seeds = np.random.default_rng(seed % 997).integers(0, n, 200)
    stream = P.KeyedRng(seed).derive(1, 0, 3).derive(2, 7)
    cfg = P.SamplingConfig(fanouts=fanouts, batch_size=len(seeds))
    got = P.sample_batch(g, seeds, cfg, stream)
    want = O.sample_batch(g.row_offsets, g.col_indices, n, seeds, fanouts, stream.key)
    for hop, (s, off, nbr) in zip(got.hops, want):
        assert np.array_equal(hop.sources, s)
        assert np.array_equal(hop.offsets, off)
        assert np.array_equal(hop.neighbors, nbr)
    assert np.array_equal(got.distinct_vertices(), O.distinct_vertices(seeds, want))
