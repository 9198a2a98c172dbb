"""Input validation and capacity handling on the device path (reference errors:
sampling.py:128-131 ValueError('invalid seed vertex id'))."""

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


def _setup(n=30_000, cap=None, sparse=False):
    import paper_2305_16588_b200 as P
    from paper_2305_16588_b200.cache import FeatureStore
    from paper_2305_16588_b200.graph import synthetic_features_device
    from paper_2305_16588_b200.pipeline import SampleGatherPipeline

    g = P.generate_synthetic(n, 12, 1.2, seed=4)
    pool = np.arange(0, n, 7, dtype=np.int64)
    cfg = P.SamplingConfig(fanouts=(10, 5), batch_size=256)
    store = FeatureStore.resident(synthetic_features_device(0, n, 64))
    pipe = SampleGatherPipeline(g, cfg, store, len(pool), window=4, feat_rows_cap=cap, sparse_visited=sparse)
    return P, g, pool, cfg, pipe


@pytest.mark.parametrize("sparse", [False, True])
def test_unique_capacity_overflow_is_reported_and_recoverable(sparse):
    """A batch with more distinct ids than feat_rows_cap: nothing is written past the
    cap, ucount keeps the true count, check_capacity raises, and the visited sets are
    still cleared so the next epoch (same buffers) is exact."""
    P, g, pool, cfg, pipe = _setup(cap=300, sparse=sparse)
    sp = pipe.sampler
    guard = sp.unique.new_full((sp.W + 1, sp.ucap), -7)  # canary row right after the buffer
    sp.unique = guard[: sp.W]
    gs = P.KeyedRng(3).derive(0, 0, 0)
    pipe.run_epoch(pipe.plan_epoch(pool, gs))
    torch.cuda.synchronize()
    assert int(sp.ucount[: sp.W].max()) > sp.ucap
    assert bool((guard[sp.W] == -7).all()), "compaction wrote past the unique capacity"
    with pytest.raises(OverflowError):
        pipe.check_capacity(reset=True)
    with pytest.raises(OverflowError):
        pipe.window_to_host(sp.W)
    assert int(sp.bitmap.count_nonzero()) == 0, "visited bitmaps were not cleared after an overflow"
    if sp.summary is not None:
        assert int(sp.summary.count_nonzero()) == 0

    # the same buffers with a capacity that fits: exact vs the oracle
    _, g2, pool2, cfg2, ok = _setup(sparse=sparse)
    seen = []
    shuffled = pool2[O.permutation(gs.derive(1).key, len(pool2))]

    def check(p, w0, nbw):
        for bi in range(nbw):
            b = w0 + bi
            seeds = shuffled[b * 256 : (b + 1) * 256]
            hops = O.sample_batch(g2.row_offsets, g2.col_indices, g2.num_vertices, seeds, (10, 5),
                                  gs.derive(2, b).key)
            u = int(p.sampler.ucount[bi])
            assert np.array_equal(p.sampler.unique[bi, :u].cpu().numpy(), O.distinct_vertices(seeds, hops))
            seen.append(b)

    ok.run_epoch(ok.plan_epoch(pool2, gs), on_window=check)
    assert ok.check_capacity() <= ok.sampler.ucap
    assert len(seen) == -(-len(pool2) // 256)


def test_invalid_seed_ids_raise_before_the_device():
    P, g, pool, cfg, pipe = _setup()
    gs = P.KeyedRng(1).derive(0, 0, 0)
    for bad in (np.append(pool, g.num_vertices), np.append(pool, -1)):
        with pytest.raises(ValueError, match="invalid seed vertex id"):
            pipe.plan_epoch(bad, gs)
        with pytest.raises(ValueError, match="invalid seed vertex id"):
            pipe.plan_epoch(torch.from_numpy(bad).cuda(), gs)
    layout = P.block_layout(1, 1)
    with pytest.raises(ValueError, match="invalid seed vertex id"):
        P.run_sampling_epoch(g, [np.array([0, g.num_vertices + 5])], layout, cfg, 1, 0)
    with pytest.raises(ValueError, match="invalid seed vertex id"):
        P.sample_batch(g, [3, g.num_vertices], cfg, gs)
