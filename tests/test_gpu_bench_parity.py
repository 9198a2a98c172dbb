"""Parity at the exact configuration bench.py times.

C2 (BASELINE configs[1]): 2.4M vertices, degree 26, fanouts [15,10,5], batch 1024, the
whole 235-batch epoch as one window, 65,536-row unique/gather capacity, each epoch one
CUDA-graph replay (SampleGatherPipeline.run_epoch_graph) — bench.build_inputs and the
same constructor arguments. Two epochs; in each, 8 batches (first, second, spread
through the epoch, and the partial last one) are compared with the oracle: seeds,
per-hop offsets and neighbours, sorted distinct vertices, relabelled ids and gathered
feature rows, bit for bit (sampling.py:84-143, :73-75)."""

import math
import multiprocessing as mp
import sys
from pathlib import Path

import numpy as np
import pytest

import gnncache_oracle as O

pytestmark = pytest.mark.gpu


def local_ids(t):
    """Relabelled ids as int64 (the sampler stores u16 in int16 when a window's batches fit)."""
    from paper_2305_16588_b200.sampling import local_ids as decode

    return decode(t)
torch = pytest.importorskip("torch")

ROOT = Path(__file__).resolve().parents[1]
_STATE = {}


def _oracle_batch(args):
    b, gkey = args
    g, shuffled, fan, B, dim = (_STATE[k] for k in ("g", "shuffled", "fan", "B", "dim"))
    seeds = shuffled[b * B : (b + 1) * B]
    hops = O.sample_batch(g.row_offsets, g.col_indices, g.num_vertices, seeds, fan, O.derive(gkey, 2, b))
    uniq = O.distinct_vertices(seeds, hops)
    return b, seeds, hops, uniq


def test_bench_c2_pipeline_matches_oracle():
    sys.path.insert(0, str(ROOT))
    import bench

    from paper_2305_16588_b200 import KeyedRng, SamplingConfig, derive_seed
    from paper_2305_16588_b200.cache import FeatureStore
    from paper_2305_16588_b200.graph import synthetic_features_device
    from paper_2305_16588_b200.pipeline import SampleGatherPipeline

    torch.cuda.set_device(0)
    C = bench.CONFIG
    g, pools, layout = bench.build_inputs(C["num_vertices"], 1)
    pool = pools[0]
    cfg = SamplingConfig(fanouts=tuple(C["fanouts"]), batch_size=C["batch_size"],
                         seed=derive_seed(C["master_seed"], 0x10))
    dim = C["feature_dim"]
    store = FeatureStore.resident(synthetic_features_device(0, g.num_vertices, dim))
    nb = math.ceil(len(pool) / cfg.batch_size)
    assert nb == 235 and len(pool) % cfg.batch_size  # the last batch is partial
    pipe = SampleGatherPipeline(g, cfg, store, len(pool), window=nb, feat_rows_cap=65536, lanes=1)
    root = KeyedRng(cfg.seed)
    check = [0, 1, 2, 58, 117, 175, 233, 234]
    for epoch in (3, 4):  # timed epochs of the default bench (after 3 warm-up epochs)
        gs = root.derive(epoch, 0, 0)
        pipe.run_epoch_graph(pipe.plan_epoch(pool, gs))
        torch.cuda.synchronize()
        pipe.check_capacity(reset=True)
        sp = pipe.sampler
        shuffled = np.asarray(pool)[O.permutation(gs.derive(1).key, len(pool))]
        _STATE.update(g=g, shuffled=shuffled, fan=tuple(C["fanouts"]), B=cfg.batch_size, dim=dim)
        with mp.get_context("fork").Pool(min(len(check), mp.cpu_count())) as workers:
            want = workers.map(_oracle_batch, [(b, gs.key) for b in check])
        counts = sp.counts[:, :nb].cpu().numpy()
        for b, seeds, hops, uniq in want:
            assert counts[0, b] == len(seeds)
            assert np.array_equal(sp.seeds[b, : len(seeds)].cpu().numpy().view(np.uint32), seeds)
            u = int(sp.ucount[b])
            assert u == len(uniq) <= pipe.feat_cap
            assert np.array_equal(sp.unique[b, :u].cpu().numpy().view(np.uint32), uniq)
            assert np.array_equal(local_ids(sp.local_seeds[b, : len(seeds)]).cpu().numpy(), O.relabel(uniq, seeds))
            for h, (_, off, nbr) in enumerate(hops):
                t = int(counts[h + 1, b])
                assert t == len(nbr), (epoch, b, h)
                assert np.array_equal(sp.offsets[h][b, : len(off)].cpu().numpy(), off), (epoch, b, h)
                assert np.array_equal(sp.nbrs[h][b, :t].cpu().numpy().view(np.uint32), nbr), (epoch, b, h)
                assert np.array_equal(local_ids(sp.local_nbrs[h][b, :t]).cpu().numpy(), O.relabel(uniq, nbr)), (epoch, b, h)
            assert np.array_equal(pipe.features[b, :u].cpu().numpy(), O.synthetic_features(uniq, dim)), (epoch, b)
