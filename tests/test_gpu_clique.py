"""The partitioned clique cache across processes (north-star configuration, scaled down).

World-size 2 and 3 process groups share the one GPU of the test box (gloo for the
collectives — NCCL refuses two ranks on one device; the CUDA IPC mapping of peer slabs
works across processes on one device exactly as across GPUs). Each rank presamples its
own tablet, the hotness rows are merged, every rank derives the plan, fills only its
own slabs from a node-shared host table, maps its peers' slabs, and runs a validation
epoch through the three tiers. Checked against the unmodified reference (oracle/_ref):
the same plan (alpha, estimate, per-GPU assignment), every batch's sampled sub-graph and
gathered rows bit-exact (oracle port), and each rank's measured tier counters equal to
the reference simulator's TrafficReport for that GPU (simulator.py:132-228)."""

import os
import socket
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
N, DEG, DIM, FANOUTS, BATCH = 120_000, 14, 128, (25, 10), 512
BUDGET_FRAC = 0.06  # per GPU; the clique budget is world x this


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(world):
    import paper_2305_16588_b200 as P
    from paper_2305_16588_b200.partition import single_clique_partitioning

    g = P.generate_synthetic(N, DEG, 1.2, seed=P.derive_seed(11, 1))
    train = P.select_training_set(g, 0.1, seed=P.derive_seed(11, 2))
    layout = P.block_layout(world, world)
    pools = P.assign_tablets(P.split_intra_clique(train, single_clique_partitioning(g), layout), layout)
    feat = P.FeatureSpec(DIM)
    budget = int(BUDGET_FRAC * (g.num_edges * 4 + 8 * N + N * feat.row_bytes)) * world
    spec = P.HardwareSpec(layout, clique_budget_bytes=budget)
    cfg = P.SamplingConfig(fanouts=FANOUTS, batch_size=BATCH, presample_epochs=1, seed=P.derive_seed(11, 4))
    return g, train, layout, pools, feat, spec, cfg


def _rank_main(rank, world, port, shm_name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]
    try:
        import torch.distributed as dist

        import paper_2305_16588_b200 as P
        from paper_2305_16588_b200.clique import build_clique_cache
        from paper_2305_16588_b200.graph import synthetic_features_device
        from paper_2305_16588_b200.hostmem import shared_host_table
        from paper_2305_16588_b200.pipeline import SampleGatherPipeline

        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        g, train, layout, pools, feat, spec, cfg = _inputs(world)
        host = shared_host_table(shm_name, (N, DIM), torch.float32, rank,
                                 fill=lambda t: t.copy_(synthetic_features_device(0, N, DIM)),
                                 barrier=dist.barrier)
        cr = build_clique_cache(g, pools[rank], layout, cfg, feat, spec, host.tensor, rank=rank, world=world)
        val_seed = P.derive_seed(11, 5)
        pool = pools[rank]
        pipe = SampleGatherPipeline(g, cfg, cr.features, len(pool), window=7, topology=cr.topology)
        gs = P.KeyedRng(val_seed).derive(0, 0, rank)
        shuffled = np.asarray(pool)[O.permutation(gs.derive(1).key, len(pool))]
        bad = []

        def check(p, w0, nbw):
            sp = p.sampler
            torch.cuda.synchronize()
            counts = sp.counts[:, :nbw].cpu().numpy()
            for bi in range(nbw):
                b = w0 + bi
                seeds = shuffled[b * BATCH : (b + 1) * BATCH]
                hops = O.sample_batch(g.row_offsets, g.col_indices, N, seeds, FANOUTS, gs.derive(2, b).key)
                uniq = O.distinct_vertices(seeds, hops)
                u = int(sp.ucount[bi])
                ok = np.array_equal(sp.unique[bi, :u].cpu().numpy().view(np.uint32), uniq)
                for h, (_, off, nbr) in enumerate(hops):
                    t = int(counts[h + 1, bi])
                    ok &= np.array_equal(sp.nbrs[h][bi, :t].cpu().numpy().view(np.uint32), nbr)
                    ok &= np.array_equal(sp.offsets[h][bi, : len(off)].cpu().numpy(), off)
                    ok &= np.array_equal(local_ids(sp.local_nbrs[h][bi, :t]).cpu().numpy(), O.relabel(uniq, nbr))
                ok &= np.array_equal(p.features[bi, :u].cpu().numpy(), O.synthetic_features(uniq, DIM))
                if not ok:
                    bad.append(b)

        cr.topology.reset_counters()
        cr.features.reset_counters()
        pipe.run_epoch(pipe.plan_epoch(pool, gs), on_window=check)
        torch.cuda.synchronize()
        out = {
            "rank": rank, "bad": bad, "alpha": cr.plan.alpha, "est_total": cr.estimate.total_txns,
            "topo": cr.topology.tier_counts(), "feat": cr.features.tier_counts(),
            "topo_vertices": [np.asarray(v) for v in cr.assignment.topo_vertices],
            "feat_vertices": [np.asarray(v) for v in cr.assignment.feat_vertices],
            "txn_total": cr.sampling_txn_total,
        }
        dist.barrier()  # peers stop reading this rank's slabs before it exits
        q.put(out)
    except Exception as exc:
        import traceback

        q.put(f"rank {rank}: {exc}\n{traceback.format_exc()}")
    finally:
        import torch.distributed as dist

        if dist.is_initialized():
            dist.destroy_process_group()


def _reference(world):
    """The unmodified reference's plan and validation-epoch TrafficReport."""
    ref = ROOT / "oracle" / "_ref"
    if not (ref / "gnncache" / "__init__.py").exists():
        pytest.skip("oracle/_ref not built (python oracle/build_ref.sh or __graft_entry__.build())")
    sys.path.insert(0, str(ref))
    import gnncache as R

    import paper_2305_16588_b200 as P

    g, train, layout, pools, feat, spec, cfg = _inputs(world)
    rg = R.CsrGraph(g.num_vertices, g.num_edges, g.row_offsets, g.col_indices)
    rlayout = R.block_layout(world, world)
    rparts = R.Partitioning(np.zeros(N, dtype=np.int32), 1)
    rtrain = R.select_training_set(rg, 0.1, seed=P.derive_seed(11, 2))
    assert np.array_equal(rtrain.vertex_ids, train.vertex_ids)
    tablets = R.split_intra_clique(rtrain, rparts, rlayout)
    rspec = R.HardwareSpec(rlayout, clique_budget_bytes=spec.clique_budget_bytes)
    rfeat = R.FeatureSpec(DIM)
    rcfg = R.SamplingConfig(fanouts=FANOUTS, batch_size=BATCH, presample_epochs=1, seed=cfg.seed)
    hot = R.run_presampling(rg, tablets, rlayout, rcfg, rspec)[0]
    orders = R.build_candidate_orders(hot)
    plan, est = R.search_optimal_plan(orders, rspec.clique_budget_bytes, 0.01, rg, rfeat, rspec,
                                      hot.sampling_txn_total)
    asg = R.materialize_assignment([orders], [plan], rlayout, rg, rfeat, rspec)
    rpools = R.assign_tablets(tablets, rlayout)
    rep = R.simulate_epoch(rg, rpools, rcfg, asg, rlayout, rspec, rfeat, seed=P.derive_seed(11, 5))
    return hot, plan, est, asg, rep


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_clique_across_processes(world):
    import torch.multiprocessing as mp

    from paper_2305_16588_b200.planner import feature_row_transactions

    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    name = f"gc_test_clique_{os.getpid()}_{port}"
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        results = [q.get(timeout=600) for _ in range(world)]
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.is_alive():
                p.kill()
        if os.path.exists(f"/dev/shm/{name}"):
            os.unlink(f"/dev/shm/{name}")
    errs = [r for r in results if isinstance(r, str)]
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs)
    results.sort(key=lambda r: r["rank"])
    hot, plan, est, asg, rep = _reference(world)
    row_txns = feature_row_transactions(*_inputs(world)[4:6])
    for r in results:
        g = r["rank"]
        assert r["bad"] == [], f"rank {g}: batches {r['bad']} differ from the oracle"
        assert r["txn_total"] == hot.sampling_txn_total
        assert r["alpha"] == plan.alpha and r["est_total"] == est.total_txns
        for k in range(world):
            assert np.array_equal(r["topo_vertices"][k], asg.topo_vertices[k])
            assert np.array_equal(r["feat_vertices"][k], asg.feat_vertices[k])
        t, f = r["topo"], r["feat"]
        assert t["reads_local"] == rep.topo_local_hits[g]
        assert t["reads_peer"] == rep.topo_peer_hits[g]
        assert t["reads_local"] + t["reads_peer"] + t["reads_host"] == rep.topo_reads[g]
        assert t["host_txn"] == rep.sampling_cpu_txn[g]
        assert f["local"] == rep.feat_local_hits[g] and f["peer"] == rep.feat_peer_hits[g]
        assert f["host"] * row_txns == rep.feature_cpu_txn[g]
        # the partitioned cache is exercised on every tier
        assert t["reads_peer"] > 0 and f["peer"] > 0 and f["host"] > 0 and f["local"] > 0
