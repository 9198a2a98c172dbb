"""Multi-process (gloo, CPU) tests of the exchange steps of the N>1 path."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, fn, *args):
    port = _free_port()
    ctx = mp.get_context("fork")  # CPU-only children: no CUDA state to inherit
    q = ctx.Queue()
    procs = [ctx.Process(target=_entry, args=(r, world, port, fn, args, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    errs = [r for r in results if isinstance(r, str)]
    assert not errs, errs
    return sorted(results, key=lambda r: r[0])


def _entry(rank, world, port, fn, args, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        q.put((rank, fn(rank, world, *args)))
    except Exception as exc:  # surface the failure to the parent
        import traceback

        q.put(f"rank {rank}: {exc}\n{traceback.format_exc()}")
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def _merge(rank, world, rows_t, rows_f):
    from paper_2305_16588_b200.distributed import merge_hotness

    tt, to, ft, fo = merge_hotness(torch.from_numpy(rows_t[rank]), torch.from_numpy(rows_f[rank]), rank)
    return tt.numpy(), to.numpy(), ft.numpy(), fo.numpy()


@pytest.mark.parametrize("world", [2, 4])
def test_merge_hotness_equals_colsum_and_first_argmax(world):
    from paper_2305_16588_b200.distributed import rows_numpy_merge_reference

    rng = np.random.default_rng(world)
    n = 5000
    rows_t = rng.integers(0, 4, size=(world, n)).astype(np.int64)  # many ties: first argmax matters
    rows_f = rng.integers(0, 2**40, size=(world, n)).astype(np.int64)
    rows_f[:, :50] = 7  # all-equal columns -> owner 0
    res = _run(world, _merge, rows_t, rows_f)
    want_tt, want_to = rows_numpy_merge_reference(rows_t)
    want_ft, want_fo = rows_numpy_merge_reference(rows_f)
    for _, (tt, to, ft, fo) in res:
        assert np.array_equal(tt, want_tt) and np.array_equal(to, want_to)
        assert np.array_equal(ft, want_ft) and np.array_equal(fo, want_fo)
        assert (fo[:50] == 0).all()


def _merge_golden(rank, world, ht, hf):
    from paper_2305_16588_b200.distributed import merge_hotness

    tt, to, ft, fo = merge_hotness(torch.from_numpy(ht[rank]), torch.from_numpy(hf[rank]), rank)
    return tt.numpy(), to.numpy(), ft.numpy(), fo.numpy()


def test_merge_reproduces_reference_candidate_totals_and_owners(golden):
    g = golden("planner")
    res = _run(4, _merge_golden, g["HT"], g["HF"])
    for _, (tt, to, ft, fo) in res:
        assert np.array_equal(tt, g["topo_totals"]) and np.array_equal(to, g["topo_owner"])
        assert np.array_equal(ft, g["feat_totals"]) and np.array_equal(fo, g["feat_owner"])


def _exchange(rank, world):
    from paper_2305_16588_b200.distributed import exchange_addresses

    local = [f"slab{rank}", f"offs{rank}"]
    export = lambda t: f"handle:{t}".encode()  # noqa: E731  stand-in for a CUDA IPC handle
    imp = lambda b: b.decode().replace("handle:", "mapped:")  # noqa: E731
    return exchange_addresses(local, rank, world, export=export, import_=imp)


def test_slab_address_exchange():
    res = _run(3, _exchange)
    for rank, table in res:
        for g in range(3):
            prefix = "" if g == rank else "mapped:"
            assert table[g] == [f"{prefix}slab{g}", f"{prefix}offs{g}"]


def _timing(rank, world):
    from paper_2305_16588_b200.distributed import max_over_ranks, sum_over_ranks

    return max_over_ranks(1.5 + rank), sum_over_ranks(10 * (rank + 1))


def test_max_over_ranks_timing_reduction():
    res = _run(2, _timing)
    assert [r[1] for r in res] == [(2.5, 30), (2.5, 30)]


def test_tablets_shard_training_set_disjointly(golden):
    """Per-rank seed pools (split_intra_clique + assign_tablets) equal the reference's."""
    import paper_2305_16588_b200 as P
    from paper_2305_16588_b200.partition import Partitioning

    g = golden("planner")
    train = P.TrainingSet(g["train_ids"], 0.1)
    n = int(g["train_ids"].max()) + 1
    layout = P.block_layout(4, 4)
    pools = P.assign_tablets(P.split_intra_clique(train, Partitioning(np.zeros(n + 10, np.int32), 1), layout), layout)
    for gi in range(4):
        assert np.array_equal(pools[gi], g[f"pool{gi}"])
    allids = np.concatenate(pools)
    assert len(np.unique(allids)) == len(allids) == len(train)
