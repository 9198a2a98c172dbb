"""Inter-clique LDG partition (gc_partition_ldg, host C++ in the library) against the
reference's own partitions (tests/golden/partition.npz and policies.npz, made by
tests/golden/make_golden.py from partition.py:85-166). Runs on CPU: the BFS root
order comes from the oracle's permutation (the product computes it on the device)."""

import numpy as np
import pytest

import gnncache_oracle as O


def _roots(seed, n):
    return O.permutation(O.derive(int(seed), 0x5EED), n)


def _graph(ro, ci):
    from paper_2305_16588_b200.graph import CsrGraph

    return CsrGraph(len(ro) - 1, len(ci), ro, ci)


@pytest.fixture(scope="module")
def lib():
    from paper_2305_16588_b200 import _lib

    return _lib.load_library()


def test_ldg_matches_reference_partitions(golden, lib):
    from paper_2305_16588_b200.partition import Partitioning, edge_cut_ratio, ldg_assign, ldg_capacity

    g = golden("partition")
    graphs = {}
    for k, (gi, parts, eps100, passes, seed) in enumerate(g["cases"]):
        if gi not in graphs:
            graphs[gi] = _graph(g[f"g{gi}_ro"], g[f"g{gi}_ci"])
        graph = graphs[gi]
        cap = ldg_capacity(graph.num_vertices, int(parts), eps100 / 100.0)
        got, cuts = ldg_assign(graph, int(parts), cap, _roots(seed, graph.num_vertices), int(passes), lib=lib)
        assert np.array_equal(got, g[f"c{k}"]), (gi, parts, eps100, passes, seed)
        assert edge_cut_ratio(graph, Partitioning(got, int(parts))) == float(g[f"c{k}_cut"][0])
        assert np.bincount(got, minlength=int(parts)).max() <= cap
        assert (cuts[:, 1] <= cuts[:, 0]).all()


def test_ldg_matches_policy_pipeline_partitions(golden, lib):
    from paper_2305_16588_b200.partition import ldg_assign, ldg_capacity

    g = golden("policies")
    graph = _graph(g["graph_ro"], g["graph_ci"])
    seed = O.derive(5, 0x52)  # derive_seed(5, 0x52), make_golden.policy_vectors
    checked = 0
    for key in list(g):
        if "_part" not in key or key.endswith("_part1"):
            continue
        parts = int(key.split("_part")[1])
        cap = ldg_capacity(graph.num_vertices, parts, 0.05)
        got, _ = ldg_assign(graph, parts, cap, _roots(seed, graph.num_vertices), 2, lib=lib)
        assert np.array_equal(got, g[key]), key
        checked += 1
    assert checked >= 2


def test_ldg_argument_errors(lib):
    from paper_2305_16588_b200.partition import ldg_assign

    graph = _graph(np.array([0, 1, 2, 2], dtype=np.uint64), np.array([1, 2], dtype=np.uint32))
    with pytest.raises(ValueError):
        ldg_assign(graph, 2, 1, np.arange(3), lib=lib)  # capacity * parts < n
    with pytest.raises(ValueError):
        ldg_assign(graph, 2, 2, np.array([0, 0, 1]), lib=lib)  # not a permutation
    with pytest.raises(ValueError):
        ldg_assign(graph, 4, 2, np.arange(3), lib=lib)  # more parts than vertices


def test_dump_formats(tmp_path):
    """dump_partitioning / dump_tablets write the reference's text lines
    (partition.py:221-232): "v p" per vertex; "v clique gpu" per training vertex."""
    import paper_2305_16588_b200 as P

    part = P.Partitioning(np.array([1, 0, 2, 2, 0], dtype=np.int32), 3)
    P.dump_partitioning(part, tmp_path / "p.txt")
    assert (tmp_path / "p.txt").read_text() == "".join(f"{v} {p}\n" for v, p in enumerate([1, 0, 2, 2, 0]))
    layout = P.block_layout(4, 2)
    tabs = P.TabletAssignment(((np.array([3, 9]), np.array([], dtype=np.int64)), (np.array([1]), np.array([4, 7]))))
    P.dump_tablets(tabs, layout, tmp_path / "t.txt")
    want = "".join(f"{v} {ci} {li}\n" for ci in range(2) for li in range(2) for v in tabs.tablets[ci][li])
    assert (tmp_path / "t.txt").read_text() == want
