"""Persisted inputs, byte for byte against files the reference itself wrote
(tests/golden/formats.npz from make_golden.py --formats): the LGCSR1 graph format
(graph.py:112-141) and the u32 hotness dump (sampling.py:292-326). CPU only."""

import numpy as np
import pytest


def _graph(golden):
    from paper_2305_16588_b200 import CsrGraph

    d = golden("formats")
    return d, CsrGraph(len(d["graph_ro"]) - 1, len(d["graph_ci"]), d["graph_ro"], d["graph_ci"])


def test_save_csr_is_byte_identical_to_the_reference(golden, tmp_path):
    from paper_2305_16588_b200 import generate_synthetic, save_csr

    d, g = _graph(golden)
    save_csr(g, tmp_path / "a.lgcsr")
    assert (tmp_path / "a.lgcsr").read_bytes() == d["lgcsr1_bytes"].tobytes()
    # the same file from our own generator run (same seed): the generator is pinned too
    save_csr(generate_synthetic(600, 7, 1.1, seed=21), tmp_path / "b.lgcsr")
    assert (tmp_path / "b.lgcsr").read_bytes() == d["lgcsr1_bytes"].tobytes()


def test_load_csr_reads_the_reference_file(golden, tmp_path):
    from paper_2305_16588_b200 import load_csr

    d, _ = _graph(golden)
    p = tmp_path / "ref.lgcsr"
    p.write_bytes(d["lgcsr1_bytes"].tobytes())
    g = load_csr(p)
    assert g.num_vertices == len(d["graph_ro"]) - 1 and g.num_edges == len(d["graph_ci"])
    assert np.array_equal(g.row_offsets, d["graph_ro"]) and np.array_equal(g.col_indices, d["graph_ci"])
    assert g.row_offsets.dtype == np.uint64 and g.col_indices.dtype == np.uint32
    assert not g.col_indices.flags.writeable


def test_load_csr_error_classes(golden, tmp_path):
    """The reference's distinct error classes (graph.py:19-59, tests/test_graph.py:23-91)."""
    from paper_2305_16588_b200.graph import (ColumnRangeError, GraphFormatError, HeaderError,
                                             OffsetMonotonicityError, TruncatedArrayError, load_csr)

    d, _ = _graph(golden)
    raw = bytearray(d["lgcsr1_bytes"].tobytes())
    n = len(d["graph_ro"]) - 1
    head = 6 + 16

    def load(data):
        p = tmp_path / "x.lgcsr"
        p.write_bytes(bytes(data))
        return load_csr(p)

    with pytest.raises(HeaderError):
        load(b"LGCSR")
    with pytest.raises(HeaderError):
        load(b"LGCSR2" + raw[6:])
    with pytest.raises(TruncatedArrayError):
        load(raw[: head + 8 * n])  # offsets cut short
    with pytest.raises(TruncatedArrayError):
        load(raw[:-4])  # one column missing
    with pytest.raises(TruncatedArrayError):
        load(raw + b"\0")
    bad = bytearray(raw)
    bad[head + 8 : head + 16] = (10**6).to_bytes(8, "little")  # offsets[1] > offsets[2]
    with pytest.raises(OffsetMonotonicityError):
        load(bad)
    bad = bytearray(raw)
    bad[head + 8 * (n + 1) : head + 8 * (n + 1) + 4] = (n + 3).to_bytes(4, "little")
    with pytest.raises(ColumnRangeError):
        load(bad)
    for cls in (HeaderError, TruncatedArrayError, OffsetMonotonicityError, ColumnRangeError):
        assert issubclass(cls, GraphFormatError) and issubclass(cls, ValueError)


def _matrices(d):
    from paper_2305_16588_b200 import HotnessMatrices

    return [HotnessMatrices(int(d[f"hot{c}_id"][0]), d[f"hot{c}_topo"].copy(), d[f"hot{c}_feat"].copy(),
                            int(d[f"hot{c}_txn"][0])) for c in range(int(d["num_cliques"][0]))]


def test_write_hotness_is_byte_identical_to_the_reference(golden, tmp_path):
    from paper_2305_16588_b200 import write_hotness

    d = golden("formats")
    write_hotness(tmp_path / "h.bin", _matrices(d))
    assert (tmp_path / "h.bin").read_bytes() == d["hotness_bytes"].tobytes()


def test_read_hotness_reads_the_reference_dump(golden, tmp_path):
    from paper_2305_16588_b200 import read_hotness

    d = golden("formats")
    p = tmp_path / "ref.bin"
    p.write_bytes(d["hotness_bytes"].tobytes())
    got = read_hotness(p)
    want = _matrices(d)
    assert len(got) == len(want) == 2
    for a, b in zip(got, want):
        assert a.clique_id == b.clique_id and a.sampling_txn_total == b.sampling_txn_total
        assert a.topo_hotness.dtype == np.int64 and a.clique_size == b.clique_size
        assert np.array_equal(a.topo_hotness, b.topo_hotness) and np.array_equal(a.feat_hotness, b.feat_hotness)


def test_write_hotness_overflow(tmp_path):
    from paper_2305_16588_b200 import HotnessMatrices, write_hotness

    h = HotnessMatrices(0, np.array([[1 << 32]], dtype=np.int64), np.zeros((1, 1), np.int64), 0)
    with pytest.raises(OverflowError):
        write_hotness(tmp_path / "o.bin", [h])


def test_offsets_from_counts_rebuilds_packed_offsets():
    """window_to_host(compact_ids=True) ships each hop's offsets as u8 per-position
    counts; offsets_from_counts restores the packed int32 layout (each batch from 0),
    empty batches included."""
    from paper_2305_16588_b200.pipeline import offsets_from_counts

    rng = np.random.default_rng(5)
    sizes = [3, 0, 7, 1]
    segs = [rng.integers(0, 16, s).astype(np.uint8) for s in sizes]
    cptr = np.concatenate(([0], np.cumsum(sizes))).astype(np.int64)
    off, optr = offsets_from_counts(np.concatenate(segs), cptr)
    want = np.concatenate([np.concatenate(([0], np.cumsum(s, dtype=np.int64))) for s in segs]).astype(np.int32)
    assert off.dtype.is_floating_point is False and np.array_equal(off.numpy(), want)
    assert np.array_equal(optr, np.concatenate(([0], np.cumsum(np.array(sizes) + 1))))
