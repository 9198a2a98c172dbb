"""NVLink topology layer (hardware.py of the reference) against the reference's own
outputs (tests/golden/hardware.npz): clique detection incl. tie-breaking between
maximum cliques and heterogeneous layouts, and the config file format."""

import numpy as np
import pytest


def test_detect_cliques_matches_reference(golden):
    import paper_2305_16588_b200 as P

    g = golden("hardware")
    for k in range(int(g["count"][0])):
        m = P.NvlinkMatrix(g[f"m{k}"])
        size = int(g[f"m{k}_size"][0])
        if size < 0:
            with pytest.raises(P.HeterogeneousTopologyError):
                P.detect_cliques(m)
            continue
        lay = P.detect_cliques(m)
        assert lay.clique_size == size
        assert np.array_equal(np.array([x for c in lay.cliques for x in c]), g[f"m{k}_cliques"]), k


def test_hardware_config_roundtrip(golden, tmp_path):
    import paper_2305_16588_b200 as P

    g = golden("hardware")
    spec = P.HardwareSpec(P.block_layout(8, 4), 123456, 128)
    P.save_hardware_config(spec, tmp_path / "hw.txt")
    assert (tmp_path / "hw.txt").read_text() == str(g["saved_text"][0])
    back = P.load_hardware_config(tmp_path / "hw.txt")
    assert back == spec
    assert P.validate_spec(back) == []
    bad = P.HardwareSpec(P.block_layout(2, 2), 0, 48, uint32_bytes=0)
    assert P.validate_spec(bad) == ["budget must be positive", "cache line not a power of two",
                                    "uint32_bytes must be positive"]
    (tmp_path / "bad.txt").write_text("gpu_count: 2\nnvlink_matrix:\n1 1\n")
    with pytest.raises(ValueError):
        P.load_hardware_config(tmp_path / "bad.txt")  # no clique_budget_bytes
    (tmp_path / "c.txt").write_text("# box\ngpu_count: 4\nclique_budget_bytes: 10  # bytes\nnvlink_matrix:\n"
                                    "1 1 0 0\n1 1 0 0\n0 0 1 1\n0 0 1 1\n")
    assert P.load_hardware_config(tmp_path / "c.txt").layout == P.block_layout(4, 2)
    with pytest.raises(ValueError):
        P.NvlinkMatrix(np.array([[1, 1], [0, 1]], dtype=bool))
    assert P.detect_cliques(P.block_matrix(8, 8)) == P.block_layout(8, 8)
