"""generate_synthetic_device: the reference generator's CSR (graph.py:144-177), bit for
bit, from the device PCG64 jump-ahead + searchsorted kernel (gc_synth_zipf_targets)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _device():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("n,deg,skew,seed", [(2, 1, 1.2, 0), (3, 5, 0.0, 1), (1000, 10, 1.2, 3), (50_000, 14, 1.0, 9),
                                             (77_777, 3, 2.5, 2**63 + 5)])
def test_device_generator_matches_numpy_generator(n, deg, skew, seed):
    import paper_2305_16588_b200 as P

    a = P.generate_synthetic(n, deg, skew, seed)
    b = P.generate_synthetic_device(n, deg, skew, seed)
    assert b.num_vertices == a.num_vertices and b.num_edges == a.num_edges
    assert np.array_equal(a.row_offsets, b.row_offsets)
    assert np.array_equal(a.col_indices, b.col_indices)
    # the primed device placements hold the same arrays
    dev = b.device("hbm")
    assert np.array_equal(dev.col_indices.cpu().numpy().view(np.uint32), a.col_indices)


def test_device_generator_at_c2_shape():
    """BASELINE configs[1]: 2.4M vertices, degree 26 (62.4M draws), the bench's seed."""
    import paper_2305_16588_b200 as P

    seed = P.derive_seed(7, 1)
    a = P.generate_synthetic(2_400_000, 26, 1.2, seed)
    b = P.generate_synthetic_device(2_400_000, 26, 1.2, seed)
    assert np.array_equal(a.col_indices, b.col_indices)


def test_device_generator_matches_the_reference_itself():
    """Against the unmodified reference built into oracle/_ref (when present)."""
    import sys
    from pathlib import Path

    ref = Path(__file__).resolve().parents[1] / "oracle" / "_ref"
    if not (ref / "gnncache").exists():
        pytest.skip("oracle/_ref not built")
    sys.path.insert(0, str(ref))
    import gnncache

    import paper_2305_16588_b200 as P

    r = gnncache.generate_synthetic(30_000, 12, 1.2, seed=1234)
    b = P.generate_synthetic_device(30_000, 12, 1.2, seed=1234)
    assert np.array_equal(r.col_indices, b.col_indices) and np.array_equal(r.row_offsets, b.row_offsets)
