"""Host logic of the measured-bandwidth cost objective (no GPU needed)."""

import numpy as np
import pytest

from paper_2305_16588_b200.bandwidth import MeasuredBandwidths, estimate_seconds, spearman
from paper_2305_16588_b200.graph import FeatureSpec
from paper_2305_16588_b200.hardware import HardwareSpec, block_layout
from paper_2305_16588_b200.planner import TrafficEstimate

scipy_stats = pytest.importorskip("scipy.stats")


@pytest.mark.parametrize("seed", range(5))
def test_spearman_matches_scipy_with_ties(seed):
    rng = np.random.default_rng(seed)
    a = rng.integers(0, 12, 40).astype(float)
    b = a * 0.5 + rng.integers(0, 6, 40)
    assert spearman(a, b) == pytest.approx(scipy_stats.spearmanr(a, b).statistic, abs=1e-12)


def test_estimate_seconds_and_json_roundtrip():
    spec = HardwareSpec(block_layout(1, 1), clique_budget_bytes=1 << 20)
    feat = FeatureSpec(128)
    est = TrafficEstimate(1000.0, 8 * 50, 1400.0, 0.5, 50, 10, 20)
    bw = MeasuredBandwidths(2.0, 8.0, 6000.0, None, "unit test")
    want = 1000 * 64 / 2e9 + 50 * 512 / 8e9
    assert estimate_seconds(est, feat, spec, bw) == pytest.approx(want, rel=1e-15)
    assert MeasuredBandwidths.from_json(bw.to_json()) == bw
