"""Host-side bench logic that needs no GPU: three-tier window balancing."""

import importlib.util
import math
from pathlib import Path

import pytest

_spec = importlib.util.spec_from_file_location("bench", Path(__file__).resolve().parents[1] / "bench.py")
bench = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(bench)


@pytest.mark.parametrize("nb,window,want", [
    (10840, 1536, 1549),  # C3: 7 equal windows instead of 7 x 1536 + 88
    (10254, 1024, 1026),  # C4
    (6348, 1024, 907),    # C5: rounding down to 6 windows would exceed the window by > 2%
    (1355, 1536, 1355),   # one window per rank at 8 ranks
    (3, 1536, 3),
    (1, 1, 1),
    (4096, 1024, 1024),   # already equal
])
def test_balanced_window(nb, window, want):
    win = bench.balanced_window(nb, window)
    assert win == want
    k = math.ceil(nb / win)
    assert win <= max(1.02 * window, 1) and win <= nb
    assert nb - (k - 1) * win > 0  # no empty window
    assert (k - 1) * win < nb <= k * win


def test_balanced_window_sweep():
    for nb in range(1, 3000, 7):
        for window in (1, 5, 64, 256, 1000):
            win = bench.balanced_window(nb, window)
            k = math.ceil(nb / win)
            assert 1 <= win <= min(nb, math.floor(1.02 * window) + 1)
            last = nb - (k - 1) * win
            assert 0 < last <= win and win - last < k  # equal up to rounding
