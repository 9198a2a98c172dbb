"""Trainer host logic on CPU: the stacked-level forward (one segment mean and one GEMM
pair per layer) equals the level-by-level walk of the sampled position tree."""

import numpy as np
import pytest
import torch
import torch.nn.functional as F


def _per_level_forward(model, batch):
    """Reference walk: h[level] = act(layer(h[level], mean(h[level + 1] children)))."""
    L = len(model.layers)
    h = [batch.features[t] for t in batch.local]
    for li in range(L):
        h = [F.relu(model.layers[li](h[lvl], h[lvl + 1], batch.offsets[lvl])) for lvl in range(L - li)]
    return model.classifier(h[0])


@pytest.mark.parametrize("layer", ["sage", "gcn"])
@pytest.mark.parametrize("fanouts", [(4, 3, 2), (5,), (3, 0)])
def test_stacked_levels_equal_level_walk(layer, fanouts):
    from paper_2305_16588_b200.train import GraphSAGE, TreeBatch

    rng = np.random.default_rng(len(fanouts))
    U, D = 400, 12
    feats = torch.randn(U, D, generator=torch.Generator().manual_seed(3))
    sizes = [25]
    local = [torch.from_numpy(rng.integers(0, U, 25))]
    offsets = []
    for f in fanouts:
        take = rng.integers(0, f + 1, sizes[-1])  # ragged, with empty segments
        off = np.concatenate(([0], np.cumsum(take)))
        offsets.append(torch.from_numpy(off))
        sizes.append(int(off[-1]))
        local.append(torch.from_numpy(rng.integers(0, U, sizes[-1])))
    batch = TreeBatch(feats, local, offsets, torch.from_numpy(rng.integers(0, 5, 25)))
    torch.manual_seed(1)
    model = GraphSAGE(D, 8, 5, len(fanouts), layer=layer)
    with torch.no_grad():
        got = model(batch)
        want = _per_level_forward(model, batch)
    assert torch.allclose(got, want, rtol=1e-6, atol=1e-6)
