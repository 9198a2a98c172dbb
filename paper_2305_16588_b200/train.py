"""GraphSAGE training over the device-prepared mini-batches.

The reference has no trainer; Legion's backend is a PyTorch GraphSAGE/GCN
fed by the sampling server. The data-preparation kernels produce,
per batch, the sampled position tree (frontiers are not deduplicated between hops,
sampling.py:123-125): level 0 = seeds, level h+1 = hop h's neighbours with offsets
into level h. Relabel maps every position to a row of the batch's gathered feature
matrix, so the model never touches global ids:

    h0[level]  = X_batch[local_ids[level]]
    layer l    : h[level] = act(W_self h[level] + W_neigh mean(children of level+1))
                 for levels 0 .. L-1-l
    loss       = cross_entropy(classifier(h[0]), labels[seeds])

Layer GEMMs run in PyTorch (north star: tensor cores are not part of this product);
the mean aggregation is a segment reduce over the tree offsets.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.nn as nn
import torch.nn.functional as F


@dataclass
class TreeBatch:
    """One mini-batch as the model consumes it (all tensors on one device)."""

    features: torch.Tensor  # float32 [U, D] gathered rows (U distinct vertices)
    local: list  # per level: int64 [P_level] row index into `features`
    offsets: list  # per hop: int64 [P_level + 1] children offsets into the next level
    labels: torch.Tensor  # int64 [B]


def synthetic_labels(ids, num_classes: int) -> np.ndarray:
    """Deterministic class of a vertex: splitmix64(v) mod C (bench/test input)."""
    v = np.asarray(ids, dtype=np.uint64)
    with np.errstate(over="ignore"):
        v = v ^ (v >> np.uint64(30))
        v = v * np.uint64(0xBF58476D1CE4E5B9)
        v = v ^ (v >> np.uint64(27))
        v = v * np.uint64(0x94D049BB133111EB)
        v = v ^ (v >> np.uint64(31))
    return (v % np.uint64(num_classes)).astype(np.int64)


def segment_mean(x: torch.Tensor, offsets: torch.Tensor) -> torch.Tensor:
    """Mean of x over consecutive segments [offsets[i], offsets[i+1]); empty -> 0."""
    lengths = offsets[1:] - offsets[:-1]
    if x.shape[0] == 0:
        return x.new_zeros((lengths.shape[0], x.shape[1]))
    return torch.segment_reduce(x, "mean", lengths=lengths, unsafe=True, initial=0.0)


def segment_mean_gather(x: torch.Tensor, idx: torch.Tensor, offsets: torch.Tensor) -> torch.Tensor:
    """segment_mean(x[idx], offsets) without materialising x[idx]: on the device one
    kernel (gc_segment_mean_gather) reads the rows straight from x. No gradient flows
    to x (the gathered feature rows are inputs)."""
    segs = offsets.shape[0] - 1
    if not x.is_cuda:
        return segment_mean(x[idx], offsets)
    from . import _lib

    x = x.detach().contiguous()
    idx = idx.to(torch.int64).contiguous()
    offsets = offsets.to(torch.int64).contiguous()
    out = torch.empty((segs, x.shape[1]), dtype=torch.float32, device=x.device)
    _lib.check(_lib.lib().gc_segment_mean_gather(x.data_ptr(), x.shape[1], idx.data_ptr(), offsets.data_ptr(), segs,
                                                 out.data_ptr(), _lib.stream_handle()), "segment_mean_gather")
    return out


class SAGELayer(nn.Module):
    def __init__(self, d_in: int, d_out: int):
        super().__init__()
        self.lin_self = nn.Linear(d_in, d_out)
        self.lin_neigh = nn.Linear(d_in, d_out, bias=False)

    def forward(self, h_self, h_children, offsets, x=None, idx=None):
        """h_children = None with (x, idx): the children are rows x[idx] (first layer)."""
        agg = segment_mean(h_children, offsets) if h_children is not None else segment_mean_gather(x, idx, offsets)
        return self.lin_self(h_self) + self.lin_neigh(agg)


class GCNLayer(nn.Module):
    """Graph convolution on a sampled tree: h' = W (h_self + sum of children) / (deg + 1) + b
    — the mean over the closed neighbourhood (self loop included), one weight matrix."""

    def __init__(self, d_in: int, d_out: int):
        super().__init__()
        self.lin = nn.Linear(d_in, d_out)

    def forward(self, h_self, h_children, offsets, x=None, idx=None):
        deg = (offsets[1:] - offsets[:-1]).to(h_self.dtype).unsqueeze(1)
        mean = segment_mean(h_children, offsets) if h_children is not None else segment_mean_gather(x, idx, offsets)
        agg = mean * deg  # segment sum (0 for empty segments)
        return self.lin((h_self + agg) / (deg + 1.0))


class GraphSAGE(nn.Module):
    """L-layer mean-aggregator GraphSAGE on sampled position trees (layer="gcn": the
    same tree walk with GCNLayer, BASELINE configs[3]'s GCN)."""

    def __init__(self, d_in: int, hidden: int, num_classes: int, num_layers: int, layer: str = "sage"):
        super().__init__()
        dims = [d_in] + [hidden] * num_layers
        kind = {"sage": SAGELayer, "gcn": GCNLayer}[layer]
        self.layers = nn.ModuleList(kind(dims[i], dims[i + 1]) for i in range(num_layers))
        self.classifier = nn.Linear(hidden, num_classes)

    def forward(self, batch: TreeBatch) -> torch.Tensor:
        """Levels are stacked row-wise (level 0, 1, ...), so each layer is one segment
        mean and one GEMM pair over all the levels it updates: layer l's outputs for
        levels 0..L-1-l are a row prefix of the stack and their children (levels
        1..L-l) a contiguous row range; the children offsets of every level are
        rebased into that range once per batch."""
        L = len(self.layers)
        x = batch.features
        c = [0]
        for t in batch.local:
            c.append(c[-1] + t.numel())  # c[k] = positions in levels < k
        offs = torch.cat([batch.offsets[lvl][:-1] + (c[lvl + 1] - c[1]) for lvl in range(L)] +
                         [batch.offsets[L - 1][-1:] + (c[L] - c[1])])
        # first layer: the children's mean is taken straight from the gathered rows
        # (the leaf level, 5x the positions of the level above, is never materialised)
        # under autocast the distinct rows are cast once (U rows), not per position
        xs = x.to(torch.get_autocast_dtype("cuda")) if x.is_cuda and torch.is_autocast_enabled("cuda") else x
        h = F.relu(self.layers[0](xs[torch.cat(batch.local[:L])], None, offs, x=x, idx=torch.cat(batch.local[1:])))
        for li in range(1, L):
            top = c[L - li]  # rows updated by this layer: levels 0 .. L-1-li
            h = F.relu(self.layers[li](h[:top], h[c[1] : c[L - li + 1]], offs[: top + 1]))
        return self.classifier(h[: c[1]])


def tree_batch_from_window(pipe, b: int, labels: torch.Tensor, counts=None, ucount=None) -> TreeBatch:
    """View batch b of the pipeline's current window as a TreeBatch (device tensors;
    u32 ids widen to int64 for indexing). labels: int64 [n] class per vertex;
    counts/ucount: the window's host copies of the per-batch sizes (else read here)."""
    sp = pipe.sampler
    counts = sp.counts[:, b].tolist() if counts is None else [int(c) for c in counts[:, b]]
    u = int(sp.ucount[b].item()) if ucount is None else int(ucount[b])
    feats = pipe.features[b, :u]
    local = [sp.local_seeds[b, : counts[0]].long()]
    offsets = []
    for h in range(sp.H):
        local.append(sp.local_nbrs[h][b, : counts[h + 1]].long())
        offsets.append(sp.offsets[h][b, : counts[h] + 1].long())
    seeds = sp.seeds[b, : counts[0]].long() & 0xFFFFFFFF
    return TreeBatch(feats, local, offsets, labels[seeds])


PRECISIONS = ("fp32", "bf16")


def train_step(model: GraphSAGE, opt: torch.optim.Optimizer, batch: TreeBatch, precision: str = "fp32") -> torch.Tensor:
    """One SGD step. precision="bf16": the layer GEMMs run under bf16 autocast on the
    tensor cores (weights, gathered rows, the neighbour means and the loss stay fp32)."""
    if precision not in PRECISIONS:
        raise ValueError(f"precision must be one of {PRECISIONS}")
    opt.zero_grad(set_to_none=True)
    if precision == "bf16" and batch.features.is_cuda:
        with torch.autocast("cuda", dtype=torch.bfloat16):
            logits = model(batch)
        loss = F.cross_entropy(logits.float(), batch.labels)
    else:
        loss = F.cross_entropy(model(batch), batch.labels)
    loss.backward()
    opt.step()
    return loss.detach()


def train_epoch(pipe, plan, model: GraphSAGE, opt, labels: torch.Tensor, max_batches: int | None = None,
                precision: str = "fp32") -> list:
    """Sample the epoch window by window on the device and train on every batch in
    order; returns the per-batch losses (device scalars)."""
    losses = []

    def consume(p, w0, nbw):
        counts = p.sampler.counts[:, :nbw].cpu().numpy()  # one sync per window for the sizes
        ucount = p.sampler.ucount[:nbw].cpu().numpy()
        if nbw and int(ucount.max()) > p.sampler.ucap:
            raise OverflowError(f"a batch has {int(ucount.max())} distinct vertices but the gather capacity "
                                f"is {p.sampler.ucap}: raise feat_rows_cap")
        for b in range(nbw):
            if max_batches is not None and len(losses) >= max_batches:
                return
            losses.append(train_step(model, opt, tree_batch_from_window(p, b, labels, counts, ucount), precision))

    pipe.run_epoch(plan, on_window=consume)
    return losses
