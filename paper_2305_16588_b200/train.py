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

from .sampling import local_ids


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
    local = [local_ids(sp.local_seeds[b, : counts[0]])]
    offsets = []
    for h in range(sp.H):
        local.append(local_ids(sp.local_nbrs[h][b, : counts[h + 1]]))
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


# ---------------------------------------------------------------------------------------
# TreeTrainer: the same model and SGD step with a hand-written forward and backward.
_MM_OUT_DTYPE = [None]  # does torch.mm(..., out_dtype=) work here (decided once, outside graph capture)


def _mm_f32_into(out: torch.Tensor, a: torch.Tensor, b: torch.Tensor) -> None:
    """out = a @ b in fp32, written in place when torch supports it (no extra copy)."""
    if a.dtype == torch.float32:
        torch.mm(a, b, out=out)
        return
    if _MM_OUT_INTO[0] is None:
        try:
            torch.mm(a[:1], b[:, :1], out_dtype=torch.float32, out=torch.empty((1, 1), device=a.device))
            _MM_OUT_INTO[0] = True
        except (RuntimeError, TypeError):
            _MM_OUT_INTO[0] = False
    if _MM_OUT_INTO[0]:
        torch.mm(a, b, out_dtype=torch.float32, out=out)
    else:
        out.copy_(_mm_f32(a, b))


_MM_OUT_INTO = [None]


def _splitk_parts(rows: int) -> int:
    """Row chunks of the fp32 weight-gradient GEMM (split-K): one torch.mm over 170K rows
    leaves cuBLAS's SIMT kernel a handful of output tiles; tools/splitk_probe.py."""
    return 32 if rows >= 65536 else (8 if rows >= 8192 else 1)


def _dw_split_into(out: torch.Tensor, g: torch.Tensor, A: torch.Tensor, part: torch.Tensor) -> None:
    """out = g^T A in fp32 as P strided-batched GEMMs over row chunks plus a fixed-order
    sum of the P partials (deterministic; remainder rows added last)."""
    P, rows = part.shape[0], g.shape[0]
    ch = rows // P
    gv = g.as_strided((P, ch, g.shape[1]), (ch * g.stride(0), g.stride(0), 1))
    av = A.as_strided((P, ch, A.shape[1]), (ch * A.stride(0), A.stride(0), 1))
    torch.bmm(gv.transpose(1, 2), av, out=part)
    torch.sum(part, 0, out=out)
    if P * ch < rows:
        out.addmm_(g[P * ch :].t(), A[P * ch :])


def _mm_f32(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """a @ b accumulated and returned in fp32 (bf16 operands stay on the tensor cores)."""
    if a.dtype == torch.float32:
        return a @ b
    if _MM_OUT_DTYPE[0] is None:
        try:
            torch.mm(a[:1], b[:, :1], out_dtype=torch.float32)
            _MM_OUT_DTYPE[0] = True
        except (RuntimeError, TypeError):
            _MM_OUT_DTYPE[0] = False
    return torch.mm(a, b, out_dtype=torch.float32) if _MM_OUT_DTYPE[0] else (a @ b).float()


class TreeTrainer:
    """Training steps of a GraphSAGE / GCN model on the pipeline's windows, B200-native.

    Every position of the sampled tree has exactly one parent, so the whole backward is
    gathers, no atomics: layer l's neighbour aggregation (gc_tree_aggregate) writes
    A_l = [h_self, mean(h_children), 1] (GCN: [closed-neighbourhood mean, 1]) and one
    cuBLAS GEMM with the bias folded into the weights (W_ext = [W | b]) gives the
    pre-activations z_{l+1}; ReLU is applied when the next layer reads them, and the
    backward mask is z > 0. Backward: dW_ext = g^T A_l (the bias gradient is the ones
    column's), dA = g W and gc_tree_aggregate_backward, which routes dA back to each
    position from its own row and its parent's (fused with the mask). The first layer
    reads its inputs straight from the window's gathered feature rows through the
    relabelled ids. Batch b is staged (gc_tree_stage) into padded fixed-shape buffers —
    padded positions have no children and no parent, padded seeds no label — so the whole
    step (stage, forward, backward, SGD) is one CUDA graph, replayed for every batch with
    the batch index read from device memory: no host work and no sync per batch.

    The model's parameters become views into one flat fp32 buffer laid out as the GEMMs
    want it (a layer's self/neighbour weights and bias are column blocks of W_ext); the
    gradients live in a matching flat buffer, so across ranks (DDP) one all-reduce per
    step (NCCL, or gloo for the CPU tests) averages them over the ranks that had a batch
    — a rank whose tablet ran out of batches joins each step with a zero gradient.
    Semantics are GraphSAGE.forward + F.cross_entropy + torch.optim.SGD(lr) (no
    momentum), which tests/test_gpu_train.py checks step by step."""

    def __init__(self, model: GraphSAGE, sampler, labels: torch.Tensor, lr: float, precision: str = "fp32",
                 use_graph: bool = True, group=None):
        import torch.distributed as dist

        from . import _lib

        if precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {PRECISIONS}")
        self.model, self.sp, self.lr = model, sampler, float(lr)
        self.layers = list(model.layers)
        L = len(self.layers)
        if L != sampler.H:
            raise ValueError("the model needs one layer per sampled hop")
        if not sampler.relabel:
            raise ValueError("the trainer needs relabelled windows (SampleGatherPipeline(relabel=True))")
        self.mode = 0 if isinstance(self.layers[0], SAGELayer) else 1
        self.act = torch.bfloat16 if precision == "bf16" else torch.float32
        self.dt = 1 if precision == "bf16" else 0
        self.L = L
        caps = list(sampler.caps)
        self.base = [0]
        for c in caps:
            self.base.append(self.base[-1] + c)
        P = self.base[-1]
        dev = "cuda"
        i32 = torch.int32
        self.b_dev = torch.zeros(1, dtype=i32, device=dev)
        self.loc = torch.zeros(P, dtype=i32, device=dev)
        self.cbeg = torch.zeros(max(self.base[L], 1), dtype=i32, device=dev)
        self.cdeg = torch.zeros(max(self.base[L], 1), dtype=i32, device=dev)
        self.level_counts = torch.zeros(L + 1, dtype=i32, device=dev)
        self.caps_c = (_lib.I64 * (L + 1))(*caps)
        self.labels_b = torch.zeros(caps[0], dtype=torch.int64, device=dev)
        src = _lib.GcTreeSrc()
        src.hops = L
        src.counts = sampler.counts.data_ptr()
        src.counts_stride = sampler.counts.stride(0)
        levels = [sampler.local_seeds] + list(sampler.local_nbrs)
        for k, t in enumerate(levels):
            src.local[k] = t.data_ptr()
            src.local_stride[k] = t.stride(0)
            src.caps[k] = caps[k]
        for h, t in enumerate(sampler.offsets):
            src.offsets[h] = t.data_ptr()
            src.offsets_stride[h] = t.stride(0)
        src.seeds = sampler.seeds.data_ptr()
        src.seeds_stride = sampler.seeds.stride(0)
        self.labels = labels.to(device=dev, dtype=torch.int64).contiguous()
        src.labels = self.labels.data_ptr()
        src.local_bits = sampler.local_bits
        self.src = src
        # per layer: input width d, aggregate width cols (2d SAGE / d GCN), + ones column
        # (the bias), padded to 8 so every row is 16-byte aligned in bf16
        self.shape = []
        for layer in self.layers:
            if isinstance(layer, SAGELayer):
                hid, d = layer.lin_self.weight.shape
                cols = 2 * d
            else:
                hid, d = layer.lin.weight.shape
                cols = d
            self.shape.append((d, cols, (cols + 1 + 7) // 8 * 8, hid))
        # flat parameters: W_ext of every layer [hid, ext], then the classifier W, b
        cls = model.classifier
        sizes = [hid * ext for (_, _, ext, hid) in self.shape] + [cls.weight.numel(), cls.bias.numel()]
        n = sum(sizes)
        self.flat = torch.zeros(n, dtype=torch.float32, device=dev)
        self.gflat = torch.zeros(n + 1, dtype=torch.float32, device=dev)  # + ranks contributing this step
        # the activation-type copy of the parameters the GEMMs read (bf16 runs), refreshed
        # by one cast per step
        self.flat_act = self.flat if self.act == torch.float32 else torch.empty(n, dtype=self.act, device=dev)
        self.W, self.dW, self.W_act = [], [], []
        o = 0
        with torch.no_grad():
            for layer, (d, cols, ext, hid) in zip(self.layers, self.shape):
                W = self.flat[o : o + hid * ext].view(hid, ext)
                self.dW.append(self.gflat[o : o + hid * ext].view(hid, ext))
                self.W_act.append(self.flat_act[o : o + hid * ext].view(hid, ext))
                o += hid * ext
                if isinstance(layer, SAGELayer):
                    parts = [(layer.lin_self.weight, W[:, :d]), (layer.lin_neigh.weight, W[:, d : 2 * d]),
                             (layer.lin_self.bias, W[:, cols])]
                else:
                    parts = [(layer.lin.weight, W[:, :d]), (layer.lin.bias, W[:, cols])]
                for param, view in parts:
                    view.copy_(param.detach())
                    param.data = view
                self.W.append(W)
            k = cls.weight.numel()
            self.Wc = self.flat[o : o + k].view_as(cls.weight)
            self.dWc = self.gflat[o : o + k].view_as(cls.weight)
            self.Wc.copy_(cls.weight.detach())
            cls.weight.data = self.Wc
            o += k
            k = cls.bias.numel()
            self.bc = self.flat[o : o + k]
            self.dbc = self.gflat[o : o + k]
            self.bc.copy_(cls.bias.detach())
            cls.bias.data = self.bc
        self.gflat[n] = 1.0
        # activations: A_l [base_{L-l}, ext] with the ones column; z_{l+1} [base_{L-l}, hid]
        self.A, self.Z = [], []
        for l, (d, cols, ext, hid) in enumerate(self.shape):
            rows = self.base[L - l]
            A = torch.zeros((rows, ext), dtype=self.act, device=dev)
            A[:, cols] = 1.0
            self.A.append(A)
            self.Z.append(torch.zeros((rows, hid), dtype=self.act, device=dev))
        # split-K partials of the fp32 weight gradients (bf16 runs use the tensor cores)
        self.dW_parts = []
        for l, (d, cols, ext, hid) in enumerate(self.shape):
            P = _splitk_parts(self.base[L - l]) if self.act == torch.float32 else 1
            self.dW_parts.append(torch.empty((P, hid, ext), dtype=torch.float32, device=dev) if P > 1 else None)
        self.loss = torch.zeros((), dtype=torch.float32, device=dev)
        # classifier head (gc_tree_head): gradient w.r.t. the top layer's pre-activations
        # of the seed rows, and the kernel's work buffer
        from . import _lib as _L

        ncls, hid_top = self.Wc.shape
        self.g_top = torch.empty((self.base[1], hid_top), dtype=self.act, device=dev)
        self.head_work = torch.empty(int(_L.lib().gc_tree_head_work_floats(self.base[1], ncls, hid_top)),
                                     dtype=torch.float32, device=dev)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.backend = dist.get_backend(group) if self.world > 1 else None
        self.use_graph = use_graph
        self._graphs = None
        self._graph_feats = None
        self.steps = 0

    # ------------------------------------------------------------------ one step
    def _fwd_bwd(self) -> None:
        from . import _lib

        lib, s = _lib.lib(), _lib.stream_handle()
        L, act = self.L, self.act
        _lib.check(lib.gc_tree_stage(self.src, self.b_dev.data_ptr(), self.loc.data_ptr(), self.cbeg.data_ptr(),
                                     self.cdeg.data_ptr(), self.level_counts.data_ptr(), self.labels_b.data_ptr(), s),
                   "tree_stage")
        feats = self._features
        dim = feats.shape[-1]
        if act == torch.float32:
            Wa = self.W
        else:  # one cast of the whole parameter buffer; the layers' weights are views into it
            self.flat_act.copy_(self.flat)
            Wa = self.W_act
        for l in range(L):
            d, cols, ext, hid = self.shape[l]
            A, rows = self.A[l], self.base[L - l]
            if l == 0:  # children rows straight from the gathered features of batch b
                _lib.check(lib.gc_tree_aggregate(feats.data_ptr(), 0, dim, dim, self.loc.data_ptr(),
                                                 self.cbeg.data_ptr(), self.cdeg.data_ptr(), rows, self.mode,
                                                 A.data_ptr(), self.dt, A.stride(0), self.b_dev.data_ptr(),
                                                 feats.stride(0) // dim, s), "tree_aggregate")
            else:  # ReLU of the previous layer's pre-activations, applied as they are read
                z = self.Z[l - 1]
                _lib.check(lib.gc_tree_aggregate(z.data_ptr(), self.dt, z.stride(0), z.shape[1], None,
                                                 self.cbeg.data_ptr(), self.cdeg.data_ptr(), rows, self.mode + 2,
                                                 A.data_ptr(), self.dt, A.stride(0), None, 0, s), "tree_aggregate")
            torch.mm(A, Wa[l].t(), out=self.Z[l])
        # classifier head in one native call: relu, logits (activation-type operands, fp32
        # sums), cross entropy averaged over the batch's real seeds (level_counts[0]; padded
        # seeds carry label -100), dWc, dbc and the gradient g w.r.t. the seed rows of z
        B = self.base[1]
        ztop = self.Z[L - 1][:B]
        ncls, hid_top = self.Wc.shape
        _lib.check(lib.gc_tree_head(ztop.data_ptr(), self.dt, ztop.stride(0), hid_top, B, self.Wc.data_ptr(),
                                    self.bc.data_ptr(), ncls, self.labels_b.data_ptr(), self.level_counts.data_ptr(),
                                    self.loss.data_ptr(), self.dWc.data_ptr(), self.dbc.data_ptr(),
                                    self.g_top.data_ptr(), self.g_top.stride(0), self.head_work.data_ptr(),
                                    self.head_work.numel(), s), "tree_head")
        g = self.g_top
        for l in range(L - 1, -1, -1):
            d, cols, ext, hid = self.shape[l]
            # the ones column of A gives the bias gradient
            if self.dW_parts[l] is not None:
                _dw_split_into(self.dW[l], g, self.A[l], self.dW_parts[l])
            else:
                _mm_f32_into(self.dW[l], g.t(), self.A[l])
            if l == 0:
                break
            dA = g @ Wa[l][:, :cols]
            z = self.Z[l - 1]
            g_in = torch.empty_like(z)
            _lib.check(lib.gc_tree_aggregate_backward(dA.data_ptr(), self.dt, dA.stride(0), z.shape[1], self.mode,
                                                      self.cbeg.data_ptr(), self.cdeg.data_ptr(), dA.shape[0],
                                                      z.shape[0], z.data_ptr(), z.stride(0), g_in.data_ptr(),
                                                      g_in.stride(0), L - l + 1, self.caps_c,
                                                      self.level_counts.data_ptr(), s), "tree_aggregate_backward")
            g = g_in

    def _update(self) -> None:
        n = self.flat.numel()
        if self.world > 1:
            self.flat.sub_(self.gflat[:n] * (self.lr / self.gflat[n].clamp(min=1.0)))
        else:
            self.flat.add_(self.gflat[:n], alpha=-self.lr)

    def _allreduce(self) -> None:
        import torch.distributed as dist

        if self.backend == "nccl":
            dist.all_reduce(self.gflat, group=self.group)
        else:
            host = self.gflat.cpu()
            dist.all_reduce(host, group=self.group)
            self.gflat.copy_(host)

    def _capture(self) -> None:
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm-up outside the capture (cuBLAS handles, lazy init)
            for _ in range(2):
                self._fwd_bwd()
        torch.cuda.current_stream().wait_stream(side)
        g1 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1):
            self._fwd_bwd()
            if self.world == 1:
                self._update()
        g2 = None
        if self.world > 1:
            g2 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g2):
                self._update()
        self._graphs = (g1, g2)

    def step(self, features: torch.Tensor, b: int | None) -> torch.Tensor:
        """One SGD step on batch b of the sampler's current window (features: the
        window's gathered rows [W, ucap, D]); b=None: this rank has no batch left this
        step and joins the gradient all-reduce with zeros. Returns the loss (device)."""
        self._features = features
        if b is None:
            self.gflat.zero_()
            self._allreduce()
            self._update()
            self.gflat[-1] = 1.0
            return self.loss
        self.b_dev.fill_(int(b))
        if not self.use_graph:
            self._fwd_bwd()
            if self.world > 1:
                self._allreduce()
            self._update()
            if self.world > 1:
                self.gflat[-1] = 1.0
        else:
            if self._graphs is None or self._graph_feats != features.data_ptr():
                self._graph_feats = features.data_ptr()
                self._capture()
            g1, g2 = self._graphs
            g1.replay()
            if g2 is not None:
                self._allreduce()
                g2.replay()
                self.gflat[-1] = 1.0
        self.steps += 1
        return self.loss


def train_epoch_tree(pipe, plan, trainer: TreeTrainer, steps: int | None = None, max_batches: int | None = None):
    """One epoch through TreeTrainer: windows sampled on the device, every batch one
    graph replay; with DDP every rank runs `steps` steps (the max over ranks; ranks out
    of batches join with zero gradients). Returns the per-batch losses as one device
    tensor (no host sync inside the epoch)."""
    losses = []

    def consume(p, w0, nbw):
        if p.sampler is not trainer.sp:
            raise ValueError("the trainer was built on another window sampler (use lanes=1)")
        for b in range(nbw):
            if max_batches is not None and len(losses) >= max_batches:
                return
            losses.append(trainer.step(p.features, b).clone())

    pipe.run_epoch(plan, on_window=consume)
    for _ in range(len(losses), steps or 0):
        trainer.step(pipe.features, None)
    pipe.check_capacity(reset=True)
    return torch.stack(losses) if losses else torch.zeros(0, device="cuda")
