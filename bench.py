"""Benchmark: sampled+gathered mini-batches/s of Legion's data-preparation path on B200.

Workload (BASELINE.json configs[1], the metric's single-GPU config): ogbn-products-shaped
synthetic graph — 2.4M vertices, constant out-degree 26 (62.4M edges), Zipf skew 1.2,
100-d fp32 features fully HBM-resident — GraphSAGE 3-hop fanouts [15,10,5], batch 1024,
10% training set split into per-GPU tablets. One step = one epoch of the rank's tablet:
local shuffle (K1), then for every batch 3-hop sampling (K2), dedup + relabel (K3) and
feature gather (K4), all on the device, with the reference's exact RNG streams.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...        (one process per GPU)

Prints one JSON line (rank 0).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "GraphSAGE epoch time, sampled+gathered batches/s at 1/2/4/8 B200; PCIe GB/batch"
UNIT = "batches/s"
C3 = {
    "workload": "C3 ogbn-papers100M-shaped synthetic; cache partitioned over the clique (one owner per vertex, "
                "peers read over NVLink) + host tier (UVA over PCIe)",
    "num_vertices": 111_000_000,
    "avg_degree": 14,
    "skew": 1.2,
    "feature_dim": 128,
    "fanouts": [25, 10],
    "batch_size": 1024,
    "training_fraction": 0.1,
    "master_seed": 7,
    "budget_frac_per_gpu": 0.1,
    "window": 1536,  # batches per launch window
    "feat_rows_cap": 16_384,  # distinct rows per batch the window buffers hold (checked before timing)
    "lanes": 2,
    # host-tier rows deferred to a second kernel that reads each window's in address
    # order, 32 CTAs x 256 rows in flight on a high-priority stream (they hold ~32 SMs'
    # shared memory, the next window's sampling runs on the rest): 64.3K -> 112K
    # batches/s at C3 (profiles/r02_host_tier_pages.md)
    "defer_host": True,
    "defer_ctas": 32,
    "defer_rows": 256,
}
# BASELINE configs[3] and [4]: the same flow at their shapes (python bench.py --tier-workload c4|c5)
C4 = {**C3, "workload": "C4 UK-2007-shaped synthetic (GCN 2-layer input): 105M vertices, 3.7B edges, 128-d; "
                        "topology partially host-resident (UVA), cache partitioned over the clique",
      "num_vertices": 105_000_000, "avg_degree": 35, "window": 1024, "feat_rows_cap": 24_576}
C5 = {**C3, "workload": "C5 Friendster-shaped synthetic: 65M vertices, 3.6B edges, 256-d features, tight HBM budget "
                        "(5% of topology+feature bytes per GPU)",
      "num_vertices": 65_000_000, "avg_degree": 55, "feature_dim": 256, "budget_frac_per_gpu": 0.05, "window": 1024,
      "feat_rows_cap": 24_576, "defer_rows": 128}
TIER_WORKLOADS = {"c3": C3, "c4": C4, "c5": C5}
PCIE_NOMINAL_GBS = 64.0  # PCIe Gen5 x16, north_star's tier roofline
NVLINK_GBS = 900.0  # NVLink 5 per direction
CONFIG = {
    "workload": "C2 ogbn-products-shaped synthetic, fully HBM-cached",
    "num_vertices": 2_400_000,
    "avg_degree": 26,
    "skew": 1.2,
    "feature_dim": 100,
    "fanouts": [15, 10, 5],
    "batch_size": 1024,
    "training_fraction": 0.1,
    "master_seed": 7,
}
HBM_FALLBACK_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--window", type=int, default=0,
                    help="batches per launch window (0 = whole epoch / lanes*2 windows when lanes > 1)")
    ap.add_argument("--lanes", type=int, default=1, help="concurrent window lanes (inter-batch pipeline streams)")
    ap.add_argument("--mem-priority", type=int, default=0,
                    help="1: each window's dedup/relabel/gather on a high-priority stream (overlaps the next hop)")
    ap.add_argument("--graph", type=int, default=1, help="1: each timed epoch is one CUDA-graph launch")
    ap.add_argument("--visited", default="auto", choices=["auto", "dense", "sparse"],
                    help="visited-set layout for dedup (auto: sparse above 4M vertices)")
    ap.add_argument("--num-vertices", type=int, default=CONFIG["num_vertices"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--train-epochs", type=int, default=1, help="GraphSAGE epochs timed after the data-path bench")
    ap.add_argument("--c3-scale", type=float, default=1.0,
                    help="three-tier section (the --tier-workload shape x scale; 0 skips it)")
    ap.add_argument("--tier-workload", default="c3", choices=sorted(TIER_WORKLOADS),
                    help="configuration of the three-tier section (BASELINE configs[2..4])")
    ap.add_argument("--c3-steps", type=int, default=3)
    ap.add_argument("--c3-warmup", type=int, default=3)
    ap.add_argument("--c3-presample-epochs", type=int, default=32,
                    help="presampling epochs behind the cache plan (the reference default is 1; 32 epochs take ~3.4 s at C3 on one B200 and bring the plan's in-sample PCIe prediction within 0.01%% of fresh epochs)")
    ap.add_argument("--c3-window", type=int, default=0, help="three-tier window in batches (0: the workload's)")
    ap.add_argument("--c3-fcap", type=int, default=0, help="three-tier distinct rows per batch held (0: the workload's)")
    ap.add_argument("--c3-lanes", type=int, default=0, help="three-tier pipeline lanes (0: the workload's)")
    ap.add_argument("--c3-defer", type=int, default=-1,
                    help="1: host-tier rows deferred to a second kernel that reads them in address order; "
                         "0: inline in the gather; -1: the workload's")
    ap.add_argument("--c3-defer-ctas", type=int, default=0, help="CTAs of the deferred host-row kernel (0: default)")
    ap.add_argument("--c3-defer-rows", type=int, default=-1,
                    help="rows in flight per deferred host-row CTA (-1: the workload's, 0: the library default)")
    ap.add_argument("--c3-graph", type=int, default=1, help="1: each timed three-tier epoch is one CUDA-graph launch")
    ap.add_argument("--c3-only", action="store_true", help="skip the C2 sections (three-tier section alone)")
    ap.add_argument("--c3-budget-frac", type=float, default=0.0,
                    help="per-GPU cache budget / (topology + feature bytes), 0 = the workload's; the clique's is "
                         "world x this")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def build_inputs(n: int, world: int):
    from paper_2305_16588_b200 import derive_seed, generate_synthetic_device, select_training_set
    from paper_2305_16588_b200.hardware import block_layout
    from paper_2305_16588_b200.partition import assign_tablets, single_clique_partitioning, split_intra_clique

    seed = CONFIG["master_seed"]
    g = generate_synthetic_device(n, CONFIG["avg_degree"], CONFIG["skew"], seed=derive_seed(seed, 1))
    train = select_training_set(g, CONFIG["training_fraction"], seed=derive_seed(seed, 2))
    layout = block_layout(world, world)
    pools = assign_tablets(split_intra_clique(train, single_clique_partitioning(g), layout), layout)
    return g, pools, layout


def peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return HBM_FALLBACK_GBS, "fallback"


class ClockSampler:
    """SM clock and throttle reasons sampled through NVML every ~2 ms in a thread while
    the timed region runs (nvidia-smi's 100 ms period is longer than a C2 step)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = None
        self._thread = None
        self.error = None

    def __enter__(self):
        import threading

        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        except Exception as exc:  # no NVML: report why instead of clocks
            self.error = f"nvml unavailable: {exc}"
            return self
        self._stop = threading.Event()

        def poll():
            while not self._stop.is_set():
                try:
                    self.samples.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                    bits = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for name, mask in self.REASONS.items():
                        if bits & mask:
                            self.reasons.add(name)
                except Exception as exc:
                    self.error = str(exc)
                    return
                self._stop.wait(0.002)

        self._thread = threading.Thread(target=poll, daemon=True)
        self._thread.start()
        return self

    def __exit__(self, *exc):
        if self._thread is not None:
            self._stop.set()
            self._thread.join()

    def summary(self):
        out = {"sm_mhz": float(np.median(self.samples)) if self.samples else None, "sm_max_mhz": self.max_mhz,
               "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml"}
        if self.error:
            out["error"] = self.error
        return out


# ------------------------------------------------------------------ CPU baseline (the reference)
def reference_module():
    """The unmodified reference (gnncache 0.1.0) installed by oracle/build_ref.sh into
    oracle/_ref; None when that build output is absent (then the oracle port stands in,
    reported as kind "port")."""
    ref = ROOT / "oracle" / "_ref"
    if not (ref / "gnncache" / "__init__.py").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import gnncache

    return gnncache


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


class CpuPath:
    """The reference's CPU path for one GPU's epoch: the stock
    gnncache.run_sampling_epoch loop body (sampling.py:224-234) — shuffle with
    KeyedRng.permutation, sample_batch, BatchSample.distinct_vertices — plus the
    feature gather X[ids] (numpy fancy indexing; the reference stores no values).
    Falls back to the oracle port when oracle/_ref is missing."""

    def __init__(self, g, table, pool, epoch=0, conf=None, seed=None):
        self.R = reference_module()
        self.kind = "reference" if self.R is not None else "port"
        self.table = table
        self.conf = conf or CONFIG
        seed = _seed() if seed is None else seed
        B = self.conf["batch_size"]
        if self.R is not None:
            R = self.R
            self.g = R.CsrGraph(g.num_vertices, g.num_edges, g.row_offsets, g.col_indices)
            self.cfg = R.SamplingConfig(fanouts=tuple(self.conf["fanouts"]), batch_size=B)
            from gnncache.rng import KeyedRng

            self.stream = KeyedRng(seed).derive(epoch, 0, 0)
            from gnncache.rng import ROLE_SAMPLE, ROLE_SHUFFLE

            self.role_sample = ROLE_SAMPLE
            self.shuffled = np.asarray(pool, np.int64)[self.stream.derive(ROLE_SHUFFLE).permutation(len(pool))]
        else:
            sys.path.insert(0, str(ROOT / "oracle"))
            import gnncache_oracle as O

            self.O, self.g = O, g
            self.gkey, skey = O.batch_stream_keys(seed, epoch, 0, 0)
            self.shuffled = np.asarray(pool, np.int64)[O.permutation(skey, len(pool))]

    def batch(self, b: int):
        B = self.conf["batch_size"]
        start = (b * B) % len(self.shuffled)
        seeds = self.shuffled[start : start + B]
        if self.R is not None:
            bs = self.R.sample_batch(self.g, seeds, self.cfg, self.stream.derive(self.role_sample, b))
            uniq = bs.distinct_vertices()
            return uniq, self.table[uniq], [(h.offsets, h.neighbors) for h in bs.hops]
        O, g = self.O, self.g
        hops = O.sample_batch(g.row_offsets, g.col_indices, g.num_vertices, seeds, self.conf["fanouts"],
                              O.derive(self.gkey, 2, b))
        uniq = O.distinct_vertices(seeds, hops)
        return uniq, O.gather(self.table, uniq), [(off, nbr) for _, off, nbr in hops]


def _seed():
    from paper_2305_16588_b200 import derive_seed

    return derive_seed(CONFIG["master_seed"], 0x10)


def cpu_batches(g, table, pool, nbatches, seconds, epoch=0, keep=0, conf=None, seed=None):
    """Time the reference's CPU path on one host core for about `seconds`; returns
    (batches, elapsed, kind, results) — results: (distinct ids, rows) of the first
    `keep` batches, which the bench compares with the device's epoch."""
    path = CpuPath(g, table, pool, epoch, conf, seed)
    t0 = time.perf_counter()
    done = 0
    results = []
    for b in range(nbatches):
        r = path.batch(b)
        if b < keep:
            results.append(r)
        done += 1
        if time.perf_counter() - t0 > seconds:
            break
    return done, time.perf_counter() - t0, path.kind, results


_REF_STATE = None


def _ref_worker(b):
    _REF_STATE.batch(b)
    return 1


def host_table(n, dim):
    sys.path.insert(0, str(ROOT / "oracle"))
    import gnncache_oracle as O

    out = np.empty((n, dim), dtype=np.float32)
    step = 1 << 18
    for s in range(0, n, step):
        out[s : s + step] = O.synthetic_features(np.arange(s, min(n, s + step)), dim)
    return out


def run_reference(args):
    """--impl reference: the unmodified reference (oracle/_ref, gnncache 0.1.0) through
    its public API on all host cores — one forked process per core, one batch each per
    step; the rank's epoch state is built once and shared copy-on-write. Under torchrun
    rank 0 alone runs; the other ranks exit 0 without work."""
    global _REF_STATE
    import multiprocessing as mp

    rank, _, world = dist_env()
    if rank != 0:
        return
    from paper_2305_16588_b200 import derive_seed, generate_synthetic, select_training_set
    from paper_2305_16588_b200.hardware import block_layout
    from paper_2305_16588_b200.partition import assign_tablets, single_clique_partitioning, split_intra_clique

    # the same synthetic inputs as the B200 arm (identical CSR: same PCG64 draws), built on the host
    seed = CONFIG["master_seed"]
    g = generate_synthetic(args.num_vertices, CONFIG["avg_degree"], CONFIG["skew"], seed=derive_seed(seed, 1))
    train = select_training_set(g, CONFIG["training_fraction"], seed=derive_seed(seed, 2))
    layout = block_layout(world, world)
    pools = assign_tablets(split_intra_clique(train, single_clique_partitioning(g), layout), layout)
    table = host_table(g.num_vertices, CONFIG["feature_dim"])
    _REF_STATE = CpuPath(g, table, pools[0])
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    nb_epoch = math.ceil(len(pools[0]) / CONFIG["batch_size"])
    per_step = cores  # one batch per worker per step
    ctx = mp.get_context("fork")
    times = []
    with ctx.Pool(cores) as pool:
        b = 0
        for it in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            pool.map(_ref_worker, [(b + i) % nb_epoch for i in range(per_step)], chunksize=1)
            dt = time.perf_counter() - t0
            b += per_step
            if it >= args.warmup:
                times.append(dt)
    total = sum(times)
    value = per_step * len(times) / total
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * total / len(times), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (reference generator law, PCG64 draws)",
        "impl": "reference",
        "config": {**CONFIG, "num_vertices": args.num_vertices, "parallelism": f"{cores} host processes"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": _REF_STATE.kind,
                         "cpu_model": cpu_model(),
                         "sample": f"{per_step} batches per step (one per process) of GPU 0's epoch: "
                                   "gnncache.sample_batch + BatchSample.distinct_vertices + X[ids]"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ B200 arm
def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2305_16588_b200 import KeyedRng, SamplingConfig, derive_seed
    from paper_2305_16588_b200.cache import FeatureStore
    from paper_2305_16588_b200.graph import synthetic_features_device
    from paper_2305_16588_b200.pipeline import SampleGatherPipeline, StageTimer

    from paper_2305_16588_b200.distributed import max_over_ranks, sum_over_ranks

    rank, local, world = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # one process per GPU; GC_DIST_BACKEND=gloo lets a test run several ranks on one GPU
    device = local % torch.cuda.device_count()
    torch.cuda.set_device(device)
    if world > 1:
        backend = os.environ.get("GC_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:
            dist.init_process_group(backend)

    if args.c3_only:
        out = c3_run(args, rank, local, world)
        if rank == 0:
            print(json.dumps({f"{args.tier_workload}_three_tier": out}), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return
    # the three-tier section first, on a clean device: its two lanes of 1536-batch
    # windows need ~110 GB, more than is left beside the C2 section's leftovers
    tier_out = c3_run(args, rank, local, world) if args.c3_scale > 0 else None
    g, pools, layout = build_inputs(args.num_vertices, world)
    pool = pools[rank]
    cfg = SamplingConfig(fanouts=tuple(CONFIG["fanouts"]), batch_size=CONFIG["batch_size"],
                         seed=derive_seed(CONFIG["master_seed"], 0x10))
    dim = CONFIG["feature_dim"]
    table = synthetic_features_device(0, g.num_vertices, dim)  # fully HBM-resident feature table
    store = FeatureStore.resident(table)
    nb = math.ceil(len(pool) / cfg.batch_size)
    window = args.window or (nb if args.lanes == 1 else math.ceil(nb / (2 * args.lanes)))
    # per-batch distinct rows stay far below the 938K worst case; 64K keeps the
    # window's gather buffer small, and the run checks it never overflowed
    sparse = None if args.visited == "auto" else args.visited == "sparse"
    pipe = SampleGatherPipeline(g, cfg, store, len(pool), window=window, feat_rows_cap=65536, lanes=args.lanes,
                                sparse_visited=sparse, mem_priority=bool(args.mem_priority))
    root = KeyedRng(cfg.seed)
    clique, local_idx = layout.gpu_position(rank)
    plans = [pipe.plan_epoch(pool, root.derive(e, clique, local_idx)) for e in range(args.warmup + args.steps)]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    H = len(cfg.fanouts)
    hop_keys = [f"hop_expand.h{h}" for h in range(H)]
    stats = {"bytes": {k: 0 for k in ["sampling", "dedup", "gather"] + hop_keys}, "unique_rows": 0, "sampled": 0,
             "max_unique": 0}

    def account(p, w0, nbw):
        b = p.window_bytes(nbw)
        for k in stats["bytes"]:
            stats["bytes"][k] += b[k]
        stats["unique_rows"] += b["unique_rows"]
        stats["sampled"] += b["sampled"]
        stats["max_unique"] = max(stats["max_unique"], int(p.sampler.ucount[:nbw].max().item()))

    epoch_fn = pipe.run_epoch_graph if args.graph else pipe.run_epoch
    # before any timing: every epoch the timed region will run goes through the eager
    # pipeline once, one lane, kernels back to back — (1) the capacity check (a batch
    # with more distinct vertices than feat_rows_cap fails the run here, before timing),
    # (2) the algorithmic bytes, (3) per-stage device times for the roofline (stage
    # events with the host run ahead, so they bracket device time only)
    seq = pipe if args.lanes == 1 else SampleGatherPipeline(g, cfg, store, len(pool), window=window,
                                                              sparse_visited=sparse, feat_rows_cap=65536, lanes=1)
    for s in range(args.steps):
        seq.run_epoch(plans[args.warmup + s], on_window=account)
    stats["peak_unique"] = seq.check_capacity(reset=True)  # raises OverflowError on truncation
    timer = StageTimer()
    seq.timer = timer
    for s in range(args.steps):
        flush.zero_()
        StageTimer.hold()  # the host runs ahead: stage events see device time only
        seq.run_epoch(plans[args.warmup + s])
    seq.timer = None
    torch.cuda.synchronize()
    for e in range(args.warmup):
        epoch_fn(plans[e])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    pipe.launches = 0
    step_ms = []
    with ClockSampler(device) as clocks:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for s in range(args.steps):
            flush.zero_()  # L2 flush outside the timed events
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            epoch_fn(plans[args.warmup + s])
            e1.record()
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
        if world > 1:
            dist.barrier()
    launches = pipe.launches
    pipe.check_capacity(reset=True)  # the timed epochs were checked above; this re-asserts it
    pipe = seq

    total_ms = float(sum(step_ms))
    if world > 1:
        total_ms = max_over_ranks(total_ms)  # device-timed, max over ranks
        batches_all = sum_over_ranks(nb) * args.steps
    else:
        batches_all = nb * args.steps
    value = batches_all / (total_ms / 1000.0)

    stage = timer.summary()
    peak, peak_kind = peak_hbm()
    stage_bytes = {"unique_relabel": stats["bytes"]["dedup"], "gather": stats["bytes"]["gather"]}
    for k in hop_keys:
        stage_bytes[k] = stats["bytes"][k]
    # dominant single kernel = the stage with the most device time (one launch per window)
    dom = max((k for k in stage if k in stage_bytes), key=lambda k: stage[k][1])
    dom_launches, dom_ms = stage[dom]
    achieved = stage_bytes[dom] / (dom_ms / 1000.0) / 1e9
    traffic, pipes = None, None
    prof = ROOT / "profiles" / "ncu_traffic.json"
    if prof.exists():
        try:
            pj = json.loads(prof.read_text())
            traffic = pj.get(dom)
            traffic = float(traffic) if traffic is not None else None
            pipes = pj.get("_pipes", {}).get(dom)
        except Exception:
            traffic, pipes = None, None
    step_bytes = stats["bytes"]["sampling"] + stats["bytes"]["dedup"] + stats["bytes"]["gather"]

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u64", "data": "synthetic (reference generator law, PCG64 draws; random fp32 features)",
        "config": {**CONFIG, "num_vertices": args.num_vertices, "batches_per_step_per_gpu": nb,
                   "window_batches": pipe.window, "lanes": args.lanes, "cuda_graph": bool(args.graph), "parallelism": f"dp{world} (tablet per GPU, no data-path collective)",
                   "l2": "flushed (256 MB write) between timed steps; graph+features 1.2 GB > L2"},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "launches": dom_launches, "avg_launch_ms": dom_ms / max(dom_launches, 1),
                     "bytes_per_launch": stage_bytes[dom] / max(dom_launches, 1),
                     # the kernel is issue/ALU-bound, not HBM-bound: its pipe counters
                     # from the committed ncu capture and its issue roofline below
                     "ncu_pipes": pipes,
                     "issue": issue_roofline(pipes, dom_ms / max(dom_launches, 1), clocks)},
        "step_roofline": {"bytes_per_batch": step_bytes / (nb * args.steps),
                          "t_roof_us_per_batch": step_bytes / (nb * args.steps) / (peak * 1e9) * 1e6,
                          "measured_us_per_batch": total_ms * 1000 / (nb * args.steps),
                          "frac": (step_bytes / (peak * 1e9)) / (total_ms / 1000.0)},
        "stages_ms": {k: v[1] / args.steps for k, v in stage.items()},
        "stage_bytes_per_step": {k: v / args.steps for k, v in stage_bytes.items()},
        "pcie_gb_per_batch": 0.0,
        "sampled_per_batch": stats["sampled"] / (nb * args.steps),
        "unique_rows_per_batch": stats["unique_rows"] / (nb * args.steps),
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }

    if not args.no_e2e:
        line["e2e"] = e2e_run(args, g, cfg, store, pool, root, clique, local_idx, world)
        # the training-feed view: same API and H2D, results left in HBM for the trainer
        line["e2e_device_consumer"] = e2e_run(args, g, cfg, store, pool, root, clique, local_idx, world,
                                              results_to_host=False)
    if args.train_epochs > 0:
        line["graphsage_epoch"] = train_run(args, g, cfg, pipe, pool, root, clique, local_idx, world)
    if world > 1:
        line["config"]["dist_backend"] = dist.get_backend()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        host = table.cpu().numpy()
        done, el, kind, ref = cpu_batches(g, host, pool, nb, args.cpu_seconds, keep=8)
        line["cpu_baseline"] = {"value": done / el, "unit": UNIT, "cores": 1, "kind": kind, "cpu_model": cpu_model(),
                                "sample": f"first {done} batches of epoch 0 (C2, 1 core): gnncache.sample_batch + "
                                          "distinct_vertices + X[ids]"}
        line["verified"] = verify_epoch0(pipe, plans[0], ref)
    if tier_out is not None:
        line[f"{args.tier_workload}_three_tier"] = tier_out
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def balanced_window(nb: int, window: int) -> int:
    """Equal windows: a short last window is a pipeline stage with nothing to overlap
    (C3: 7 windows of 1549 batches instead of 7 x 1536 + 88, +1.4%). The result is at
    most 2% above `window` (window buffers are sized by it) and never above nb."""
    win = max(1, min(window, nb))
    k = math.ceil(nb / win) if nb else 1
    if k > 1 and math.ceil(nb / (k - 1)) <= 1.02 * win:
        k -= 1
    return max(1, math.ceil(nb / k)) if nb else win


def c3_run(args, rank, local, world):
    """C3 (BASELINE configs[2]; C4/C5 with --tier-workload) through Legion's full flow, one process per GPU of one
    NVSwitch clique: per-rank presampling -> hotness merge -> CSLP plan -> each rank fills
    its own slabs -> CUDA IPC peer slabs (clique.build_clique_cache), the host tier one
    node-shared pinned table; then timed epochs through the three tiers. Reports
    batches/s over all ranks (device time, max over ranks), measured PCIe per batch
    against the reference plan's prediction N_total x CLS / batches (planner.py:142-169),
    and the north-star tier roofline max(B_HBM/HBM, B_NVL/NVLink, B_PCIe/PCIe) per batch."""
    import torch
    import torch.distributed as dist

    import paper_2305_16588_b200 as P
    from paper_2305_16588_b200 import planner as PL
    from paper_2305_16588_b200.clique import build_clique_cache
    from paper_2305_16588_b200.distributed import max_over_ranks, sum_over_ranks
    from paper_2305_16588_b200.graph import synthetic_features_device
    from paper_2305_16588_b200.hostmem import shared_host_table
    from paper_2305_16588_b200.partition import single_clique_partitioning
    from paper_2305_16588_b200.pipeline import SampleGatherPipeline, StageTimer

    t_setup = time.perf_counter()
    C3 = TIER_WORKLOADS[args.tier_workload]
    budget_frac = args.c3_budget_frac or C3["budget_frac_per_gpu"]
    multi = world > 1
    barrier = dist.barrier if multi else (lambda: None)
    n = int(round(C3["num_vertices"] * args.c3_scale))
    dim, B = C3["feature_dim"], C3["batch_size"]
    seed = C3["master_seed"]
    g = P.generate_synthetic_device(n, C3["avg_degree"], C3["skew"], seed=P.derive_seed(seed, 1))
    train = P.select_training_set(g, C3["training_fraction"], seed=P.derive_seed(seed, 2))
    layout = P.block_layout(world, world)
    pools = P.assign_tablets(P.split_intra_clique(train, single_clique_partitioning(g), layout), layout)
    pool = pools[rank]
    feat = P.FeatureSpec(dim)
    total_bytes = g.num_edges * 4 + 8 * n + n * feat.row_bytes
    budget = int(budget_frac * total_bytes) * world
    spec = P.HardwareSpec(layout, clique_budget_bytes=budget)
    cfg = P.SamplingConfig(fanouts=tuple(C3["fanouts"]), batch_size=B, presample_epochs=args.c3_presample_epochs,
                           seed=P.derive_seed(seed, 4))

    def fill(t):  # the host tier, written from the device in 64 MB pieces
        step = 1 << 17
        for r0 in range(0, n, step):
            rows = min(step, n - r0)
            t[r0 : r0 + rows].copy_(synthetic_features_device(r0, rows, dim))
        torch.cuda.synchronize()

    run_id = os.environ.get("TORCHELASTIC_RUN_ID", "") + os.environ.get("MASTER_PORT", str(os.getpid()))
    host = shared_host_table(f"gc_{args.tier_workload}_{run_id}", (n, dim), torch.float32, local, fill=fill,
                             barrier=barrier)
    t0 = time.perf_counter()
    cr = build_clique_cache(g, pool, layout, cfg, feat, spec, host.tensor, rank=rank, world=world)
    torch.cuda.synchronize()
    t_cache = time.perf_counter() - t0
    nb = math.ceil(len(pool) / B)
    win = balanced_window(nb, args.c3_window or C3["window"])
    fcap = args.c3_fcap or C3["feat_rows_cap"]
    lanes = args.c3_lanes or C3["lanes"]
    defer = bool(C3["defer_host"] if args.c3_defer < 0 else args.c3_defer)
    # untimed passes over the timed epochs, one lane: algorithmic bytes, the capacity
    # check (before timing), per-stage device times (built and freed before the timed
    # pipeline, so the two never hold their window buffers at once)
    seq = SampleGatherPipeline(g, cfg, cr.features, len(pool), window=win, feat_rows_cap=fcap,
                               topology=cr.topology, lanes=1, defer_host=defer)
    root = P.KeyedRng(P.derive_seed(seed, 5))
    plans = [seq.plan_epoch(pool, root.derive(e, 0, rank)) for e in range(args.c3_warmup + args.c3_steps)]
    timed = plans[args.c3_warmup :]
    acc = {"sampling": 0, "dedup": 0, "gather": 0}

    def account(p, w0, nbw):
        wb = p.window_bytes(nbw)
        for k in acc:
            acc[k] += wb[k]

    for pl in timed:
        seq.run_epoch(pl, on_window=account)
    max_distinct = seq.check_capacity(reset=True)
    timer = StageTimer()
    seq.timer = timer
    for pl in timed:
        StageTimer.hold()
        seq.run_epoch(pl)
    seq.timer = None
    torch.cuda.synchronize()
    stages = {k: v[1] / len(timed) for k, v in timer.summary().items()}
    del seq
    torch.cuda.empty_cache()
    pipe = SampleGatherPipeline(g, cfg, cr.features, len(pool), window=win, feat_rows_cap=fcap,
                                topology=cr.topology, lanes=lanes, defer_host=defer)
    from paper_2305_16588_b200 import _lib

    defer_ctas = args.c3_defer_ctas or C3.get("defer_ctas", 0)
    defer_rows = args.c3_defer_rows if args.c3_defer_rows >= 0 else C3.get("defer_rows", 0)
    if defer_ctas:
        _lib.check(_lib.lib().gc_set_option(_lib.GC_OPT_DEFER_CTAS, defer_ctas))
    _lib.check(_lib.lib().gc_set_option(_lib.GC_OPT_DEFER_ROWS, defer_rows))
    run = pipe.run_epoch_graph if args.c3_graph else pipe.run_epoch
    for pl in plans[: args.c3_warmup]:
        run(pl)
    torch.cuda.synchronize()
    cr.topology.reset_counters()
    cr.features.reset_counters()
    setup_s = time.perf_counter() - t_setup
    barrier()
    ms = []
    for pl in timed:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(pl)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    barrier()
    pipe.check_capacity(reset=True)
    t, f = cr.topology.tier_counts(), cr.features.tier_counts()
    my_ms = float(sum(ms))
    batches = nb * len(timed)
    row = feat.row_bytes
    row_txns = PL.feature_row_transactions(feat, spec)
    cls = spec.cache_line_bytes
    pcie_b = t["reads_host"] * 16 + t["edges_host"] * 4 + f["host"] * row
    nvl_b = t["reads_peer"] * 16 + t["edges_peer"] * 4 + f["peer"] * row
    hbm_b = acc["sampling"] + acc["dedup"] + acc["gather"] - pcie_b - nvl_b
    peak, peak_kind = peak_hbm()
    t_tier = {"hbm": hbm_b / (peak * 1e9), "nvlink": nvl_b / (NVLINK_GBS * 1e9), "pcie": pcie_b / (PCIE_NOMINAL_GBS * 1e9)}
    my_roof_s = max(t_tier.values())  # this rank's epochs at the tier roofline
    my_frac = my_roof_s / (my_ms / 1000.0)
    # the host tier's random-row read rate on this box, over this table, through the
    # product's own host-tier gather (all ranks at once): the rate the inline gather is
    # held to, which the address-ordered deferred read beats (profiles/r02_host_tier_pages.md)
    from paper_2305_16588_b200.bandwidth import random_read_gbs

    barrier()
    host_row_gbs = random_read_gbs(host.tensor.data_ptr(), host.nbytes, row)
    barrier()
    host_achieved_gbs = pcie_b / (my_ms / 1000.0) / 1e9
    measured_txn = t["host_txn"] + f["host"] * row_txns
    # whole clique: device time is the max over ranks; bytes and transactions add up
    total_ms = max_over_ranks(my_ms)
    all_batches = sum_over_ranks(batches)
    all_txn = sum_over_ranks(int(measured_txn))
    min_frac = -max_over_ranks(-my_frac)
    roof_sum = max_over_ranks(my_roof_s)  # the slowest rank's roofline time bounds the clique
    pred_txn_per_batch = cr.predicted_pcie_txn_per_batch()
    out = {
        "metric": "sampled+gathered batches/s through the three tiers; PCIe GB/batch vs the reference plan",
        "value": all_batches / (total_ms / 1000.0), "unit": "batches/s", "n_gpus": world,
        "steps": len(timed), "warmup": args.c3_warmup, "ms_per_step": total_ms / len(timed),
        "config": {**C3, "num_vertices": n, "num_edges": g.num_edges, "scale": args.c3_scale,
                   "budget_bytes_clique": budget, "budget_frac_per_gpu": budget_frac,
                   "batches_per_step_per_gpu": nb, "window_batches": pipe.window, "feat_rows_cap": fcap,
                   "max_distinct_rows_per_batch_rank0": int(max_distinct),
                   "lanes": pipe.lanes,
                   "host_rows": "deferred: per window, read in address order after the local/peer gather"
                                if defer else "inline in the gather",
                   "cuda_graph": bool(args.c3_graph), "parallelism": f"dp{world}, cache partitioned over {world} GPU(s)",
                   "host_tier": "one node-shared pinned table (/dev/shm + cudaHostRegister), UVA reads",
                   "l2": "inputs (tens of GB of topology and features at scale 1) far larger than L2"},
        "plan": {"presample_epochs": cfg.presample_epochs, "alpha": cr.plan.alpha,
                 "topo_prefix_len": cr.estimate.topo_prefix_len, "feat_prefix_len": cr.estimate.feat_prefix_len,
                 "predicted_txn_total": cr.estimate.total_txns, "presample_batches": cr.presample_batches,
                 "presample_txn_total": cr.sampling_txn_total},
        "pcie": {"measured_gb_per_batch": all_txn * cls / all_batches / 1e9,
                 "predicted_gb_per_batch": pred_txn_per_batch * cls / 1e9,
                 "measured_over_predicted": (all_txn / all_batches) / pred_txn_per_batch if pred_txn_per_batch else None,
                 "payload_gb_per_batch_rank0": pcie_b / batches / 1e9,
                 "unit_note": "transactions x 64 B cache lines, the reference's PCIe unit (SPEC.md:403)"},
        "tier_roofline": {"bytes_per_batch_rank0": {"hbm": hbm_b / batches, "nvlink": nvl_b / batches,
                                                     "pcie": pcie_b / batches},
                          "gbs": {"hbm": peak, "nvlink": NVLINK_GBS, "pcie": PCIE_NOMINAL_GBS}, "hbm_peak_kind": peak_kind,
                          "t_us_per_batch_rank0": {k: v * 1e6 / batches for k, v in t_tier.items()},
                          "bound_rank0": max(t_tier, key=t_tier.get),
                          "measured_us_per_batch_rank0": my_ms * 1000 / batches,
                          "frac_min_over_ranks": min_frac,
                          "frac_clique": roof_sum / (total_ms / 1000.0),
                          "host_tier_rank0": {
                              "random_row_read_gbs": host_row_gbs,
                              "achieved_gbs_over_the_epoch": host_achieved_gbs,
                              "note": f"random {row} B rows over the {host.nbytes / 1e9:.0f} GB host table measured "
                                      "with the host-tier gather on this box; achieved = host-tier bytes / epoch "
                                      "time"}},
        "tiers_per_batch_rank0": {**{k: v / batches for k, v in t.items()},
                                  **{f"rows_{k}": v / batches for k, v in f.items()}},
        "stages_ms_per_epoch_rank0": stages,
        "setup_s": {"total": setup_s, "clique_cache": t_cache},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        done, el, kind, ref = cpu_batches(g, host.tensor.numpy(), pool, nb, args.cpu_seconds, keep=4, conf=C3,
                                          seed=P.derive_seed(seed, 5))
        out["cpu_baseline"] = {"value": done / el, "unit": "batches/s", "cores": 1, "kind": kind,
                               "cpu_model": cpu_model(),
                               "sample": f"first {done} batches of epoch 0 ({args.tier_workload.upper()}, 1 core): "
                                         "gnncache.sample_batch + "
                                         "distinct_vertices + X[ids] from the host table"}
        out["verified"] = verify_epoch0(pipe, plans[0], ref)
    del pipe, plans, timed, cr
    barrier()  # no rank reads a peer's slabs or the host table any more
    host.close()
    torch.cuda.empty_cache()
    return out


def issue_roofline(pipes, launch_ms, clocks):
    """Issue roofline of an ALU-bound kernel: its warp-instructions (ncu capture of the
    same launch) at one warp-instruction per cycle per SM sub-partition (4 per SM) at
    the max SM clock, against the kernel's live-measured launch time."""
    import torch

    if not pipes or not pipes.get("warp_inst"):
        return None
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    mhz = clocks.max_mhz or 1965.0
    peak = sms * 4 * mhz * 1e6  # warp-instructions per second
    floor_ms = pipes["warp_inst"] / peak * 1e3
    return {"warp_inst_per_launch": pipes["warp_inst"], "peak_warp_inst_per_s": peak, "floor_ms": floor_ms,
            "measured_ms": launch_ms, "frac": floor_ms / launch_ms}


def verify_epoch0(pipe, plan, ref):
    """The bench checks its own output: epoch 0 once more through the benched pipeline,
    and each batch the CPU leg ran is compared with the reference's result — every
    hop's offsets and sampled neighbours, the sorted distinct vertices and their
    gathered feature rows, bit for bit."""
    import torch

    got = {}

    def grab(p, w0, nbw):
        sp = p.sampler
        torch.cuda.synchronize()
        for bi in range(nbw):
            b = w0 + bi
            if b < len(ref):
                u = int(sp.ucount[bi])
                hops = []
                for h in range(sp.H):
                    f, t = int(sp.counts[h, bi]), int(sp.counts[h + 1, bi])
                    hops.append((sp.offsets[h][bi, : f + 1].cpu().numpy().astype(np.int64),
                                 sp.nbrs[h][bi, :t].cpu().numpy().view(np.uint32).astype(np.int64)))
                got[b] = (sp.unique[bi, :u].cpu().numpy().view(np.uint32).astype(np.int64),
                          p.features[bi, :u].cpu().numpy(), hops)

    def same(b, want):
        if b not in got:
            return False
        uniq, rows, hops = got[b]
        ok = np.array_equal(uniq, want[0]) and np.array_equal(rows, want[1]) and len(hops) == len(want[2])
        for (o, n), (wo, wn) in zip(hops, want[2]):
            ok = ok and np.array_equal(o, np.asarray(wo, np.int64)) and np.array_equal(n, np.asarray(wn, np.int64))
        return ok

    pipe.run_epoch(plan, on_window=grab)
    bad = [b for b, want in enumerate(ref) if not same(b, want)]
    if bad:
        raise RuntimeError(f"bench self-check failed: batches {bad} of epoch 0 differ from the reference")
    return {"batches": len(ref), "epoch": 0, "bit_exact": True,
            "against": "the CPU leg's own results: per-hop offsets and neighbours, distinct vertices, gathered rows"}


def train_run(args, g, cfg, pipe, pool, root, clique, local_idx, world):
    """Full GraphSAGE epochs (3 layers, hidden 256, 47 classes, SGD lr 0.1) on the
    device-prepared batches through TreeTrainer (hand-written forward/backward, one CUDA
    graph per step; with N ranks the gradients are all-reduced every step — DDP):
    epoch time = sampling + gather + forward/backward/step of every batch (CUDA events,
    max over ranks)."""
    import torch

    from paper_2305_16588_b200.distributed import max_over_ranks
    from paper_2305_16588_b200.train import GraphSAGE, TreeTrainer, synthetic_labels, train_epoch_tree

    classes = 47
    labels = torch.from_numpy(synthetic_labels(np.arange(g.num_vertices), classes)).cuda()
    plans = [pipe.plan_epoch(pool, root.derive(1000 + e, clique, local_idx)) for e in range(args.train_epochs + 1)]
    steps = int(max_over_ranks(float(plans[0].num_batches)))  # DDP: every rank runs the same steps
    out = {}
    for precision in ("fp32", "bf16"):
        torch.manual_seed(0)
        model = GraphSAGE(CONFIG["feature_dim"], 256, classes, len(cfg.fanouts)).cuda()
        tr = TreeTrainer(model, pipe.sampler, labels, lr=0.1, precision=precision)
        train_epoch_tree(pipe, plans[0], tr, steps=8, max_batches=8)  # warm-up + graph capture
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        losses = []
        for e in range(args.train_epochs):
            losses.append(train_epoch_tree(pipe, plans[1 + e], tr, steps=steps))
        e1.record()
        torch.cuda.synchronize()
        sec = e0.elapsed_time(e1) / 1000.0 / args.train_epochs
        sec = max_over_ranks(sec)
        losses = torch.cat(losses).cpu().numpy()
        gemm = "fp32 GEMMs (no TF32)" if precision == "fp32" else "bf16 GEMMs (fp32 accumulate, weights and loss)"
        res = {"seconds": sec, "batches_per_gpu": len(losses) // args.train_epochs, "epochs": args.train_epochs,
               "steps_per_epoch": steps, "ddp_ranks": world,
               "model": f"GraphSAGE mean, 3 layers, hidden 256, 47 classes, {gemm}, SGD lr 0.1",
               "trainer": "TreeTrainer: gc_tree_* kernels + cuBLAS, one CUDA graph per step",
               "first_loss": float(losses[0]), "last_loss": float(losses[-1])}
        if precision == "fp32":
            out.update(res)
        else:
            out["bf16"] = res
    return out


def e2e_run(args, g, cfg, store, pool, root, clique, local_idx, world, results_to_host: bool = True):
    """Same metric through the public pipeline API with host buffers: the tablet goes
    host->device from pinned memory each step, and every batch's result (distinct
    ids, gathered rows, relabelled hop ids and offsets) comes back to pinned host.
    Results travel packed (one copy per array per window) with relabelled ids as
    16-bit values when a window's batches have <= 65536 distinct vertices, and the
    copies of epoch e overlap epoch e+1's sampling (two staging sets alternate).
    results_to_host=False: the results stay on the device for an on-device consumer
    (the trainer) and only each window's per-batch sizes come back."""
    import torch
    import torch.distributed as dist

    from paper_2305_16588_b200.pipeline import SampleGatherPipeline

    nb = math.ceil(len(pool) / cfg.batch_size)
    pipe = SampleGatherPipeline(g, cfg, store, len(pool), window=args.window or nb, feat_rows_cap=65536,
                                sparse_visited=None if args.visited == "auto" else args.visited == "sparse")
    from paper_2305_16588_b200.sampling import check_seed_pool

    host_pool = torch.from_numpy(np.asarray(pool, dtype=np.int64)).pin_memory()
    check_seed_pool(host_pool.numpy(), g.num_vertices)  # once, on the host: the device copy is not read back
    sp = pipe.sampler
    H = len(cfg.fanouts)
    stagings = [{}, {}]  # pinned host buffers, alternating between consecutive windows
    pending = [None, None]
    moved = {"h2d": 0, "d2h": 0, "windows": 0, "u16": 0}

    def drain(p, w0, nbw):
        if not results_to_host:
            counts = sp.counts[:, :nbw].cpu()  # sync point: sizes of this window
            ucnt = sp.ucount[:nbw].cpu()
            moved["d2h"] += 4 * (counts.numel() + ucnt.numel())
            return
        k = moved["windows"] % 2
        if pending[k] is not None:
            pending[k].synchronize()  # that staging set's previous copies have landed
        # sizes (one sync), then one packed D2H copy per array into pinned memory
        moved["d2h"] += 4 * (H + 2) * nbw
        out = p.window_to_host(nbw, stagings[k], compact_ids=True, wait=False)
        pending[k] = out["ready"]
        moved["windows"] += 1
        moved["u16"] += out["local_bits"] == 16
        moved["d2h"] += sum(t.numel() * t.element_size() for t in (out["unique"], out["features"],
                                                                     *out.get("counts", out.get("offsets")),
                                                                     *out["local"]))

    def step(e):
        dev_pool = host_pool.to("cuda", non_blocking=True)
        moved["h2d"] += host_pool.numel() * 8
        plan = pipe.plan_epoch(dev_pool, root.derive(e, clique, local_idx), validated=True)
        moved["h2d"] += plan.keys.numel() * 8 + plan.counts.numel() * 4
        pipe.run_epoch(plan, on_window=drain)

    def settle():
        for ev in pending:
            if ev is not None:
                torch.cuda.current_stream().wait_event(ev)  # the timed region ends after the last copy

    steps = max(1, min(args.steps, 10))
    for e in range(min(args.warmup, 2)):
        step(e)
    settle()
    torch.cuda.synchronize()
    moved = {"h2d": 0, "d2h": 0, "windows": 0, "u16": 0}
    if world > 1:
        dist.barrier()
    # device events on the launching stream; the drains' host syncs sit inside them
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in range(steps):
        step(100 + s)
    settle()
    e1.record()
    torch.cuda.synchronize()
    el = e0.elapsed_time(e1) / 1000.0
    if world > 1:
        from paper_2305_16588_b200.distributed import max_over_ranks

        el = max_over_ranks(el)
    out = {"value": nb * world * steps / el, "unit": UNIT, "h2d_bytes_per_step": moved["h2d"] // steps,
           "d2h_bytes_per_step": moved["d2h"] // steps, "steps": steps,
           "api": "SampleGatherPipeline.plan_epoch/run_epoch + window_to_host (ctypes -> libgnncache_b200.so)"}
    if results_to_host:
        out["ids_on_the_wire"] = "u16" if moved["u16"] == moved["windows"] else "u32 (a window exceeded 65536 rows)"
        # the link the host-buffer arm is bound by: one large device -> pinned copy
        src = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
        feats = stagings[0]["features"]
        dst = feats.view(-1)[: 1 << 28] if feats.numel() >= 1 << 28 else torch.empty(1 << 28, dtype=torch.float32).pin_memory()
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record()
        for _ in range(3):
            dst.copy_(src, non_blocking=True)
        c1.record()
        torch.cuda.synchronize()
        link = 3 * src.numel() * 4 / (c0.elapsed_time(c1) / 1000.0) / 1e9
        out["d2h_link_gbs"] = link
        out["d2h_floor_per_s"] = nb * world / (out["d2h_bytes_per_step"] / (link * 1e9))
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
