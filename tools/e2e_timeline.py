"""Timeline of the e2e arm's device work (torch.profiler trace events): copies vs kernels.
Usage: python tools/e2e_timeline.py"""
import json
import math
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2305_16588_b200 import KeyedRng, SamplingConfig, derive_seed  # noqa: E402
from paper_2305_16588_b200.cache import FeatureStore  # noqa: E402
from paper_2305_16588_b200.graph import synthetic_features_device  # noqa: E402

torch.cuda.set_device(0)
C = bench.CONFIG
g, pools, layout = bench.build_inputs(C["num_vertices"], 1)
pool = pools[0]
cfg = SamplingConfig(fanouts=tuple(C["fanouts"]), batch_size=C["batch_size"], seed=derive_seed(C["master_seed"], 0x10))
store = FeatureStore.resident(synthetic_features_device(0, g.num_vertices, C["feature_dim"]))


class A:
    steps, warmup, window, visited = 4, 2, 0, "auto"


root = KeyedRng(cfg.seed)
bench.e2e_run(A, g, cfg, store, pool, root, 0, 0, 1)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    r = bench.e2e_run(A, g, cfg, store, pool, root, 0, 0, 1)
print(json.dumps({k: v for k, v in r.items() if k != "api"}))
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    if e.time_range.elapsed_us() > 200 or "Memcpy" in e.name:
        print(f"{(e.time_range.start - t0) / 1000:9.2f} ms  {e.time_range.elapsed_us() / 1000:8.2f} ms  {e.name[:70]}")
