"""Where TreeTrainer's step time goes (torch.profiler over eager steps, C2 shape).
Usage: python tools/train_tree_profile.py [fp32|bf16]"""
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
from paper_2305_16588_b200.pipeline import SampleGatherPipeline  # noqa: E402
from paper_2305_16588_b200.train import GraphSAGE, TreeTrainer, synthetic_labels, train_epoch_tree  # noqa: E402

torch.cuda.set_device(0)
C = bench.CONFIG
g, pools, layout = bench.build_inputs(C["num_vertices"], 1)
pool = pools[0]
cfg = SamplingConfig(fanouts=tuple(C["fanouts"]), batch_size=C["batch_size"], seed=derive_seed(C["master_seed"], 0x10))
store = FeatureStore.resident(synthetic_features_device(0, g.num_vertices, C["feature_dim"]))
nb = math.ceil(len(pool) / cfg.batch_size)
pipe = SampleGatherPipeline(g, cfg, store, len(pool), window=nb, feat_rows_cap=65536)
plan = pipe.plan_epoch(pool, KeyedRng(cfg.seed).derive(0, 0, 0))
model = GraphSAGE(C["feature_dim"], 256, 47, 3).cuda()
labels = torch.from_numpy(synthetic_labels(np.arange(g.num_vertices), 47)).cuda()
prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
tr = TreeTrainer(model, pipe.sampler, labels, lr=0.1, precision=prec, use_graph=False)
train_epoch_tree(pipe, plan, tr, max_batches=5)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    train_epoch_tree(pipe, plan, tr, max_batches=20)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30, max_name_column_width=90))
