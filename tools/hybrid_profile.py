"""Kernel time breakdown of the C5 hybrid step on one GPU (torch.profiler / CUPTI).
Usage: python tools/hybrid_profile.py [staleness] [steps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_05897_b200 import hps  # noqa: E402
from paper_2111_05897_b200 import workloads as W  # noqa: E402
from paper_2111_05897_b200.hybrid import HybridTrainer  # noqa: E402

tau = int(sys.argv[1]) if len(sys.argv) > 1 else 4
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = W.Config("c5p", 16384, 26, 20_000_000, 64, "adagrad", "mean")
dev = torch.device("cuda", 0)
table = hps.ShardSet(cfg.shards, cfg.dim, cfg.table_capacity(), hps.ADAGRAD, salts=cfg.salts())
data = []
for m in range(5):
    b = W.make_batch(cfg, m)
    x, y = W.make_dense_inputs(cfg, b)
    data.append(tuple(torch.from_numpy(a).to(dev) for a in
                      (b.ids.view(np.int64), b.offsets.view(np.int32), x, y)))
tr = HybridTrainer(table, 26, W.C5_NON_ID, hidden=W.C5_HIDDEN, staleness=tau)
for i in range(10):
    tr.step(*data[i % 5])
tr.sync()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(steps):
        tr.step(*data[i % 5])
    tr.sync()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30, max_name_column_width=70))
