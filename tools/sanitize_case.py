"""Small shapes of every device path, for compute-sanitizer (memcheck / racecheck /
synccheck): register / pull / push (small and large plans, hot rows), the PS surface
(lookup, apply with delays, LRU eviction on both paths), checkpoints, the p2p exchange at
world 1 (exact and codec). Usage: compute-sanitizer --tool memcheck python tools/sanitize_case.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_05897_b200 import hps  # noqa: E402
from paper_2111_05897_b200 import workloads as W  # noqa: E402

dev = torch.device("cuda:0")
rng = np.random.default_rng(0)
S, D = 4, 16
salts = [W.mix64_int(7 + s) for s in range(S)]

# batch surface: small plan, then a large plan with hot rows (> 4096 repeated listings)
t = hps.ShardSet(S, D, 1 << 14, hps.ADAGRAD, salts=salts, device=0)
ew = hps.EmbeddingWorker(t, hps.MEAN)
for B, F, per, space in [(64, 4, 6, 300), (600, 4, 12, 40)]:
    ids, offs = W.random_csr(rng, B, F, per, space)
    g = (rng.standard_normal((B, F, D)) * 0.1).astype(np.float32)
    ew.register_batch(torch.from_numpy(ids.view(np.int64)).to(dev),
                      torch.from_numpy(offs.view(np.int32)).to(dev), B, F)
    ew.serve_pull()
    ew.apply_backward(torch.from_numpy(g).to(dev), 0.05, 1 if B == 64 else 2)
torch.cuda.synchronize()
t.sync()

# PS surface: lookup, tracked apply with delays, untracked apply
ids = rng.integers(0, 500, 200).astype(np.uint64)
t.lookup(ids)
ok, dl = t.apply_gradients(ids, np.ones((200, D), np.float32), np.zeros(200, np.uint64), 0.1, 3)
t.apply_gradients_map({1: np.ones(D, np.float32)}, 0.1)

# checkpoints
img = t.save_checkpoint(0)
t2 = hps.ShardSet(S, D, 1 << 14, hps.ADAGRAD, salts=salts, device=0)
t2.load_checkpoint([t.save_checkpoint(s) for s in range(S)])

# LRU: parallel path and the sequential evicting path
lru = hps.ShardSet(2, D, 0, hps.ADAGRAD, salts=salts[:2], lru_shard_capacity=16)
for k in range(8):
    lru.lookup(rng.integers(0, 80, 20).astype(np.uint64))
    i2 = rng.integers(0, 80, 10).astype(np.uint64)
    lru.apply_gradients(i2, np.ones((10, D), np.float32), np.zeros(10, np.uint64), 0.1, k + 1)
lru.load_checkpoint([lru.save_checkpoint(0), lru.save_checkpoint(1)])

# exchange, world 1 (p2p transport; exact and codec)
import torch.distributed as dist  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29517")
dist.init_process_group("gloo", rank=0, world_size=1)
from paper_2111_05897_b200.sharded import ShardedEmbeddingWorker  # noqa: E402

for kappa in (0.0, 1024.0):
    tab = hps.ShardSet(8, D, 1 << 14, hps.ADAGRAD, salts=[W.mix64_int(7 + s) for s in range(8)])
    sw = ShardedEmbeddingWorker(tab, hps.MEAN, max_ids=4096, codec_kappa=kappa)
    for step in range(2):
        ids, offs = W.random_csr(rng, 32, 3, 4, 100)
        sw.register_batch(torch.from_numpy(ids.view(np.int64)).to(dev),
                          torch.from_numpy(offs.view(np.int32)).to(dev), 32, 3)
        sw.serve_pull()
        sw.apply_backward(torch.from_numpy((rng.standard_normal((32, 3, D)) * 0.1)
                                           .astype(np.float32)).to(dev), 0.05, step + 1)
    torch.cuda.synchronize()
    tab.sync()
dist.destroy_process_group()
print("sanitize case done")
