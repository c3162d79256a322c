"""Per-phase device time of the sharded step (diagnostic; torchrun, N ranks).
Each phase is bracketed by CUDA events on the current stream; prints rank 0's means."""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_05897_b200 import hps  # noqa: E402
from paper_2111_05897_b200 import workloads as W  # noqa: E402
from paper_2111_05897_b200.sharded import ShardedEmbeddingWorker  # noqa: E402

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
cfg = W.sharded_config(world)
cfg.rows = int(os.environ.get("ROWS_PER_GPU", 125_000_000)) * world
D, F, B, S = cfg.dim, cfg.features, cfg.batch, cfg.shards
rows = cfg.table_capacity()
table = hps.ShardSet(S, D, int(rows / world * 1.05) + (1 << 20), hps.ADAGRAD, salts=cfg.salts())
hb = [W.make_batch(cfg, 1000 * rank + m) for m in range(3)]
bs = [(torch.from_numpy(h.ids.view(np.int64)).to(dev), torch.from_numpy(h.offsets.view(np.int32)).to(dev)) for h in hb]
grads = torch.rand((B, F, D), device=dev) * 0.02 - 0.01
transport = os.environ.get("TRANSPORT", "nccl")
ew = ShardedEmbeddingWorker(table, hps.MEAN, transport=transport,
                            max_ids=max(int(h.N) for h in hb))
pooled = torch.empty((B, F, D), device=dev)
ops = ew.ops
names = ["route", "cnt1", "a2a_ids", "lookup", "a2a_rows", "pool", "pairs", "cnt2", "a2a_pos",
         "a2a_con", "apply"] if transport == "nccl" else ["fwd", "pool", "bwd"]
acc = {n: 0.0 for n in names}
wall = 0.0
steps = 12
for it in range(steps + 3):
    ids, offs = bs[it % 3]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    ev[0].record()
    if transport == "p2p":
        ew.register_batch(ids, offs, B, F); ev[1].record()
        ew.serve_pull(out_pooled=pooled); ev[2].record()
        ew.apply_backward(grads, 0.05, it + 1); ev[3].record()
        torch.cuda.synchronize()
        if it >= 3:
            wall += time.perf_counter() - t0
            for k, n in enumerate(names):
                acc[n] += ev[k].elapsed_time(ev[k + 1])
        continue
    send, counts = ops.route(ids, offs, B, F); ev[1].record()
    sc, rc = ew._exchange_counts(counts); ev[2].record()
    rid = ew._a2a(send[:sum(sc)], sc, rc); ev[3].record()
    rows_, ver = ops.lookup(rid); ev[4].record()
    back = ew._a2a(rows_, rc, sc); ev[5].record()
    ops.pool(back, B, F, pooled); ev[6].record()
    pos, con, pc = ops.pairs(grads, ids.numel()); ev[7].record()
    psc, prc = ew._exchange_counts(pc); ev[8].record()
    P = sum(psc)
    rpos = ew._a2a(pos[:P], psc, prc); ev[9].record()
    rcon = ew._a2a(con[:P], psc, prc); ev[10].record()
    ops.apply_pairs(rid, ver, rc, rpos, rcon, prc, 0.05, it + 1, table.epoch(), hps.ASYNC)
    ev[11].record()
    torch.cuda.synchronize()
    if it >= 3:
        wall += time.perf_counter() - t0
        for k, n in enumerate(names):
            acc[n] += ev[k].elapsed_time(ev[k + 1])
table.sync()
# library-side regions of the p2p step (events on the stream, eager steps)
prof = {}
if transport == "p2p":
    table.profile(True)
    for it in range(6):
        ids, offs = bs[it % 3]
        ew.register_batch(ids, offs, B, F)
        ew.serve_pull()
        ew.apply_backward(grads, 0.05, 1000 + it)
    torch.cuda.synchronize()
    for r in ("x_route", "x_barrier", "x_owner_probe", "x_owner_gather", "x_pairs", "x_emit",
              "x_owner_apply", "plan", "sort_small", "sort", "check", "update", "update_multi"):
        ms_, cnt_ = table.profile_get(r)
        prof[r] = ms_ / 6
    table.profile(False)
if rank == 0:
    tot = sum(acc.values()) / steps
    print(f"transport={transport} world={world} per-step device {tot:.3f} ms, wall {1000 * wall / steps:.3f} ms")
    for n in names:
        print(f"  {n:9s} {acc[n] / steps:7.3f} ms")
    for r, v in prof.items():
        print(f"    region {r:15s} {v:7.3f} ms/step")
dist.destroy_process_group()
