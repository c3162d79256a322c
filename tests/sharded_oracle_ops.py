"""TEST INFRASTRUCTURE: the local steps of a sharded step restated on the CPU (numpy +
the oracle's C restatement as the owner table), with the same interface as
paper_2111_05897_b200.sharded.DeviceOps. Lets tests drive ShardedEmbeddingWorker's
collective sequencing over a gloo process group without a GPU. Never used by the product.

Restates embedding_worker.hpp:541-557 (pooling) and :726-775 (per-sample fan-out) for the
rows returned by the owners."""
from __future__ import annotations

import numpy as np
import torch

from paper_2111_05897_b200 import hps


class OracleOps:
    def __init__(self, orc, world: int, shard_count: int, dim: int, agg: str = "mean"):
        self.orc = orc
        self.world = world
        self.S = shard_count
        self.D = dim
        self.mean = agg == "mean"

    # distinct ids grouped by owner; first-occurrence order inside an owner's segment
    def route(self, ids, offsets, B, F):
        ids = ids.numpy().view(np.uint64)
        self.offsets = offsets.numpy().astype(np.int64)
        self.B, self.F = B, F
        owner = np.array([hps.route_shard(int(i), self.S) % self.world for i in ids], np.int64)
        seen = {}
        segs = [[] for _ in range(self.world)]
        for i, d in zip(ids, owner):
            if int(i) not in seen:
                seen[int(i)] = (int(d), len(segs[d]))
                segs[d].append(int(i))
        counts = [len(s) for s in segs]
        base = np.concatenate([[0], np.cumsum(counts)])
        self.pos = np.array([base[seen[int(i)][0]] + seen[int(i)][1] for i in ids], np.int64)
        self.dest_of_pos = np.repeat(np.arange(self.world), counts)
        self.base = base
        send = np.array([i for s in segs for i in s], np.uint64)
        return torch.from_numpy(send.view(np.int64).copy()), counts

    def lookup(self, recv_ids):
        ids = recv_ids.numpy().view(np.uint64)
        rows, ver = self.orc.lookup(ids)
        return torch.from_numpy(rows), torch.from_numpy(ver.view(np.int64).copy())

    def pool(self, rows, B, F, out=None):
        rows = rows.numpy()
        res = np.zeros((B, F, self.D), np.float32)
        for sg in range(B * F):
            a, e = self.offsets[sg], self.offsets[sg + 1]
            if e == a:
                continue
            acc = np.zeros(self.D, np.float64)
            for i in range(a, e):
                acc = acc + rows[self.pos[i]].astype(np.float64)
            scale = 1.0 / float(e - a) if self.mean else 1.0
            res[sg // F, sg % F] = (acc * scale).astype(np.float32)
        t = torch.from_numpy(res)
        if out is not None:
            out.copy_(t)
            return out
        return t

    def pairs(self, grads, n_ids):
        g = grads.numpy().reshape(self.B * self.F, self.D)
        per_dest = [[] for _ in range(self.world)]  # (sample, pos, contribution)
        for b in range(self.B):
            acc = {}
            order = []
            for f in range(self.F):
                sg = b * self.F + f
                a, e = self.offsets[sg], self.offsets[sg + 1]
                scale = 1.0 / float(e - a) if (self.mean and e > a) else 1.0
                for i in range(a, e):
                    p = int(self.pos[i])
                    if p not in acc:
                        acc[p] = np.zeros(self.D, np.float64)
                        order.append(p)
                    acc[p] = acc[p] + g[sg].astype(np.float64) * scale
            for p in order:
                d = int(self.dest_of_pos[p])
                per_dest[d].append((p - int(self.base[d]), acc[p].astype(np.float32)))
        counts = [len(x) for x in per_dest]
        flat = [x for d in per_dest for x in d]
        pos = np.array([p for p, _ in flat], np.int32)
        con = np.stack([c for _, c in flat]) if flat else np.zeros((0, self.D), np.float32)
        return torch.from_numpy(pos), torch.from_numpy(con), counts

    def apply_pairs(self, recv_ids, recv_versions, id_counts, pair_pos, contrib, pair_counts, lr,
                    step_tag, epoch, flags=0):
        rid = recv_ids.numpy().view(np.uint64)
        rv = recv_versions.numpy().view(np.uint64)
        ib = np.concatenate([[0], np.cumsum(id_counts)])
        ids, vers = [], []
        k = 0
        for r, pc in enumerate(pair_counts):
            for _ in range(pc):
                j = ib[r] + int(pair_pos[k])
                assert j < ib[r + 1]
                ids.append(rid[j])
                vers.append(rv[j])
                k += 1
        ok, _ = self.orc.apply(np.array(ids, np.uint64), contrib.numpy(),
                               np.array(vers, np.uint64), lr, step_tag, epoch)
        return ok


class EpochOnly:
    """Stand-in for the table handle the worker asks for its epoch."""

    def __init__(self, orc):
        self.orc = orc

    def epoch(self):
        return self.orc.epoch
