"""The hybrid training step: embedding lookup +
dense tower + synchronous dense all-reduce + embedding update, with bounded staleness.

Reference semantics (``Orchestrator::train_loop`` orchestrator.hpp:799-830, hybrid
mode; ``NnWorker::complete_slot`` staleness gate nn_worker.hpp:390-393;
``StepClock`` staleness.hpp:95-200):

  step s:  pull(s)  -- reads see every embedding update of steps <= s-1-tau
           dense forward/backward(s), all-reduce mean of the dense gradient, SGD
           push(s)   -- per-sample embedding gradients, applied in SampleId order

With tau = 0 this is the sync pipeline (pull(s+1) after push(s)). With tau > 0 the
reference lets the embedding path run ahead of the dense tower by up to tau steps.

B200 realisation. All table operations of a trainer go to ONE embedding stream, in an
order that fixes the staleness exactly: ``register+pull(s), push(s-tau)``. The dense
tower runs on a second stream (cuBLAS fp32 GEMMs) and hands its
per-sample embedding gradients back through events. So with tau >= 1 the HBM-bound
embedding work of steps s-tau .. s+1 overlaps the dense compute of step s, while the
table never sees two operations at once (no torn rows, no shared-plan races) and every
run is deterministic. tau + 1 embedding-worker handles (batches in flight) keep each
step's plan and read versions until its push (``protect_reads`` snapshots the read
versions a later mutation would otherwise hide).

Multi-GPU: the dense gradient goes through ``dense.allreduce_mean`` (the reference's
canonical mean, bit-exact) and the embeddings through hash-sharded workers
(``sharded.ShardedEmbeddingWorker``): one per in-flight batch (tau + 1, each with its own
exchange arena and device barriers), used round-robin like the local worker handles. The
owners apply in the exchange's fresh mode, so the staleness delay statistics of the
sharded path count the batch's own step only (values and versions are exact).
"""
from __future__ import annotations

from . import hps
from .dense import DenseTower, allreduce_mean


class HybridTrainer:
    """One NN worker + its embedding worker(s) on one GPU (rank of ``group``)."""

    def __init__(self, table: hps.ShardSet, groups: int, non_id_dim: int, hidden=(64, 32),
                 dense_lr: float = 0.05, embedding_lr: float = 0.05, staleness: int = 0,
                 aggregation: int = hps.MEAN, init_seed: int = 0, group=None,
                 sharded_worker=None, device_step: bool = False, sharded_workers=None):
        import torch

        if staleness < 0:
            raise hps.ConfigError("staleness must be >= 0")
        if sharded_worker is not None:
            sharded_workers = [sharded_worker]
        if sharded_workers is not None and len(sharded_workers) != staleness + 1:
            raise hps.ConfigError("sharded training needs one embedding worker per batch in "
                                  f"flight: {staleness + 1} for staleness {staleness}")
        self.torch = torch
        self.table = table
        self.F = groups
        self.D = table.embedding_dim
        self.non_id_dim = non_id_dim
        self.tau = staleness
        self.dense_lr = dense_lr
        self.embedding_lr = embedding_lr
        self.group = group
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.tower = DenseTower(groups * self.D + non_id_dim, hidden, init_seed, self.device)
        self.sharded = sharded_workers
        self.workers = [] if sharded_workers is not None else \
            [hps.EmbeddingWorker(table, aggregation) for _ in range(staleness + 1)]
        self.emb_stream = torch.cuda.Stream()
        self.dense_stream = torch.cuda.Stream()
        self.step_no = 0
        # device_step: step tags come from the table's device counter (one per push), so
        # a CUDA graph of a step advances them on every replay
        self.flags = hps.ASYNC | (hps.DEVICE_STEP if device_step else 0)
        self.pending = []  # (step, worker slot, batch) pushes held back by the window
        self._bufs = {}
        # sticky device flag: some step's loss or dense gradient was non-finite (the
        # reference raises DivergenceError there, dense_nn.hpp:233,268, and the training
        # loop aborts, orchestrator.hpp:786-788); reported by check() / flush()
        self._diverged = torch.zeros((), dtype=torch.bool, device=self.device)

    # -- buffers: one per in-flight batch ----------------------------------------------
    def _buf(self, k: int, B: int):
        key = (k, B)
        if key not in self._bufs:
            t = self.torch
            self._bufs[key] = dict(
                # local workers pull into this buffer; sharded workers hand out a view of
                # their exchange arena instead
                pooled=None if self.sharded is not None else
                t.empty((B, self.F, self.D), dtype=t.float32, device=self.device),
                grads=t.empty((B, self.F, self.D), dtype=t.float32, device=self.device),
                pulled=t.cuda.Event(), graded=t.cuda.Event())
        return self._bufs[key]

    def _push(self, s: int, k: int, B: int):
        b = self._buf(k, B)
        t = self.torch
        # Under CUDA-graph capture (one graph per step) the dense step of an earlier step
        # belongs to an earlier graph launch, which completes before this one starts: the
        # event dependency is implied (and may not cross captures).
        if not (t.cuda.is_current_stream_capturing() and s != self.step_no):
            self.emb_stream.wait_event(b["graded"])
        g = b["grads"]  # per-sample embedding gradients, [B][F][D]
        with t.cuda.stream(self.emb_stream):
            if self.sharded is not None:
                self.sharded[k].apply_backward(g, self.embedding_lr, s + 1, flags=self.flags)
            else:
                self.workers[k].apply_backward(g, self.embedding_lr, s + 1, flags=self.flags,
                                               stream=self.emb_stream)

    def step(self, ids, offsets, non_id, labels):
        """One hybrid step on device inputs (CSR ids/offsets [B*F+1], non_id [B, nd],
        labels [B]). Returns the step's mean loss as a device scalar (not synchronised)."""
        t = self.torch
        B = labels.shape[0]
        s = self.step_no
        k = s % (self.tau + 1)
        b = self._buf(k, B)
        main = t.cuda.current_stream()
        # the caller's inputs: wait for what main has queued so far (main itself never
        # waits on the trainer's streams inside a step, so step s+1's embedding work is
        # not serialised behind step s's dense work)
        self.emb_stream.wait_stream(main)
        self.dense_stream.wait_stream(main)
        for x_ in (ids, offsets):
            x_.record_stream(self.emb_stream)
        for x_ in (non_id, labels):
            x_.record_stream(self.dense_stream)
        # embedding stream: register + pull(s), then the push tau steps behind
        with t.cuda.stream(self.emb_stream):
            if self.sharded is not None:
                w = self.sharded[k]
                w.register_batch(ids, offsets, B, self.F)
                # zero-copy view of the exchange's pooled buffer: valid until this worker's
                # next forward, tau + 1 steps later, after the dense step consumed it
                b["view"] = w.serve_pull()
            else:
                w = self.workers[k]
                w.register_batch(ids, offsets, B, self.F, stream=self.emb_stream)
                w.serve_pull(out_pooled=b["pooled"], stream=self.emb_stream)
            b["pulled"].record(self.emb_stream)
        # dense stream: forward/backward, synchronous dense all-reduce, SGD
        with t.cuda.stream(self.dense_stream):
            self.dense_stream.wait_event(b["pulled"])
            pooled = b["view"] if self.sharded is not None else b["pooled"]
            # the dense input [pooled | non-id] as two column blocks (no concatenated copy)
            loss, _, _ = self.tower.forward_backward(
                [pooled.reshape(B, -1), non_id], labels, input_grad=b["grads"].view(B, -1),
                input_cols=self.F * self.D)
            g = allreduce_mean(self.tower.grad, self.group)
            finite = t.isfinite(g).all()
            self._diverged |= ~(finite & t.isfinite(loss))
            self.tower.sgd_step(g, self.dense_lr, finite=finite)
            b["graded"].record(self.dense_stream)
        self.pending.append((s, k, B))
        if len(self.pending) > self.tau:
            self._push(*self.pending.pop(0))
        self.step_no += 1
        return loss  # on the dense stream: call sync() before reading it

    def sync(self):
        """Makes the caller's current stream wait for everything issued so far."""
        main = self.torch.cuda.current_stream()
        main.wait_stream(self.dense_stream)
        main.wait_stream(self.emb_stream)

    def check(self):
        """Raises DivergenceError if any step so far saw a non-finite loss or dense
        gradient (its dense update was skipped; host round trip, not capturable). The
        embedding side reports its own rejections through ``table.sync()``."""
        t = self.torch
        self.dense_stream.synchronize()
        if bool(self._diverged.item()):
            self._diverged.zero_()
            raise hps.DivergenceError("hybrid step: non-finite loss or dense gradient; the "
                                      "dense update of that step was not applied")

    def flush(self):
        """Issues the pushes still held back by the staleness window, then reports a
        diverged dense step (check())."""
        while self.pending:
            self._push(*self.pending.pop(0))
        self.sync()
        self.check()
