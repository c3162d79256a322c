#!/usr/bin/env python
"""Benchmark of the embedding lookup+update hot path (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

One step = one batch of the config's synthetic workload through the embedding worker:
register (route, probe / lazy init, per-row apply order), pull (gather + fp64
pooling) and push (validation + fp64 fan-out + ordered fused Adagrad update), i.e.
SURVEY.md §8(d). The table is pre-warmed (every row of the 100M-row table exists,
M = 0 lazy inits in the timed region). Inputs rotate over --batches distinct
batches whose per-step footprint (rows RMW + grads + pooled > 400 MB) is larger
than L2, so no L2 flush is needed between steps.

Rank 0 prints ONE JSON line. --impl reference times the reference's own CPU path
(oracle/_ref/libhps_ref.so, the reference headers compiled unmodified) on the
box's host cores on bounded samples of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c5"])
    p.add_argument("--staleness", type=int, default=None,
                   help="c5: embedding staleness (default 4 on one GPU; 0 when sharded)")
    p.add_argument("--batches", type=int, default=8, help="distinct batches cycled")
    p.add_argument("--e2e-steps", type=int, default=10)
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--soak-seconds", type=float, default=2.0)
    p.add_argument("--no-graph", action="store_true", help="eager launches instead of CUDA graphs")
    p.add_argument("--no-pipeline", action="store_true",
                   help="C2: register each batch in line instead of beside the previous push")
    p.add_argument("--prefetch-priority", type=int, default=0,
                   help="sharded: stream priority of the next batch's prefetch (0 = lowest)")
    p.add_argument("--step-priority", type=int, default=0,
                   help="sharded: stream priority of the captured step (-1 = above the prefetch)")
    p.add_argument("--e2e-slots", type=int, default=2,
                   help="e2e leg: batches in flight (pinned staging / device buffer sets)")
    p.add_argument("--no-defer-plan-join", action="store_true",
                   help="pipelined steps: join the next batch's plan at its register (A/B)")
    p.add_argument("--register-priority", type=int, default=0,
                   help="stream priority of the next batch's register (0: the step's own; "
                        "-1 = above it measured slower once the check streams, "
                        "profiles/r2_check_probe_ab.txt)")
    p.add_argument("--register-after", default="push", choices=["push", "pull"],
                   help="the next batch's register starts after the previous push (beside "
                        "this step's pull and push) or after this step's pull (beside its push)")
    p.add_argument("--timeline", default="",
                   help="write a CUPTI kernel timeline of a few graph replays to this file")
    p.add_argument("--codec-kappa", type=float, default=0.0,
                   help="N > 1, p2p: kappa-scaled binary16 payloads on NVLink (the reference's "
                        "compress_values; lossy, opt-in); 0 = exact fp32 (default)")
    p.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                   help="N > 1: NVLink peer writes (p2p) or NCCL all-to-alls")
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def nproc():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi samples every 200 ms while the timed region (+ soak) runs."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)
        return self.summary()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() in ("active", "1", "0x1"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- reference arm / cpu baseline


def reference_run(cfg, B_sample, steps, warmup, threads, seconds_cap=None, legs=False):
    """The reference's own path (EmbeddingWorker -> LocalHub -> PsShardService ->
    PsShard, sync order: pull on `threads` threads, ordered single-thread push) on the
    config's batches, compiled from the unmodified headers (oracle/_ref). Like the GPU
    arm, the timed steps cycle over a few distinct batches whose ids were created before
    timing (no lazy inits inside the timed region); the table holds those rows.
    Returns (samples/s, steps timed, rows held, extra legs)."""
    import oracle as O
    from paper_2111_05897_b200 import workloads as W

    M = 2
    batches = [W.make_batch(cfg, 10_000 + m, batch=B_sample) for m in range(M)]
    grads = [W.make_grads(cfg, B_sample, m) for m in range(M)]
    uniq = np.unique(np.concatenate([b.ids for b in batches]))
    shard = (W.mix64(uniq) % np.uint64(cfg.shards)).astype(np.int64)
    per_shard = int(np.bincount(shard, minlength=cfg.shards).max() * 1.25) + 1024
    ref = O.Reference(cfg.salts(), per_shard, cfg.dim, cfg.optimizer, cfg.aggregation,
                      cfg.features)
    for s_ in range(cfg.shards):  # pre-warm: every id the timed steps list exists
        ref.shard_lookup(s_, uniq[shard == s_])
    times = []
    t_start = time.perf_counter()
    for s in range(steps + warmup):
        b, g = batches[s % M], grads[s % M]
        off = b.offsets.astype(np.uint64)
        t0 = time.perf_counter()
        ref.step(b.B, b.ids, off, g, cfg.lr, s + 1, True, threads=threads)
        dt = time.perf_counter() - t0
        if s >= warmup:
            times.append(dt)
        if seconds_cap and time.perf_counter() - t_start > seconds_cap and len(times) >= 1:
            break
    value = B_sample * len(times) / sum(times)
    extra = {}
    if legs:
        # hybrid semantics: the same steps with the push on `threads` threads at once
        ht = []
        for s in range(3):
            b, g = batches[s % M], grads[s % M]
            off = b.offsets.astype(np.uint64)
            t0 = time.perf_counter()
            ref.step(b.B, b.ids, off, g, cfg.lr, 100 + s, True, threads=threads,
                     push_threads=True)
            ht.append(time.perf_counter() - t0)
        extra["hybrid_push_samples_per_s"] = B_sample * len(ht) / sum(ht)
        # raw PsShard::lookup / apply_gradients (the CPU data-structure upper bound), one
        # thread per shard (ctypes releases the GIL), rows of one batch
        import concurrent.futures as cf

        ids0 = np.unique(batches[0].ids)
        sh0 = (W.mix64(ids0) % np.uint64(cfg.shards)).astype(np.int64)
        parts = [ids0[sh0 == s_] for s_ in range(cfg.shards)]
        with cf.ThreadPoolExecutor(max_workers=min(threads, cfg.shards)) as ex:
            t0 = time.perf_counter()
            vers = list(ex.map(lambda s_: ref.shard_lookup(s_, parts[s_])[1], range(cfg.shards)))
            t_look = time.perf_counter() - t0
            gr = [np.full((len(p_), cfg.dim), 1e-3, np.float32) for p_ in parts]
            t0 = time.perf_counter()
            list(ex.map(lambda s_: ref.shard_apply(s_, parts[s_], gr[s_], vers[s_], cfg.lr,
                                                   1000, 0), range(cfg.shards)))
            t_app = time.perf_counter() - t0
        extra["ps_lookup_rows_per_s"] = len(ids0) / t_look
        extra["ps_apply_rows_per_s"] = len(ids0) / t_app
        extra["ps_threads"] = min(threads, cfg.shards)
    return value, len(times), int(len(uniq)), extra


def run_reference_arm(args):
    from paper_2111_05897_b200 import workloads as W

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = W.CONFIGS["c2" if args.config == "c5" else args.config]
    B_sample = cfg.batch
    cores = nproc()
    value, n, rows, extra = reference_run(cfg, B_sample, args.steps, args.warmup, cores,
                                          legs=True)
    conf = workload_config(cfg, args)
    conf["rows"] = rows
    conf["reference_rows_note"] = (f"the reference's PsShards hold the {rows} rows the timed "
                                   f"batches list (created before timing, as the GPU arm's "
                                   f"pre-warm); the GPU table holds {cfg.table_capacity()}")
    line = {
        "impl": "reference", "metric": "embedding lookup+update samples/sec", "value": value,
        "unit": "samples/s", "n_gpus": args.gpus, "steps": n, "warmup": args.warmup,
        "ms_per_step": 1000.0 * B_sample / value, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 (fp64 pooling/fan-out)", "data": "synthetic",
        "config": conf,
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": "reference",
                         "sample": f"{n} steps x {B_sample} samples of {cfg.name} (2 distinct "
                                   f"batches, pre-warmed rows), pull on {cores} threads + "
                                   f"ordered single-thread push, reference headers via "
                                   f"oracle/_ref"},
        "legs": extra,
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(cfg, args):
    d = {"workload": f"{cfg.name}: batch {cfg.batch}, {cfg.features} "
                     f"{'multi-hot' if cfg.multi_hot else 'one-hot'} features, "
                     f"{cfg.rows // 1_000_000}M-row table dim {cfg.dim}, {cfg.optimizer}, "
                     f"{cfg.aggregation} pooling, staleness 0",
         "global_batch": cfg.batch * args.gpus, "rows": cfg.table_capacity(), "dim": cfg.dim,
         "features": cfg.features, "logical_shards": cfg.shards,
         "parallelism": f"replicas{args.gpus}" if args.gpus > 1 else "single",
         "l2": "per-step footprint > L2 (126 MB); no flush",
         "table": "in-order step tags, latest-bump-tag delays (no HPS_TABLE_TAG_RING)"}
    return d


# ---------------------------------------------------------------- C5: the hybrid step


def hybrid_cpu_baseline(cfg, B_s, steps=3):
    """C5 on the reference's own CPU code (oracle/_ref: EmbeddingWorker -> PsShardService
    -> PsShard pull on all threads, the reference's DenseNet batch_forward_backward and
    sgd_step, the ordered push), on a bounded sample: B_s samples of the C5 shape per step,
    the rows they list created first. Returns (samples/s, cores, sample description)."""
    import oracle as O
    from paper_2111_05897_b200 import workloads as W

    hb = W.make_batch(cfg, 20_000, batch=B_s)
    x, y = W.make_dense_inputs(cfg, hb)
    D, F = cfg.dim, cfg.features
    uniq = np.unique(hb.ids)
    shard = (W.mix64(uniq) % np.uint64(cfg.shards)).astype(np.int64)
    per_shard = int(np.bincount(shard, minlength=cfg.shards).max() * 1.25) + 1024
    ref = O.Reference(cfg.salts(), per_shard, D, cfg.optimizer, cfg.aggregation, F)
    for s_ in range(cfg.shards):
        ref.shard_lookup(s_, uniq[shard == s_])
    dims = [F * D + W.C5_NON_ID, *W.C5_HIDDEN]
    params = O.ref_dense_init(dims, 0)
    cores = nproc()
    off = hb.offsets.astype(np.uint64)
    times = []
    for s in range(steps + 1):
        t0 = time.perf_counter()
        pooled, _, _ = ref.step(B_s, hb.ids, off, None, 0.0, s + 1, True, threads=cores,
                                pull=True, push=False)
        inputs = np.concatenate([pooled.reshape(B_s, F * D), x], axis=1)
        _, _, dg, ig = O.ref_dense_fwd_bwd(dims, params, inputs, y)
        params = O.ref_sgd_step(params, dg, cfg.lr)
        g = np.ascontiguousarray(ig[:, :F * D].reshape(B_s, F, D))
        ref.step(B_s, hb.ids, off, g, cfg.lr, s + 1, True, threads=cores, pull=False,
                 push=True)
        if s > 0:
            times.append(time.perf_counter() - t0)
    return (B_s * len(times) / sum(times), cores,
            f"{len(times)} steps x {B_s} samples of the C5 shape (pre-warmed rows): pull on "
            f"{cores} threads, DenseNet {dims}+1 fwd/bwd + SGD, ordered push (oracle/_ref)")


def run_hybrid(args, world, rank, local, dev):
    """C5: embedding lookup + dense tower (1677 -> 64 -> 32 -> 1, fp32 cuBLAS) + the
    reference's canonical dense all-reduce + embedding update (HybridTrainer), bounded
    staleness (default 4: the embedding stream runs up to 4 steps ahead of the dense
    stream). One GPU: local table. N GPUs: the hash-sharded table (one exchange per batch
    in flight) and the dense gradient all-reduced every step."""
    import torch
    import torch.distributed as dist

    from paper_2111_05897_b200 import hps
    from paper_2111_05897_b200 import workloads as W
    from paper_2111_05897_b200.hybrid import HybridTrainer
    from paper_2111_05897_b200.sharded import ShardedEmbeddingWorker

    if world > 1:
        cfg = W.sharded_config(world)
        tau = W.C5_STALENESS if args.staleness is None else args.staleness
    else:
        cfg = W.CONFIGS["c5"]
        tau = W.C5_STALENESS if args.staleness is None else args.staleness
    D, F, B, S = cfg.dim, cfg.features, cfg.batch, cfg.shards
    rows = cfg.table_capacity()
    cap = int(rows / world * 1.01) + (1 << 20) if world > 1 else rows
    # in-order step tags (one pipeline, device step counter): each row's latest bump tag
    # counts delays exactly, no tag ring needed (it would refuse out-of-order tags)
    table = hps.ShardSet(S, D, cap, hps.ADAGRAD, salts=cfg.salts(), device=local,
                         tag_ring=False)
    stream = torch.cuda.current_stream()
    t0 = time.perf_counter()
    chunk = 1 << 23
    for a in range(0, rows, chunk):
        n = min(chunk, rows - a)
        ids = torch.arange(a, a + n, dtype=torch.int64, device=dev)
        if world > 1:
            ids = ids[(hps.route(ids, S, stream=stream).to(torch.int64) % world) == rank]
        table.lookup(ids, stream=stream)
    torch.cuda.synchronize()
    prewarm_s = time.perf_counter() - t0
    M = args.batches
    data = []
    for m in range(M):
        hb = W.make_batch(cfg, 1000 * rank + m)
        x, y = W.make_dense_inputs(cfg, hb)
        data.append(tuple(torch.from_numpy(a).to(dev) for a in
                          (hb.ids.view(np.int64), hb.offsets.view(np.int32), x, y)))
    sharded = None
    if world > 1:  # one hash-sharded worker (exchange arena) per batch in flight
        sharded = [ShardedEmbeddingWorker(table, hps.MEAN, transport=args.transport,
                                          max_ids=max(int(d[0].numel()) for d in data))
                   for _ in range(tau + 1)]
    use_graph = not args.no_graph
    tr = HybridTrainer(table, F, W.C5_NON_ID, hidden=W.C5_HIDDEN, dense_lr=cfg.lr,
                       embedding_lr=cfg.lr, staleness=tau, sharded_workers=sharded,
                       device_step=use_graph)
    torch.backends.cuda.matmul.allow_tf32 = False  # fp32 dense tower, as the reference
    it = 0
    # (at least one eager step per in-flight batch: every worker's exchange arena and
    # buffers exist before the steps are captured)
    for _ in range(max(args.warmup, tau + 1)):
        tr.step(*data[it % M])
        it += 1
    tr.sync()
    torch.cuda.synchronize()
    table.sync()
    # e2e (before the graphs are captured: eager steps, the trainer's pipeline state
    # carries on into the captured cycle): the same steps through the trainer's API with HOST inputs -- every step's ids,
    # offsets, dense features and labels copied in from pinned memory (K buffer sets, a
    # set reused only after the step that read it has finished) and the step's loss read
    # back to the host
    e2e = None
    if args.e2e_steps > 0:
        K = tau + 2
        hsets = []
        for m in range(M):
            hb = W.make_batch(cfg, 1000 * rank + m)
            x_, y_ = W.make_dense_inputs(cfg, hb)
            hsets.append([torch.from_numpy(a).pin_memory() for a in
                          (hb.ids.view(np.int64), hb.offsets.view(np.int32), x_, y_)])
        dsets = [[torch.empty_like(h, device=dev) for h in hsets[0]] for _ in range(K)]
        done = [torch.cuda.Event() for _ in range(K)]
        h_loss = torch.empty(args.e2e_steps, dtype=torch.float32).pin_memory()
        nbytes = sum(h.numel() * h.element_size() for h in hsets[0])
        for e_ in done:
            e_.record(stream)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for j in range(args.e2e_steps):
            k = j % K
            stream.wait_event(done[k])
            for dbuf, hbuf in zip(dsets[k], hsets[(it + j) % M]):
                n_ = hbuf.numel()
                dbuf[:n_].copy_(hbuf, non_blocking=True)
            loss = tr.step(*dsets[k])
            tr.sync()  # (the step's streams joined: set k is free again after this point)
            done[k].record(stream)
            h_loss[j:j + 1].copy_(loss.reshape(1), non_blocking=True)
        torch.cuda.synchronize()
        _ = float(h_loss[-1])
        e_ms = (time.perf_counter() - w0) * 1000.0 / args.e2e_steps
        if world > 1:
            t = torch.tensor([e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        it += args.e2e_steps
        table.sync()
        e2e = {"value": world * B * 1000.0 / e_ms, "unit": "samples/s",
               "h2d_bytes_per_step": int(nbytes), "d2h_bytes_per_step": 4,
               "path": "HybridTrainer.step on device buffers fed from pinned host memory "
                       "every step (eager launches, one trainer sync per step)"}
    # One CUDA graph per step of the cycle (lcm of the batch count and tau + 1: the step
    # index picks the batch and the in-flight slot): register + pull(s) and push(s-tau) on
    # the embedding stream, the dense step on the dense stream, forked and joined inside
    # the graph -- so push(s-tau) overlaps dense(s) without host launch overhead.
    graphs, losses_g, graph_launches = [], [], []
    if use_graph:
        cyc = M * (tau + 1) // math.gcd(M, tau + 1)
        cs = torch.cuda.Stream()
        with torch.cuda.stream(cs):
            for j in range(cyc):
                g = torch.cuda.CUDAGraph()
                l0 = hps.launch_count()
                with torch.cuda.graph(g, stream=cs, capture_error_mode="thread_local"):
                    losses_g.append(tr.step(*data[(it + j) % M]))
                    tr.sync()
                graph_launches.append(hps.launch_count() - l0)
                graphs.append(g)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def run_step(i):
        if graphs:
            graphs[(i - it0) % len(graphs)].replay()
            return losses_g[(i - it0) % len(graphs)]
        return tr.step(*data[i % M])

    it0 = it
    for _ in range(len(graphs) or 2):
        run_step(it)
        it += 1
    tr.sync()
    torch.cuda.synchronize()
    table.sync()
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = hps.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    losses = []
    for _ in range(args.steps):
        v = run_step(it)
        losses.append(v.clone() if graphs else v)
        it += 1
    tr.sync()
    e1.record(stream)
    torch.cuda.synchronize()
    launches = hps.launch_count() - l0
    if graphs:  # replays do not pass through the host launch counter
        launches = sum(graph_launches[(i - it0) % len(graphs)] for i in range(it - args.steps, it))
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if not graphs:
        tr.flush()
    torch.cuda.synchronize()
    tr.check()  # a diverged dense step (non-finite loss / gradient) fails the run
    table.sync()
    loss_vals = [float(v) for v in losses]
    value = world * B * 1000.0 / ms
    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v_, c_, smp = hybrid_cpu_baseline(cfg, 1024)
        cpu_base = {"value": v_, "unit": "samples/s", "cores": c_, "kind": "reference",
                    "sample": smp}
    if rank == 0:
        params = tr.tower.param_count
        line = {
            "metric": "hybrid training samples/sec (embedding lookup+update + dense tower)",
            "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 (fp64 pooling/fan-out)",
            "data": "synthetic (teacher labels)",
            "config": {"workload": f"c5: batch {B}/GPU, {F} one-hot features, "
                                   f"{rows // 1_000_000}M-row table dim {D}, adagrad, mean "
                                   f"pooling, staleness {tau}, dense 1677-64-32-1 fp32 SGD, "
                                   f"canonical all-reduce",
                       "global_batch": B * world, "dense_params": params,
                       "parallelism": f"dp{world} + hash-sharded embeddings" if world > 1
                       else "single", "staleness": tau},
            "loss_first_last": [loss_vals[0], loss_vals[-1]],
            "gpu_launches": launches, "clocks": clk, "prewarm_s": prewarm_s,
            "cpu_baseline": cpu_base, "e2e": e2e,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        # the graphs hold NCCL work: release them, then leave without tearing the
        # communicator down under them
        graphs.clear()
        torch.cuda.synchronize()
        dist.barrier()
        sys.stdout.flush()
        os._exit(0)


# ---------------------------------------------------------------- our arm, N > 1 (sharded)


def run_sharded(args, world, rank, local, dev):
    """C4: the table hash-sharded over the N GPUs (owner = route_shard(id, S) % N), one
    embedding worker per GPU with its own batch, NCCL all-to-all of ids, rows and
    (position, contribution) pairs per step (paper_2111_05897_b200/sharded.py)."""
    import torch
    import torch.distributed as dist

    from paper_2111_05897_b200 import hps
    from paper_2111_05897_b200 import workloads as W
    from paper_2111_05897_b200.sharded import ShardedEmbeddingWorker

    cfg = W.sharded_config(world)
    D, F, B = cfg.dim, cfg.features, cfg.batch
    S = cfg.shards
    rows = cfg.table_capacity()
    cap = int(rows / world * 1.01) + (1 << 20)
    # in-order step tags (one pipeline, device step counter): each row's latest bump tag
    # counts delays exactly, no tag ring needed (it would refuse out-of-order tags)
    table = hps.ShardSet(S, D, cap, hps.ADAGRAD, salts=cfg.salts(), device=local,
                         tag_ring=False)
    stream = torch.cuda.current_stream()
    # pre-warm: each rank creates the rows it owns (M = 0 lazy inits while timing)
    t0 = time.perf_counter()
    chunk = 1 << 24
    for a in range(0, rows, chunk):
        n = min(chunk, rows - a)
        ids = torch.arange(a, a + n, dtype=torch.int64, device=dev)
        sh = hps.route(ids, S, stream=stream).to(torch.int64)
        owned = ids[(sh % world) == rank]
        table.lookup(owned, stream=stream)
    torch.cuda.synchronize()
    prewarm_s = time.perf_counter() - t0

    M = args.batches
    host_batches = [W.make_batch(cfg, 1000 * rank + m) for m in range(M)]
    batches = [(torch.from_numpy(hb.ids.view(np.int64)).to(dev),
                torch.from_numpy(hb.offsets.view(np.int32)).to(dev), hb.N) for hb in host_batches]
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    grads = [((torch.rand((B, F, D), generator=gen, device=dev) * 2 - 1) * cfg.grad_scale)
             for _ in range(M)]
    pooled = torch.empty((B, F, D), dtype=torch.float32, device=dev)
    max_n = max(b[2] for b in batches)
    ew = ShardedEmbeddingWorker(table, hps.MEAN, transport=args.transport, max_ids=max_n,
                                codec_kappa=args.codec_kappa)
    tag = [0]

    p2p = args.transport == "p2p"

    def eager_step(i):
        ids, offs, _ = batches[i % M]
        ew.register_batch(ids, offs, B, F)
        # p2p: the pooled batch stays in the exchange arena (zero-copy view)
        ew.serve_pull(out_pooled=None if p2p else pooled)
        tag[0] += 1
        # p2p: step tags from the table's device counter (graph replays advance it)
        ew.apply_backward(grads[i % M], cfg.lr, tag[0],
                          flags=hps.ASYNC | (hps.DEVICE_STEP if p2p else 0))

    it = 0
    for _ in range(args.warmup):
        eager_step(it)
        it += 1
    torch.cuda.synchronize()
    table.sync()
    # Pipelined sync steps (p2p, default): two exchanges alternate; the next batch's
    # routing + pair plan (phase 1 of its forward: no barrier, no table access) runs on
    # a second stream beside this batch's owner lookup, pull and backward.
    pipe = p2p and not args.no_pipeline and M % 2 == 0
    ews = [ew, ShardedEmbeddingWorker(table, hps.MEAN, transport=args.transport,
                                      max_ids=max_n, codec_kappa=args.codec_kappa)] \
        if pipe else []
    side = torch.cuda.Stream(priority=args.prefetch_priority) if pipe else None

    def pipe_step(i):
        cur = torch.cuda.current_stream()
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            ids1, offs1, _ = batches[(i + 1) % M]
            ews[(i + 1) % 2].prefetch(ids1, offs1, B, F)
        w = ews[i % 2]
        w.register_prefetched()
        w.serve_pull(out_pooled=None)
        tag[0] += 1
        w.apply_backward(grads[i % M], cfg.lr, tag[0], flags=hps.ASYNC | hps.DEVICE_STEP)
        cur.wait_stream(side)

    if pipe:
        ids0, offs0, _ = batches[it % M]
        ews[it % 2].prefetch(ids0, offs0, B, F)
        for _ in range(2):
            pipe_step(it)
            it += 1
        torch.cuda.synchronize()
        table.sync()
    # p2p: the whole sharded step (route, peer writes, device barriers, owner apply) is
    # stream-ordered without host round trips -> one CUDA graph per input batch.
    graphs, graph_launches, cycle = [], [], []
    it_g = it
    if p2p and not args.no_graph:
        cs = torch.cuda.Stream(priority=args.step_priority)
        for m in range(M):
            g = torch.cuda.CUDAGraph()
            l0 = hps.launch_count()
            with torch.cuda.graph(g, stream=cs, capture_error_mode="thread_local"):
                if pipe:
                    pipe_step(it_g + m)
                else:
                    eager_step(m)
            graph_launches.append(hps.launch_count() - l0)
            graphs.append(g)
        if pipe:  # and one graph of the whole cycle of M steps (no graph boundaries)
            g = torch.cuda.CUDAGraph()
            l0 = hps.launch_count()
            with torch.cuda.graph(g, stream=cs, capture_error_mode="thread_local"):
                for m in range(M):
                    pipe_step(it_g + m)
            cycle.append((g, hps.launch_count() - l0))
        torch.cuda.synchronize()
        dist.barrier()

    def step(i):
        if graphs:
            graphs[(i - it_g) % M if pipe else i % M].replay()
        elif pipe:
            pipe_step(i)
        else:
            eager_step(i)

    def run_steps(i, n):
        """Steps i .. i+n-1 (the cycle graph where a cycle starts); returns launches."""
        launches = 0
        while n > 0:
            k = (i - it_g) % M
            if cycle and k == 0 and n >= M:
                cycle[0][0].replay()
                launches += cycle[0][1]
                i, n = i + M, n - M
            else:
                step(i)
                launches += graph_launches[k if pipe else i % M] if graphs else 0
                i, n = i + 1, n - 1
        return launches

    for _ in range(2):
        step(it)
        it += 1
    torch.cuda.synchronize()
    table.sync()
    clocks = ClockSampler(local)
    clocks.start()
    dist.barrier()
    torch.cuda.synchronize()
    l0 = hps.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    x_ids = x_pairs = 0
    g_launches = 0
    if graphs:
        g_launches = run_steps(it, args.steps)
        it += args.steps
    else:
        for _ in range(args.steps):
            step(it)
            it += 1
            if args.transport == "nccl":
                x_ids += sum(c for d, c in enumerate(ew.send_counts) if d != rank)
                x_pairs += sum(c for d, c in enumerate(ew.pair_counts) if d != rank)
    e1.record(stream)
    dist.barrier()
    torch.cuda.synchronize()
    launches = hps.launch_count() - l0
    if graphs:  # replays do not pass through the host launch counter
        launches = g_launches
    ms = e0.elapsed_time(e1) / args.steps
    t_soak = time.perf_counter()
    while time.perf_counter() - t_soak < args.soak_seconds:
        step(it)
        it += 1
        torch.cuda.synchronize()
    clk = clocks.stop()
    table.sync()
    if args.timeline:  # every rank replays (the steps are collective); one file per rank
        write_timeline(f"{args.timeline}.r{rank}", step, it, 4)
        it += 4
        table.sync()
    t = torch.tensor([ms], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = world * B * 1000.0 / ms

    # off-rank bytes each GPU sends per step (ids out + rows back + pairs out) ~ NVLink
    N_avg = float(np.mean([b[2] for b in batches]))
    if args.transport == "nccl":
        U_avg = float(x_ids) / args.steps  # distinct ids this rank sent off-rank per step
        P_avg = float(x_pairs) / args.steps
    else:  # one-hot over >= 125M rows per GPU: ~every listing distinct, uniform owners
        U_avg = P_avg = N_avg * (world - 1) / world
    row_b = (2 * D + 4) if args.codec_kappa else 4 * D  # binary16 payload + f32 scale
    nvl_bytes = 8 * U_avg + row_b * U_avg + (4 + row_b) * P_avg
    O_ = D
    uniq = float(N_avg)  # one-hot over 125M rows per GPU: ~all listings distinct
    bytes_step = (8 * N_avg + 8 * N_avg + 12 * uniq + 4 * D * uniq + 4 * B * F * D +
                  4 * B * F * D + 8 * (D + O_) * uniq)
    peak, peak_kind = peaks()

    # e2e: host (pinned) inputs copied in and the pooled output copied out every step
    hb = host_batches[0]
    h_ids = torch.from_numpy(hb.ids.view(np.int64)).pin_memory()
    h_offs = torch.from_numpy(hb.offsets.view(np.int32)).pin_memory()
    h_grads = grads[0].cpu().pin_memory()
    h_pooled = torch.empty((B, F, D), dtype=torch.float32).pin_memory()
    d_ids = torch.empty_like(batches[0][0])
    d_offs = torch.empty_like(batches[0][1])
    d_grads = torch.empty_like(grads[0])

    def e2e_step():
        d_ids.copy_(h_ids, non_blocking=True)
        d_offs.copy_(h_offs, non_blocking=True)
        ew.register_batch(d_ids, d_offs, B, F)
        h_pooled.copy_(ew.serve_pull(out_pooled=None if p2p else pooled), non_blocking=True)
        d_grads.copy_(h_grads, non_blocking=True)
        tag[0] += 1
        ew.apply_backward(d_grads, cfg.lr, tag[0],
                          flags=hps.ASYNC | (hps.DEVICE_STEP if p2p else 0))

    e2e = None
    if args.e2e_steps > 0:
        e2e_step()
        dist.barrier()
        torch.cuda.synchronize()
        q0 = torch.cuda.Event(enable_timing=True)
        q1 = torch.cuda.Event(enable_timing=True)
        q0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        q1.record(stream)
        torch.cuda.synchronize()
        e_ms = q0.elapsed_time(q1) / args.e2e_steps
        t = torch.tensor([e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
        e2e = {"value": world * B * 1000.0 / e_ms, "unit": "samples/s",
               "h2d_bytes_per_step": int(8 * hb.N + 4 * (B * F + 1) + 4 * B * F * D),
               "d2h_bytes_per_step": int(4 * B * F * D),
               "path": "ShardedEmbeddingWorker with pinned host inputs/outputs per rank"}

    if rank == 0:
        line = {
            "metric": "embedding lookup+update samples/sec", "value": value,
            "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 (fp64 pooling/fan-out)", "data": "synthetic",
            "config": {"workload": f"c4: per-GPU batch {B}, {F} one-hot features, "
                                   f"{rows // 1_000_000}M-row table dim {D} hash-sharded over "
                                   f"{world} GPUs ({S} logical shards), adagrad, mean pooling, "
                                   f"staleness 0, " + ("NVLink peer-write exchange" if
                                   args.transport == "p2p" else "NCCL all-to-all exchange") +
                                   (f", binary16 payload codec (kappa {args.codec_kappa:g}, "
                                    f"lossy)" if args.codec_kappa else ", exact fp32 payloads"),
                       "global_batch": B * world, "rows": rows, "dim": D, "features": F,
                       "logical_shards": S, "parallelism": f"sharded{world}",
                       "l2": "per-step footprint > L2 (126 MB); no flush"},
            "hbm": {"algorithmic_bytes_per_step_per_gpu": bytes_step,
                    "achieved_gbs_per_gpu": bytes_step / (ms * 1e-3) / 1e9,
                    "frac_of_peak": bytes_step / (ms * 1e-3) / 1e9 / peak},
            "roofline": {"bound": "hbm", "kernel": "whole step (per GPU)",
                         "achieved": bytes_step / (ms * 1e-3) / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": bytes_step / (ms * 1e-3) / 1e9 / peak,
                         "traffic": None, "peak_source": peak_kind},
            "nvlink": {"transport": args.transport,
                       "offrank_bytes_per_step_per_gpu": nvl_bytes,
                       "achieved_gbs_per_direction": nvl_bytes / (ms * 1e-3) / 1e9,
                       "frac_of_900": nvl_bytes / (ms * 1e-3) / 1e9 / 900.0},
            "cpu_baseline": None, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk, "prewarm_s": prewarm_s,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def write_timeline(path, step, it, n):
    """Kernel start/end times (CUPTI via torch.profiler) of n replays of the timed step:
    where the step's time goes between and beside the kernels."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(n):
            step(it + i)
        torch.cuda.synchronize()
    evs = []
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() >= 0:
            evs.append((e.time_range.start, e.time_range.end, e.name))
    evs.sort()
    t0 = evs[0][0] if evs else 0
    with open(path, "w") as f:
        for a_, b_, nm in evs:
            f.write(f"{a_ - t0:10.2f} {b_ - a_:8.2f}  {nm[:90]}\n")
    print(f"timeline: {len(evs)} kernels over {n} steps -> {path}", file=sys.stderr)


# ---------------------------------------------------------------- e2e (host buffers)


def run_e2e_local(args, table, agg, cfg, host_batches, grads, stream, dev, B, F, D):
    import torch

    from paper_2111_05897_b200 import hps

    K = args.e2e_slots
    ews = [hps.EmbeddingWorker(table, agg) for _ in range(K)]
    M = min(len(host_batches), K)
    nmax = max(hb.N for hb in host_batches[:M])
    h_ids = [torch.from_numpy(hb.ids.view(np.int64)).pin_memory() for hb in host_batches[:M]]
    h_offs = [torch.from_numpy(hb.offsets.view(np.int32)).pin_memory()
              for hb in host_batches[:M]]
    h_grads = [grads[m].cpu().pin_memory() for m in range(M)]
    h_pooled = [torch.empty((B, F, D), dtype=torch.float32).pin_memory() for _ in range(K)]
    d_ids = [torch.empty(nmax, dtype=torch.int64, device=dev) for _ in range(K)]
    d_offs = [torch.empty(B * F + 1, dtype=torch.int32, device=dev) for _ in range(K)]
    d_grads = [torch.empty((B, F, D), dtype=torch.float32, device=dev) for _ in range(K)]
    d_pooled = [torch.empty((B, F, D), dtype=torch.float32, device=dev) for _ in range(K)]
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    ev = lambda: torch.cuda.Event()
    in_ready, g_ready, pooled_ready = [ev() for _ in range(K)], [ev() for _ in range(K)], \
        [ev() for _ in range(K)]
    push_done, out_done = [ev() for _ in range(K)], [ev() for _ in range(K)]
    for e_ in push_done + out_done:
        e_.record(stream)
    ns = [0]

    def stage_in(s):  # H2D of step s into slot s % K, once that slot's last user is done
        k, m = s % K, s % M
        with torch.cuda.stream(h2d):
            h2d.wait_event(push_done[k])
            n = h_ids[m].numel()
            d_ids[k][:n].copy_(h_ids[m], non_blocking=True)
            d_offs[k].copy_(h_offs[m], non_blocking=True)
            in_ready[k].record(h2d)
            d_grads[k].copy_(h_grads[m], non_blocking=True)
            g_ready[k].record(h2d)

    def step(s):
        k, m = s % K, s % M
        n = h_ids[m].numel()
        stream.wait_event(in_ready[k])
        ews[k].register_batch(d_ids[k][:n], d_offs[k], B, F, stream=stream)
        stream.wait_event(out_done[k])  # the slot's previous pooled batch reached the host
        ews[k].serve_pull(out_pooled=d_pooled[k], stream=stream)
        pooled_ready[k].record(stream)
        with torch.cuda.stream(d2h):
            d2h.wait_event(pooled_ready[k])
            h_pooled[k].copy_(d_pooled[k], non_blocking=True)
            out_done[k].record(d2h)
        stream.wait_event(g_ready[k])
        ews[k].apply_backward(d_grads[k], cfg.lr, flags=hps.ASYNC | hps.DEVICE_STEP,
                              stream=stream)
        push_done[k].record(stream)
        stage_in(s + 1)

    s0 = 0
    stage_in(s0)
    for _ in range(3):  # warm-up
        step(s0)
        s0 += 1
    torch.cuda.synchronize()
    table.sync()
    q0 = torch.cuda.Event(enable_timing=True)
    q1 = torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    q0.record(stream)
    for _ in range(args.e2e_steps):
        step(s0)
        s0 += 1
    stream.wait_stream(d2h)
    q1.record(stream)
    torch.cuda.synchronize()
    _ = float(h_pooled[(s0 - 1) % K][0, 0, 0])  # the host reads the last result
    wall_ms = (time.perf_counter() - w0) * 1000 / args.e2e_steps
    e_ms = max(q0.elapsed_time(q1) / args.e2e_steps, wall_ms)
    table.sync()
    hb = host_batches[0]
    return {"value": B * 1000.0 / e_ms, "unit": "samples/s",
            "h2d_bytes_per_step": int(8 * hb.N + 4 * (B * F + 1) + 4 * B * F * D),
            "d2h_bytes_per_step": int(4 * B * F * D),
            "path": "hps_batch_register/pull/push on device buffers fed from pinned host "
                    "memory every step (H2D of step s+1 and D2H of step s on two copy "
                    "streams, overlapped)"}


# ---------------------------------------------------------------- our arm


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    import torch
    import torch.distributed as dist

    from paper_2111_05897_b200 import hps
    from paper_2111_05897_b200 import workloads as W

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if args.config == "c5":
        run_hybrid(args, world, rank, local, dev)
        return
    if world > 1:
        run_sharded(args, world, rank, local, dev)
        return
    cfg = W.CONFIGS[args.config]
    D, F, B = cfg.dim, cfg.features, cfg.batch
    opt = hps.ADAGRAD if cfg.optimizer == "adagrad" else hps.SGD
    agg = hps.MEAN if cfg.aggregation == "mean" else hps.SUM
    cap = cfg.table_capacity()
    # in-order step tags (one pipeline, device step counter): each row's latest bump tag
    # counts delays exactly, no tag ring needed (it would refuse out-of-order tags)
    table = hps.ShardSet(cfg.shards, D, cap, opt, salts=cfg.salts(), device=local,
                         tag_ring=False)
    stream = torch.cuda.current_stream()

    # -- pre-warm: every row of the table exists before timing (M = 0 misses).
    t0 = time.perf_counter()
    chunk = 1 << 23
    buf = torch.empty((chunk, D), dtype=torch.float32, device=dev)
    for a in range(0, cap, chunk):
        n = min(chunk, cap - a)
        ids = torch.arange(a, a + n, dtype=torch.int64, device=dev)
        table.lookup(ids, out_values=buf[:n], stream=stream)
    torch.cuda.synchronize()
    prewarm_s = time.perf_counter() - t0

    # -- inputs: M distinct batches, resident in HBM
    M = args.batches
    host_batches = [W.make_batch(cfg, 1000 * rank + m) for m in range(M)]
    batches = []
    uniq = []
    for hb in host_batches:
        ids = torch.from_numpy(hb.ids.view(np.int64)).to(dev)
        offs = torch.from_numpy(hb.offsets.view(np.int32)).to(dev)
        batches.append((ids, offs, hb.N))
        uniq.append(len(np.unique(hb.ids)))
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    grads = [((torch.rand((B, F, D), generator=gen, device=dev) * 2 - 1) * cfg.grad_scale)
             for _ in range(M)]
    pooled = torch.empty((B, F, D), dtype=torch.float32, device=dev)
    ew = hps.EmbeddingWorker(table, agg)

    def eager_step(i, s=None):
        s = s or stream
        ids, offs, n = batches[i % M]
        ew.register_batch(ids, offs, B, F, stream=s)
        ew.serve_pull(out_pooled=pooled, stream=s)
        # step tags come from the table's device step counter, so graph replays
        # advance them exactly like eager calls would
        ew.apply_backward(grads[i % M], cfg.lr, flags=hps.ASYNC | hps.DEVICE_STEP, stream=s)

    it = 0
    for _ in range(args.warmup):
        eager_step(it)
        it += 1
    torch.cuda.synchronize()
    table.sync()

    # Pipelined sync steps (default): the next batch's register (probe, plan, sorts --
    # latency-bound, no row data) runs on a second stream beside this batch's pull and
    # push, like the reference's register_sample buffering upcoming samples while the
    # current step trains; every pull still follows the previous push (exact sync
    # semantics: the next pull is issued after this push on the main stream). Two
    # embedding-worker handles alternate; each batch has its own plan bitmaps.
    pipe = not args.no_pipeline and M % 2 == 0
    ews = [hps.EmbeddingWorker(table, agg) for _ in range(2)] if pipe else []
    side = torch.cuda.Stream(priority=args.register_priority) if pipe else None
    # the next batch's plan (its sort) is joined by its push, not by its register: the
    # next pooling does not wait for it (hps_batch_defer_plan_join); a graph capture that
    # ends before the push joins it itself (join_pending below)
    defer = pipe and not args.no_defer_plan_join
    for w_ in ews:
        w_.defer_plan_join(defer)

    def join_pending(i_last):
        if defer:  # the batch the capture's last step registered
            ews[(i_last + 1) % 2].join_plan(stream=torch.cuda.current_stream())

    def pipe_step(i, s):
        nxt = i + 1
        w = ews[i % 2]
        ids1, offs1, _ = batches[nxt % M]
        if args.register_after == "pull":
            w.serve_pull(out_pooled=pooled, stream=s)
        side.wait_stream(s)
        ews[nxt % 2].register_batch(ids1, offs1, B, F, stream=side)
        if args.register_after == "push":
            w.serve_pull(out_pooled=pooled, stream=s)
        w.apply_backward(grads[i % M], cfg.lr, flags=hps.ASYNC | hps.DEVICE_STEP, stream=s)
        s.wait_stream(side)

    if pipe:
        ids0, offs0, _ = batches[it % M]
        ews[it % 2].register_batch(ids0, offs0, B, F, stream=stream)
        for _ in range(2):
            pipe_step(it, stream)
            it += 1
        torch.cuda.synchronize()
        table.sync()

    # CUDA graphs: one of the whole cycle of M input batches (M pipelined steps replayed
    # without host launch overhead and without graph boundaries between them), one per
    # PAIR of batches and one per batch for step counts that do not fill a cycle.
    graphs, graph_launches = [], []
    pairs, pair_launches = [], []
    cycle = []
    it_g = it
    if not args.no_graph:
        cap = torch.cuda.Stream(priority=args.step_priority)
        for m in range(M):
            g = torch.cuda.CUDAGraph()
            l0 = hps.launch_count()
            with torch.cuda.graph(g, stream=cap, capture_error_mode="thread_local"):
                if pipe:
                    pipe_step(it_g + m, torch.cuda.current_stream())
                    join_pending(it_g + m)
                else:
                    eager_step(m, torch.cuda.current_stream())
            graph_launches.append(hps.launch_count() - l0)
            graphs.append(g)
        if pipe:
            for m in range(0, M, 2):
                g = torch.cuda.CUDAGraph()
                l0 = hps.launch_count()
                with torch.cuda.graph(g, stream=cap, capture_error_mode="thread_local"):
                    pipe_step(it_g + m, torch.cuda.current_stream())
                    pipe_step(it_g + m + 1, torch.cuda.current_stream())
                    join_pending(it_g + m + 1)
                pair_launches.append(hps.launch_count() - l0)
                pairs.append(g)
            if M > 2:  # and one graph of all M batches' steps
                g = torch.cuda.CUDAGraph()
                l0 = hps.launch_count()
                with torch.cuda.graph(g, stream=cap, capture_error_mode="thread_local"):
                    for m in range(M):
                        pipe_step(it_g + m, torch.cuda.current_stream())
                    join_pending(it_g + M - 1)
                cycle.append((g, hps.launch_count() - l0))
        torch.cuda.synchronize()

    def step(i):
        if graphs:
            graphs[(i - it_g) % M if pipe else i % M].replay()
        elif pipe:
            pipe_step(i, stream)
        else:
            eager_step(i)

    def run_steps(i, n):
        """Steps i .. i+n-1 (pair graphs where a pair starts); returns launches issued."""
        launches = 0
        while n > 0:
            k = (i - it_g) % M
            if cycle and k == 0 and n >= M:
                cycle[0][0].replay()
                launches += cycle[0][1]
                i, n = i + M, n - M
            elif pairs and k % 2 == 0 and n >= 2:
                pairs[k // 2].replay()
                launches += pair_launches[k // 2]
                i, n = i + 2, n - 2
            else:
                step(i)
                launches += graph_launches[k if pipe else i % M] if graphs else 0
                i, n = i + 1, n - 1
        return launches

    for _ in range(2):
        step(it)
        it += 1
    torch.cuda.synchronize()
    table.sync()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # -- timed region (device time, CUDA events on the launching stream)
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    l0 = hps.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    g_launches = run_steps(it, args.steps)
    it += args.steps
    e1.record(stream)
    barrier()
    launches = hps.launch_count() - l0
    if graphs:  # replays do not pass through the host launch counter
        launches = g_launches
    ms = e0.elapsed_time(e1) / args.steps
    # soak: keep the same step running so the clock sampler sees >= soak-seconds under load
    t_soak = time.perf_counter()
    while time.perf_counter() - t_soak < args.soak_seconds:
        for _ in range(10):
            step(it)
            it += 1
        torch.cuda.synchronize()
    clk = clocks.stop()
    table.sync()  # surfaces any deferred data-dependent error of the timed steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * B * 1000.0 / ms

    if args.timeline:
        write_timeline(args.timeline, step, it, 4)
        it += 4

    # -- per-kernel timing pass (same steps, events around each region)
    table.profile(True)
    for _ in range(args.steps):
        eager_step(it)  # events need the host-side launch sequence (no graph)
        it += 1
    torch.cuda.synchronize()
    regions = {}
    for r in ("probe", "plan", "sort_small", "sort", "pool", "check", "update", "update_multi"):
        tot, cnt = table.profile_get(r)
        regions[r] = (tot / max(cnt, 1), cnt)
    table.profile(False)

    # -- algorithmic bytes
    N_avg = float(np.mean([b[2] for b in batches]))
    U_avg = float(np.mean(uniq))
    O_ = D if opt == hps.ADAGRAD else 0
    bytes_step = (8 * N_avg + 8 * N_avg + 12 * U_avg + 4 * D * U_avg + 4 * B * F * D +
                  4 * B * F * D + 8 * (D + O_) * U_avg)
    kernel_bytes = {
        "update": 4 * B * F * D + 8 * (D + O_) * U_avg,
        "pool": 4 * D * U_avg + 4 * B * F * D + 4 * N_avg,
        "probe": 8 * N_avg + 12 * U_avg + 4 * N_avg,
        "check": 4 * B * F * D,
    }
    peak, peak_kind = peaks()
    dom = max(("update", "pool", "probe", "check"), key=lambda r: regions[r][0])
    dom_ms = regions[dom][0]
    achieved = kernel_bytes[dom] / (dom_ms * 1e-3) / 1e9 if dom_ms > 0 else None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(cfg.name, {}).get(dom)
        except Exception:
            traffic = None

    # -- e2e through the public API, inputs from and results to pinned HOST memory: every
    # step copies its ids, offsets and gradients in and its pooled embeddings out, inside
    # the timed region. Two in-flight slots: the H2D copies of step s+1 (one copy
    # stream) and the D2H copy of step s (another) overlap each other and the compute
    # (PCIe is full duplex) -- the same double buffering a trainer feeding the table from
    # host memory would use.
    e2e = None
    if args.e2e_steps > 0:
        e2e = run_e2e_local(args, table, agg, cfg, host_batches, grads, stream, dev, B, F, D)
        if world > 1:
            t = torch.tensor([1000.0 * B / e2e["value"]], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e["value"] = world * B * 1000.0 / float(t.item())

    # -- CPU baseline: the reference on this box's host cores (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cores = nproc()
            B_s = cfg.batch
            v, n, rows, _ = reference_run(cfg, B_s, steps=100, warmup=1, threads=cores,
                                          seconds_cap=args.cpu_seconds)
            cpu = {"value": v, "unit": "samples/s", "cores": cores, "kind": "reference",
                   "sample": f"{n} steps x {B_s} samples of {cfg.name} (2 distinct batches, "
                             f"their {rows} rows created before timing) through the reference "
                             f"EmbeddingWorker/PsShard (oracle/_ref), pull on {cores} threads + "
                             f"ordered single-thread push"}
        except Exception as e:  # report, never fake
            cpu = {"value": None, "unit": "samples/s", "cores": nproc(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": "embedding lookup+update samples/sec", "value": value,
            "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 (fp64 pooling/fan-out)", "data": "synthetic",
            "config": dict(workload_config(cfg, args),
                           schedule=("sync steps; each batch registered (probe + plan) beside "
                                     "the previous batch's push, its pull after that push"
                                     if pipe else "sync steps, in line")),
            "hbm": {"algorithmic_bytes_per_step": bytes_step,
                    "achieved_gbs": bytes_step / (ms * 1e-3) / 1e9,
                    "frac_of_peak": bytes_step / (ms * 1e-3) / 1e9 / peak,
                    "N": N_avg, "U": U_avg},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": (achieved / peak) if achieved else None,
                         "traffic": traffic, "peak_source": peak_kind,
                         "algorithmic_bytes_per_launch": kernel_bytes[dom],
                         "ms_per_launch": dom_ms},
            "kernels_ms": {k: round(v[0], 4) for k, v in regions.items()},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk, "prewarm_s": prewarm_s,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
