"""Replays the committed reference fixtures (tests/golden/*.npz) through an
implementation -- the C restatement (CPU) or the CUDA path through the C ABI -- and
compares bit-for-bit. Fixtures were produced by the reference itself
(tests/golden/make_golden.py)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SYNC_CASES = ["c1_two_steps", "ragged_mean_adagrad_e2", "ragged_sum_adagrad_d5"]


def load(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False)
    return {k: z[k] for k in z.files}


def _s(x):
    return str(x) if not isinstance(x, np.ndarray) else str(x.item())


def replay_oracle(case):
    import oracle as O

    d = load(case)
    orc = O.Restatement(d["salts"], int(d["D"]), _s(d["opt"]))
    agg = _s(d["agg"])
    F = int(d["F"])
    has_step = bool(d["has_step"])
    for s in range(int(d["steps"])):
        B = int(d[f"B_{s}"])
        ids, offs = d[f"ids_{s}"], d[f"offsets_{s}"].astype(np.uint64)
        pooled, rv = orc.pull_batch(B, F, ids, offs, agg)
        assert pooled.tobytes() == d[f"pooled_{s}"].tobytes(), f"{case}: pooled step {s}"
        assert (rv == d[f"rv_{s}"]).all(), f"{case}: read versions step {s}"
        ok, _ = orc.push_batch(B, F, ids, offs, d[f"grads_{s}"], float(d["lr"]),
                               s + 1 if has_step else 0, read_versions=rv,
                               sample_keys=d[f"sids_{s}"], agg=agg)
        assert ok
    w, a, v, present = orc.peek(d["final_ids"])
    assert present.all()
    assert w.tobytes() == d["final_w"].tobytes(), f"{case}: final w"
    assert a.tobytes() == d["final_acc"].tobytes(), f"{case}: final acc"
    assert (v == d["final_ver"]).all(), f"{case}: final versions"
    assert orc.counters()["size"] == len(d["final_ids"])


def replay_gpu(case, device_arrays=False):
    """The CUDA path through the C ABI (EmbeddingWorker batch surface)."""
    import torch

    from paper_2111_05897_b200 import hps

    d = load(case)
    D, F = int(d["D"]), int(d["F"])
    opt = hps.ADAGRAD if _s(d["opt"]) == "adagrad" else hps.SGD
    agg = hps.MEAN if _s(d["agg"]) == "mean" else hps.SUM
    table = hps.ShardSet(len(d["salts"]), D, 1 << 16, opt, salts=d["salts"])
    ew = hps.EmbeddingWorker(table, agg)
    has_step = bool(d["has_step"])
    for s in range(int(d["steps"])):
        B = int(d[f"B_{s}"])
        ids, offs, sids, grads = d[f"ids_{s}"], d[f"offsets_{s}"], d[f"sids_{s}"], d[f"grads_{s}"]
        rv = np.zeros(len(ids), np.uint64)
        if device_arrays:
            dev = torch.device("cuda:0")
            ids_t = torch.from_numpy(ids.view(np.int64)).to(dev)
            offs_t = torch.from_numpy(offs.view(np.int32)).to(dev)
            sids_t = torch.from_numpy(sids.view(np.int64)).to(dev)
            ew.register_batch(ids_t, offs_t, B, F, sample_keys=sids_t)
            pooled_t = torch.empty((B, F, D), dtype=torch.float32, device=dev)
            rv_t = torch.empty(len(ids), dtype=torch.int64, device=dev)
            ew.serve_pull(out_pooled=pooled_t, out_read_versions=rv_t)
            pooled = pooled_t.cpu().numpy()
            rv = rv_t.cpu().numpy().view(np.uint64)
            ok = ew.apply_backward(torch.from_numpy(grads).to(dev), float(d["lr"]),
                                   s + 1 if has_step else 0)
        else:
            ew.register_batch(ids, offs, B, F, sample_keys=sids)
            pooled = ew.serve_pull(out_read_versions=rv)
            ok = ew.apply_backward(grads, float(d["lr"]), s + 1 if has_step else 0)
        assert pooled.tobytes() == d[f"pooled_{s}"].tobytes(), f"{case}: pooled step {s}"
        assert (rv == d[f"rv_{s}"]).all(), f"{case}: read versions step {s}"
        assert ok
    w, a, v, present = table.peek(d["final_ids"])
    assert present.all()
    np.testing.assert_array_equal(w, d["final_w"], err_msg=f"{case}: final w")
    np.testing.assert_array_equal(a, d["final_acc"], err_msg=f"{case}: final acc")
    assert (v == d["final_ver"]).all(), f"{case}: final versions"
    assert table.size() == len(d["final_ids"])
    c = table.counters()
    assert c.misses == len(d["final_ids"])
    if has_step:
        assert c.delay_hist[0] > 0 and sum(c.delay_hist[1:]) == 0  # sync mode: all delays 0
