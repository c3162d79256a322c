"""Multi-rank sharded step: every rank's pooled output, and the rows,
optimizer state and versions each owner holds after several steps, equal the oracle
driven with the whole global batch in ascending-SampleId order (bit-exact).

CPU: the collective sequencing of ShardedEmbeddingWorker over gloo (world 2 and 3) with
the local steps restated on the CPU (tests/sharded_oracle_ops.py).
GPU: the same case through libhps.so + NCCL (world 1 on one GPU; world 2 when two GPUs
are visible)."""
import pytest

from sharded_case import run_world


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_sequencing_gloo(world):
    res = run_world(world, "gloo", use_device=False)
    assert sorted(r for r, _, _ in res) == list(range(world))
    for r, status, n in res:
        assert status == "ok", status


def test_sharded_sequencing_gloo_sum_sgd():
    res = run_world(2, "gloo", use_device=False, agg="sum", opt="sgd")
    for r, status, n in res:
        assert status == "ok", status


TRANSPORTS = ["p2p", "nccl"]


@pytest.mark.gpu
@pytest.mark.parametrize("transport", TRANSPORTS)
def test_sharded_device_world1(transport):
    res = run_world(1, "nccl", use_device=True, transport=transport)
    assert res[0][1] == "ok", res[0][1]


@pytest.mark.gpu
@pytest.mark.parametrize("transport", TRANSPORTS)
@pytest.mark.parametrize("D", [64, 5])
def test_sharded_device_world1_nonfinite_rejected(D, transport):
    """A non-finite contribution at step 1: the owner applies nothing of that step (the
    sources validate while emitting on the p2p path, the owner's check on nccl); the
    steps before and after match the oracle that skipped it."""
    res = run_world(1, "nccl", use_device=True, D=D, steps=3, nan_step=1, transport=transport)
    assert res[0][1] == "ok", res[0][1]


@pytest.mark.gpu
@pytest.mark.parametrize("transport", TRANSPORTS)
@pytest.mark.parametrize("D", [64, 5])
def test_sharded_device_world1_large_plan(D, transport):
    """More than 4096 listings of repeated ids: the device-gated radix-sort path."""
    res = run_world(1, "nccl", use_device=True, B=1500, F=4, D=D, space=2500, steps=2,
                    transport=transport)
    assert res[0][1] == "ok", res[0][1]


@pytest.mark.gpu
@pytest.mark.parametrize("transport", TRANSPORTS)
@pytest.mark.parametrize("agg,opt", [("mean", "adagrad"), ("sum", "sgd")])
def test_sharded_device_world2(agg, opt, transport):
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    res = run_world(2, "nccl", use_device=True, agg=agg, opt=opt, transport=transport)
    for r, status, n in res:
        assert status == "ok", status


@pytest.mark.gpu
@pytest.mark.parametrize("transport", TRANSPORTS)
def test_sharded_device_world2_large_plan(transport):
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    res = run_world(2, "nccl", use_device=True, B=800, F=4, D=16, space=2000, steps=2,
                    transport=transport)
    for r, status, n in res:
        assert status == "ok", status


@pytest.mark.gpu
@pytest.mark.parametrize("agg,opt", [("mean", "adagrad"), ("sum", "sgd")])
@pytest.mark.parametrize("D", [64, 5])
def test_sharded_p2p_two_ranks(agg, opt, D):
    """Two ranks over the NVLink peer transport -- on two GPUs when the box has them, else
    both processes on one GPU (CUDA IPC arenas, device barriers, gloo only for the handle
    exchange): the multi-rank exchange, barriers and SampleId ordering run on a 1-GPU box
    too. Bit-exact vs the global-batch oracle."""
    res = run_world(2, "gloo", use_device=True, agg=agg, opt=opt, D=D, transport="p2p",
                    timeout=400)
    for r, status, n in res:
        assert status == "ok", status


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2])
@pytest.mark.parametrize("agg,opt,D", [("mean", "adagrad", 64), ("sum", "sgd", 8)])
def test_sharded_p2p_value_codec_matches_reference(world, agg, opt, D):
    """Codec mode (hps_exchange_set_codec, kappa 1024): rows and contributions cross the
    exchange as kappa-scaled binary16; pooled outputs and the owners' rows, accumulators
    and versions equal the reference run with PsShardService(compress) and
    EmbeddingWorkerConfig::compress_values (oracle/_ref), bit for bit."""
    res = run_world(world, "gloo", use_device=True, agg=agg, opt=opt, D=D, transport="p2p",
                    codec=1024.0, timeout=400)
    for r, status, n in res:
        assert status == "ok", status


@pytest.mark.gpu
@pytest.mark.parametrize("world", [4, 8])
def test_sharded_p2p_wide_world(world):
    """World 4 and 8 over the peer transport, ranks sharing the visible GPUs round-robin
    (8 processes on one GPU on a 1-GPU box): the wide exchange -- 8 id regions and pair
    segments per owner, 8-way device barriers, SampleId order across 8 sources -- bit-exact
    vs the global-batch oracle."""
    res = run_world(world, "gloo", use_device=True, transport="p2p", B=8, steps=2,
                    timeout=600)
    assert sorted(r for r, _, _ in res) == list(range(world))
    for r, status, n in res:
        assert status == "ok", status


@pytest.mark.gpu
def test_sharded_p2p_two_ranks_large_plan_and_graph():
    """Two ranks (one GPU if need be): the radix-sort plan of repeated ids, then a CUDA
    graph of the p2p step replayed on new inputs."""
    res = run_world(2, "gloo", use_device=True, B=800, F=4, D=16, space=2000, steps=2,
                    transport="p2p", timeout=400)
    for r, status, n in res:
        assert status == "ok", status
    res = run_world(2, "gloo", use_device=True, transport="p2p", graph=True, steps=4, B=16,
                    timeout=400)
    for r, status, n in res:
        assert status == "ok", status


@pytest.mark.gpu
def test_sharded_pipelined_prefetch_two_ranks():
    """bench.py's pipelined sharded schedule with two ranks (sharing GPU 0 on a 1-GPU box)."""
    from sharded_case import run_pipelined_world

    res = run_pipelined_world(2, D=8)
    assert all(r[1] == "ok" for r in res), [r[1] for r in res]


@pytest.mark.gpu
def test_sharded_p2p_cuda_graph_replay():
    """The peer-transport step has no host round trip: captured once in a CUDA graph and
    replayed on new inputs it stays bit-exact (device barrier epochs and step tags)."""
    import torch

    world = 2 if torch.cuda.device_count() >= 2 else 1
    res = run_world(world, "nccl", use_device=True, transport="p2p", graph=True, steps=4, B=16)
    for r, status, n in res:
        assert status == "ok", status


@pytest.mark.gpu
def test_apply_pairs_rejects_positions_outside_the_source_segment():
    """A pair naming an id outside its source's segment fails the whole apply
    (HPS_E_PROTOCOL) and leaves every row untouched."""
    import numpy as np
    import torch

    import oracle as O
    from paper_2111_05897_b200 import hps
    from paper_2111_05897_b200.sharded import DeviceOps

    dev = torch.device("cuda:0")
    salts = [O.mix64(7 + s) for s in range(4)]
    table = hps.ShardSet(4, 8, 1 << 12, hps.SGD, salts=salts)
    ops = DeviceOps(table, 1, hps.SUM)
    ids = torch.tensor([11, 12, 13], dtype=torch.int64, device=dev)
    rows, ver = ops.lookup(ids)
    torch.cuda.synchronize()
    before = table.peek(np.array([11, 12, 13], np.uint64))[0]
    pos = torch.tensor([0, 5], dtype=torch.int32, device=dev)  # 5 is outside [0, 3)
    con = torch.ones((2, 8), dtype=torch.float32, device=dev)
    with pytest.raises(hps.ProtocolError):
        ops.apply_pairs(ids, ver, [3], pos, con, [2], 0.5, 1, table.epoch(), flags=0)
    after = table.peek(np.array([11, 12, 13], np.uint64))[0]
    assert before.tobytes() == after.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("world,tau", [(1, 2), (2, 0), (2, 2)])
def test_sharded_hybrid_staleness(world, tau):
    """HybridTrainer over tau + 1 hash-sharded workers: owners' rows bit-exact vs the
    oracle driven with the recorded embedding gradients in staleness order; the dense
    replicas identical (canonical all-reduce)."""
    import torch

    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    from sharded_case import run_hybrid_world

    res = run_hybrid_world(world, tau=tau)
    assert all(r[1] == "ok" for r in res), [r[1] for r in res]


@pytest.mark.gpu
@pytest.mark.parametrize("world,D", [(1, 8), (2, 8), (2, 64)])
def test_sharded_pipelined_prefetch(world, D):
    """Two exchanges alternate; the next batch is prefetched (routed, pairs planned) on a
    second stream beside this batch's forward completion, pull and backward: bit-exact
    with the oracle in sync order."""
    import torch

    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    from sharded_case import run_pipelined_world

    res = run_pipelined_world(world, D=D)
    assert all(r[1] == "ok" for r in res), [r[1] for r in res]
