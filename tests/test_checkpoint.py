"""HPS1 checkpoints of the device table: the reference's on-disk
contract (PsShard::save_checkpoint / load_checkpoint / recover_from_checkpoint,
embedding_ps.hpp:209-402; its tests test_embedding_ps.cpp:243-391).

GPU: images written by the device table are byte-identical to the reference's when the
reference's recency order is its insertion order, and otherwise carry the same rows,
accumulators and versions (the reference loads them and trains on identically); images
written by the reference load into the device table bit-exactly; corrupt images are
rejected before anything changes.
"""
import struct

import numpy as np
import pytest

from conftest import cuda_available

import oracle as O
from paper_2111_05897_b200 import workloads as W

def _salts(S, base=7):
    return [W.mix64_int(base + s) for s in range(S)]


def test_reference_image_layout_for_insertion_ordered_touches():
    """CPU: the reference's own image when every step touches one new id -- slots in
    first-touch order, recency chain newest (head) -> oldest (tail): the canonical order
    the device table writes."""
    S, D, cap = 1, 4, 64
    ref = O.Reference(_salts(S), cap, D, "adagrad", "mean", groups=1)
    ids = [11, 5, 42, 7]
    for k, i in enumerate(ids):
        ref.step(1, np.array([i], np.uint64), np.array([0, 1], np.uint64),
                 np.full((1, 1, D), 0.25, np.float32), 0.1, k + 1, True)
    img = ref.shard_export(0)
    hwm, head, tail, free_head, live = struct.unpack_from("<5I", img, 24)
    assert (hwm, head, tail, free_head, live) == (4, 3, 0, 0xFFFFFFFF, 4)
    assert list(np.frombuffer(img, np.uint64, 4, 64)) == ids
    prev = np.frombuffer(img, np.uint32, 4, 64 + 32)
    nxt = np.frombuffer(img, np.uint32, 4, 64 + 48)
    assert list(prev) == [1, 2, 3, 0xFFFFFFFF] and list(nxt) == [0xFFFFFFFF, 0, 1, 2]


def _device_table(S, D, cap, opt="adagrad", salts=None):
    from paper_2111_05897_b200 import hps

    return hps.ShardSet(S, D, cap, hps.ADAGRAD if opt == "adagrad" else hps.SGD,
                        salts=salts or _salts(S), device=0)


def _run_device(table, stream, F, lr, agg="mean"):
    from paper_2111_05897_b200 import hps

    ew = hps.EmbeddingWorker(table, hps.MEAN if agg == "mean" else hps.SUM)
    for k, (ids, offs, g) in enumerate(stream):
        B = len(offs) - 1
        B //= F
        ew.register_batch(ids, offs, B, F)
        ew.serve_pull()
        assert ew.apply_backward(g, lr, k + 1)
    table.sync()


def _run_reference(ref, stream, F, lr, start=0):
    """Steps tagged start+1, start+2, ... (the step tag drives the version bumps)."""
    for k, (ids, offs, g) in enumerate(stream):
        B = (len(offs) - 1) // F
        ref.step(B, ids, offs.astype(np.uint64), g, lr, start + k + 1, True)


def _stream(steps, B, F, D, seed=3, id_space=300):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(steps):
        ids, offs = W.random_csr(rng, B, F, 3, id_space)
        g = (rng.standard_normal((B, F, D)) * 0.1).astype(np.float32)
        out.append((ids, offs, g))
    return out


def _device_state(table, ids):
    w, a, v, present = table.peek(ids)
    assert present.all()
    return w, a, v


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available(), reason="needs a GPU")
@pytest.mark.parametrize("opt,D", [("adagrad", 16), ("adagrad", 64), ("sgd", 8)])
def test_checkpoint_bytes_identical_to_reference(opt, D):
    S, cap = 3, 256
    rng = np.random.default_rng(1)
    ids = rng.permutation(1000)[:40].astype(np.uint64)
    stream = [(np.array([i], np.uint64), np.array([0, 1], np.uint32),
               (rng.standard_normal((1, 1, D)) * 0.1).astype(np.float32)) for i in ids]
    ref = O.Reference(_salts(S), cap, D, opt, "mean", groups=1)
    _run_reference(ref, stream, 1, 0.05)
    table = _device_table(S, D, 4096, opt)
    _run_device(table, stream, 1, 0.05)
    for s in range(S):
        assert table.save_checkpoint(s, shard_capacity=cap) == ref.shard_export(s)


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available(), reason="needs a GPU")
@pytest.mark.parametrize("D", [16, 64])
def test_reference_images_load_bit_exact_and_train_on(D):
    S, F, cap = 4, 3, 4096
    stream = _stream(6, 32, F, D)
    ref = O.Reference(_salts(S), cap, D, "adagrad", "mean", groups=F)
    _run_reference(ref, stream[:5], F, 0.05)
    images = [ref.shard_export(s) for s in range(S)]
    table = _device_table(S, D, 8192)
    table.load_checkpoint(images)
    want = ref.state()
    ids = np.array(sorted(want), np.uint64)
    w, a, v = _device_state(table, ids)
    assert w.tobytes() == np.stack([want[int(i)][0] for i in ids]).tobytes()
    assert a.tobytes() == np.stack([want[int(i)][1] for i in ids]).tobytes()
    assert (v == np.array([want[int(i)][2] for i in ids])).all()
    assert table.epoch() == 0
    # one more step on both sides: identical (the loaded versions drive the delays)
    _run_reference(ref, stream[5:], F, 0.05, start=5)
    from paper_2111_05897_b200 import hps

    ew = hps.EmbeddingWorker(table, hps.MEAN)
    ids5, offs5, g5 = stream[5]
    ew.register_batch(ids5, offs5, 32, F)
    ew.serve_pull()
    assert ew.apply_backward(g5, 0.05, 6)
    want = ref.state()
    ids = np.array(sorted(want), np.uint64)
    w, a, v = _device_state(table, ids)
    assert w.tobytes() == np.stack([want[int(i)][0] for i in ids]).tobytes()
    assert a.tobytes() == np.stack([want[int(i)][1] for i in ids]).tobytes()
    assert (v == np.array([want[int(i)][2] for i in ids])).all()


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available(), reason="needs a GPU")
def test_device_images_load_into_reference():
    S, F, D, cap = 4, 3, 16, 4096
    stream = _stream(6, 32, F, D, seed=9)
    table = _device_table(S, D, 8192)
    _run_device(table, stream[:5], F, 0.05)
    ref = O.Reference(_salts(S), cap, D, "adagrad", "mean", groups=F)
    _run_reference(ref, stream[:5], F, 0.05)
    images = [table.save_checkpoint(s, shard_capacity=cap) for s in range(S)]
    # same content as the reference's own images
    got = {}
    for im in images:
        got.update(O.parse_hps1(im)["rows"])
    want = ref.state()
    assert sorted(got) == sorted(want)
    for i, (w, a, v) in want.items():
        assert got[i][0].tobytes() == w.tobytes() and got[i][1].tobytes() == a.tobytes()
        assert got[i][2] == v
    # the reference adopts them (parse + restore validation) and trains on identically
    ref2 = O.Reference(_salts(S), cap, D, "adagrad", "mean", groups=F)
    for s, im in enumerate(images):
        ref2.shard_import(s, im, validate_only=True)
        ref2.shard_import(s, im)
    _run_reference(ref, stream[5:], F, 0.05, start=5)
    # ref2's shards recovered into epoch 1 (max(live, image) + 1)
    _run_reference_epoch(ref2, stream[5:], F, 0.05, start=5)
    a1, a2 = ref.state(), ref2.state()
    assert sorted(a1) == sorted(a2)
    for i in a1:
        assert a1[i][0].tobytes() == a2[i][0].tobytes()
        assert a1[i][1].tobytes() == a2[i][1].tobytes()
        assert a1[i][2] == a2[i][2]


def _run_reference_epoch(ref, stream, F, lr, start):
    ref.set_epoch(1)
    _run_reference(ref, stream, F, lr, start)


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available(), reason="needs a GPU")
def test_corrupt_images_rejected_and_table_unchanged():
    from paper_2111_05897_b200 import hps

    S, F, D = 2, 2, 8
    stream = _stream(3, 16, F, D, seed=5)
    src = _device_table(S, D, 4096)
    _run_device(src, stream, F, 0.05)
    good = [src.save_checkpoint(s) for s in range(S)]
    dst = _device_table(S, D, 4096)
    _run_device(dst, _stream(1, 8, F, D, seed=77), F, 0.05)
    probe = np.arange(0, 300, dtype=np.uint64)
    before = dst.peek(probe)

    def bad(mut, shard=0):
        b = bytearray(good[shard])
        mut(b)
        return bytes(b)

    def flip_body(b):
        b[80] ^= 0x10

    def magic(b):
        b[0:4] = b"HPS2"

    def version(b):
        b[4] = 2

    cases = [bad(flip_body), bad(magic), bad(version), good[0][:40], good[0][:-4]]
    for c in cases:
        with pytest.raises(hps.CheckpointCorruptError):
            dst.load_checkpoint([good[1], c])
    other = _device_table(S, 16, 4096).save_checkpoint(0)  # D = 16 image into a D = 8 table
    with pytest.raises(hps.CheckpointCorruptError):
        dst.load_checkpoint([other])
    foreign = _device_table(S, D, 4096, salts=_salts(S, base=99)).save_checkpoint(0)
    with pytest.raises(hps.ConfigError):
        dst.load_checkpoint([foreign])
    after = dst.peek(probe)
    for x, y in zip(before, after):
        assert np.asarray(x).tobytes() == np.asarray(y).tobytes()
    # a good set still loads, and recover advances the epoch past the live one
    e0 = dst.epoch()
    dst.load_checkpoint(good, recover=True)
    assert dst.epoch() == max(e0, 0) + 1
    ids = np.unique(np.concatenate([s[0] for s in stream]))
    w1, a1, v1, _ = src.peek(ids)
    w2, a2, v2, _ = dst.peek(ids)
    assert w1.tobytes() == w2.tobytes() and a1.tobytes() == a2.tobytes() and (v1 == v2).all()
    # a push tagged with the pre-recovery epoch is dropped (embedding_ps.hpp:142-145)
    ew = hps.EmbeddingWorker(dst, hps.MEAN)
    ids0, offs0, g0 = stream[0]
    ew.register_batch(ids0, offs0, 16, F)
    ew.serve_pull()
    assert not ew.apply_backward(g0, 0.05, 9, epoch=e0)
