"""The C restatement reproduces every committed reference fixture bit-for-bit (CPU)."""
import numpy as np
import pytest

import golden_cases as G
import oracle as O

pytestmark = pytest.mark.usefixtures("oracle_built")


@pytest.mark.parametrize("case", G.SYNC_CASES)
def test_restatement_replays_reference_fixture(case):
    G.replay_oracle(case)


def test_mix64_route_init_vectors():
    d = G.load("mix64_init")
    for x, m in zip(d["x"], d["mix"]):
        assert O.mix64(int(x)) == int(m)
    for i, x in enumerate(d["x"]):
        for j, s in enumerate(d["route_s"]):
            assert O.route_shard(int(x), int(s)) == int(d["routes"][i, j])
    for dim in (1, 4, 5, 16, 64):
        for i, x in enumerate(d["x"]):
            assert O.init_row(int(x), int(d["salt"]), dim).tobytes() == d[f"init_{dim}"][i].tobytes()


def test_compress_indices_fixture():
    d = G.load("compress_indices")
    res = O.compress_indices(int(d["B"]), int(d["G"]), d["ids"], d["offsets"].astype(np.uint64))
    for g, (u, posts) in enumerate(res):
        assert (u == d[f"unique_{g}"]).all()
        assert [len(p) for p in posts] == list(d[f"post_len_{g}"])
        flat = np.concatenate(posts) if posts else np.zeros(0, np.uint16)
        assert (flat == d[f"postings_{g}"]).all()
