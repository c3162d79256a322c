"""The reference's lossy value codec on the device (codec.hpp:
30-103, 208-261; the reference's own cases test_codec.cpp:121-226).

CPU: the numpy restatement pinned against the reference (compiled in oracle/_ref) on
random rows across 60 binades, zero rows, signed zeros and subnormals.
GPU: hps.compress_values / decompress_values bit-identical to the reference, host and
device buffers; the reference's error cases.
"""
import numpy as np
import pytest

from conftest import cuda_available

import oracle as O


def _rows(seed=0, n=64, d=64):
    rng = np.random.default_rng(seed)
    v = (rng.standard_normal((n, d)) * np.exp(rng.uniform(-30, 30, (n, 1)))).astype(np.float32)
    v[3] = 0.0
    v[4, :5] = -0.0
    v[5] = np.float32(1e-30)  # tiny but normal: scale stays finite
    v[6, ::2] = 0.0
    v[7] = np.float32(3.0e38) * np.sign(v[7])  # near FLT_MAX
    return v


def test_restatement_matches_reference():
    import warnings

    v = _rows()
    s1, p1 = O.ref_compress_values(v)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        s2, p2 = O.compress_values_np(v)
    assert s1.tobytes() == s2.tobytes() and p1.tobytes() == p2.tobytes()
    assert O.ref_decompress_values(s1, p1).tobytes() == O.decompress_values_np(s2, p2).tobytes()


def test_reference_roundtrip_bound():
    """||v - decompress(compress(v))||_inf <= ||v||_inf * 2^-11 (codec.hpp:208-213)."""
    v = _rows(1)
    s, p = O.ref_compress_values(v)
    back = O.ref_decompress_values(s, p)
    bound = np.abs(v).max(axis=1, keepdims=True) * 2.0**-11
    assert (np.abs(back - v) <= bound).all()


gpu = pytest.mark.skipif(not cuda_available(), reason="needs a GPU")


@pytest.mark.gpu
@gpu
@pytest.mark.parametrize("d", [64, 16, 5, 1, 100])
def test_device_codec_bit_exact(d):
    import torch

    from paper_2111_05897_b200 import hps

    v = _rows(2, 300, d)
    s_ref, p_ref = O.ref_compress_values(v)
    s, p = hps.compress_values(v)  # host buffers
    assert s.tobytes() == s_ref.tobytes() and p.tobytes() == p_ref.tobytes()
    out = hps.decompress_values(s, p)
    assert out.tobytes() == O.ref_decompress_values(s_ref, p_ref).tobytes()
    dv = torch.from_numpy(v).cuda()  # device buffers
    ds, dp = hps.compress_values(dv)
    assert ds.cpu().numpy().tobytes() == s_ref.tobytes()
    assert dp.cpu().numpy().view(np.uint16).tobytes() == p_ref.tobytes()
    do = hps.decompress_values(ds, dp)
    assert do.cpu().numpy().tobytes() == out.tobytes()
    # kappa other than the default
    s2, p2 = hps.compress_values(v, kappa=30000.0)
    s2r, p2r = O.ref_compress_values(v, 30000.0)
    assert s2.tobytes() == s2r.tobytes() and p2.tobytes() == p2r.tobytes()


@pytest.mark.gpu
@gpu
def test_device_codec_errors():
    from paper_2111_05897_b200 import hps

    with pytest.raises(hps.PreconditionError):  # test_codec.cpp:210-212
        hps.compress_values(np.array([[1.0, np.inf]], np.float32))
    with pytest.raises(hps.PreconditionError):
        hps.compress_values(np.array([[np.nan]], np.float32))
    with pytest.raises(hps.PreconditionError):  # :213
        hps.compress_values(np.array([[1.0]], np.float32), kappa=0.0)
    s, p = hps.compress_values(np.array([[1.0, -2.0]], np.float32))
    for bad in (0.0, -1.0, np.inf, np.nan):  # :215-225
        with pytest.raises(hps.ProtocolError):
            hps.decompress_values(np.array([bad], np.float32), p)
    with pytest.raises(hps.ProtocolError):  # non-finite payload value
        hps.decompress_values(s, np.array([[0x7C00, 0]], np.uint16))
