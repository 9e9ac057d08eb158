"""CSVD / CSVH / CSVI readers and writers (formats.py): byte compatibility with
the reference's own writers and readers (tensor_io.py:136-189,
cluster_index.py:398-479) and its error behaviour."""

import os
import struct
import sys

import numpy as np
import pytest

from paper_2511_21702_b200 import formats as F, workload as wl


@pytest.fixture(scope="module")
def small():
    T = wl.synth_vocab(600, 24, 6, 0.4, 3)
    ix = wl.fast_index(T, 6, 2)
    aug = wl.fast_index(T, 6, 2, mode="bias_augmented")
    return T, ix, aug


def _same_index(a, b):
    assert (a.mode, a.vocab_size, a.hidden_dim, a.bias_depth, a.fingerprint) == \
           (b.mode, b.vocab_size, b.hidden_dim, b.bias_depth, b.fingerprint)
    assert np.array_equal(a.perm, b.perm)
    for x, y in zip(a.clusters, b.clusters):
        assert np.array_equal(x.centroid, y.centroid)
        assert (x.centroid_norm, x.radius, x.angular, x.max_bias, x.max_norm, x.min_norm, x.start, x.end) == \
               (y.centroid_norm, y.radius, y.angular, y.max_bias, y.max_norm, y.min_norm, y.start, y.end)
        assert tuple(x.bias_topm) == tuple(y.bias_topm)


def test_round_trip(tmp_path, small):
    T, ix, aug = small
    F.save_table(T, tmp_path / "t.csvd")
    T2 = F.load_table(tmp_path / "t.csvd")
    assert np.array_equal(T2.weights_f64(), T.weights_f64()) and np.array_equal(T2.bias, T.bias)
    for idx in (ix, aug):
        F.save_index(idx, tmp_path / "i.csvi")
        _same_index(F.load_index(tmp_path / "i.csvi"), idx)
    q = wl.generate_queries(5, 24, "random", 1).astype(np.float32).astype(np.float64)
    F.save_queries(q, tmp_path / "q.csvh")
    assert np.array_equal(F.load_queries(tmp_path / "q.csvh"), q)


def test_errors(tmp_path, small):
    T, ix, _ = small
    p = tmp_path / "t.csvd"
    F.save_table(T, p)
    data = p.read_bytes()
    (tmp_path / "bad").write_bytes(b"XXXX" + data[4:])
    with pytest.raises(F.BadMagicError):
        F.load_table(tmp_path / "bad")
    (tmp_path / "ver").write_bytes(data[:4] + struct.pack("<I", 2) + data[8:])
    with pytest.raises(F.VersionMismatchError):
        F.load_table(tmp_path / "ver")
    (tmp_path / "trunc").write_bytes(data[:-3])
    with pytest.raises(F.TruncatedPayloadError):
        F.load_table(tmp_path / "trunc")
    (tmp_path / "trail").write_bytes(data + b"\0")
    with pytest.raises(F.TruncatedPayloadError):
        F.load_table(tmp_path / "trail")
    nan = bytearray(data)
    nan[32:36] = struct.pack("<f", float("nan"))
    (tmp_path / "nan").write_bytes(bytes(nan))
    with pytest.raises(F.NonFiniteEntryError):
        F.load_table(tmp_path / "nan")
    F.save_index(ix, tmp_path / "i.csvi")
    with pytest.raises(F.TruncatedPayloadError):
        (tmp_path / "i2").write_bytes((tmp_path / "i.csvi").read_bytes()[:-1])
        F.load_index(tmp_path / "i2")


def _reference():
    path = "/root/reference/pkg/src"
    if not os.path.isdir(path):
        return None
    sys.path.insert(0, path)
    try:
        import csvd
        return csvd
    except Exception:  # pragma: no cover
        return None
    finally:
        sys.path.remove(path)


def test_byte_compatible_with_reference(tmp_path, small):
    csvd = _reference()
    if csvd is None:
        pytest.skip("reference not importable on this host")
    from csvd import cluster_index as RC, tensor_io as RT
    T, ix, aug = small
    # ours -> reference reader
    F.save_table(T, tmp_path / "a.csvd")
    RTab = RT.load_embedding_table(tmp_path / "a.csvd")
    assert np.array_equal(RTab.weights, T.weights_f64()) and np.array_equal(RTab.bias, T.bias)
    for idx in (ix, aug):
        F.save_index(idx, tmp_path / "a.csvi")
        R = RC.load_index(tmp_path / "a.csvi")
        _same_index(R, idx)
        # reference writer -> ours, byte for byte identical files
        RC.save_index(R, tmp_path / "b.csvi")
        assert (tmp_path / "a.csvi").read_bytes() == (tmp_path / "b.csvi").read_bytes()
        _same_index(F.load_index(tmp_path / "b.csvi"), idx)
    RT.save_embedding_table(RTab, tmp_path / "b.csvd")
    assert (tmp_path / "a.csvd").read_bytes() == (tmp_path / "b.csvd").read_bytes()
