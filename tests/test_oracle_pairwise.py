"""Pins the oracle's C pairwise GEMV (oracle/pairwise.c) to numpy's own
add-reduce, bit for bit: out[r] = (rows[r] * h).sum() -- the reference's
csvd._linalg.gemv_rows (/root/reference/pkg/src/csvd/_linalg.py:25-37) --
for every d in 1..600 and the BASELINE / edge lengths up to 16385, with f32
(widened exactly), bf16 and f64 rows; and l2_norm (_linalg.py:40-43)."""
import numpy as np
import pytest

import csvd_oracle as O
from paper_2511_21702_b200 import workload as wl

LONG = [1000, 1023, 1024, 1025, 2047, 2048, 2049, 3584, 3585, 4095, 4096, 4097, 8192, 8193, 12288, 16384, 16385]


def _case(d, seed, rows=3):
    rng = np.random.default_rng(seed)
    w32 = rng.standard_normal((rows, d)).astype(np.float32)
    h = rng.standard_normal(d)
    return w32, h


def test_every_short_length():
    for d in range(1, 601):
        w32, h = _case(d, d)
        want = (w32.astype(np.float64) * h).sum(axis=1)
        got = O.gemv_rows(w32, h)
        assert np.array_equal(got, want), d


@pytest.mark.parametrize("d", LONG)
def test_long_lengths_and_dtypes(d):
    w32, h = _case(d, 7 + d)
    assert np.array_equal(O.gemv_rows(w32, h), (w32.astype(np.float64) * h).sum(axis=1))
    w64 = w32.astype(np.float64) * 1.0000001  # not f32-exact: centroid-like rows
    assert np.array_equal(O.gemv_rows(w64, h), (w64 * h).sum(axis=1))
    b16 = wl.f32_to_bf16_bits(w32)
    wide = wl.bf16_bits_to_f32(b16).astype(np.float64)
    assert np.array_equal(O.gemv_rows(b16, h), (wide * h).sum(axis=1))
    assert O.l2_norm(h) == np.sqrt((h * h).sum())
