"""The workload generators the parity tests and the bench rely on reproduce
the reference's bits: synth_vocab (tensor_io.py:192-216), generate_queries
(bench.py:183-209) and the table fingerprint (tensor_io.py:219-226); the fast
index passes the reference's own validate_index
(cluster_index.py:344-395).  Compared with the reference itself where it is
importable (this build container); skipped on the GPU box."""
import os
import sys

import numpy as np
import pytest

from paper_2511_21702_b200 import workload as wl

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="needs the reference importable")


@pytest.fixture(scope="module")
def csvd():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import csvd as c
    import csvd.bench  # noqa: F401
    return c


@pytest.mark.parametrize("V,d,modes,spread,seed", [(3000, 64, 30, 0.05, 1), (2048, 96, 16, 0.3, 5)])
def test_synth_vocab_and_fingerprint_bit_equal(csvd, V, d, modes, spread, seed):
    ref = csvd.synth_vocab(V, d, modes, spread, seed)
    ours = wl.synth_vocab(V, d, modes, spread, seed)
    assert np.array_equal(ref.weights, ours.weights.astype(np.float64))
    assert np.array_equal(ref.bias, ours.bias)
    assert wl.table_fingerprint(ours) == csvd.tensor_io.table_fingerprint(ref)


@pytest.mark.parametrize("model", ["contextual", "random"])
def test_generate_queries_bit_equal(csvd, model):
    T = wl.synth_vocab(2000, 64, 20, 0.05, 1)
    ix = wl.fast_index(T, 20, 2)
    ref = csvd.bench.generate_queries(25, 64, model, 7, centroids=ix.centroids, noise=0.3, zipf_exponent=1.1)
    ours = wl.generate_queries(25, 64, model, 7, centroids=ix.centroids, noise=0.3, zipf_exponent=1.1)
    assert np.array_equal(ref, ours)


def test_fast_index_passes_reference_validation(csvd, tmp_path):
    from csvd.cluster_index import load_index
    from paper_2511_21702_b200 import formats
    ref_table = csvd.synth_vocab(4000, 32, 25, 0.05, 1)
    T = wl.synth_vocab(4000, 32, 25, 0.05, 1)
    ix = wl.fast_index(T, 25, 3, fingerprint=wl.table_fingerprint(T))
    formats.save_index(ix, tmp_path / "ix.csvi")  # byte-identical with the reference's writer
    ref_ix = load_index(tmp_path / "ix.csvi")
    rep = csvd.validate_index(ref_ix, ref_table)
    assert getattr(rep, "ok", True) and not getattr(rep, "violations", None), rep
