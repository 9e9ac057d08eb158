"""GPU offline clustering (build_index_gpu, the B200 counterpart of
csvd.build_index, cluster_index.py:282-341): a valid partition with the
reference's statistics and ordering, for every bound mode, and decoding with
the index it builds is exact against the oracle."""
import numpy as np
import pytest

import csvd_oracle as O
from conftest import TRANS_RTOL, assert_outcome, has_gpu
from test_gpu_batch import _fields

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a GPU")]


@pytest.mark.parametrize("mode", ["euclidean", "spherical", "bias_augmented"])
def test_build_index_gpu_valid_and_exact_decode(mode):
    import paper_2511_21702_b200 as P
    from paper_2511_21702_b200 import workload as wl
    T = wl.synth_vocab(6000, 128, 30, 0.2, 1)
    ix = P.build_index_gpu(T, 60, mode=mode, iters=12, seed=0)
    assert ix.n_clusters == 60 and ix.mode == mode
    perm = np.asarray(ix.perm)
    assert np.array_equal(np.sort(perm), np.arange(T.vocab_size))  # a partition
    sizes = np.asarray(ix.sizes)
    assert (sizes > 0).all() and (np.diff(sizes) <= 0).all()  # size-descending order
    # the statistics are the reference's arithmetic on this partition
    ref = wl.index_from_assignment(T, np.repeat(np.arange(60), sizes)[np.argsort(perm)], mode=mode)
    assert np.array_equal(np.asarray(ref.centroids), np.asarray(ix.centroids))
    assert np.array_equal(np.asarray(ref.radii), np.asarray(ix.radii))
    d = T.hidden_dim
    H = np.vstack([wl.generate_queries(3, d, "contextual", 7, centroids=np.asarray(ix.centroids)[:, :d]),
                   wl.generate_queries(1, d, "random", 8)])
    cfg = P.DecodeConfig(k=10)
    for i, h in enumerate(H):
        assert_outcome(P.decode_step(T, ix, h, cfg), _fields(O.decode_step(T, ix, h, cfg)), rtol=TRANS_RTOL,
                       where=f"{mode}[{i}]", exact_bounds=mode != "spherical")


def test_build_index_gpu_errors():
    import paper_2511_21702_b200 as P
    from paper_2511_21702_b200 import workload as wl
    T = wl.synth_vocab(500, 32, 5, 0.2, 1)
    for kw in (dict(n_clusters=0), dict(n_clusters=501), dict(n_clusters=5, iters=0), dict(n_clusters=5, m=0),
               dict(n_clusters=5, mode="cosine")):
        with pytest.raises(ValueError):
            P.build_index_gpu(T, **kw)
