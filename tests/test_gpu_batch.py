"""GPU: batched decode (B queries, one graph replay, concurrent lanes) equals
B independent reference decode_step calls, query by query."""

import numpy as np
import pytest

import csvd_oracle as O
from conftest import TRANS_RTOL, assert_outcome, has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a GPU")]


def _fields(o):
    st = o.stats
    return dict(ids=o.token_ids, logits=o.logits, kind=o.status.kind, fallback=o.fallback_used,
                sub_size=st["sub_size"], clusters_opened=st["clusters_opened"], heap_pops=st["heap_pops"],
                flops_sparse=st["flops_sparse"], flops_bounds=st["flops_bounds"], eps=o.status.epsilon_achieved,
                u_max=o.status.u_max, topk_min=o.status.topk_min, rho=st["rho"], xi=st["xi"], ratio=st["ratio"])


@pytest.mark.parametrize("B,dtype", [(16, "bf16"), (5, "f32"), (1, "f32")])
def test_batch_equals_independent_steps(B, dtype):
    import paper_2511_21702_b200 as P
    from paper_2511_21702_b200 import workload as wl
    d = 3584
    T = wl.synth_vocab(24000, d, 96, 0.3, 1, dtype=dtype)
    ix = wl.fast_index(T, 96, 3)
    H = np.vstack([wl.generate_queries(B - B // 4, d, "contextual", 7, centroids=ix.centroids),
                   wl.generate_queries(B // 4, d, "random", 8)]) if B > 1 else \
        wl.generate_queries(1, d, "contextual", 7, centroids=ix.centroids)
    for cfg in (P.DecodeConfig(k=10, epsilon=1e-3, targets=("softmax_eps",)), P.DecodeConfig(k=10)):
        outs = P.decode_step_batch(T, ix, H, cfg)
        assert len(outs) == B
        for b in range(B):
            exp = O.decode_step(T, ix, H[b], cfg)
            assert_outcome(outs[b], _fields(exp), rtol=TRANS_RTOL, where=f"B={B} {dtype} q{b}")
        # the same queries one by one through the single-query path
        for b in range(min(B, 3)):
            one = P.decode_step(T, ix, H[b], cfg)
            assert np.array_equal(one.token_ids, outs[b].token_ids)
            assert np.array_equal(one.logits, outs[b].logits)


@pytest.mark.parametrize("mode", ["spherical", "bias_augmented"])
def test_batch_other_bound_modes(mode):
    """Spherical (batched dots + cone bound in the lanes) and bias-augmented
    (d+1 bound rows: no batched bounds, forked lanes with their own bounds)."""
    import paper_2511_21702_b200 as P
    from paper_2511_21702_b200 import workload as wl
    d = 512
    T = wl.synth_vocab(12000, d, 60, 0.3, 1)
    ix = wl.fast_index(T, 60, 2, mode=mode)
    H = np.vstack([wl.generate_queries(5, d, "contextual", 7, centroids=ix.centroids[:, :d]),
                   wl.generate_queries(2, d, "random", 8)])
    for cfg in (P.DecodeConfig(k=10), P.DecodeConfig(k=5, epsilon=1e-2, targets=("softmax_eps",))):
        outs = P.decode_step_batch(T, ix, H, cfg)
        for b in range(len(H)):
            exp = O.decode_step(T, ix, H[b], cfg)
            assert_outcome(outs[b], _fields(exp), rtol=TRANS_RTOL, where=f"{mode} q{b}",
                           exact_bounds=mode != "spherical")


@pytest.mark.parametrize("d,B", [(512, 9), (4096, 13), (8192, 7), (3584, 1)])
def test_batch_bounds_tree_per_dimension(d, B):
    """Batched dots (chain-per-lane register blocks, partial query groups,
    slice trees of depth 0..4) give every query the single-query outcome."""
    import paper_2511_21702_b200 as P
    from paper_2511_21702_b200 import workload as wl
    T = wl.synth_vocab(6000, d, 40, 0.3, 1)
    ix = wl.fast_index(T, 40, 3)
    H = np.vstack([wl.generate_queries(B - B // 3, d, "contextual", 7, centroids=ix.centroids),
                   wl.generate_queries(B // 3, d, "random", 8)])
    cfg = P.DecodeConfig(k=10)
    outs = P.decode_step_batch(T, ix, H, cfg)
    for b in range(B):
        assert_outcome(outs[b], _fields(O.decode_step(T, ix, H[b], cfg)), rtol=TRANS_RTOL, where=f"d={d} q{b}")
