"""GPU parity at the BASELINE configurations' full sizes (c2 single step, c3
batched), against the oracle on the same inputs.  Slow-ish (table synthesis
dominates), so few queries; the bench repeats the c2 check on its own stream."""

import numpy as np
import pytest

import csvd_oracle as O
from conftest import TRANS_RTOL, assert_outcome, has_gpu
from test_gpu_batch import _fields

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a GPU")]


def test_c2_llama3_head_full_size():
    import paper_2511_21702_b200 as P
    from paper_2511_21702_b200 import workload as wl
    V, d, C, g = 128256, 4096, 1024, 16
    T = wl.synth_vocab(V, d, C // g, 0.3, 1)
    ix = wl.fast_index(T, C // g, g)
    q = np.vstack([wl.generate_queries(5, d, "contextual", 7, centroids=ix.centroids),
                   wl.generate_queries(1, d, "random", 8)])
    for cfg in (P.DecodeConfig(k=10), P.DecodeConfig(k=10, k_max=1200)):
        for i, h in enumerate(q):
            assert_outcome(P.decode_step(T, ix, h, cfg), _fields(O.decode_step(T, ix, h, cfg)), rtol=TRANS_RTOL,
                           where=f"c2[{cfg.k_max},{i}]")


def test_c3_qwen_head_batched_full_size():
    import paper_2511_21702_b200 as P
    from paper_2511_21702_b200 import workload as wl
    V, d, C = 151552, 3584, 2273
    T = wl.synth_vocab(V, d, C, 0.3, 1, dtype="bf16")
    ix = wl.fast_index(T, C, 1)
    H = wl.generate_queries(16, d, "contextual", 7, centroids=ix.centroids)
    cfg = P.DecodeConfig(k=10, epsilon=1e-3, targets=("softmax_eps",))
    outs = P.decode_step_batch(T, ix, H, cfg)
    for b, h in enumerate(H):
        assert_outcome(outs[b], _fields(O.decode_step(T, ix, h, cfg)), rtol=TRANS_RTOL, where=f"c3[{b}]")


def test_c4_llama70b_head_batched_full_size():
    """configs[3] on one B200: Llama-3 70B head V=128256 d=8192 C=1024, B=64."""
    import paper_2511_21702_b200 as P
    from paper_2511_21702_b200 import workload as wl
    V, d, C, g, B = 128256, 8192, 1024, 16, 64
    T = wl.synth_vocab(V, d, C // g, 0.3, 1)
    ix = wl.fast_index(T, C // g, g)
    H = np.vstack([wl.generate_queries(B - 4, d, "contextual", 7, centroids=ix.centroids),
                   wl.generate_queries(4, d, "random", 8)])
    cfg = P.DecodeConfig(k=10)
    outs = P.decode_step_batch(T, ix, H, cfg)
    for b in range(B):
        assert_outcome(outs[b], _fields(O.decode_step(T, ix, H[b], cfg)), rtol=TRANS_RTOL, where=f"c4[{b}]")


@pytest.fixture(scope="module")
def c5():
    from paper_2511_21702_b200 import workload as wl
    V, d, C, g = 256000, 3584, 3840, 16
    T = wl.synth_vocab(V, d, C // g, 0.3, 1, dtype="bf16")
    ix = wl.fast_index(T, C // g, g)
    H = np.vstack([wl.generate_queries(124, d, "contextual", 7, centroids=ix.centroids),
                   wl.generate_queries(4, d, "random", 8)])
    return T, ix, H


@pytest.mark.parametrize("B", [1, 16, 64, 128])
def test_c5_gemma2_head_batch_sweep_full_size(c5, B):
    """configs[4] on one B200: Gemma2 head V=256000 d=3584 C=3840 bf16, the
    B = 1..128 sweep (the lane grid shrinks to one CTA per query at B=128)."""
    import paper_2511_21702_b200 as P
    T, ix, H = c5
    Hb = H[-B:] if B < 4 else np.vstack([H[:B - 4], H[-4:]])
    cfg = P.DecodeConfig(k=10)
    outs = P.decode_step_batch(T, ix, Hb, cfg)
    for b in range(B):
        assert_outcome(outs[b], _fields(O.decode_step(T, ix, Hb[b], cfg)), rtol=TRANS_RTOL, where=f"c5 B={B} [{b}]")
