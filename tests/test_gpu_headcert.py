"""GPU: the head step's certification from row-CTA segment records
(headstep.cuh head_certify_seg) against the oracle, over the cases it treats
specially: k beyond the register-list limit of the older certifiers (32),
k = 1, every target order, top-p, ties of the decision prefix, and the
determinism of the fixed-order reductions (rho bit-identical across runs).

Reference semantics: decode.py:192-210 / 312-343, certify.py:73-164."""

import numpy as np
import pytest

import csvd_oracle as O
from conftest import TRANS_RTOL, assert_outcome, has_gpu
import paper_2511_21702_b200 as P
from paper_2511_21702_b200 import workload as wl

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a GPU")]


def _fields(o):
    st = o.stats
    return dict(ids=o.token_ids, logits=o.logits, kind=o.status.kind, fallback=o.fallback_used,
                sub_size=st["sub_size"], clusters_opened=st["clusters_opened"], heap_pops=st["heap_pops"],
                flops_sparse=st["flops_sparse"], flops_bounds=st["flops_bounds"], eps=o.status.epsilon_achieved,
                u_max=o.status.u_max, topk_min=o.status.topk_min, rho=st["rho"], xi=st["xi"], ratio=st["ratio"])


@pytest.fixture(scope="module")
def case():
    T = wl.synth_vocab(32000, 4096, 64, 0.3, 1)
    ix = wl.fast_index(T, 64, 4)
    q = np.vstack([wl.generate_queries(5, 4096, "contextual", 7, centroids=ix.centroids),
                   wl.generate_queries(1, 4096, "random", 8)])
    return T, ix, q


@pytest.mark.parametrize("k", [1, 2, 33, 64, 150])
def test_head_k_range_vs_oracle(case, k):
    T, ix, q = case
    for cfg in (P.DecodeConfig(k=k), P.DecodeConfig(k=k, epsilon=0.02, targets=("softmax_eps", "topk"))):
        for i, h in enumerate(q):
            exp = O.decode_step(T, ix, h, cfg)
            got = P.decode_step(T, ix, h, cfg)
            assert_outcome(got, _fields(exp), rtol=TRANS_RTOL, where=f"k={k},{cfg.targets},{i}")


@pytest.mark.parametrize("targets", [("topk",), ("softmax_eps",), ("topp",), ("topp", "topk"),
                                     ("softmax_eps", "topp", "topk")])
def test_head_target_orders_vs_oracle(case, targets):
    T, ix, q = case
    for eps in (0.2, 0.05, 1e-3):
        cfg = P.DecodeConfig(k=10, epsilon=eps, targets=targets)
        for i, h in enumerate(q):
            exp = O.decode_step(T, ix, h, cfg)
            got = P.decode_step(T, ix, h, cfg)
            assert_outcome(got, _fields(exp), rtol=TRANS_RTOL, where=f"{targets},eps={eps},{i}")


def test_head_certification_is_deterministic(case):
    """Segment records are reduced in a fixed order: repeated steps give the
    same bits everywhere, rho and epsilon_achieved included."""
    T, ix, q = case
    cfg = P.DecodeConfig(k=10, epsilon=0.05)
    for h in q[:3]:
        a = P.decode_step(T, ix, h, cfg)
        for _ in range(3):
            b = P.decode_step(T, ix, h, cfg)
            assert np.array_equal(a.token_ids, b.token_ids)
            assert np.array_equal(a.logits.view(np.int64), b.logits.view(np.int64))
            assert np.float64(a.stats.rho).tobytes() == np.float64(b.stats.rho).tobytes()
            assert np.float64(a.status.epsilon_achieved).tobytes() == np.float64(b.status.epsilon_achieved).tobytes()
            assert a.status.topk_min == b.status.topk_min and a.stats.clusters_opened == b.stats.clusters_opened


def test_head_duplicate_logits_kth(case):
    """Duplicate rows (equal logits across clusters) at the k-th position: the
    candidate selection must return the tied value, as np.partition does."""
    T, ix, _ = case
    W = np.array(T.weights, dtype=np.float32, copy=True)
    # every row of the first 4000 repeated once: each logit appears twice
    W[4000:8000] = W[:4000]
    T2 = type(T)(weights=W, bias=np.zeros(W.shape[0]))
    ix2 = wl.fast_index(T2, 64, 4)
    q = wl.generate_queries(4, 4096, "contextual", 9, centroids=ix2.centroids)
    for k in (1, 10, 40):
        cfg = P.DecodeConfig(k=k)
        for i, h in enumerate(q):
            exp = O.decode_step(T2, ix2, h, cfg)
            got = P.decode_step(T2, ix2, h, cfg)
            assert_outcome(got, _fields(exp), rtol=TRANS_RTOL, where=f"dup k={k},{i}")


def test_device_step_reads_h_in_place(case):
    """csvd_step_device with caller-owned device queries (the head graph's
    kernel reads h where it lies, re-pointed per call): outcomes equal the
    host API's, whichever buffer each step's h comes from."""
    import ctypes

    import torch
    from paper_2511_21702_b200 import _lib
    T, ix, q = case
    ctx = P.prepare(T, ix)
    lib = _lib.load()
    cfg = P.DecodeConfig(k=10, epsilon=0.05)
    ccfg = ctx.make_config(cfg)
    hq = torch.from_numpy(np.ascontiguousarray(q)).cuda()
    ids_p, log_p, res_p = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    lib.csvd_outputs(ctx._ctx, ctypes.byref(ids_p), ctypes.byref(log_p), ctypes.byref(res_p))
    sp = ctypes.c_void_p()
    lib.csvd_stream(ctx._ctx, ctypes.byref(sp))
    for rep in range(2):
        for i in [0, 1, 2, 1, 0, 3, 3]:
            h = hq[i] if rep == 0 else hq[i].clone()  # the same pointers again / fresh buffers
            assert lib.csvd_step_device(ctx._ctx, h.data_ptr(), ctypes.byref(ccfg), sp) == 0
            torch.cuda.synchronize()
            exp = P.decode_step(T, ix, q[i], cfg)
            n = exp.stats.sub_size
            r = _lib.Result()
            ctypes.memmove(ctypes.byref(r), _d2h(res_p.value, ctypes.sizeof(_lib.Result), np.uint8).ctypes.data,
                           ctypes.sizeof(_lib.Result))
            assert int(r.sub_size) == n, (rep, i)
            assert np.array_equal(_d2h(ids_p.value, n, np.int64), exp.token_ids), (rep, i)
            assert np.array_equal(_d2h(log_p.value, n, np.float64).view(np.int64), exp.logits.view(np.int64)), (rep, i)


def _d2h(ptr, n, dtype):
    try:
        from cuda.bindings import runtime as rt
    except ImportError:  # older cuda-python layout
        from cuda import cudart as rt
    out = np.empty(n, dtype=dtype)
    err, = rt.cudaMemcpy(out.ctypes.data, ptr, out.nbytes, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
    assert int(err) == 0, err
    return out
