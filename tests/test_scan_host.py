"""The certification scan state machine (csrc/scan.cuh) reproduces the
reference's decode loop, run on the HOST through the extension's test hook.

The device runs the same template code (one warp, lanes in lockstep); here it
is fed per-cluster summaries computed by the oracle, so any mismatch is a bug
in the step-driver restatement itself (k_max check, check order, partial
expand, relax-eps, 64-merge recompute, batch-select selection, heap_pops,
tightness), independent of the kernels.  No GPU needed.
"""

import ctypes

import numpy as np
import pytest

import csvd_oracle as O
from conftest import GoldenCase, close, golden_names
from paper_2511_21702_b200 import _lib
from paper_2511_21702_b200.engine import config_struct

KIND = {0: "topk_exact", 1: "softmax_eps", 2: "topp_mass"}
PH_DONE, PH_DENSE = 2, 3


def _inputs(case, h, U):
    ix = case.index
    C = ix.n_clusters
    order = np.lexsort((np.arange(C), -U)).astype(np.int32)
    sizes = np.asarray(ix.sizes)
    cum = np.concatenate([[0], np.cumsum(sizes[order])]).astype(np.int32)
    logsz = np.log(sizes)
    lrh = np.empty(C + 1)
    opened = np.zeros(C, dtype=bool)
    for p in range(C + 1):
        un = ~opened
        lrh[p] = O.logsumexp(logsz[un] + U[un]) if un.any() else -np.inf
        if p < C:
            opened[order[p]] = True
    return order, cum, lrh


def _summaries(case, h, order, k):
    ix, T = case.index, case.table
    C = ix.n_clusters
    K = 16
    while K < k:
        K *= 2
    lse = np.empty(C)
    mn = np.empty(C)
    mx = np.empty(C)
    topk = np.full((C, K), -np.inf)
    S = []
    for q, c in enumerate(order):
        members = ix.members(int(c))
        lg = O.gemv_rows(T.weights, np.asarray(h, dtype=np.float64), sel=members, bias=T.bias)
        S.append(lg)
        lse[q] = O.logsumexp(lg)
        mn[q] = lg.min()
        mx[q] = lg.max()
        srt = -np.sort(-lg)[:k]
        topk[q, :srt.size] = srt
    return lse, mn, mx, np.ascontiguousarray(topk), K, np.concatenate(S)


@pytest.mark.parametrize("name", golden_names())
def test_host_scan_matches_reference(name):
    lib = _lib.load()
    case = GoldenCase(name)
    ix = case.index
    C, V, d = ix.n_clusters, ix.vocab_size, ix.hidden_dim
    n = 0
    for st in case.steps():
        if n >= 60:
            break
        n += 1
        exp = case.expected(st["i"])
        U = exp["U"]
        order, cum, lrh = _inputs(case, st["h"], U)
        cfg = st["cfg"]
        variant = 0 if st["variant"] == "incremental" else 1
        c = config_struct(cfg, V, st["k_max"], variant)
        lse, mn, mx, topk, K, S = _summaries(case, st["h"], order, cfg.k)
        p_sel = 0
        if variant == 1:
            p_sel = len(O.select_by_bound(order, np.asarray(ix.sizes), c.k_max))
        res = _lib.Result()
        pf = ctypes.c_int()
        ph = ctypes.c_int()
        Uo = np.ascontiguousarray(U[order])
        args = [np.ascontiguousarray(a) for a in (cum, Uo, lrh, lse, mn, mx, topk, S)]
        rc = lib.csvd_test_scan_host(ctypes.byref(c), C, V, d, *[a.ctypes.data for a in args[:7]], K,
                                     args[7].ctypes.data, p_sel, ctypes.byref(res), ctypes.byref(pf),
                                     ctypes.byref(ph))
        assert rc == 0
        where = f"{name}[{st['i']}]"
        if exp["fallback"] == "full_vocab":
            assert ph.value == PH_DENSE, where
            # the chain reached FullVocab: the device dense phase decides the
            # step, which the reference reports as exact top-k over all V
            assert exp["kind"] == "topk_exact" and exp["sub_size"] == V, where
            continue
        assert ph.value == PH_DONE, where
        assert KIND[res.kind] == exp["kind"], where
        assert _lib.FB_NAMES[res.fallback] == exp["fallback"], where
        assert res.sub_size == exp["sub_size"], where
        assert res.clusters_opened == exp["clusters_opened"], where
        assert res.heap_pops == exp["heap_pops"], where
        assert res.u_max == exp["u_max"], where
        assert res.topk_min == exp["topk_min"], where
        assert close(res.xi, exp["xi"], 0.0), where
        assert close(res.rho, exp["rho"], 1e-12), where
        assert close(res.epsilon_achieved, exp["eps"], 1e-12), where
