"""Known-answer tests restated from the reference's own test suite, run on
the oracle (CPU, always) and on the CUDA path (`-m gpu`).

Each case cites the reference test it restates; the expected values are that
test's assertions (known answers), not a comparison between the two backends.
Indexes are built with workload.index_from_assignment (the reference's
_cluster_stats arithmetic, cluster_index.py:254-279) from the partition the
reference's k-means finds on these separable tables.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import has_gpu  # noqa: F401
from paper_2511_21702_b200 import types as T
from paper_2511_21702_b200 import workload as wl

import csvd_oracle as O  # checker


def unit_queries(n, d, seed):  # reference tests/conftest.py:43-46
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((n, d))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


class Oracle:
    name = "oracle"

    def step(self, table, index, h, cfg, batchselect=False):
        o = (O.decode_step_batchselect if batchselect else O.decode_step)(table, index, h, cfg)
        return dict(kind=o.status.kind, eps=o.status.epsilon_achieved, u_max=o.status.u_max,
                     kth=o.status.topk_min, fb=o.fallback_used, ids=o.token_ids, logits=o.logits,
                     opened=o.stats["clusters_opened"], pops=o.stats["heap_pops"], rho=o.stats["rho"],
                     sub=o.stats["sub_size"])

    def bounds(self, index, h):
        return O.cluster_bounds(index, h).values

    def dense(self, table, h):
        logits, _, order = O.dense_logits(table, h)
        return logits, order


class Gpu:
    name = "gpu"

    def __init__(self):
        import paper_2511_21702_b200 as P
        self.P = P

    def step(self, table, index, h, cfg, batchselect=False):
        P = self.P
        o = (P.decode_step_batchselect if batchselect else P.decode_step)(table, index, h, cfg)
        return dict(kind=o.status.kind, eps=o.status.epsilon_achieved, u_max=o.status.u_max,
                    kth=o.status.topk_min, fb=o.fallback_used, ids=o.token_ids, logits=o.logits,
                    opened=o.stats.clusters_opened, pops=o.stats.heap_pops, rho=o.stats.rho,
                    sub=o.stats.sub_size)

    def bounds(self, index, h):
        return self.P.cluster_bounds(index, h).values

    def dense(self, table, h):
        r = self.P.dense_logits(table, h)
        return r.logits, r.order


BACKENDS = [pytest.param("oracle", id="oracle"), pytest.param("gpu", id="gpu", marks=pytest.mark.gpu)]


@pytest.fixture(params=BACKENDS)
def be(request):
    return Oracle() if request.param == "oracle" else Gpu()


def _table(rows, bias=None):
    w = np.asarray(rows, dtype=np.float64)
    return T.EmbeddingTable(weights=w, bias=np.zeros(w.shape[0]) if bias is None else np.asarray(bias, float))


def test_euclidean_formula_value(be):
    # reference tests/test_bounds.py:31-41: centroid (1,0), radius 0.5, max bias
    # 0.1 (an f64 bias that is not f32-exact), U = 2 + 1 + 0.1
    t = _table([[1.5, 0.0], [0.5, 0.0]], [0.1, -0.3])
    ix = wl.index_from_assignment(t, np.array([0, 0]))
    assert ix.clusters[0].radius == 0.5 and ix.clusters[0].max_bias == 0.1
    u = be.bounds(ix, np.array([2.0, 0.0]))
    assert abs(u[0] - 3.1) <= 1e-12
    # the logits carry the exact f64 bias (tensor_io.py:69-94)
    out = be.step(t, ix, np.array([2.0, 0.0]), T.DecodeConfig(k=2, targets=("topk",), k_max=2))
    assert out["logits"].tolist() == [3.0 + 0.1, 1.0 - 0.3] and out["ids"].tolist() == [0, 1]


def test_singleton_bound_is_exact_logit(be):
    # reference tests/test_bounds.py:44-53: a singleton's bound IS its logit, bitwise
    t = wl.synth_vocab(6, 5, 3, 0.4, 9, dtype="f64")
    t = T.EmbeddingTable(weights=t.weights, bias=np.zeros(6))
    ix = wl.index_from_assignment(t, np.arange(6))
    h = unit_queries(1, 5, 0)[0]
    u = be.bounds(ix, h)
    logits, _ = be.dense(t, h)
    for c in range(6):
        assert u[c] == logits[int(ix.perm[ix.starts[c]])]


@pytest.mark.parametrize("b_row, certified_after", [(2.5, 1), (3.0, 2)])
def test_topk_strict_dominance_and_tie(be, b_row, certified_after):
    # reference tests/test_certify.py:33-47 at the decode level: after opening
    # {5, 3} (k = 2) the next bound is a singleton's exact logit; 2.5 < 3
    # certifies, the tie 3.0 == 3.0 must not (strict <)
    t = _table([[5.0, 0.0], [3.0, 0.0], [b_row, 0.0]])
    ix = wl.index_from_assignment(t, np.array([0, 0, 1]))
    out = be.step(t, ix, np.array([1.0, 0.0]), T.DecodeConfig(k=2, targets=("topk",), k_max=3))
    assert out["kind"] == "topk_exact" and out["fb"] is None
    assert out["opened"] == certified_after and out["pops"] == certified_after
    assert out["kth"] == 3.0
    assert out["u_max"] == (b_row if certified_after == 1 else -math.inf)


def test_softmax_worked_example(be):
    # reference tests/test_certify.py:62-71 at the decode level: one computed
    # token at logit 0, one unopened pair bounded at b: rho = 2e^b / (1 + 2e^b)
    b = -4.5
    t = _table([[0.0, 0.0], [b, 0.0], [b, 0.0]])
    ix = wl.index_from_assignment(t, np.array([0, 1, 1]))
    out = be.step(t, ix, np.array([1.0, 0.0]), T.DecodeConfig(k=1, epsilon=0.05, targets=("softmax_eps",), k_max=3))
    want = 2 * math.exp(b) / (1 + 2 * math.exp(b))
    assert out["kind"] == "softmax_eps" and out["opened"] == 1
    assert out["rho"] == pytest.approx(want, rel=1e-12)
    assert out["eps"] == pytest.approx(want, rel=1e-12)


@pytest.mark.parametrize("scale, certified", [(0.999, True), (1.001, False)])
def test_topp_threshold(be, scale, certified):
    # reference tests/test_certify.py:97-105: certified iff delta <= eps/(1-eps)
    # (1/19 at eps = 0.05); a singleton at log(delta) is the whole residual
    thr = 0.05 / 0.95
    lb = float(np.float32(math.log(thr * scale)))
    t = _table([[0.0, 0.0], [lb, 0.0]])
    ix = wl.index_from_assignment(t, np.array([0, 1]))
    out = be.step(t, ix, np.array([1.0, 0.0]), T.DecodeConfig(k=1, epsilon=0.05, targets=("topp",), k_max=2))
    delta = math.exp(lb)
    if certified:
        assert out["kind"] == "topp_mass" and out["opened"] == 1
        assert out["eps"] == pytest.approx(delta / (1 + delta), rel=1e-12)
    else:  # opens the singleton; nothing left unopened: delta = 0
        assert out["kind"] == "topp_mass" and out["opened"] == 2 and out["eps"] == 0.0


def test_single_cluster_opens_everything(be):
    # reference tests/test_decode.py:52-60
    t = wl.synth_vocab(500, 16, 10, 0.05, 3, dtype="f64")
    ix = wl.index_from_assignment(t, np.zeros(500, dtype=np.int64))
    out = be.step(t, ix, unit_queries(1, 16, 0)[0], T.DecodeConfig(k=5, k_max=500))
    assert out["sub"] == 500 and out["fb"] is None and out["rho"] == 0.0 and out["pops"] == 1


def test_dominant_cluster_single_pop(be):
    # reference tests/test_decode.py:63-83
    rng = np.random.default_rng(3)
    a = np.zeros((30, 4)) + [10.0, 0, 0, 0] + 0.05 * rng.standard_normal((30, 4))
    b = np.zeros((30, 4)) + [-10.0, 0, 0, 0] + 0.05 * rng.standard_normal((30, 4))
    t = T.EmbeddingTable(weights=np.vstack([a, b]).astype(np.float32).astype(np.float64), bias=np.zeros(60))
    ix = wl.index_from_assignment(t, np.repeat([0, 1], 30))
    h = np.array([1.0, 0.0, 0.0, 0.0])
    cfg = T.DecodeConfig(k=1, targets=("topk",), k_max=60)
    logits, order = be.dense(t, h)
    out = be.step(t, ix, h, cfg)
    assert out["kind"] == "topk_exact" and out["pops"] == 1 and out["opened"] == 1
    assert out["ids"][np.argmax(out["logits"])] == order[0]
    bat = be.step(t, ix, h, cfg, batchselect=True)
    assert bat["kind"] == "topk_exact" and bat["ids"][np.argmax(bat["logits"])] == order[0]


def test_dense_tie_order(be):
    # reference tests/test_oracle.py:43-46: (logit desc, id asc)
    t = T.EmbeddingTable(weights=np.zeros((4, 2)), bias=np.array([1.0, 2.0, 2.0, 0.0]))
    _, order = be.dense(t, np.zeros(2))
    assert list(order) == [1, 2, 0, 3]


def test_tied_bounds_open_by_id(be):
    # constructed ties: clusters with identical rows have identical bounds, so
    # the opening order falls back to the cluster id (np.lexsort((ids, -U)),
    # decode.py:166).  Every backend must match the oracle's sequence exactly.
    rng = np.random.default_rng(5)
    base = rng.standard_normal((8, 32)).astype(np.float32).astype(np.float64)
    rows = np.vstack([base, base, base[:4], rng.standard_normal((20, 32)).astype(np.float32)])
    t = T.EmbeddingTable(weights=rows, bias=np.zeros(rows.shape[0]))
    assign = np.concatenate([np.repeat([0, 1], 8), np.full(4, 2), 3 + np.arange(20) // 5])
    ix = wl.index_from_assignment(t, assign)
    for h in unit_queries(6, 32, 11):
        u = be.bounds(ix, h)
        want = Oracle().step(t, ix, h, T.DecodeConfig(k=3, k_max=rows.shape[0]))
        got = be.step(t, ix, h, T.DecodeConfig(k=3, k_max=rows.shape[0]))
        assert np.array_equal(got["ids"], want["ids"]) and np.array_equal(got["logits"], want["logits"])
        assert got["kind"] == want["kind"] and got["opened"] == want["opened"] and got["u_max"] == want["u_max"]
        assert np.array_equal(u, O.cluster_bounds(ix, h).values)
