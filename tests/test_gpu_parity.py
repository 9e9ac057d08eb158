"""GPU parity: the CUDA path through the C ABI vs the reference's own outputs
(golden fixtures) and vs the oracle at larger sizes.

Bar (BASELINE north star + SURVEY §8c): token ids (as a sequence), logits
(f64 bit patterns), certificate kind, fallback level, clusters opened,
heap pops, u_max, k-th logit, xi and the bound vector are bit-exact;
rho / epsilon_achieved within 1e-12 relative (transcendentals, ~1 ulp).
"""

import numpy as np
import pytest

import csvd_oracle as O
from conftest import TRANS_RTOL, GoldenCase, assert_outcome, close, golden_names, has_gpu
import paper_2511_21702_b200 as P
from paper_2511_21702_b200 import workload as wl

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a GPU")]


@pytest.mark.parametrize("name", golden_names())
def test_decode_matches_reference_goldens(name):
    case = GoldenCase(name)
    T, ix = case.table, case.index
    for st in case.steps():
        fn = P.decode_step if st["variant"] == "incremental" else P.decode_step_batchselect
        out = fn(T, ix, st["h"], st["cfg"], k_max=st["k_max"])
        assert_outcome(out, case.expected(st["i"]), rtol=TRANS_RTOL, where=f"{name}[{st['i']}]",
                       exact_bounds=ix.mode != "spherical")


@pytest.mark.parametrize("name", golden_names())
def test_bounds_match_reference_goldens(name):
    case = GoldenCase(name)
    ix = case.index
    seen = set()
    for st in case.steps():
        key = (int(np.flatnonzero((case.z["queries"] == st["h"]).all(axis=1))[0]), st["cfg"].slack_mode)
        if key in seen:
            continue
        seen.add(key)
        exp = case.expected(st["i"])
        b = P.cluster_bounds(ix, st["h"], slack_mode=st["cfg"].slack_mode)
        if ix.mode == "spherical":  # acos/cos: ulp-level libm differences
            np.testing.assert_allclose(b.values, exp["U"], rtol=1e-12, atol=0)
        else:
            assert np.array_equal(b.values, exp["U"]), f"{name}: bounds not bit-equal"
        assert b.query_norm == exp["qn"]
        if ix.mode == "spherical":
            assert abs(b.slack - exp["slack"]) <= 1e-12 * abs(exp["slack"])
        else:
            assert b.slack == exp["slack"]


@pytest.mark.parametrize("name", golden_names())
def test_dense_matches_reference_goldens(name):
    case = GoldenCase(name)
    for i, ref in enumerate(case.z["dense"]):
        r = P.dense_logits(case.table, case.z["queries"][i])
        assert np.array_equal(r.logits, ref)


def _c1_like(V=32000, d=4096, n_modes=128, g=2, dtype="f32"):
    T = wl.synth_vocab(V, d, n_modes, 0.3, 1, dtype=dtype)
    ix = wl.fast_index(T, n_modes, g)
    return T, ix


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_c1_shape_vs_oracle(dtype):
    """c1 shape (V=32000, d=4096, C=256): GPU vs oracle, mixed workloads."""
    T, ix = _c1_like(dtype=dtype)
    q = np.vstack([wl.generate_queries(6, 4096, "contextual", 7, centroids=ix.centroids),
                   wl.generate_queries(2, 4096, "random", 8)])
    cfgs = [P.DecodeConfig(k=10), P.DecodeConfig(k=10, epsilon=1e-3, targets=("softmax_eps",)),
            P.DecodeConfig(k=10, k_max=600)]
    for ci, cfg in enumerate(cfgs):
        for i, h in enumerate(q):
            exp = O.decode_step(T, ix, h, cfg)
            got = P.decode_step(T, ix, h, cfg)
            e = _fields(exp)
            assert_outcome(got, e, rtol=TRANS_RTOL, where=f"c1[{dtype},{ci},{i}]")


def _fields(o):
    st = o.stats
    return dict(ids=o.token_ids, logits=o.logits, kind=o.status.kind, fallback=o.fallback_used,
                sub_size=st["sub_size"], clusters_opened=st["clusters_opened"], heap_pops=st["heap_pops"],
                flops_sparse=st["flops_sparse"], flops_bounds=st["flops_bounds"], eps=o.status.epsilon_achieved,
                u_max=o.status.u_max, topk_min=o.status.topk_min, rho=st["rho"], xi=st["xi"], ratio=st["ratio"])


def test_many_clusters_64_merge_recompute():
    """g=80 clusters per mode: certification needs > 64 opens, crossing the
    full log_z recompute every 64th merge (certify.py:79-83)."""
    T = wl.synth_vocab(20000, 512, 4, 0.05, 1)
    ix = wl.fast_index(T, 4, 80)
    q = wl.generate_queries(4, 512, "contextual", 7, centroids=ix.centroids)
    for cfg in (P.DecodeConfig(k=10), P.DecodeConfig(k=5, epsilon=1e-2, targets=("softmax_eps",))):
        for i, h in enumerate(q):
            exp = O.decode_step(T, ix, h, cfg)
            got = P.decode_step(T, ix, h, cfg)
            assert exp.stats["clusters_opened"] >= 1
            assert_outcome(got, _fields(exp), rtol=1e-11, where=f"g80[{i}]")


def test_errors_mirror_reference():
    T, ix = _c1_like(V=2000, d=512, n_modes=20, g=1)
    h = wl.generate_queries(1, 512, "random", 1)[0]
    with pytest.raises(P.ConfigError):
        P.decode_step(T, ix, h, P.DecodeConfig(k=0))
    with pytest.raises(P.ConfigError):
        P.decode_step(T, ix, h, P.DecodeConfig(epsilon=1.5))
    with pytest.raises(ValueError):
        P.decode_step(T, ix, h[:10], P.DecodeConfig())
    bad = wl.index_from_assignment(T, np.arange(2000) % 20)
    bad.fingerprint = b"x" * 32
    with pytest.raises(P.ConfigError):
        P.decode_step(T, bad, h, P.DecodeConfig())


def test_head_fast_path_and_general_path_agree():
    """The kernel orders clusters two ways: the head fast path (only clusters
    whose bound beats the best-logit estimate, sorted by one warp) and the full
    block sort.  first_wave_tokens > 0 forces the full sort.  Both must equal
    the oracle, including steps where the head is exhausted (partial expand
    past it, tight budgets) and where it is too large (random queries)."""
    from paper_2511_21702_b200 import _lib
    T, ix = _c1_like(V=32000, d=4096, n_modes=64, g=4)
    q = np.vstack([wl.generate_queries(4, 4096, "contextual", 7, centroids=ix.centroids),
                   wl.generate_queries(2, 4096, "random", 8)])
    ctx = P.prepare(T, ix)
    cfgs = [P.DecodeConfig(k=10), P.DecodeConfig(k=10, k_max=300), P.DecodeConfig(k=3, k_max=150),
            P.DecodeConfig(k=16)]
    for ci, cfg in enumerate(cfgs):
        for i, h in enumerate(q):
            e = _fields(O.decode_step(T, ix, h, cfg))
            for fwt in (0, 1):
                c = ctx.make_config(cfg, first_wave_tokens=fwt)
                assert c.variant == _lib.VARIANT_INCREMENTAL
                got = ctx.step(h, c)
                assert_outcome(got, e, rtol=TRANS_RTOL, where=f"head[{ci},{i},fwt={fwt}]")


def test_budgeted_decoder_sequence_matches_oracle():
    """The adaptive budget in front of the step (decode.py:404-431): the same
    controller trajectory and outcomes as the oracle run with the controller's
    k_max, over a query stream that mixes certified steps and fallbacks."""
    T, ix = _c1_like(V=32000, d=4096, n_modes=64, g=4)
    q = np.vstack([wl.generate_queries(10, 4096, "contextual", 7, centroids=ix.centroids),
                   wl.generate_queries(3, 4096, "random", 8)])
    cfg = P.DecodeConfig(k=10, adaptive_enabled=True, alpha=0.5, rho_target=0.05, ema_half_life=3.0,
                         warmup_steps=2)
    dec = P.BudgetedDecoder(T, ix, cfg, initial_k_max=700)
    ctl = P.AdaptiveBudget(cfg, ix.vocab_size, 700)
    for t, h in enumerate(q):
        km = ctl.effective_k_max(t)
        exp = O.decode_step(T, ix, h, cfg, k_max=km)
        got = dec.step(h)
        assert_outcome(got, _fields(exp), rtol=TRANS_RTOL, where=f"budget[{t}] k_max={km}")
        ctl.observe(exp.fallback_used is not None)
        assert dec.ctl.k_max == ctl.k_max


def test_files_to_device_step(tmp_path):
    """CSVD + CSVI files -> mapped table + index -> resident context -> step."""
    from paper_2511_21702_b200 import formats as F
    T, ix = _c1_like(V=8000, d=512, n_modes=40, g=2)
    F.save_table(T, tmp_path / "t.csvd")
    F.save_index(ix, tmp_path / "i.csvi")
    T2, ix2, ctx = F.prepare_files(tmp_path / "t.csvd", tmp_path / "i.csvi")
    q = wl.generate_queries(3, 512, "contextual", 7, centroids=ix.centroids)
    cfg = P.DecodeConfig(k=10)
    for i, h in enumerate(q):
        assert_outcome(P.decode_step(T2, ix2, h, cfg), _fields(O.decode_step(T, ix, h, cfg)), rtol=TRANS_RTOL,
                       where=f"files[{i}]")


@pytest.mark.parametrize("mode", ["euclidean", "spherical"])
def test_refined_bias_bound_matches_oracle_and_reference_rules(mode):
    """refined_bias_bound (bounds.py:187-220): no exclusion gives the plain bound,
    excluding the top tabled token gives geom + the second tabled bias, and
    excluding every tabled token falls back to the exact remaining max (with
    `bias`) or the m-th tabled value (without)."""
    T = wl.synth_vocab(3000, 64, 12, 0.4, 3)
    ix = wl.fast_index(T, 12, 2, mode=mode)
    h = wl.generate_queries(1, 64, "random", 4)[0]
    U = O.cluster_bounds(ix, h).values
    for c in range(ix.n_clusters):
        meta = ix.clusters[c]
        geom = U[c] - meta.max_bias
        tol = 0.0 if mode == "euclidean" else 1e-12
        assert close(P.refined_bias_bound(ix, c, h, set()), U[c], tol)
        if len(meta.bias_topm) >= 2:
            got = P.refined_bias_bound(ix, c, h, {meta.bias_topm[0][1]})
            assert close(got, geom + meta.bias_topm[1][0], tol)
        tabled = {t for _, t in meta.bias_topm}
        members = [int(t) for t in ix.members(c)]
        if len(members) > len(tabled):
            rest = max(T.bias[t] for t in members if t not in tabled)
            assert close(P.refined_bias_bound(ix, c, h, tabled, bias=T.bias), geom + rest, tol)
            assert close(P.refined_bias_bound(ix, c, h, tabled), geom + meta.bias_topm[-1][0], tol)
        assert P.refined_bias_bound(ix, c, h, set(members)) == float("-inf")


def test_tie_ambiguous_flag():
    """A softmax decision exactly at its threshold (eps = the reference's rho at
    the certifying prefix) is flagged as an ulp-level tie; a clear margin is not."""
    import paper_2511_21702_b200 as P
    from paper_2511_21702_b200 import workload as wl
    T = wl.synth_vocab(20000, 512, 40, 0.3, 1)
    ix = wl.fast_index(T, 40, 4)
    h = wl.generate_queries(1, 512, "contextual", 7, centroids=ix.centroids)[0]
    base = P.DecodeConfig(k=10, epsilon=0.05, targets=("softmax_eps",))
    exp = O.decode_step(T, ix, h, base)
    assert exp.status.kind == "softmax_eps"
    out = P.decode_step(T, ix, h, base)
    assert not out.stats.tie_ambiguous
    tie = P.DecodeConfig(k=10, epsilon=float(exp.stats["rho"]), targets=("softmax_eps",))
    out = P.decode_step(T, ix, h, tie)
    assert out.stats.tie_ambiguous
