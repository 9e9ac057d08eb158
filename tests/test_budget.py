"""Caller-side budget control (decode.py:385-462): known answers from the
reference's own tests (tests/test_decode.py:234-276), plus a randomized
comparison against the reference itself when it is importable here."""

import math
import os
import sys

import numpy as np
import pytest

import paper_2511_21702_b200 as P


def test_adapt_budget_known_answers():  # tests/test_decode.py:234-241
    cfg = P.DecodeConfig(k=10, alpha=0.01, rho_target=0.02)
    assert P.adapt_budget(1000, 0.12, cfg, 5000) == 1001
    assert P.adapt_budget(1000, 0.02, cfg, 5000) == 1000
    assert P.adapt_budget(10, 0.0, cfg, 5000) == 10
    assert P.adapt_budget(4999, 1.0, cfg, 5000) == 5000


def test_warmup_known_answers():  # tests/test_decode.py:244-249
    cfg = P.DecodeConfig(k=5, warmup_steps=4, warmup_factor=2.0)
    assert P.warmup_k_max(cfg, 100, 0, 5000) == 200
    assert P.warmup_k_max(cfg, 100, 3, 5000) == 200
    assert P.warmup_k_max(cfg, 100, 4, 5000) == 100
    assert P.warmup_k_max(cfg, 3000, 0, 5000) == 5000


def test_controller_behaviour():  # tests/test_decode.py:252-267
    cfg = P.DecodeConfig(k=5, adaptive_enabled=True, alpha=0.01, rho_target=0.02)
    ctl = P.AdaptiveBudget(cfg, vocab_size=5000, initial_k_max=100)
    assert ctl.k_max == 100
    for _ in range(50):
        ctl.observe(True)
    assert ctl.ema > 0.2 and ctl.k_max > 100
    for _ in range(2000):
        ctl.observe(False)
    assert ctl.ema < 1e-4
    settled = ctl.k_max
    for _ in range(4000):
        ctl.observe(False)
    assert ctl.k_max < settled


def test_flop_report_known_answers():  # tests/test_decode.py:270-276
    r = P.flop_report(50257, 12288, 2000, 9000)
    assert r.flops_full == 2 * 50257 * 12288
    assert abs(r.flops_full - 1.235e9) / 1.235e9 < 1e-3
    assert P.flop_report(5000, 64, 0, 5000).speedup_proxy == 1.0
    assert P.flop_report(10, 4, 0, 0).speedup_proxy == math.inf


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


def test_controller_trajectory_equals_reference():
    csvd = _reference()
    if csvd is None:
        pytest.skip("reference not importable on this host")
    rng = np.random.default_rng(3)
    for alpha, target, hl in ((0.01, 0.02, 100.0), (0.2, 0.1, 7.0)):
        kw = dict(k=5, adaptive_enabled=True, alpha=alpha, rho_target=target, ema_half_life=hl)
        a = P.AdaptiveBudget(P.DecodeConfig(**kw), 5000, 300)
        b = csvd.AdaptiveBudget(csvd.DecodeConfig(**kw), 5000, 300)
        for t in range(3000):
            fired = bool(rng.random() < 0.15)
            a.observe(fired)
            b.observe(fired)
            assert a.k_max == b.k_max and a.effective_k_max(t % 9) == b.effective_k_max(t % 9)
            assert a.ema == b.ema
    for _ in range(2000):
        k_t, obs = int(rng.integers(1, 6000)), float(rng.random())
        cfg = P.DecodeConfig(k=3, alpha=float(rng.random()), rho_target=float(rng.random()) * 0.2)
        rcfg = csvd.DecodeConfig(k=3, alpha=cfg.alpha, rho_target=cfg.rho_target)
        assert P.adapt_budget(k_t, obs, cfg, 5000) == csvd.adapt_budget(k_t, obs, rcfg, 5000)
