"""Caller-side budget control and FLOP accounting around the step.

Restates the reference's host-side helpers that feed `decode_step` its k_max
(§8a row 25):

* `adapt_budget`   one-shot multiplicative update toward the target fallback
                   rate, clamped to [k, V]                       decode.py:385-394
* `warmup_k_max`   widened budget for the first steps of a sequence
                                                                decode.py:397-401
* `AdaptiveBudget` EMA controller with a float-held budget       decode.py:404-431
* `flop_report`, `flop_accounting`  2 FLOPs per multiply-add      decode.py:434-462

`BudgetedDecoder` is the loop a serving caller runs: the controller's
effective k_max per step, the B200 step, then the observed fallback.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .types import resolved_k_max


def _round_half_up(x: float) -> int:
    return int(math.floor(x + 0.5))


def adapt_budget(k_t: int, rho_fall_observed: float, cfg, vocab_size: int) -> int:
    """Budget times (1 + alpha (observed - target)), rounded half up and
    clamped to [k, V]: more budget when fallbacks run hot."""
    proposed = _round_half_up(k_t * (1.0 + cfg.alpha * (rho_fall_observed - cfg.rho_target)))
    return max(cfg.k, min(vocab_size, proposed))


def warmup_k_max(cfg, k_max: int, step: int, vocab_size: int) -> int:
    """k_max x warmup_factor (capped at V) while step < warmup_steps."""
    if step >= cfg.warmup_steps:
        return k_max
    return min(vocab_size, _round_half_up(k_max * cfg.warmup_factor))


class AdaptiveBudget:
    """EMA of the fallback indicator (half-life cfg.ema_half_life steps)
    drives a budget held in floating point, so small drifts accumulate."""

    def __init__(self, cfg, vocab_size: int, initial_k_max: int | None = None):
        self.cfg = cfg
        self.vocab_size = vocab_size
        self._budget = float(resolved_k_max(cfg, vocab_size) if initial_k_max is None else initial_k_max)
        self._decay = 0.5 ** (1.0 / cfg.ema_half_life)
        self.ema = 0.0

    @property
    def k_max(self) -> int:
        return max(self.cfg.k, min(self.vocab_size, _round_half_up(self._budget)))

    def effective_k_max(self, step: int) -> int:
        return warmup_k_max(self.cfg, self.k_max, step, self.vocab_size)

    def observe(self, fallback_fired: bool) -> None:
        self.ema = self._decay * self.ema + (1.0 - self._decay) * (1.0 if fallback_fired else 0.0)
        if not self.cfg.adaptive_enabled:
            return
        b = self._budget * (1.0 + self.cfg.alpha * (self.ema - self.cfg.rho_target))
        self._budget = min(float(self.vocab_size), max(float(self.cfg.k), b))


@dataclass(frozen=True)
class FlopReport:
    flops_bounds: int
    flops_sparse: int
    flops_full: int
    speedup_proxy: float


def flop_report(vocab_size: int, hidden_dim: int, n_clusters: int, sub_size: int,
                bounds_dim: int | None = None) -> FlopReport:
    bd = hidden_dim if bounds_dim is None else bounds_dim
    fb, fs, ff = 2 * n_clusters * bd, 2 * sub_size * hidden_dim, 2 * vocab_size * hidden_dim
    return FlopReport(fb, fs, ff, ff / (fb + fs) if fb + fs else math.inf)


def flop_accounting(outcome, table, index) -> FlopReport:
    bd = index.hidden_dim + (1 if index.mode == "bias_augmented" else 0)
    return flop_report(table.vocab_size, table.hidden_dim, index.n_clusters, outcome.stats.sub_size, bd)


class BudgetedDecoder:
    """A decoding loop with the adaptive budget in front of the B200 step:
    step t runs with k_max = controller.effective_k_max(t), then the
    controller observes whether a fallback fired."""

    def __init__(self, table, index, cfg, initial_k_max: int | None = None):
        from . import engine
        self.table, self.index, self.cfg = table, index, cfg
        self.ctl = AdaptiveBudget(cfg, index.vocab_size, initial_k_max)
        self._ctx = engine.prepare(table, index)
        self.t = 0

    def step(self, h):
        k_max = self.ctl.effective_k_max(self.t)
        out = self._ctx.step(h, self._ctx.make_config(self.cfg, k_max))
        out.stats.step = self.t
        self.ctl.observe(out.fallback_used is not None)
        self.t += 1
        return out
