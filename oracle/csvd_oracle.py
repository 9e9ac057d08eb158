"""ORACLE -- TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference CSV-Decode output-layer hot path
(`/root/reference/pkg/src/csvd/`), used as the parity checker by `tests/`,
by `__graft_entry__.smoke()` and as the `cpu_baseline` / `--impl reference`
arm of `bench.py`.  The product package (`paper_2511_21702_b200`) never
imports this module; its CUDA path fails loudly when its extension is absent.

Parity pinning: this restatement is checked bit-for-bit against outputs of
the reference itself (imported from /root/reference in the build container)
by `tests/golden/make_golden.py` -> `tests/golden/*.npz`, and against the
reference's own known-answer tests (restated in tests/test_kat.py, run on the oracle and the GPU).

Arithmetic is numpy float64 in the reference's order; the row reductions go
through the C restatement in `oracle/pairwise.c` (multi-threaded, bit-equal to
numpy's pairwise add-reduce) when `oracle/_build/libcsvd_oracle.so` is built,
otherwise through numpy itself (identical bits, slower).

Inputs are duck-typed: any object with the reference's field names works --
the reference's own EmbeddingTable / ClusterIndex / DecodeConfig, or the
product's mirrors of them.  W may be held as float64 (reference), float32 or
bf16 bit patterns (uint16); all are f32-exact so the arithmetic is unchanged.
"""

from __future__ import annotations

import ctypes
import hashlib
import math
import os
import struct
from dataclasses import dataclass, field

import numpy as np

NEG_INF = float("-inf")
_RECOMPUTE_EVERY = 64  # certify.py:31
_F32_EPS = float(np.finfo(np.float32).eps)  # bounds.py:42
_THETA_PAD = 4e-12  # bounds.py:92

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _lib():
    """Load the C restatement (oracle/_build/libcsvd_oracle.so) if built."""
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "_build", "libcsvd_oracle.so")
        if os.path.exists(path):
            lib = ctypes.CDLL(path)
            lib.oracle_gemv_rows.restype = None
            lib.oracle_gemv_rows.argtypes = [
                ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                ctypes.c_void_p, ctypes.c_int,
            ]
            lib.oracle_l2_norm.restype = ctypes.c_double
            lib.oracle_l2_norm.argtypes = [ctypes.c_void_p, ctypes.c_int64]
            lib.oracle_sum.restype = ctypes.c_double
            lib.oracle_sum.argtypes = [ctypes.c_void_p, ctypes.c_int64]
            _LIB = lib
        else:
            _LIB = False
    return _LIB or None


_THREADS = int(os.environ.get("CSVD_ORACLE_THREADS", "0"))


def set_threads(n: int) -> None:
    global _THREADS
    _THREADS = int(n)


def _dtype_code(a: np.ndarray) -> int:
    if a.dtype == np.float32:
        return 0
    if a.dtype == np.uint16:
        return 1
    if a.dtype == np.float64:
        return 2
    raise TypeError(f"unsupported row dtype {a.dtype}")


def _widen(a: np.ndarray) -> np.ndarray:
    """Exact widening of stored rows to float64 (bf16 bits -> f32 -> f64)."""
    if a.dtype == np.uint16:
        return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return np.asarray(a, dtype=np.float64)


# ---------------------------------------------------------------------------
# L0: fixed-order numerics  (_linalg.py)
# ---------------------------------------------------------------------------

def gemv_rows(rows: np.ndarray, h: np.ndarray, sel=None, bias=None) -> np.ndarray:
    """`(rows[sel] * h).sum(axis=1) (+ bias[sel])`  -- _linalg.py:25-37, decode.py:171.

    Bit-equal whichever engine runs it (C restatement or numpy)."""
    rows = np.ascontiguousarray(rows)
    if rows.ndim == 1:
        rows = rows[None, :]
    h = np.ascontiguousarray(h, dtype=np.float64)
    if rows.shape[1] != h.shape[0]:
        raise ValueError(f"dimension mismatch: rows d={rows.shape[1]}, h d={h.shape[0]}")
    n = rows.shape[0] if sel is None else len(sel)
    lib = _lib()
    if lib is not None:
        out = np.empty(n, dtype=np.float64)
        sel_a = None if sel is None else np.ascontiguousarray(sel, dtype=np.int64)
        bias_a = None if bias is None else np.ascontiguousarray(bias)
        lib.oracle_gemv_rows(
            rows.ctypes.data, _dtype_code(rows), n, rows.shape[1],
            None if sel_a is None else sel_a.ctypes.data, h.ctypes.data,
            None if bias_a is None else bias_a.ctypes.data,
            0 if bias_a is None else _dtype_code(bias_a),
            out.ctypes.data, _THREADS,
        )
        return out
    r = _widen(rows if sel is None else rows[np.asarray(sel)])
    out = (r * h).sum(axis=1)
    if bias is not None:
        b = _widen(np.asarray(bias))
        out = out + (b if sel is None else b[np.asarray(sel)])
    return out


def l2_norm(v: np.ndarray) -> float:
    """sqrt((v*v).sum())  -- _linalg.py:40-43."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    return float(np.sqrt((v * v).sum()))


def logsumexp(values: np.ndarray) -> float:
    """Max-shifted logsumexp, -inf for empty  -- _linalg.py:46-60."""
    values = np.asarray(values, dtype=np.float64)
    if values.size == 0:
        return NEG_INF
    m = float(values.max())
    if m == NEG_INF:
        return NEG_INF
    if np.isposinf(m):
        return float("inf")
    return m + float(np.log(np.exp(values - m).sum()))


# ---------------------------------------------------------------------------
# fingerprint  (tensor_io.py:219-226)
# ---------------------------------------------------------------------------

def table_fingerprint(weights: np.ndarray, bias: np.ndarray) -> bytes:
    h = hashlib.sha256()
    h.update(b"CSVD")
    h.update(struct.pack("<QQ", weights.shape[0], weights.shape[1]))
    h.update(_widen(weights).astype("<f4").tobytes() if weights.dtype != np.float32
             else weights.astype("<f4").tobytes())
    h.update(np.asarray(bias).astype("<f4").tobytes())
    return h.digest()


# ---------------------------------------------------------------------------
# L2: bounds  (bounds.py)
# ---------------------------------------------------------------------------

@dataclass
class OBounds:
    values: np.ndarray
    mode: str
    query_norm: float
    slack: float


def _augment_query(index, h):
    """bounds.py:67-76."""
    h = np.ascontiguousarray(h, dtype=np.float64)
    if index.mode == "bias_augmented":
        if h.shape == (index.hidden_dim,):
            h = np.concatenate([h, [1.0]])
        elif h.shape != (index.hidden_dim + 1,):
            raise ValueError(f"query must have length {index.hidden_dim}")
    elif h.shape != (index.hidden_dim,):
        raise ValueError(f"query must have length {index.hidden_dim}")
    return h


def _slack_for(values, slack_mode):
    """bounds.py:58-64."""
    if slack_mode == "none":
        return 0.0
    if slack_mode == "f32":
        return 4.0 * _F32_EPS * float(np.abs(values).max(initial=1.0))
    raise ValueError(f"unknown slack mode {slack_mode!r}")


def _euclidean_raw(index, h, qn, sel):
    """bounds.py:79-83: (<mu,h> + R*||h||) + maxb, each op rounded in order."""
    raw = gemv_rows(index.centroids[sel], h) + index.radii[sel] * qn
    if index.mode == "euclidean":
        raw = raw + index.max_biases[sel]
    return raw


def _cone_raw(index, h, qn, sel):
    """bounds.py:95-118 (spherical cone bound)."""
    cnorms = index.centroid_norms[sel]
    radii = index.radii[sel]
    angulars = index.angulars[sel]
    max_norms = index.max_norms[sel]
    min_norms = index.min_norms[sel]
    dots = gemv_rows(index.centroids[sel], h)
    geom = np.empty(dots.shape[0])
    nz = cnorms > 0
    exact = nz & (radii == 0.0)
    cone = nz & ~exact
    if qn > 0:
        cos_phi = np.clip(dots[cone] / (cnorms[cone] * qn), -1.0, 1.0)
        gamma = np.cos(np.maximum(0.0, np.arccos(cos_phi) - (angulars[cone] + _THETA_PAD)))
        geom[cone] = qn * np.maximum(max_norms[cone] * gamma, min_norms[cone] * gamma)
    else:
        geom[cone] = 0.0
    geom[exact] = dots[exact]
    geom[~nz] = radii[~nz] * qn
    return geom + index.max_biases[sel]


def raw_bounds_subset(index, h, qn, cluster_ids):
    """bounds.py:121-128."""
    h = _augment_query(index, h)
    if index.mode == "spherical":
        return _cone_raw(index, h, qn, cluster_ids)
    return _euclidean_raw(index, h, qn, cluster_ids)


def cluster_bounds(index, h, query_norm=None, slack_mode="none") -> OBounds:
    """bounds.py:131-184 (euclidean / bias_augmented / spherical-cone)."""
    h = _augment_query(index, h)
    if query_norm is None:
        query_norm = l2_norm(h)
    sel = slice(None)
    raw = _cone_raw(index, h, query_norm, sel) if index.mode == "spherical" else \
        _euclidean_raw(index, h, query_norm, sel)
    eta = _slack_for(raw, slack_mode)
    vals = raw + eta
    if not np.isfinite(vals).all():  # BoundVector.__post_init__, bounds.py:53-55
        raise ValueError("bounds must be finite")
    return OBounds(values=vals, mode=index.mode, query_norm=query_norm, slack=eta)


# ---------------------------------------------------------------------------
# L3/L4: certificates + engine  (certify.py, decode.py)
# ---------------------------------------------------------------------------

@dataclass
class OStatus:
    kind: str
    epsilon_achieved: float
    u_max: float
    topk_min: float


@dataclass
class OOutcome:
    token_ids: np.ndarray
    logits: np.ndarray
    status: OStatus
    fallback_used: str | None
    stats: dict
    opened: list = field(default_factory=list)  # cluster ids in opening order
    bounds: np.ndarray | None = None
    order: np.ndarray | None = None


def _fallback_name(lv) -> str:
    name = getattr(lv, "name", None)
    if name is None:
        raise ValueError(f"unknown fallback level {lv!r}")
    return name


class _Ctx:
    """Restates decode._StepContext (decode.py:147-265) + certify.CertState
    (certify.py:56-111)."""

    def __init__(self, table, index, h, cfg, k_max, bounds=None):
        self.W = table.weights
        self.b = table.bias
        self.index = index
        self.h = np.ascontiguousarray(h, dtype=np.float64)
        self.cfg = cfg
        self.k_max = k_max
        self.bounds = bounds if bounds is not None else cluster_bounds(
            index, self.h, slack_mode=getattr(cfg, "slack_mode", "none"))
        C = index.n_clusters
        self.C = C
        self.V = index.vocab_size
        self.opened_mask = np.zeros(C, dtype=bool)
        self.opened: list = []
        self._ids: list = []
        self._logits: list = []
        self.token_ids = np.empty(0, dtype=np.int64)
        self.logits = np.empty(0, dtype=np.float64)
        self.log_z = NEG_INF
        self._merges = 0
        self.log_sizes = np.log(index.sizes)  # certify.py:119 np.log(sizes[...])
        self.log_rhat = self._residual()
        self.heap_pops = 0
        self.order = np.lexsort((np.arange(C), -self.bounds.values))  # decode.py:166
        self.cursor = 0

    # certify.residual_log_rhat, certify.py:114-119
    def _residual(self):
        un = ~self.opened_mask
        if not un.any():
            return NEG_INF
        return logsumexp(self.log_sizes[un] + self.bounds.values[un])

    # decode.open_cluster, decode.py:169-176 + CertState.merge_cluster certify.py:73-83
    def open_cluster(self, c):
        idx = self.index
        s, e = int(idx.starts[c]), int(idx.ends[c])
        members = idx.perm[s:e]
        logits = gemv_rows(self.W, self.h, sel=members, bias=self.b)
        self.opened.append(int(c))
        self._ids.append(np.asarray(members, dtype=np.int64))
        self._logits.append(logits)
        self.token_ids = np.concatenate(self._ids)
        self.logits = np.concatenate(self._logits)
        self._merges += 1
        if self._merges % _RECOMPUTE_EVERY == 0:
            self.log_z = logsumexp(self.logits)
        else:
            self.log_z = float(np.logaddexp(self.log_z, logsumexp(logits)))
        self.opened_mask[c] = True
        self.log_rhat = self._residual()

    def open_next_by_bound(self):  # decode.py:178-185
        while self.cursor < self.C:
            c = int(self.order[self.cursor])
            self.cursor += 1
            if not self.opened_mask[c]:
                self.open_cluster(c)
                return True
        return False

    def n(self):
        return self.token_ids.size

    def topk_min(self, k=None):  # certify.py:85-88
        k = self.cfg.k if k is None else k
        n = self.n()
        if n < k:
            return NEG_INF
        return float(np.partition(self.logits, n - k)[n - k])

    def rho(self):  # certify.py:93-99
        if self.log_rhat == NEG_INF:
            return 0.0
        if self.log_z == NEG_INF:
            return 1.0
        return 1.0 / (1.0 + math.exp(self.log_z - self.log_rhat))

    def delta(self):  # certify.py:101-107
        if self.log_rhat == NEG_INF:
            return 0.0
        if self.log_z == NEG_INF:
            return math.inf
        return math.exp(self.log_rhat - self.log_z)

    def u_max_unopened(self):  # decode.py:187-190
        if self.opened_mask.all():
            return NEG_INF
        return float(self.bounds.values[~self.opened_mask].max())

    def topk_decision(self):  # certify.topk_certified, certify.py:128-139
        k = self.cfg.k
        if self.n() < k:
            return False, NEG_INF, NEG_INF
        kth = self.topk_min()
        if self.opened_mask.all():
            return True, NEG_INF, kth
        u_max = self.u_max_unopened()
        return u_max < kth, u_max, kth

    def softmax_decision(self, eps):  # certify.py:147-153
        if not 0 < eps < 1:
            raise ValueError(f"epsilon must lie in (0, 1), got {eps}")
        if self.n() == 0:
            return False, 1.0
        r = self.rho()
        return r <= eps, r

    def topp_decision(self, eps):  # certify.py:156-164
        if not 0 < eps < 1:
            raise ValueError(f"epsilon must lie in (0, 1), got {eps}")
        if self.n() == 0:
            return False, 1.0
        dl = self.delta()
        mass = dl / (1.0 + dl) if math.isfinite(dl) else 1.0
        return dl <= eps / (1.0 - eps), mass

    def check_targets(self, eps):  # decode.py:192-210
        for t in self.cfg.targets:
            if t == "topk":
                ok, u, kth = self.topk_decision()
                if ok:
                    return OStatus("topk_exact", 0.0, u, kth)
            elif t == "softmax_eps":
                ok, r = self.softmax_decision(eps)
                if ok:
                    return OStatus("softmax_eps", r, self.u_max_unopened(), self.topk_min())
            elif t == "topp":
                ok, r = self.topp_decision(eps)
                if ok:
                    return OStatus("topp_mass", r, self.u_max_unopened(), self.topk_min())
        return None

    def bounds_dim(self):
        return self.index.hidden_dim + (1 if self.index.mode == "bias_augmented" else 0)

    def tightness(self):  # certify.py:172-184
        if self.n() < 2 or self.opened_mask.all():
            return math.nan
        lo = float(self.logits.min())
        hi = float(self.logits.max())
        u = self.u_max_unopened()
        if u <= lo:
            return 1.0
        return (hi - lo) / (u - lo)

    def outcome(self, status, fb):  # decode.py:212-237
        n = self.n()
        stats = dict(
            sub_size=n, ratio=n / self.V, clusters_opened=len(self.opened),
            xi=self.tightness(), cert_kind=status.kind, fallback=fb, rho=self.rho(),
            flops_sparse=2 * n * self.index.hidden_dim,
            flops_bounds=2 * self.C * self.bounds_dim(), heap_pops=self.heap_pops,
        )
        return OOutcome(self.token_ids, self.logits, status, fb, stats, list(self.opened),
                        self.bounds.values, self.order)

    def full_vocab_outcome(self):  # decode.py:239-262
        V = self.V
        logits = gemv_rows(self.W, self.h, bias=self.b)
        k = self.cfg.k
        kth = float(np.partition(logits, V - k)[V - k])
        status = OStatus("topk_exact", 0.0, NEG_INF, kth)
        stats = dict(
            sub_size=V, ratio=1.0, clusters_opened=self.C, xi=math.nan,
            cert_kind=status.kind, fallback="full_vocab", rho=0.0,
            flops_sparse=2 * V * self.index.hidden_dim,
            flops_bounds=2 * self.C * self.bounds_dim(), heap_pops=self.heap_pops,
        )
        return OOutcome(np.arange(V, dtype=np.int64), logits, status, "full_vocab", stats,
                        list(self.opened), self.bounds.values, self.order)


def _apply_fallback(level, ctx):  # decode.py:268-298
    name = _fallback_name(level)
    if name == "partial_expand":
        for _ in range(level.delta_c):
            if not ctx.open_next_by_bound():
                break
        st = ctx.check_targets(ctx.cfg.epsilon)
        return None if st is None else ctx.outcome(st, "partial_expand")
    if name == "relax_eps":
        relaxed = min(ctx.cfg.epsilon * level.factor, 1.0 - 1e-12)
        for t in ctx.cfg.targets:
            if t == "softmax_eps":
                ok, r = ctx.softmax_decision(relaxed)
                if ok:
                    return ctx.outcome(OStatus("softmax_eps", r, ctx.u_max_unopened(),
                                               ctx.topk_min()), "relax_eps")
            elif t == "topp":
                ok, r = ctx.topp_decision(relaxed)
                if ok:
                    return ctx.outcome(OStatus("topp_mass", r, ctx.u_max_unopened(),
                                               ctx.topk_min()), "relax_eps")
        return None
    if name == "full_vocab":
        return ctx.full_vocab_outcome()
    raise ValueError(f"unknown fallback level {level!r}")


def _run_fallback_chain(ctx):  # decode.py:301-309
    levels = list(ctx.cfg.fallback)
    if not any(_fallback_name(lv) == "full_vocab" for lv in levels):
        levels.append(_FV)
    for lv in levels:
        out = _apply_fallback(lv, ctx)
        if out is not None:
            return out
    raise AssertionError("full_vocab level is total")


class _FullVocabLevel:
    name = "full_vocab"


_FV = _FullVocabLevel()


def resolved_k_max(cfg, V):  # decode.py:99-102
    return max(cfg.k, V // 2) if cfg.k_max is None else cfg.k_max


def validate_cfg(cfg, V):  # decode.py:104-115 (raises ValueError subclasses)
    kinds = ("topk", "softmax_eps", "topp")
    if not cfg.targets or any(t not in kinds for t in cfg.targets):
        raise ValueError(f"targets must be a non-empty subset of {kinds}")
    if not 1 <= cfg.k <= V:
        raise ValueError(f"need 1 <= k <= V, got k={cfg.k}, V={V}")
    km = resolved_k_max(cfg, V)
    if not cfg.k <= km <= V:
        raise ValueError(f"need k <= K_max <= V, got K_max={km}")
    if not 0 < cfg.epsilon < 1:
        raise ValueError(f"epsilon must lie in (0, 1), got {cfg.epsilon}")


def decode_step(table, index, h, cfg, k_max=None, check_fingerprint=False):
    """decode.py:312-343 -- incremental heap-ordered opening.

    The reference re-hashes the whole table every step (decode.py:324 ->
    tensor_io.py:219-226); pass check_fingerprint=True to restate that cost.
    """
    if check_fingerprint and index.fingerprint != table_fingerprint(table.weights, table.bias):
        raise ValueError("index fingerprint does not match table")
    validate_cfg(cfg, index.vocab_size)
    k_max = resolved_k_max(cfg, index.vocab_size) if k_max is None else k_max
    ctx = _Ctx(table, index, h, cfg, k_max)
    # heap pop order == lexsort order (same key, same tie-break; decode.py:329-340)
    while True:
        if ctx.n() > 0:
            st = ctx.check_targets(cfg.epsilon)
            if st is not None:
                return ctx.outcome(st, None)
        if ctx.cursor >= ctx.C:
            raise AssertionError("heap exhausted without certification")
        c = int(ctx.order[ctx.cursor])
        ctx.heap_pops += 1
        ctx.cursor += 1
        ctx.open_cluster(c)
        if ctx.n() > k_max:
            return _run_fallback_chain(ctx)


def select_by_bound(order, sizes, k_max):  # decode.py:346-359
    selected, total = [], 0
    for c in order:
        c = int(c)
        size = int(sizes[c])
        if selected and total + size > k_max:
            break
        selected.append(c)
        total += size
        if total >= k_max:
            break
    return selected


def decode_step_batchselect(table, index, h, cfg, k_max=None, bounds=None):
    """decode.py:362-382 -- one-shot select-under-budget, verify once."""
    validate_cfg(cfg, index.vocab_size)
    k_max = resolved_k_max(cfg, index.vocab_size) if k_max is None else k_max
    ctx = _Ctx(table, index, h, cfg, k_max, bounds=bounds)
    selected = select_by_bound(ctx.order, index.sizes, k_max)
    ctx.cursor = len(selected)
    for c in selected:
        ctx.open_cluster(c)
    st = ctx.check_targets(cfg.epsilon)
    if st is not None:
        return ctx.outcome(st, None)
    return _run_fallback_chain(ctx)


def sharded_decode_step(table, index, assignment, n_workers, h, cfg, k_max=None,
                        flops_per_unit=1.0, bytes_per_unit=1.0):
    """shard_sim.py:134-208: per-worker bounds, global select, verify, ledger."""
    validate_cfg(cfg, index.vocab_size)
    k_max = resolved_k_max(cfg, index.vocab_size) if k_max is None else k_max
    h = np.ascontiguousarray(h, dtype=np.float64)
    d, C, N = index.hidden_dim, index.n_clusters, n_workers
    qn = l2_norm(h if index.mode != "bias_augmented" else np.concatenate([h, [1.0]]))
    bdim = d + (1 if index.mode == "bias_augmented" else 0)
    raw = np.empty(C)
    bound_flops = np.zeros(N)
    assignment = np.asarray(assignment)
    for g in range(N):
        mine = np.flatnonzero(assignment == g)
        if mine.size:
            raw[mine] = raw_bounds_subset(index, h, qn, mine)
        bound_flops[g] = 2 * mine.size * bdim
    eta = _slack_for(raw, getattr(cfg, "slack_mode", "none"))
    bounds = OBounds(raw + eta, index.mode, qn, eta)
    out = decode_step_batchselect(table, index, h, cfg, k_max, bounds=bounds)
    loads = np.zeros(N, dtype=np.int64)
    np.add.at(loads, assignment, index.sizes)
    if out.fallback_used == "full_vocab":
        tpw = loads.astype(np.float64)
    else:
        tpw = np.zeros(N)
        for c in out.opened:
            tpw[assignment[c]] += index.sizes[c]
    sparse_flops = 2 * tpw * d
    ex = N >= 2
    bb = C * 4 if ex else 0
    bl = out.stats["sub_size"] * (d * 2 + 4) if ex else 0
    tb, tl = bb / bytes_per_unit, bl / bytes_per_unit
    ph = {"bounds": float(bound_flops.max()) / flops_per_unit + tb,
          "logits": float(sparse_flops.max()) / flops_per_unit + tl, "verify": 0.0}
    tot = sum(ph.values())
    ledger = dict(bytes_bounds_phase=bb, bytes_logits_phase=bl, phase_latencies=ph,
                  omega_comm=(tb + tl) / tot if tot > 0 else 0.0)
    return out, ledger


# ---------------------------------------------------------------------------
# oracle.py
# ---------------------------------------------------------------------------

def dense_logits(table, h):
    """oracle.py:33-41: all logits, softmax, (logit desc, id asc) order."""
    h = np.asarray(h, dtype=np.float64)
    logits = gemv_rows(table.weights, h, bias=table.bias)
    lse = logsumexp(logits)
    probs = np.exp(logits - lse)
    order = np.lexsort((np.arange(logits.size), -logits))
    return logits, probs, order
