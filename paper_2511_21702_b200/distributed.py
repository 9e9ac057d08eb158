"""Vocabulary-sharded decoding: one process per GPU, W sharded by cluster.

Reference: `csvd.shard_sim.sharded_decode_step` (shard_sim.py:134-208), an
in-process simulation of N workers whose outcome must equal the one-shot
`decode_step_batchselect` (decode.py:362-382) bit for bit
(tests/test_acceptance.py:142-161).  Here the workers are real ranks of a
`torch.distributed` group (NCCL over NVLink on the B200 box, gloo in the CPU
tests):

* every rank holds the replicated per-cluster data (centroids, radii, sizes)
  and only its own clusters' W rows (`csvd_create_shard`); it computes all C
  bounds and the global opening order itself, so the batch-select prefix, the
  bound after it and log R-hat are identical everywhere without a collective;
* each rank opens its clusters of the prefix on its GPU and reduces them to a
  merge record (`csvd_shard_open`): LSE, min, max, token count and top-k list;
* ONE all_gather of those records (k + 16 doubles per rank) gives every rank
  the certificate inputs: the k-th logit of S (union of the top-k lists),
  log Z_S (LSE of the LSEs), min/max (tightness), |S|;
* every rank then runs the same certification and fallback chain
  (check_targets decode.py:192-210, _run_fallback_chain decode.py:268-309):
  PartialExpand opens the next clusters with one more open + all_gather,
  RelaxEps is a local re-check, FullVocab runs the shard-local dense GEMV and
  merges top-k lists the same way;
* the outcome's token ids / logits (opening order) are assembled from one
  all_gather of each rank's (position, id, logit) triples.

The merge arithmetic is exact for everything the reference compares
bitwise (ids, logits, k-th logit, bounds, decisions); log Z_S is a
log-sum-exp of per-shard log-sum-exps instead of the reference's streaming
logaddexp chain, so rho / delta agree to ~1e-15 relative (tests use 1e-12).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib
from .types import CertStatus, ConfigError, DecodeOutcome, StepMetrics, resolved_k_max, validate_config

NEG_INF = float("-inf")
SH_TOPK = 16  # CSVD_SH_TOPK (include/csvd_b200.h)
(SH_LSE, SH_MIN, SH_MAX, SH_NTOK, SH_NLIST, SH_P_LO, SH_P_HI, SH_P_SEL, SH_CUM_LO, SH_CUM_HI, SH_U_NEXT,
 SH_LRH_NEXT, SH_QNORM, SH_SLACK) = range(14)


# ---------------------------------------------------------------------------
# rank-local device work (C ABI)
# ---------------------------------------------------------------------------
class DeviceShard:
    """This rank's shard on its GPU: replicated cluster data, owned W rows."""

    def __init__(self, table, index, owned: np.ndarray, device: int = 0):
        from .engine import DeviceIndex
        self.lib = _lib.load()
        self.V, self.d, self.C = int(index.vocab_size), int(index.hidden_dim), int(index.n_clusters)
        owned = np.ascontiguousarray(owned, dtype=np.uint8)
        if owned.shape != (self.C,):
            raise ValueError("owned mask must have one entry per cluster")
        self.owned = owned
        # DeviceIndex builds the descriptors; the shard constructor uploads
        # only the owned rows
        self._di = DeviceIndex(table, index, device, weights_required=True, owned=owned)
        self._ctx = self._di._ctx
        n_own = int(np.asarray(index.sizes)[owned.astype(bool)].sum())
        self.n_owned_tokens = n_own
        self._pos = np.empty(self.V, dtype=np.int64)
        self._ids = np.empty(self.V, dtype=np.int64)
        self._logits = np.empty(self.V, dtype=np.float64)

    def _check(self, rc):
        if rc != 0:
            self._di._check(rc)

    def open(self, h, cfg_struct, lo: int, hi: int):
        c = _lib.Config()
        ctypes.pointer(c)[0] = cfg_struct
        c.shard_lo, c.shard_hi = int(lo), int(hi)
        summ = np.empty(SH_TOPK + max(1, c.k), dtype=np.float64)
        n = ctypes.c_int64()
        h = np.ascontiguousarray(h, dtype=np.float64)
        self._check(self.lib.csvd_shard_open(self._ctx, h.ctypes.data, ctypes.byref(c), summ.ctypes.data,
                                             self._pos.ctypes.data, self._ids.ctypes.data,
                                             self._logits.ctypes.data, self.V, ctypes.byref(n)))
        m = n.value
        return summ, self._pos[:m].copy(), self._ids[:m].copy(), self._logits[:m].copy()

    def dense(self, h, k: int):
        summ = np.empty(SH_TOPK + max(1, k), dtype=np.float64)
        n = ctypes.c_int64()
        h = np.ascontiguousarray(h, dtype=np.float64)
        self._check(self.lib.csvd_shard_dense(self._ctx, h.ctypes.data, int(k), summ.ctypes.data,
                                              self._ids.ctypes.data, self._logits.ctypes.data, self.V,
                                              ctypes.byref(n)))
        m = n.value
        return summ, self._ids[:m].copy(), self._logits[:m].copy()

    def close(self):
        self._di.close()


# ---------------------------------------------------------------------------
# collectives
# ---------------------------------------------------------------------------
class TorchComm:
    """all_gather of small float64 / int64 vectors over a torch.distributed
    group (NCCL: staged through the rank's GPU; gloo: CPU)."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.dist, self.torch, self.group = dist, torch, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        backend = dist.get_backend(group)
        self.dev = torch.device("cuda", torch.cuda.current_device() if device is None else device) \
            if backend == "nccl" else torch.device("cpu")
        self.bytes = 0

    def all_gather(self, arr: np.ndarray) -> list:
        t = self.torch.from_numpy(np.ascontiguousarray(arr)).to(self.dev)
        out = [self.torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        self.bytes += t.numel() * t.element_size() * (self.world - 1)
        return [o.cpu().numpy() for o in out]

    def all_gather_var(self, arr: np.ndarray, n: int, counts) -> list:
        """variable-length gather: every rank already knows every count"""
        m = max(1, int(max(counts)))
        buf = np.zeros(m, dtype=arr.dtype)
        buf[:n] = arr[:n]
        parts = self.all_gather(buf)
        return [p[:int(c)] for p, c in zip(parts, counts)]


# ---------------------------------------------------------------------------
# merge + certification (identical on every rank)
# ---------------------------------------------------------------------------
class MergedState:
    """The certificate state of the opened prefix, merged over shards (the
    sharded counterpart of certify.CertState for a batch-select step)."""

    def __init__(self, k: int):
        self.k = k
        self.p = 0
        self.n = 0
        self.lses = []
        self.smin, self.smax = math.inf, NEG_INF
        self.tops = np.empty(0)
        self.u_next = NEG_INF
        self.lrh = NEG_INF
        self.C = 0

    def absorb(self, summaries):
        """Merge one open of every shard (same range on all ranks)."""
        s0 = summaries[0]
        k = self.k
        tops = [self.tops]
        for s in summaries:
            nl = int(s[SH_NLIST])
            tops.append(s[SH_TOPK:SH_TOPK + nl])
            if int(s[SH_NTOK]) > 0:
                self.lses.append(float(s[SH_LSE]))
                self.smin = min(self.smin, float(s[SH_MIN]))
                self.smax = max(self.smax, float(s[SH_MAX]))
            self.n += int(s[SH_NTOK])
        allv = np.concatenate(tops)
        self.tops = -np.sort(-allv)[:k]
        self.p = int(s0[SH_P_HI])
        self.u_next = float(s0[SH_U_NEXT])
        self.lrh = float(s0[SH_LRH_NEXT])
        if self.n != int(s0[SH_CUM_HI]):
            raise RuntimeError(f"shard merge lost tokens: {self.n} != {int(s0[SH_CUM_HI])}")

    @property
    def log_z(self) -> float:
        v = np.asarray(self.lses, dtype=np.float64)
        if v.size == 0:
            return NEG_INF
        m = float(v.max())
        if m == NEG_INF:
            return NEG_INF
        return m + math.log(float(np.exp(v - m).sum()))

    def kth(self) -> float:  # CertState.topk_min (certify.py:85-88)
        return float(self.tops[self.k - 1]) if self.n >= self.k else NEG_INF

    def rho(self) -> float:  # certify.py:93-99
        if self.lrh == NEG_INF:
            return 0.0
        lz = self.log_z
        if lz == NEG_INF:
            return 1.0
        return 1.0 / (1.0 + math.exp(lz - self.lrh))

    def delta(self) -> float:  # certify.py:101-107
        if self.lrh == NEG_INF:
            return 0.0
        lz = self.log_z
        if lz == NEG_INF:
            return math.inf
        return math.exp(self.lrh - lz)

    def u_max(self) -> float:
        return NEG_INF if self.p >= self.C else self.u_next


def check_targets(st: MergedState, cfg, epsilon: float):
    """decode._StepContext.check_targets (decode.py:192-210) on merged state."""
    for t in cfg.targets:
        if t == "topk":
            if st.n < cfg.k:
                continue
            kth = st.kth()
            if st.p >= st.C:
                return CertStatus("topk_exact", 0.0, NEG_INF, kth)
            if st.u_next < kth:
                return CertStatus("topk_exact", 0.0, st.u_next, kth)
        elif t == "softmax_eps":
            if st.n == 0:
                continue
            r = st.rho()
            if r <= epsilon:
                return CertStatus("softmax_eps", r, st.u_max(), st.kth())
        elif t == "topp":
            if st.n == 0:
                continue
            dl = st.delta()
            mass = dl / (1.0 + dl) if math.isfinite(dl) else 1.0
            if dl <= epsilon / (1.0 - epsilon):
                return CertStatus("topp_mass", mass, st.u_max(), st.kth())
        else:
            raise ConfigError(f"unknown target {t!r}")
    return None


def relaxed_check(st: MergedState, cfg, factor: float):
    """RelaxEps (decode.py:278-296): softmax / top-p only, at min(f eps, 1 - 1e-12)."""
    relaxed = min(cfg.epsilon * factor, 1.0 - 1e-12)
    for t in cfg.targets:
        if t == "softmax_eps":
            r = st.rho()
            if r <= relaxed:
                return CertStatus("softmax_eps", r, st.u_max(), st.kth())
        elif t == "topp":
            dl = st.delta()
            mass = dl / (1.0 + dl) if math.isfinite(dl) else 1.0
            if dl <= relaxed / (1.0 - relaxed):
                return CertStatus("topp_mass", mass, st.u_max(), st.kth())
    return None


def _xi(st: MergedState) -> float:
    """certify.tightness (certify.py:172-184) from merged min / max."""
    if st.n < 2 or st.p >= st.C:
        return math.nan
    lo, hi, um = st.smin, st.smax, st.u_next
    return 1.0 if um <= lo else (hi - lo) / (um - lo)


# ---------------------------------------------------------------------------
# the sharded step
# ---------------------------------------------------------------------------
class ShardedDecoder:
    """`sharded_decode_step` over a real process group.

    backend: a DeviceShard (default: built from table / index / plan for this
    rank) or any object with the same `open` / `dense` methods (the CPU tests
    use an oracle-backed one); comm: TorchComm (default) or a compatible
    object."""

    def __init__(self, table, index, plan, comm=None, backend=None, device=None):
        self.index = index
        self.plan = plan
        self.comm = comm if comm is not None else TorchComm(device=device)
        if self.comm.world != plan.n_workers:
            raise ValueError(f"plan has {plan.n_workers} workers, process group has {self.comm.world}")
        self.rank = self.comm.rank
        owned = (np.asarray(plan.assignment) == self.rank)
        if backend is None:
            import torch
            dev = (torch.cuda.current_device() if torch.cuda.is_available() else 0) if device is None else device
            backend = DeviceShard(table, index, owned, dev)
        self.backend = backend
        self.V, self.C, self.d = int(index.vocab_size), int(index.n_clusters), int(index.hidden_dim)

    def check_same_inputs(self, h, cfg, k_max):
        """Every rank must decode the same query with the same config (the
        workers of one sharded step): all_gather a digest and compare."""
        import hashlib
        m = hashlib.sha256(np.ascontiguousarray(h, dtype=np.float64).tobytes())
        m.update(repr((cfg.k, cfg.epsilon, tuple(cfg.targets), cfg.k_max, tuple(map(repr, cfg.fallback)),
                       getattr(cfg, "slack_mode", "none"), k_max)).encode())
        dig = np.frombuffer(m.digest()[:16], dtype=np.int64)
        got = self.comm.all_gather(dig)
        if any(not np.array_equal(g, dig) for g in got):
            raise ValueError("sharded step: ranks passed different queries or configs")

    def _open(self, st: MergedState, h, cs, lo, hi, parts):
        summ, pos, ids, logits = self.backend.open(h, cs, lo, hi)
        sums = self.comm.all_gather(summ)
        st.absorb(sums)
        parts.append((pos, ids, logits, [int(s[SH_NTOK]) for s in sums]))
        return sums

    def _assemble(self, parts, n):
        """One variable-length all_gather per open: (position, id, logit bits)
        packed as three int64 columns, so the logits travel bit for bit."""
        pos_l, id_l, lg_l = [], [], []
        for pos, ids, logits, counts in parts:
            mine = len(pos)
            packed = np.stack([pos.astype(np.int64), ids.astype(np.int64),
                               np.ascontiguousarray(logits, dtype=np.float64).view(np.int64)], axis=1).reshape(-1)
            got = self.comm.all_gather_var(packed, 3 * mine, [3 * c for c in counts])
            for g in got:
                g = g.reshape(-1, 3)
                pos_l.append(g[:, 0])
                id_l.append(g[:, 1])
                lg_l.append(np.ascontiguousarray(g[:, 2]).view(np.float64))
        pos = np.concatenate(pos_l) if pos_l else np.empty(0, np.int64)
        order = np.argsort(pos, kind="stable")
        if pos.size != n or not np.array_equal(pos[order], np.arange(n)):
            raise RuntimeError("sharded outputs do not tile the opened prefix")
        return np.concatenate(id_l)[order], np.concatenate(lg_l)[order]

    def step(self, h, cfg, k_max=None):
        """One sharded step -> DecodeOutcome (the batch-select outcome)."""
        from .engine import config_struct
        validate_config(cfg, self.V)
        km = resolved_k_max(cfg, self.V) if k_max is None else int(k_max)
        cs = config_struct(cfg, self.V, km, _lib.VARIANT_BATCHSELECT)
        st = MergedState(cfg.k)
        st.C = self.C
        parts = []
        sums = self._open(st, h, cs, 0, 0, parts)
        qn, slack = float(sums[0][SH_QNORM]), float(sums[0][SH_SLACK])
        status = check_targets(st, cfg, cfg.epsilon)
        fb = None
        if status is None:
            levels = list(cfg.fallback)
            if not any(getattr(lv, "name", None) == "full_vocab" for lv in levels):
                levels.append(None)  # FullVocab is always the implicit last level
            for lv in levels:
                name = getattr(lv, "name", "full_vocab") if lv is not None else "full_vocab"
                if name == "partial_expand":
                    hi = min(self.C, st.p + max(0, int(lv.delta_c)))
                    if hi > st.p:
                        self._open(st, h, cs, st.p, hi, parts)
                    status = check_targets(st, cfg, cfg.epsilon)
                elif name == "relax_eps":
                    status = relaxed_check(st, cfg, float(lv.factor))
                else:
                    return self._full_vocab(h, cfg, qn, slack)
                if status is not None:
                    fb = name
                    break
        ids, logits = self._assemble(parts, st.n)
        stats = StepMetrics(
            sub_size=st.n, ratio=st.n / self.V, clusters_opened=st.p, xi=_xi(st), cert_kind=status.kind,
            fallback=fb, rho=st.rho(), flops_sparse=2 * st.n * self.d,
            flops_bounds=2 * self.C * (self.d + (1 if self.index.mode == "bias_augmented" else 0)),
            heap_pops=0)  # batch-select pops no heap (decode.py:362-382)
        return DecodeOutcome(token_ids=ids, logits=logits, status=status, fallback_used=fb, stats=stats)

    def _full_vocab(self, h, cfg, qn, slack):
        """FullVocab (decode.py:239-262): shard-local dense GEMV, top-k merge."""
        summ, ids, logits = self.backend.dense(h, cfg.k)
        sums = self.comm.all_gather(summ)
        tops = np.concatenate([s[SH_TOPK:SH_TOPK + int(s[SH_NLIST])] for s in sums])
        kth = float(-np.sort(-tops)[cfg.k - 1])
        counts = [int(s[SH_NTOK]) for s in sums]
        packed = np.stack([ids.astype(np.int64),
                           np.ascontiguousarray(logits, dtype=np.float64).view(np.int64)], axis=1).reshape(-1)
        got = [g.reshape(-1, 2) for g in self.comm.all_gather_var(packed, 2 * len(ids), [2 * c for c in counts])]
        all_ids = np.concatenate([g[:, 0] for g in got])
        all_lg = np.concatenate([np.ascontiguousarray(g[:, 1]).view(np.float64) for g in got])
        out = np.empty(self.V, dtype=np.float64)
        out[all_ids] = all_lg
        if all_ids.size != self.V:
            raise RuntimeError("full-vocabulary shards do not cover the vocabulary")
        status = CertStatus("topk_exact", 0.0, NEG_INF, kth)
        stats = StepMetrics(
            sub_size=self.V, ratio=1.0, clusters_opened=self.C, xi=math.nan, cert_kind="topk_exact",
            fallback="full_vocab", rho=0.0, flops_sparse=2 * self.V * self.d,
            flops_bounds=2 * self.C * (self.d + (1 if self.index.mode == "bias_augmented" else 0)),
            heap_pops=0)
        return DecodeOutcome(token_ids=np.arange(self.V, dtype=np.int64), logits=out, status=status,
                             fallback_used="full_vocab", stats=stats)
