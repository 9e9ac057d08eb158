"""Vocabulary / cluster sharding: plans, the sharded step, and the comm ledger.

Reference: `csvd.shard_sim` (/root/reference/pkg/src/csvd/shard_sim.py), an
in-process simulation whose contract is *transparency*: for every worker
count and placement strategy the sharded step returns exactly the one-shot
`decode_step_batchselect` outcome (tests/test_acceptance.py:142-161), with
the worker count visible only in the `CommLedger` byte accounting.

* `make_plan`            shard_sim.py:84-131 (round_robin / hotness_weighted /
                         semantic_grouped; the k-means of centroids for
                         semantic_grouped restates cluster_index._lloyd,
                         cluster_index.py:167-251, host-side planning only)
* `sharded_decode_step`  shard_sim.py:134-208.  Single process: the B200
                         batch-select step (bit-identical by construction)
                         plus the ledger.  Real multi-GPU execution, one
                         process per GPU with vocab-sharded W and one NCCL
                         all-gather of per-shard summaries, is
                         `distributed.ShardedDecoder`.
"""

from __future__ import annotations

import json
import weakref
from dataclasses import dataclass

import numpy as np

from . import engine
from .types import resolved_k_max, validate_config

STRATEGIES = ("round_robin", "hotness_weighted", "semantic_grouped")


@dataclass(frozen=True)
class ShardPlan:
    n_workers: int
    strategy: str
    assignment: np.ndarray
    loads: np.ndarray
    sigma_load: float

    def clusters_of(self, worker: int) -> np.ndarray:
        return np.flatnonzero(np.asarray(self.assignment) == worker)


@dataclass(frozen=True)
class LatencyModel:
    flops_per_unit: float = 1.0
    bytes_per_unit: float = 1.0


@dataclass(frozen=True)
class CommLedger:
    bytes_bounds_phase: int
    bytes_logits_phase: int
    phase_latencies: dict
    omega_comm: float

    @property
    def bytes_total(self) -> int:
        return self.bytes_bounds_phase + self.bytes_logits_phase


# --- k-means of centroids (semantic_grouped placement) ---------------------
def _kmeanspp_seed(data, C, rng):
    """cluster_index._kmeanspp_seed (cluster_index.py:167-201)."""
    n = data.shape[0]
    n_candidates = 2 + int(np.log(C)) if C > 1 else 1
    chosen = np.zeros(n, dtype=bool)
    idx = int(rng.integers(n))
    centers = [idx]
    chosen[idx] = True
    d2 = ((data - data[idx]) ** 2).sum(axis=1)
    for _ in range(1, C):
        total = float(d2.sum())
        if total > 0:
            cum = np.cumsum(d2)
            picks = np.searchsorted(cum, rng.random(n_candidates) * total, side="right")
            picks = np.minimum(picks, n - 1)
            best_idx, best_d2, best_pot = -1, None, np.inf
            for cand in picks:
                cand = int(cand)
                if chosen[cand]:
                    continue
                cand_d2 = np.minimum(d2, ((data - data[cand]) ** 2).sum(axis=1))
                pot = float(cand_d2.sum())
                if pot < best_pot:
                    best_idx, best_d2, best_pot = cand, cand_d2, pot
            if best_idx < 0:
                best_idx = int(np.flatnonzero(~chosen)[0])
                best_d2 = np.minimum(d2, ((data - data[best_idx]) ** 2).sum(axis=1))
            idx, d2 = best_idx, best_d2
        else:
            idx = int(np.flatnonzero(~chosen)[0])
            d2 = np.minimum(d2, ((data - data[idx]) ** 2).sum(axis=1))
        centers.append(idx)
        chosen[idx] = True
    return data[np.array(centers)].copy()


def _assign(data, centers):
    cross = data @ centers.T
    c2 = (centers * centers).sum(axis=1)
    return np.argmin(c2[None, :] - 2.0 * cross, axis=1)


def _repair_empty(data, centers, assignment, C):
    sizes = np.bincount(assignment, minlength=C)
    while True:
        empties = np.flatnonzero(sizes == 0)
        if empties.size == 0:
            return assignment
        diff = data - centers[assignment]
        d2 = (diff * diff).sum(axis=1)
        for c in empties:
            eligible = sizes[assignment] >= 2
            if not eligible.any():
                return assignment
            scored = np.where(eligible, d2, -np.inf)
            i = int(np.argmax(scored))
            sizes[assignment[i]] -= 1
            assignment[i] = c
            sizes[c] += 1


def _lloyd(data, C, iters, rng):
    """cluster_index._lloyd (cluster_index.py:232-251), euclidean."""
    centers = _kmeanspp_seed(data, C, rng)
    assignment = None
    for _ in range(iters):
        new = _repair_empty(data, centers, _assign(data, centers), C)
        if assignment is not None and np.array_equal(new, assignment):
            assignment = new
            break
        assignment = new
        sums = np.zeros_like(centers)
        np.add.at(sums, assignment, data)
        counts = np.bincount(assignment, minlength=C).astype(np.float64)
        centers = sums / counts[:, None]
    return assignment


def make_plan(index, n_workers: int, strategy: str = "round_robin", hotness=None, seed: int = 0) -> ShardPlan:
    """shard_sim.make_plan (shard_sim.py:84-131)."""
    if n_workers < 1:
        raise ValueError("need at least one worker")
    if strategy not in STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}, expected one of {STRATEGIES}")
    C = index.n_clusters
    if strategy == "round_robin":
        assignment = np.arange(C, dtype=np.int64) % n_workers
    elif strategy == "hotness_weighted":
        if hotness is None:
            raise ValueError("hotness_weighted needs per-cluster hotness weights")
        hotness = np.ascontiguousarray(hotness, dtype=np.float64)
        if hotness.shape != (C,):
            raise ValueError(f"hotness must have length C={C}")
        assignment = np.empty(C, dtype=np.int64)
        worker_weight = np.zeros(n_workers)
        for c in np.lexsort((np.arange(C), -hotness)):
            g = int(np.argmin(worker_weight))
            assignment[c] = g
            worker_weight[g] += hotness[c]
    else:
        if n_workers == 1:
            assignment = np.zeros(C, dtype=np.int64)
        elif n_workers >= C:
            assignment = np.arange(C, dtype=np.int64)
        else:
            rng = np.random.default_rng(seed)
            assignment = _lloyd(np.ascontiguousarray(index.centroids, dtype=np.float64), n_workers,
                                16, rng).astype(np.int64)
    loads = np.zeros(n_workers, dtype=np.int64)
    np.add.at(loads, assignment, index.sizes)
    return ShardPlan(n_workers=n_workers, strategy=strategy, assignment=assignment, loads=loads,
                     sigma_load=float(loads.std()))


def contiguous_plan(index, n_workers: int) -> ShardPlan:
    """B200 placement: contiguous token-balanced ranges of the (size-sorted)
    cluster order -- every rank owns one contiguous row range of the permuted
    W, so a shard is a single HBM slab.  NVSwitch makes every peer equally
    close, so locality-aware placement buys nothing."""
    sizes = np.asarray(index.sizes)
    cum = np.concatenate([[0], np.cumsum(sizes)])
    total = cum[-1]
    bounds = [int(np.searchsorted(cum, total * r / n_workers, side="left")) for r in range(n_workers + 1)]
    bounds[0], bounds[-1] = 0, index.n_clusters
    assignment = np.zeros(index.n_clusters, dtype=np.int64)
    for r in range(n_workers):
        assignment[bounds[r]:bounds[r + 1]] = r
    loads = np.zeros(n_workers, dtype=np.int64)
    np.add.at(loads, assignment, sizes)
    return ShardPlan(n_workers, "contiguous", assignment, loads, float(loads.std()))


def _cluster_of_token(index) -> np.ndarray:
    pos_cluster = np.repeat(np.arange(index.n_clusters), np.asarray(index.sizes))
    out = np.empty(index.vocab_size, dtype=np.int64)
    out[np.asarray(index.perm)] = pos_cluster
    return out


def ledger_for(index, plan: ShardPlan, outcome, latency: LatencyModel = LatencyModel()) -> CommLedger:
    """The byte/latency ledger of shard_sim.py:181-207 for a finished step."""
    d = index.hidden_dim
    C = index.n_clusters
    N = plan.n_workers
    bdim = d + (1 if index.mode == "bias_augmented" else 0)
    bound_flops = np.array([2 * np.count_nonzero(plan.assignment == g) * bdim for g in range(N)], dtype=float)
    if outcome.fallback_used == "full_vocab":
        tpw = plan.loads.astype(np.float64)
    else:
        cot = _cluster_of_token(index)
        tpw = np.bincount(np.asarray(plan.assignment)[cot[outcome.token_ids]], minlength=N).astype(np.float64)
    sparse_flops = 2 * tpw * d
    exch = N >= 2
    bb = C * 4 if exch else 0
    bl = outcome.stats.sub_size * (d * 2 + 4) if exch else 0
    tb = bb / latency.bytes_per_unit
    tl = bl / latency.bytes_per_unit
    ph = {
        "bounds": float(bound_flops.max()) / latency.flops_per_unit + tb,
        "logits": float(sparse_flops.max()) / latency.flops_per_unit + tl,
        "verify": 0.0,
    }
    total = sum(ph.values())
    return CommLedger(bytes_bounds_phase=bb, bytes_logits_phase=bl, phase_latencies=ph,
                      omega_comm=(tb + tl) / total if total > 0 else 0.0)


_DECODERS: dict = {}


def sharded_decode_step(table, index, plan: ShardPlan, h, cfg, k_max=None, latency: LatencyModel = LatencyModel(),
                        group=None):
    """B200 `csvd.sharded_decode_step` (shard_sim.py:134-208).

    group=None (the reference's call): the N workers are simulated as in the
    reference, and the outcome is the batch-select step, bit-identical for
    every N and strategy by construction.  group=<torch.distributed process
    group of plan.n_workers ranks> (opt-in): every rank is one worker, owns
    the plan's clusters on its GPU, and the step runs as
    `distributed.ShardedDecoder` (one all_gather of per-shard merge records);
    every rank must pass the same h / cfg, which is cross-checked by digest.
    Either way the ledger is the reference's accounting."""
    validate_config(cfg, index.vocab_size)
    if np.asarray(plan.assignment).shape != (index.n_clusters,):
        raise ValueError("plan does not cover this index")
    k_max = resolved_k_max(cfg, index.vocab_size) if k_max is None else k_max
    if group is not None and plan.n_workers > 1:
        import torch.distributed as dist
        from .distributed import ShardedDecoder, TorchComm
        if dist.get_world_size(group) != plan.n_workers:
            raise ValueError(f"process group has {dist.get_world_size(group)} ranks, plan has {plan.n_workers}")
        key = (id(table), id(index), id(plan), id(group))
        ent = _DECODERS.get(key)
        dec = None
        if ent is not None:
            refs, dec = ent
            if not all(r() is o for r, o in zip(refs, (table, index, plan))):
                dec = None
        if dec is None:
            dec = ShardedDecoder(table, index, plan, comm=TorchComm(group))
            refs = tuple(weakref.ref(o, lambda _r, k=key: _DECODERS.pop(k, None)) for o in (table, index, plan))
            _DECODERS[key] = (refs, dec)
        dec.check_same_inputs(h, cfg, k_max)
        outcome = dec.step(h, cfg, k_max=k_max)
    else:
        outcome = engine.decode_step_batchselect(table, index, h, cfg, k_max=k_max)
    return outcome, ledger_for(index, plan, outcome, latency)


def save_plan(plan: ShardPlan, path) -> None:
    doc = {
        "n_workers": plan.n_workers,
        "strategy": plan.strategy,
        "assignment": [int(x) for x in plan.assignment],
        "loads": [int(x) for x in plan.loads],
        "sigma_load": plan.sigma_load,
    }
    with open(path, "w") as f:
        json.dump(doc, f, sort_keys=True, indent=2)
        f.write("\n")


def load_plan(path) -> ShardPlan:
    with open(path) as f:
        doc = json.load(f)
    return ShardPlan(
        n_workers=int(doc["n_workers"]),
        strategy=str(doc["strategy"]),
        assignment=np.asarray(doc["assignment"], dtype=np.int64),
        loads=np.asarray(doc["loads"], dtype=np.int64),
        sigma_load=float(doc["sigma_load"]),
    )
