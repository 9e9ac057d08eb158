"""Generate golden fixtures by running the REAL reference (`csvd`, imported from
/root/reference/pkg/src) on small, exactly reproducible inputs.

Run in the build container (the reference does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden.py

Inputs are regenerated on any machine from their recipe (synth_vocab is
replicated bit-for-bit by paper_2511_21702_b200.workload.synth_vocab, checked
in tests/test_workload.py); k-means indexes (reference build_index) are stored
in the fixture because rebuilding them needs the reference.  Outputs stored:
every DecodeOutcome field the parity tests compare, the bound vector, and the
reference numpy version / host SIMD flags the bits were produced with.
"""

from __future__ import annotations

import dataclasses
import json
import os
import platform
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import csvd  # noqa: E402  (the reference)
from paper_2511_21702_b200 import workload as wl  # noqa: E402

KINDS = {"topk_exact": 0, "softmax_eps": 1, "topp_mass": 2}
FBS = {None: -1, "partial_expand": 0, "relax_eps": 1, "full_vocab": 2}


def unit_queries(n, d, seed):  # reference tests/conftest.py:43-46
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((n, d))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def cfg_doc(cfg: csvd.DecodeConfig) -> dict:
    fb = []
    for lv in cfg.fallback:
        if isinstance(lv, csvd.PartialExpand):
            fb.append(["partial_expand", lv.delta_c])
        elif isinstance(lv, csvd.RelaxEps):
            fb.append(["relax_eps", lv.factor])
        else:
            fb.append(["full_vocab", 0])
    return {"k": cfg.k, "epsilon": cfg.epsilon, "targets": list(cfg.targets), "k_max": cfg.k_max,
            "fallback": fb, "slack_mode": cfg.slack_mode}


def index_arrays(ix: csvd.ClusterIndex) -> dict:
    return {
        "perm": ix.perm, "starts": ix.starts, "sizes": ix.sizes, "centroids": ix.centroids,
        "centroid_norms": ix.centroid_norms, "radii": ix.radii, "angulars": ix.angulars,
        "max_biases": ix.max_biases, "max_norms": ix.max_norms, "min_norms": ix.min_norms,
        "bias_topm": np.array([[v for pair in c.bias_topm for v in pair] + [np.nan] * (2 * ix.bias_depth - 2 * len(c.bias_topm))
                               for c in ix.clusters]),
    }


class Case:
    def __init__(self, name, table_recipe, table, index, index_recipe):
        self.name = name
        self.table_recipe = table_recipe
        self.table = table
        self.index = index
        self.index_recipe = index_recipe
        self.steps = []  # (variant, cfg_id, k_max, query_id)
        self.queries = []
        self.cfgs = []

    def add_queries(self, q):
        base = len(self.queries)
        self.queries.extend(list(q))
        return list(range(base, base + len(q)))

    def add_cfg(self, cfg):
        self.cfgs.append(cfg)
        return len(self.cfgs) - 1


def run_case(case: Case) -> dict:
    T, ix = case.table, case.index
    out = {"ids": [], "logits": [], "ptr": [0], "scal": [], "ints": [], "U": [], "qn": []}
    for variant, ci, kmax, qi in case.steps:
        cfg = case.cfgs[ci]
        h = case.queries[qi]
        if variant == "incremental":
            o = csvd.decode_step(T, ix, h, cfg, k_max=kmax)
        elif variant == "batchselect":
            o = csvd.decode_step_batchselect(T, ix, h, cfg, k_max=kmax)
        else:
            raise ValueError(variant)
        b = csvd.cluster_bounds(ix, h, slack_mode=cfg.slack_mode)
        out["ids"].append(o.token_ids)
        out["logits"].append(o.logits)
        out["ptr"].append(out["ptr"][-1] + o.token_ids.size)
        s = o.stats
        out["scal"].append([o.status.epsilon_achieved, o.status.u_max, o.status.topk_min, s.rho, s.xi,
                            s.ratio, b.query_norm, b.slack])
        out["ints"].append([KINDS[o.status.kind], FBS[o.fallback_used], s.sub_size, s.clusters_opened,
                            s.heap_pops, s.flops_sparse, s.flops_bounds])
        out["U"].append(b.values)
    arrays = {
        "ids": np.concatenate(out["ids"]) if out["ids"] else np.zeros(0, np.int64),
        "logits": np.concatenate(out["logits"]) if out["logits"] else np.zeros(0),
        "ptr": np.array(out["ptr"], dtype=np.int64),
        "scal": np.array(out["scal"], dtype=np.float64),
        "ints": np.array(out["ints"], dtype=np.int64),
        "U": np.array(out["U"], dtype=np.float64),
        "queries": np.array(case.queries, dtype=np.float64),
        "steps_variant": np.array([0 if v == "incremental" else 1 for v, _, _, _ in case.steps], dtype=np.int64),
        "steps_cfg": np.array([c for _, c, _, _ in case.steps], dtype=np.int64),
        "steps_kmax": np.array([-1 if k is None else k for _, _, k, _ in case.steps], dtype=np.int64),
        "steps_query": np.array([q for _, _, _, q in case.steps], dtype=np.int64),
    }
    if case.index_recipe is None:
        for k, v in index_arrays(ix).items():
            arrays["index_" + k] = v
        arrays["index_fingerprint"] = np.frombuffer(ix.fingerprint, dtype=np.uint8)
    # dense oracle for the first few queries
    dl = [csvd.dense_logits(T, case.queries[i]).logits for i in range(min(3, len(case.queries)))]
    arrays["dense"] = np.array(dl)
    meta = {
        "name": case.name, "table": case.table_recipe, "index": case.index_recipe, "mode": ix.mode,
        "bias_depth": ix.bias_depth, "cfgs": [cfg_doc(c) for c in case.cfgs],
        "numpy": np.__version__, "machine": platform.machine(),
        "cpu_flags": _cpu_flags(),
    }
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    return arrays


def _cpu_flags():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    fl = line.split(":")[1].split()
                    return [x for x in fl if x.startswith(("avx", "fma", "sse4"))]
    except OSError:
        pass
    return []


def base_cfgs(V):
    P, R, F = csvd.PartialExpand, csvd.RelaxEps, csvd.FullVocab
    return [
        csvd.DecodeConfig(k=5, epsilon=0.05),                                     # 0 default-ish
        csvd.DecodeConfig(k=1, targets=("topk",)),                                # 1 top-1
        csvd.DecodeConfig(k=10, epsilon=1e-3, targets=("softmax_eps",)),          # 2 eps-softmax
        csvd.DecodeConfig(k=5, epsilon=0.05, targets=("topp", "topk")),           # 3 top-p first
        csvd.DecodeConfig(k=5, epsilon=0.01, k_max=max(5, V // 50)),              # 4 tight budget -> fallback
        csvd.DecodeConfig(k=3, epsilon=1e-6, targets=("softmax_eps",), k_max=max(3, V // 40),
                          fallback=(P(2), R(2.0))),                               # 5 chain -> full_vocab
        csvd.DecodeConfig(k=50, epsilon=0.05),                                    # 6 larger k
        csvd.DecodeConfig(k=5, epsilon=0.05, slack_mode="f32"),                   # 7 f32 slack
    ]


def add_standard_steps(case: Case, qids, variants=("incremental", "batchselect"), cfg_ids=None):
    V = case.table.vocab_size
    if not case.cfgs:
        for c in base_cfgs(V):
            case.add_cfg(c)
    cfg_ids = range(len(case.cfgs)) if cfg_ids is None else cfg_ids
    for v in variants:
        for ci in cfg_ids:
            for qi in qids:
                case.steps.append((v, ci, None, qi))


def main():
    os.makedirs(HERE, exist_ok=True)
    cases = []

    # 1. reference conftest small table, three index modes (build_index k-means)
    small = csvd.synth_vocab(500, 16, 10, 0.05, 3)
    for mode in ("euclidean", "spherical", "bias_augmented"):
        ix = csvd.build_index(small, 10, mode=mode, seed=0)
        c = Case(f"small_{mode}", [500, 16, 10, 0.05, 3], small, ix, None)
        q = c.add_queries(unit_queries(6, 16, 11))
        q += c.add_queries(csvd.generate_queries(6, 16, "contextual", 7, centroids=ix.centroids))
        add_standard_steps(c, q)
        cases.append(c)

    # 2. reference conftest medium table
    med = csvd.synth_vocab(1000, 32, 20, 0.05, 5)
    ix = csvd.build_index(med, 20, seed=0)
    c = Case("medium", [1000, 32, 20, 0.05, 5], med, ix, None)
    q = c.add_queries(unit_queries(8, 32, 23))
    q += c.add_queries(4.0 * unit_queries(4, 32, 43))  # sharp softmax, PE/relax probes
    add_standard_steps(c, q)
    # k_max overrides (warmup / adaptive controller path)
    for qi in q[:4]:
        c.steps.append(("incremental", 0, 1000, qi))
        c.steps.append(("incremental", 0, 3, qi))
    cases.append(c)

    # 3. acceptance workload (tests/test_acceptance.py): V=5000, d=64, C=75
    acc = csvd.synth_vocab(5000, 64, 50, 0.05, 1)
    ix = csvd.build_index(acc, 75, seed=0)
    c = Case("acceptance", [5000, 64, 50, 0.05, 1], acc, ix, None)
    q = c.add_queries(csvd.generate_queries(12, 64, "contextual", 7, centroids=ix.centroids))
    q += c.add_queries(csvd.generate_queries(2, 64, "random", 8))
    add_standard_steps(c, q, cfg_ids=[0, 1, 2, 3, 4, 6])
    cases.append(c)

    # 4. device-regular pairwise plans (fast index, regenerated on the box):
    #    d=512 (4 leaves), 1024 (8), 2048 (16), 3584 (32x112), 4096 (32), 8192 (64)
    for V, d, n_modes, g in ((2000, 512, 20, 2), (1500, 1024, 15, 2), (1200, 2048, 12, 1),
                             (1000, 3584, 10, 2), (1200, 4096, 12, 3), (600, 8192, 6, 2)):
        t32 = wl.synth_vocab(V, d, n_modes, 0.3, 1)
        T = csvd.EmbeddingTable(weights=t32.weights.astype(np.float64), bias=t32.bias)
        mine = wl.fast_index(t32, n_modes, g)
        ix = _as_ref_index(mine)
        c = Case(f"regular_d{d}", [V, d, n_modes, 0.3, 1], T, ix, {"kind": "fast", "n_modes": n_modes, "g": g})
        q = c.add_queries(csvd.generate_queries(3, d, "contextual", 7, centroids=ix.centroids, noise=0.3))
        q += c.add_queries(csvd.generate_queries(1, d, "random", 9))
        add_standard_steps(c, q, variants=("incremental",), cfg_ids=[0, 2, 4])
        cases.append(c)

    # 5. bf16-weight variant: the reference is fed the bf16-rounded table
    t16 = wl.synth_vocab(1200, 4096, 12, 0.3, 1, dtype="bf16")
    w64 = (t16.weights.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    T = csvd.EmbeddingTable(weights=w64, bias=t16.bias)
    ix = _as_ref_index(wl.fast_index(t16, 12, 3))
    c = Case("bf16_d4096", [1200, 4096, 12, 0.3, 1, "bf16"], T, ix, {"kind": "fast", "n_modes": 12, "g": 3})
    q = c.add_queries(csvd.generate_queries(3, 4096, "contextual", 7, centroids=ix.centroids))
    add_standard_steps(c, q, variants=("incremental",), cfg_ids=[0, 2])
    cases.append(c)

    for case in cases:
        arrays = run_case(case)
        path = os.path.join(HERE, f"{case.name}.npz")
        np.savez_compressed(path, **arrays)
        mix = {}
        for kf in arrays["ints"][:, :2].tolist():
            mix[tuple(kf)] = mix.get(tuple(kf), 0) + 1
        print(f"{case.name}: {len(case.steps)} steps -> {os.path.getsize(path) / 1024:.0f} KiB  (kind,fb) mix {mix}")


def _as_ref_index(mine):
    return csvd.ClusterIndex(
        clusters=[csvd.ClusterMeta(**{f.name: getattr(cm, f.name) for f in dataclasses.fields(cm)})
                  for cm in mine.clusters],
        perm=mine.perm, mode=mine.mode, vocab_size=mine.vocab_size, hidden_dim=mine.hidden_dim,
        bias_depth=mine.bias_depth, fingerprint=mine.fingerprint)


if __name__ == "__main__":
    main()
