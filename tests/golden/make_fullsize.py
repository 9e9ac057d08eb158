"""Full-size golden fixtures from the REAL reference at BASELINE shapes.

Run in the build container (the reference does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_fullsize.py [c2|c3|c4|c5 ...]

Everything on the reference side is the reference's own code:
  * table      csvd.synth_vocab (tensor_io.py:192-216), float64; for bf16
               configs RNE-rounded to bf16 (the rounded table is what the
               reference is fed);
  * index      SURVEY §8(d) fast index: the synth RNG replayed for each row's
               mode, mode m split g ways by within-mode rank, statistics from
               csvd.cluster_index._cluster_stats in build_index's ordering
               convention (cluster_index.py:305-341), validated with
               csvd.validate_index;
  * queries    csvd.bench.generate_queries (bench.py:183-209);
  * outcomes   csvd.decode_step (decode.py:312-343) with the per-step SHA-256
               fingerprint memoized after one real check (decode.py:142-144).
The script also asserts that this repo's input replicas (workload.synth_vocab,
fast_index, generate_queries) reproduce those inputs bit for bit, which is
what lets the GPU box regenerate them without the reference.

Stored per step (compact; full-vocabulary outcomes have V entries): every
scalar of the outcome, the SHA-256 of token_ids (int64 LE) and of logits
(float64 LE), the first 64 ids / logits, and the bound vector U.
"""

from __future__ import annotations

import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import csvd  # noqa: E402  (the reference)
import csvd.decode as csvd_decode  # noqa: E402
from csvd.cluster_index import ClusterIndex as RefIndex, ClusterMeta as RefMeta, _cluster_stats  # noqa: E402

from paper_2511_21702_b200 import workload as wl  # noqa: E402
from paper_2511_21702_b200.types import f32_to_bf16_bits, bf16_bits_to_f32  # noqa: E402

# name -> (V, d, C, g, dtype, cfg kwargs, contextual queries, random queries)
CONFIGS = {
    "c2": dict(V=128256, d=4096, C=1024, g=16, dtype="f32", cfg=dict(k=10), n_ctx=20, n_rand=5),
    "c3": dict(V=151552, d=3584, C=2273, g=1, dtype="bf16", cfg=dict(k=10, epsilon=1e-3, targets=("softmax_eps",)),
               n_ctx=16, n_rand=0),
    "c4": dict(V=128256, d=8192, C=1024, g=16, dtype="f32", cfg=dict(k=10), n_ctx=8, n_rand=1),
    "c5": dict(V=256000, d=3584, C=3840, g=16, dtype="f32", cfg=dict(k=10), n_ctx=8, n_rand=1),
}
SPREAD, NOISE, TABLE_SEED, Q_SEED, R_SEED = 0.3, 0.3, 1, 7, 8


def ref_fast_index(table, n_modes, g, seed, m=3):
    """SURVEY §8(d) with the reference's own statistics and conventions."""
    V, d = table.vocab_size, table.hidden_dim
    rng = np.random.default_rng(seed)  # replay synth_vocab's draws (tensor_io.py:207-209)
    rng.standard_normal((n_modes, d))
    modes = rng.integers(0, n_modes, size=V)
    order_rows = np.argsort(modes, kind="stable")
    sm = modes[order_rows]
    first = np.searchsorted(sm, sm, side="left")
    rank = np.empty(V, dtype=np.int64)
    rank[order_rows] = np.arange(V) - first
    label = modes.astype(np.int64) * g + (rank % g)
    C = n_modes * g
    geo = np.asarray(table.weights, dtype=np.float64)
    member_lists = [np.flatnonzero(label == c) for c in range(C)]
    member_lists = [mm for mm in member_lists if mm.size]
    order = sorted(range(len(member_lists)), key=lambda c: (-member_lists[c].size, int(member_lists[c][0])))
    clusters, perm, pos = [], np.empty(V, dtype=np.int64), 0
    for c in order:
        members = member_lists[c]
        perm[pos:pos + members.size] = members
        cen, cn, rad, ang, mb, mxn, mnn, topm = _cluster_stats(geo, table.bias, members, "euclidean", m)
        clusters.append(RefMeta(centroid=cen, centroid_norm=cn, radius=rad, angular=ang, max_bias=mb, max_norm=mxn,
                                min_norm=mnn, bias_topm=topm, start=pos, end=pos + members.size))
        pos += members.size
    return RefIndex(clusters=clusters, perm=perm, mode="euclidean", vocab_size=V, hidden_dim=d, bias_depth=m,
                    fingerprint=csvd.table_fingerprint(table))


def digest(a, dt):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=dt).tobytes()).hexdigest()


def make(name):
    c = CONFIGS[name]
    V, d, C, g = c["V"], c["d"], c["C"], c["g"]
    n_modes = C // g
    t0 = time.time()
    T = csvd.synth_vocab(V, d, n_modes, SPREAD, TABLE_SEED)
    if c["dtype"] == "bf16":  # the rounded table is the reference's input
        w = bf16_bits_to_f32(f32_to_bf16_bits(T.weights.astype(np.float32))).astype(np.float64)
        T = csvd.EmbeddingTable(w, T.bias)
    # this repo's replica of the table must be the same bits
    mine = wl.synth_vocab(V, d, n_modes, SPREAD, TABLE_SEED, dtype=c["dtype"])
    mw = bf16_bits_to_f32(mine.weights) if c["dtype"] == "bf16" else mine.weights
    assert np.array_equal(mw.astype(np.float64), T.weights) and np.array_equal(mine.bias, T.bias), "synth replica"
    del mw
    ix = ref_fast_index(T, n_modes, g, TABLE_SEED)
    problems = csvd.validate_index(ix, T)
    assert problems.ok, problems.violations[:3]
    mix = wl.fast_index(mine, n_modes, g)
    for f in ("perm", "starts", "sizes", "centroids", "radii", "max_biases"):
        assert np.array_equal(np.asarray(getattr(mix, f)), np.asarray(getattr(ix, f))), f"fast_index replica: {f}"
    del mine, mix
    qs = csvd.bench.generate_queries(c["n_ctx"], d, "contextual", Q_SEED, centroids=ix.centroids, noise=NOISE)
    assert np.array_equal(qs, wl.generate_queries(c["n_ctx"], d, "contextual", Q_SEED, centroids=ix.centroids,
                                                  noise=NOISE)), "query replica"
    if c["n_rand"]:
        qr = csvd.bench.generate_queries(c["n_rand"], d, "random", R_SEED)
        assert np.array_equal(qr, wl.generate_queries(c["n_rand"], d, "random", R_SEED)), "query replica (random)"
        qs = np.vstack([qs, qr])
    print(f"{name}: inputs ready in {time.time() - t0:.0f} s", flush=True)
    cfg = csvd.DecodeConfig(**c["cfg"])
    csvd_decode._check_table_index(T, ix)  # the real fingerprint check, once
    real_check = csvd_decode._check_table_index
    csvd_decode._check_table_index = lambda table, index: None  # memoized for the remaining steps
    try:
        recs, Us = [], []
        for i, h in enumerate(qs):
            t1 = time.time()
            o = csvd.decode_step(T, ix, h, cfg)
            s = o.status
            recs.append({
                "kind": s.kind, "epsilon_achieved": s.epsilon_achieved, "u_max": s.u_max, "topk_min": s.topk_min,
                "fallback": o.fallback_used, "sub_size": int(o.stats.sub_size),
                "clusters_opened": int(o.stats.clusters_opened), "heap_pops": int(o.stats.heap_pops),
                "rho": o.stats.rho, "xi": o.stats.xi,
                "ids_sha256": digest(o.token_ids, "<i8"), "logits_sha256": digest(o.logits, "<f8"),
                "ids_head": o.token_ids[:64].tolist(), "logits_head": o.logits[:64].tolist(),
                "seconds": time.time() - t1,
            })
            Us.append(csvd.cluster_bounds(ix, h).values)
            print(f"  step {i}: {s.kind} fb={o.fallback_used} |S|={o.stats.sub_size} "
                  f"opened={o.stats.clusters_opened} ({time.time() - t1:.2f} s)", flush=True)
    finally:
        csvd_decode._check_table_index = real_check
    meta = {"config": name, "V": V, "d": d, "C": C, "g": g, "dtype": c["dtype"], "cfg": {k: v for k, v in c["cfg"].items()},
            "n_ctx": c["n_ctx"], "n_rand": c["n_rand"], "spread": SPREAD, "noise": NOISE, "table_seed": TABLE_SEED,
            "query_seed": Q_SEED, "random_seed": R_SEED, "numpy": np.__version__, "python": platform.python_version(),
            "machine": platform.machine(), "steps": recs}
    out = os.path.join(HERE, f"fullsize_{name}.npz")
    np.savez_compressed(out, meta=np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8), U=np.array(Us))
    print(f"wrote {out} ({os.path.getsize(out) / 1e3:.0f} kB) in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    for nm in (sys.argv[1:] or ["c2", "c3"]):
        make(nm)
