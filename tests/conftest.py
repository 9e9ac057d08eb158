"""Shared fixtures: golden-case loading, outcome comparison, markers.

Golden fixtures (tests/golden/*.npz) were produced by running the reference
itself (tests/golden/make_golden.py).  Tables are regenerated from their
recipe with the bit-exact synth_vocab replica; k-means indexes are stored.
"""

from __future__ import annotations

import glob
import json
import math
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from paper_2511_21702_b200 import types as T  # noqa: E402
from paper_2511_21702_b200 import workload as wl  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
KIND_NAMES = {0: "topk_exact", 1: "softmax_eps", 2: "topp_mass"}
FB_NAMES = {-1: None, 0: "partial_expand", 1: "relax_eps", 2: "full_vocab"}

# Tolerance for transcendental-derived scalars (rho, delta mass, xi):
# numpy's SIMD exp/log and CUDA's differ by ~1 ulp, so these
# compare at 1e-12 relative; everything else is bit-exact.
TRANS_RTOL = 1e-12


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def golden_names():
    """Small-case fixtures of make_golden.py (full-size ones: make_fullsize.py)."""
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if not os.path.basename(p).startswith(("fullsize_", "harness_")))


class GoldenCase:
    def __init__(self, name):
        z = np.load(os.path.join(GOLDEN, name + ".npz"))
        self.z = {k: z[k] for k in z.files}
        self.meta = json.loads(bytes(self.z["meta"]).decode())
        self.name = name
        self._table = None
        self._index = None

    @property
    def table(self):
        if self._table is None:
            r = self.meta["table"]
            dtype = "bf16" if len(r) > 5 and r[5] == "bf16" else "f32"
            self._table = wl.synth_vocab(r[0], r[1], r[2], r[3], r[4], dtype=dtype)
        return self._table

    @property
    def index(self):
        if self._index is None:
            rec = self.meta["index"]
            if rec is not None and rec["kind"] == "fast":
                self._index = wl.fast_index(self.table, rec["n_modes"], rec["g"], mode=self.meta["mode"])
            else:
                self._index = self._stored_index()
        return self._index

    def _stored_index(self):
        z = self.z
        C = z["index_starts"].shape[0]
        m = self.meta["bias_depth"]
        clusters = []
        for c in range(C):
            row = z["index_bias_topm"][c]
            topm = tuple((float(row[2 * i]), int(row[2 * i + 1])) for i in range(m) if not math.isnan(row[2 * i]))
            clusters.append(T.ClusterMeta(
                centroid=z["index_centroids"][c], centroid_norm=float(z["index_centroid_norms"][c]),
                radius=float(z["index_radii"][c]), angular=float(z["index_angulars"][c]),
                max_bias=float(z["index_max_biases"][c]), max_norm=float(z["index_max_norms"][c]),
                min_norm=float(z["index_min_norms"][c]), bias_topm=topm,
                start=int(z["index_starts"][c]), end=int(z["index_starts"][c] + z["index_sizes"][c])))
        return T.ClusterIndex(clusters=clusters, perm=z["index_perm"], mode=self.meta["mode"],
                              vocab_size=int(z["index_perm"].shape[0]),
                              hidden_dim=int(z["index_centroids"].shape[1]) - (1 if self.meta["mode"] == "bias_augmented" else 0),
                              bias_depth=m, fingerprint=bytes(z["index_fingerprint"]))

    def cfg(self, i):
        doc = self.meta["cfgs"][i]
        fb = []
        for name, arg in doc["fallback"]:
            if name == "partial_expand":
                fb.append(T.PartialExpand(int(arg)))
            elif name == "relax_eps":
                fb.append(T.RelaxEps(float(arg)))
            else:
                fb.append(T.FullVocab())
        return T.DecodeConfig(k=doc["k"], epsilon=doc["epsilon"], targets=tuple(doc["targets"]),
                              k_max=doc["k_max"], fallback=tuple(fb), slack_mode=doc["slack_mode"])

    def steps(self):
        z = self.z
        for s in range(z["steps_cfg"].shape[0]):
            km = int(z["steps_kmax"][s])
            yield dict(
                i=s,
                variant="incremental" if z["steps_variant"][s] == 0 else "batchselect",
                cfg=self.cfg(int(z["steps_cfg"][s])),
                k_max=None if km < 0 else km,
                h=z["queries"][int(z["steps_query"][s])],
            )

    def expected(self, s):
        z = self.z
        a, b = int(z["ptr"][s]), int(z["ptr"][s + 1])
        sc = z["scal"][s]
        it = z["ints"][s]
        return dict(
            ids=z["ids"][a:b], logits=z["logits"][a:b],
            kind=KIND_NAMES[int(it[0])], fallback=FB_NAMES[int(it[1])], sub_size=int(it[2]),
            clusters_opened=int(it[3]), heap_pops=int(it[4]), flops_sparse=int(it[5]), flops_bounds=int(it[6]),
            eps=float(sc[0]), u_max=float(sc[1]), topk_min=float(sc[2]), rho=float(sc[3]), xi=float(sc[4]),
            ratio=float(sc[5]), qn=float(sc[6]), slack=float(sc[7]), U=z["U"][s],
        )


def close(a: float, b: float, rtol: float) -> bool:
    if math.isnan(a) or math.isnan(b):
        return math.isnan(a) and math.isnan(b)
    if a == b:
        return True
    return abs(a - b) <= rtol * max(abs(a), abs(b))


def outcome_fields(out):
    """Normalise a product DecodeOutcome or an oracle OOutcome."""
    st = out.stats
    g = (lambda k: st[k]) if isinstance(st, dict) else (lambda k: getattr(st, k))
    return dict(
        ids=np.asarray(out.token_ids), logits=np.asarray(out.logits), kind=out.status.kind,
        fallback=out.fallback_used, sub_size=g("sub_size"), clusters_opened=g("clusters_opened"),
        heap_pops=g("heap_pops"), flops_sparse=g("flops_sparse"), flops_bounds=g("flops_bounds"),
        eps=out.status.epsilon_achieved, u_max=out.status.u_max, topk_min=out.status.topk_min,
        rho=g("rho"), xi=g("xi"), ratio=g("ratio"),
    )


def assert_outcome(out, exp, rtol=TRANS_RTOL, where="", exact_bounds=True):
    """exact_bounds=False for the spherical cone bound (acos/cos, ~1 ulp):
    u_max and xi then compare at `rtol`; every decision stays exact."""
    got = outcome_fields(out)
    for key in ("kind", "fallback", "sub_size", "clusters_opened", "heap_pops", "flops_sparse", "flops_bounds"):
        assert got[key] == exp[key], f"{where}: {key} {got[key]!r} != {exp[key]!r}"
    assert np.array_equal(got["ids"], exp["ids"]), f"{where}: token_ids differ"
    assert np.array_equal(got["logits"], exp["logits"]), f"{where}: logits not bit-equal"
    # exact comparisons (no transcendentals): bounds and k-th logit
    btol = 0.0 if exact_bounds else max(rtol, 1e-12)
    assert close(float(got["u_max"]), float(exp["u_max"]), btol), \
        f"{where}: u_max {got['u_max']!r} != {exp['u_max']!r}"
    assert got["topk_min"] == exp["topk_min"], f"{where}: topk_min differs"
    assert got["ratio"] == exp["ratio"]
    # xi = (max-min)/(u_max-min): exact inputs, exact arithmetic
    assert close(float(got["xi"]), float(exp["xi"]), btol), f"{where}: xi {got['xi']!r} vs {exp['xi']!r}"
    for key in ("eps", "rho"):
        assert close(float(got[key]), float(exp[key]), rtol), f"{where}: {key} {got[key]!r} vs {exp[key]!r}"


@pytest.fixture(scope="session")
def golden_cases():
    return {n: GoldenCase(n) for n in golden_names()}
