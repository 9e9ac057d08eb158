"""Synthetic inputs for tests and bench (NOT the hot path).

The hot path takes the offline clustering result as input; this module only
manufactures such inputs on machines where the reference is absent (the GPU
box), with the reference's own conventions so CPU and GPU see identical data:

* `synth_vocab`   -- restates tensor_io.synth_vocab (tensor_io.py:192-216):
  same RNG stream (default_rng(seed): centers, assignment, noise, bias), drawn
  in row chunks so a 128256 x 4096 table never needs a float64 copy; returns
  float32 (or bf16-rounded) weights, bit-equal to the reference's f32-exact
  float64 values.
* `fast_index`    -- SURVEY.md §8(d): replays the synth RNG to recover every
  row's mode, splits each mode into `g` clusters by within-mode rank mod g and
  computes the per-cluster statistics with the reference's `_cluster_stats`
  arithmetic (cluster_index.py:254-279) in `build_index`'s ordering convention
  (cluster_index.py:305-316: size desc, ties by smallest member id; members
  ascending).  Seconds instead of hours; `validate_index` on the result is
  clean (tests/test_workload.py).
* `index_from_assignment` -- the same for any row -> cluster assignment.
* `generate_queries` -- restates bench.generate_queries (bench.py:183-209).
"""

from __future__ import annotations

import hashlib
import struct

import numpy as np

from .types import ClusterIndex, ClusterMeta, EmbeddingTable, f32_to_bf16_bits, bf16_bits_to_f32


def table_fingerprint(table) -> bytes:
    """tensor_io.table_fingerprint (tensor_io.py:219-226), any weight dtype."""
    w = table.weights
    h = hashlib.sha256()
    h.update(b"CSVD")
    h.update(struct.pack("<QQ", w.shape[0], w.shape[1]))
    if w.dtype == np.uint16:
        h.update(bf16_bits_to_f32(w).astype("<f4").tobytes())
    else:
        h.update(np.asarray(w).astype("<f4", copy=False).tobytes())
    h.update(np.asarray(table.bias).astype("<f4").tobytes())
    return h.digest()


def synth_vocab(V: int, d: int, n_modes: int, spread: float, seed: int,
                dtype: str = "f32", chunk_rows: int = 8192) -> EmbeddingTable:
    """Gaussian-mixture table, bit-equal to the reference's synth_vocab.

    dtype: "f32" (reference values), "f64" (reference layout), or "bf16"
    (reference values RNE-rounded to bf16, stored as uint16 bit patterns --
    feed the same rounded table to the reference for the bf16 variant)."""
    if V < 1 or d < 1:
        raise ValueError("V and d must be >= 1")
    if not 1 <= n_modes <= V:
        raise ValueError(f"need 1 <= n_modes <= V, got n_modes={n_modes}, V={V}")
    if spread < 0:
        raise ValueError("spread must be non-negative")
    rng = np.random.default_rng(seed)
    centers = rng.standard_normal((n_modes, d))
    assignment = rng.integers(0, n_modes, size=V)
    w32 = np.empty((V, d), dtype=np.float32)
    for s in range(0, V, chunk_rows):
        e = min(V, s + chunk_rows)
        noise = rng.standard_normal((e - s, d))
        w32[s:e] = (centers[assignment[s:e]] + spread * noise).astype(np.float32)
    bias = rng.uniform(-1.0, 1.0, size=V).astype(np.float32).astype(np.float64)
    if dtype == "f32":
        w = w32
    elif dtype == "f64":
        w = w32.astype(np.float64)
    elif dtype == "bf16":
        w = f32_to_bf16_bits(w32)
    else:
        raise ValueError(f"unknown dtype {dtype!r}")
    return EmbeddingTable(weights=w, bias=bias)


def synth_assignment(V: int, d: int, n_modes: int, seed: int) -> np.ndarray:
    """Replay tensor_io.synth_vocab's RNG up to the mode assignment."""
    rng = np.random.default_rng(seed)
    rng.standard_normal((n_modes, d))
    return rng.integers(0, n_modes, size=V)


def _rows_f64(table, members):
    w = table.weights[members]
    if w.dtype == np.uint16:
        return bf16_bits_to_f32(w).astype(np.float64)
    return w.astype(np.float64)


def _l2(v):
    return float(np.sqrt((v * v).sum()))


def _cluster_stats(table, members, mode, m):
    """cluster_index._cluster_stats (cluster_index.py:254-279), same arithmetic."""
    rows = _rows_f64(table, members)
    if mode == "bias_augmented":
        rows = np.hstack([rows, table.bias[members][:, None]])
    centroid = rows.mean(axis=0)
    centroid_norm = _l2(centroid)
    diff = rows - centroid
    radius = float(np.sqrt((diff * diff).sum(axis=1)).max())
    row_norms = np.sqrt((rows * rows).sum(axis=1))
    max_norm = float(row_norms.max())
    min_norm = float(row_norms.min())
    if mode == "spherical":
        if centroid_norm > 0 and (row_norms > 0).all():
            cosines = np.clip((rows * centroid).sum(axis=1) / (row_norms * centroid_norm), -1.0, 1.0)
            angular = float(np.arccos(cosines).max())
        else:
            angular = float(np.pi)
    else:
        angular = 0.0
    member_bias = table.bias[members]
    max_bias = float(member_bias.max())
    order = np.lexsort((members, -member_bias))[: min(m, members.size)]
    topm = tuple((float(member_bias[i]), int(members[i])) for i in order)
    return centroid, centroid_norm, radius, angular, max_bias, max_norm, min_norm, topm


def index_from_assignment(table, assignment: np.ndarray, mode: str = "euclidean",
                          m: int = 3, fingerprint: bytes | None = None) -> ClusterIndex:
    """ClusterIndex for a given row -> cluster label array (labels need not be dense)."""
    V = table.vocab_size
    assignment = np.asarray(assignment)
    order_rows = np.argsort(assignment, kind="stable")
    labels, starts_l = np.unique(assignment[order_rows], return_index=True)
    bounds_l = list(starts_l) + [V]
    member_lists = [np.sort(order_rows[bounds_l[i]:bounds_l[i + 1]]) for i in range(len(labels))]
    order = sorted(range(len(member_lists)),
                   key=lambda c: (-member_lists[c].size, int(member_lists[c][0])))
    clusters = []
    perm = np.empty(V, dtype=np.int64)
    pos = 0
    for c in order:
        members = member_lists[c]
        start, end = pos, pos + members.size
        perm[start:end] = members
        pos = end
        st = _cluster_stats(table, members, mode, m)
        clusters.append(ClusterMeta(
            centroid=st[0], centroid_norm=st[1], radius=st[2], angular=st[3],
            max_bias=st[4], max_norm=st[5], min_norm=st[6], bias_topm=st[7],
            start=start, end=end))
    if fingerprint is None:
        fingerprint = table_fingerprint(table)
    return ClusterIndex(clusters=clusters, perm=perm, mode=mode, vocab_size=V,
                        hidden_dim=table.hidden_dim, bias_depth=m, fingerprint=fingerprint)


def fast_index(table, n_modes: int, g: int, table_seed: int = 1, mode: str = "euclidean",
               m: int = 3, fingerprint: bytes | None = None) -> ClusterIndex:
    """SURVEY.md §8(d) fast index: synth modes split g ways (C = n_modes * g)."""
    V, d = table.vocab_size, table.hidden_dim
    modes = synth_assignment(V, d, n_modes, table_seed)
    # within-mode rank (rows ascending inside each mode)
    order_rows = np.argsort(modes, kind="stable")
    sorted_modes = modes[order_rows]
    first = np.searchsorted(sorted_modes, sorted_modes, side="left")
    rank = np.empty(V, dtype=np.int64)
    rank[order_rows] = np.arange(V) - first
    label = modes.astype(np.int64) * g + (rank % g)
    return index_from_assignment(table, label, mode=mode, m=m, fingerprint=fingerprint)


def generate_queries(n: int, hidden_dim: int, model: str, seed: int,
                     centroids: np.ndarray | None = None, noise: float = 0.3,
                     zipf_exponent: float = 1.1) -> np.ndarray:
    """bench.generate_queries (bench.py:183-209), unit-norm float64."""
    rng = np.random.default_rng(seed)
    if model == "random":
        q = rng.standard_normal((n, hidden_dim))
    elif model == "contextual":
        if centroids is None:
            raise ValueError("contextual queries need cluster centroids")
        cents = np.asarray(centroids, dtype=np.float64)[:, :hidden_dim]
        C = cents.shape[0]
        weights = 1.0 / np.arange(1, C + 1) ** zipf_exponent
        weights /= weights.sum()
        picks = rng.choice(C, size=n, p=weights)
        q = cents[picks] + noise * rng.standard_normal((n, hidden_dim))
    else:
        raise ValueError(f"unknown query model {model!r}")
    norms = np.sqrt((q * q).sum(axis=1))
    norms[norms == 0] = 1.0
    return q / norms[:, None]
