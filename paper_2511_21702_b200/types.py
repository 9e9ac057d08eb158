"""Host-side mirrors of the reference's hot-path types.

Same names, fields, defaults and validation errors as the reference `csvd`
package, so code written against `csvd` runs unchanged against this package:

* `EmbeddingTable`   -- tensor_io.py:69-94
* `ClusterMeta` / `ClusterIndex` -- cluster_index.py:68-132
* `DecodeConfig`, `PartialExpand`, `RelaxEps`, `FullVocab`, `ConfigError`,
  `StepMetrics`, `DecodeOutcome` -- decode.py:63-139
* `CertStatus` -- certify.py:48-53
* `BoundVector` -- bounds.py:46-55
* `DenseResult` -- oracle.py:23-30

The functions in `engine.py` accept either these or the reference's own
objects (duck typing on the field names).

Deviation (documented in DESIGN.md): `EmbeddingTable` keeps float32 / bf16
(uint16 bit pattern) weights as given instead of promoting them to a float64
copy -- the values are identical (f32-exact) and the device upload never needs
the 2x host copy.  `weights_f64()` returns the reference's float64 view.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

NEG_INF = float("-inf")
TARGET_KINDS = ("topk", "softmax_eps", "topp")
MODES = ("euclidean", "spherical", "bias_augmented")


class ConfigError(ValueError):
    """decode.py:63-64."""


class FingerprintMismatchError(Exception):
    """cluster_index.py:59-60."""


class NonFiniteEntryError(Exception):
    """tensor_io.py:64-65 (FormatError subclass in the reference)."""


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bf16 bit pattern (finite inputs)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return rounded.astype(np.uint16)


@dataclass(frozen=True)
class EmbeddingTable:
    """Output-layer weights (V x d) plus bias (tensor_io.py:69-94).

    `weights` may be float64 (reference layout; must be f32-exact), float32,
    or uint16 holding bf16 bit patterns (the bf16-weight variant)."""

    weights: np.ndarray
    bias: np.ndarray

    def __post_init__(self):
        w = np.asarray(self.weights)
        if w.dtype not in (np.float64, np.float32, np.uint16):
            w = np.asarray(w, dtype=np.float64)
        w = np.ascontiguousarray(w)
        b = np.ascontiguousarray(np.asarray(self.bias, dtype=np.float64))
        if w.ndim != 2 or w.shape[0] < 1 or w.shape[1] < 1:
            raise ValueError(f"weights must be V x d with V,d >= 1, got shape {w.shape}")
        if b.shape != (w.shape[0],):
            raise ValueError(f"bias must have length V={w.shape[0]}, got shape {b.shape}")
        wf = bf16_bits_to_f32(w) if w.dtype == np.uint16 else w
        if not np.isfinite(wf).all() or not np.isfinite(b).all():
            raise NonFiniteEntryError("table contains non-finite entries")
        object.__setattr__(self, "weights", w)
        object.__setattr__(self, "bias", b)

    @property
    def vocab_size(self) -> int:
        return self.weights.shape[0]

    @property
    def hidden_dim(self) -> int:
        return self.weights.shape[1]

    def weights_f64(self) -> np.ndarray:
        w = self.weights
        if w.dtype == np.uint16:
            return bf16_bits_to_f32(w).astype(np.float64)
        return np.asarray(w, dtype=np.float64)


@dataclass(frozen=True)
class ClusterMeta:
    """cluster_index.py:68-83."""

    centroid: np.ndarray
    centroid_norm: float
    radius: float
    angular: float
    max_bias: float
    max_norm: float
    min_norm: float
    bias_topm: tuple
    start: int
    end: int

    @property
    def size(self) -> int:
        return self.end - self.start


@dataclass
class ClusterIndex:
    """cluster_index.py:86-132 (stacked per-cluster arrays for the hot path)."""

    clusters: list
    perm: np.ndarray
    mode: str
    vocab_size: int
    hidden_dim: int
    bias_depth: int
    fingerprint: bytes

    centroids: np.ndarray = field(init=False, repr=False)
    centroid_norms: np.ndarray = field(init=False, repr=False)
    radii: np.ndarray = field(init=False, repr=False)
    angulars: np.ndarray = field(init=False, repr=False)
    max_biases: np.ndarray = field(init=False, repr=False)
    max_norms: np.ndarray = field(init=False, repr=False)
    min_norms: np.ndarray = field(init=False, repr=False)
    sizes: np.ndarray = field(init=False, repr=False)
    starts: np.ndarray = field(init=False, repr=False)
    ends: np.ndarray = field(init=False, repr=False)
    inv_perm: np.ndarray = field(init=False, repr=False)

    def __post_init__(self):
        cs = self.clusters
        self.centroids = np.stack([c.centroid for c in cs])
        self.centroid_norms = np.array([c.centroid_norm for c in cs])
        self.radii = np.array([c.radius for c in cs])
        self.angulars = np.array([c.angular for c in cs])
        self.max_biases = np.array([c.max_bias for c in cs])
        self.max_norms = np.array([c.max_norm for c in cs])
        self.min_norms = np.array([c.min_norm for c in cs])
        self.sizes = np.array([c.size for c in cs], dtype=np.int64)
        self.starts = np.array([c.start for c in cs], dtype=np.int64)
        self.ends = np.array([c.end for c in cs], dtype=np.int64)
        self.perm = np.ascontiguousarray(self.perm, dtype=np.int64)
        inv = np.empty(self.vocab_size, dtype=np.int64)
        inv[self.perm] = np.arange(self.vocab_size)
        self.inv_perm = inv

    @property
    def n_clusters(self) -> int:
        return len(self.clusters)

    def members(self, c: int) -> np.ndarray:
        return self.perm[self.starts[c]: self.ends[c]]


@dataclass(frozen=True)
class PartialExpand:
    delta_c: int = 4
    name: str = field(default="partial_expand", init=False)


@dataclass(frozen=True)
class RelaxEps:
    factor: float = 2.0
    name: str = field(default="relax_eps", init=False)


@dataclass(frozen=True)
class FullVocab:
    name: str = field(default="full_vocab", init=False)


@dataclass(frozen=True)
class DecodeConfig:
    """decode.py:84-115 (same defaults; `validate` raises ConfigError)."""

    k: int = 10
    epsilon: float = 0.05
    targets: tuple = ("topk", "softmax_eps")
    k_max: int | None = None
    fallback: tuple = (PartialExpand(), RelaxEps(), FullVocab())
    adaptive_enabled: bool = False
    alpha: float = 0.01
    rho_target: float = 0.02
    ema_half_life: float = 100.0
    warmup_steps: int = 4
    warmup_factor: float = 2.0
    slack_mode: str = "none"

    def resolved_k_max(self, vocab_size: int) -> int:
        return resolved_k_max(self, vocab_size)

    def validate(self, vocab_size: int) -> None:
        validate_config(self, vocab_size)


def resolved_k_max(cfg, vocab_size: int) -> int:
    if cfg.k_max is None:
        return max(cfg.k, vocab_size // 2)
    return cfg.k_max


def validate_config(cfg, vocab_size: int) -> None:
    """decode.py:104-115, usable on the reference's DecodeConfig too."""
    if not cfg.targets or any(t not in TARGET_KINDS for t in cfg.targets):
        raise ConfigError(f"targets must be a non-empty subset of {TARGET_KINDS}")
    if not 1 <= cfg.k <= vocab_size:
        raise ConfigError(f"need 1 <= k <= V, got k={cfg.k}, V={vocab_size}")
    k_max = resolved_k_max(cfg, vocab_size)
    if not cfg.k <= k_max <= vocab_size:
        raise ConfigError(f"need k <= K_max <= V, got K_max={k_max}")
    if not 0 < cfg.epsilon < 1:
        raise ConfigError(f"epsilon must lie in (0, 1), got {cfg.epsilon}")
    if cfg.alpha < 0:
        raise ConfigError("alpha must be >= 0")


@dataclass(frozen=True)
class CertStatus:
    """certify.py:48-53."""

    kind: str
    epsilon_achieved: float
    u_max: float
    topk_min: float


@dataclass
class StepMetrics:
    """decode.py:118-130."""

    sub_size: int
    ratio: float
    clusters_opened: int
    xi: float
    cert_kind: str
    fallback: str | None
    rho: float
    flops_sparse: int
    flops_bounds: int
    heap_pops: int
    step: int = -1
    # B200 addition (not in the reference): a tested prefix's rho (or top-p
    # delta) was within 1e-12 relative of the threshold, i.e. the decision is
    # an ulp-level tie between the device's and numpy's exp/log
    tie_ambiguous: bool = False


@dataclass
class DecodeOutcome:
    """decode.py:133-139."""

    token_ids: np.ndarray
    logits: np.ndarray
    status: CertStatus
    fallback_used: str | None
    stats: StepMetrics


@dataclass(frozen=True)
class BoundVector:
    """bounds.py:46-55."""

    values: np.ndarray
    mode: str
    query_norm: float
    slack: float

    def __post_init__(self):
        if not np.isfinite(self.values).all():
            raise ValueError("bounds must be finite")


@dataclass(frozen=True)
class DenseResult:
    """oracle.py:23-30."""

    logits: np.ndarray
    probs: np.ndarray
    order: np.ndarray

    def topk(self, k: int) -> np.ndarray:
        return self.order[:k]


def is_nan(x: float) -> bool:
    return isinstance(x, float) and math.isnan(x)
