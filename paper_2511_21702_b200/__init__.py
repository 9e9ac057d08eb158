"""B200-native CSV-Decode output-layer hot path (drop-in for the `csvd` step API).

    from paper_2511_21702_b200 import decode_step, DecodeConfig
    out = decode_step(table, index, h, DecodeConfig(k=10))

Entry points mirror /root/reference/pkg/src/csvd/__init__.py for the hot path
(decode_step, decode_step_batchselect, sharded_decode_step, cluster_bounds,
dense_logits) and accept the reference's own table / index / config objects.
All compute runs in the sm_100a CUDA extension (include/csvd_b200.h); there
is no CPU fallback.
"""

from .types import (
    BoundVector,
    CertStatus,
    ClusterIndex,
    ClusterMeta,
    ConfigError,
    DecodeConfig,
    DecodeOutcome,
    DenseResult,
    EmbeddingTable,
    FingerprintMismatchError,
    FullVocab,
    PartialExpand,
    RelaxEps,
    StepMetrics,
)
from .engine import (
    DeviceIndex,
    clear_cache,
    cluster_bounds,
    decode_step,
    decode_step_batch,
    decode_step_batchselect,
    dense_logits,
    prepare,
    refined_bias_bound,
)
from .shard import CommLedger, LatencyModel, ShardPlan, make_plan, sharded_decode_step
from . import formats
from .cluster import build_index_gpu
from .budget import (AdaptiveBudget, BudgetedDecoder, FlopReport, adapt_budget, flop_accounting, flop_report,
                     warmup_k_max)

__version__ = "0.1.0"

__all__ = [
    "BoundVector", "CertStatus", "ClusterIndex", "ClusterMeta", "ConfigError", "DecodeConfig",
    "DecodeOutcome", "DenseResult", "EmbeddingTable", "FingerprintMismatchError", "FullVocab",
    "PartialExpand", "RelaxEps", "StepMetrics", "DeviceIndex", "clear_cache", "cluster_bounds",
    "decode_step", "decode_step_batch", "decode_step_batchselect", "dense_logits", "prepare", "refined_bias_bound", "CommLedger",
    "LatencyModel", "ShardPlan", "make_plan", "sharded_decode_step", "AdaptiveBudget", "BudgetedDecoder",
    "FlopReport", "adapt_budget", "flop_accounting", "flop_report", "warmup_k_max", "build_index_gpu",
]
