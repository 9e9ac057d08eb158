"""Random (non-contextual) c2 queries through decode_step: every step walks
the fallback chain to the full-vocabulary level (profiling helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_21702_b200 as P  # noqa: E402
from paper_2511_21702_b200 import workload as wl  # noqa: E402

T = wl.synth_vocab(128256, 4096, 64, 0.3, 1)
ix = wl.fast_index(T, 64, 16)
for h in wl.generate_queries(5, 4096, "random", 8):
    o = P.decode_step(T, ix, h, P.DecodeConfig(k=10))
    print(o.fallback_used, o.stats.clusters_opened)
