"""Run the full-vocabulary GEMV (K5) a few times at c2 shape (for ncu)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2511_21702_b200 as P  # noqa: E402
from paper_2511_21702_b200 import workload as wl  # noqa: E402

V, d = 128256, 4096
T = wl.synth_vocab(V, d, 64, 0.3, 1)
ix = wl.fast_index(T, 64, 16)
ctx = P.prepare(T, ix)
h = wl.generate_queries(1, d, "contextual", 7, centroids=ix.centroids)[0]
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    t0 = time.perf_counter()
    ctx.dense(h)
    print(f"dense host call {1e3 * (time.perf_counter() - t0):.2f} ms")
