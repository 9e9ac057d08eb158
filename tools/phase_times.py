"""Debug: per-phase device timestamps of one step (CSVD_DEBUG_TS=1)."""
import ctypes
import os
import sys

import numpy as np

os.environ["CSVD_DEBUG_TS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_21702_b200 as P  # noqa: E402
from paper_2511_21702_b200 import _lib, workload as wl  # noqa: E402

V, d, C, g = [int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (128256, 4096, 1024, 16))]
T = wl.synth_vocab(V, d, C // g, 0.3, 1)
ix = wl.fast_index(T, C // g, g)
q = wl.generate_queries(12, d, "contextual", 7, centroids=ix.centroids)
ctx = P.prepare(T, ix)
lib = _lib.load()
lib.csvd_debug_timestamps.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
cfg = P.DecodeConfig(k=10)
names = {0: "bounds start", 1: "h staged", 2: "qnorm", 3: "cta0 rows done", 4: "last cta start",
         5: "slack/keys", 6: "sorted", 7: "scans", 8: "published", 9: "bounds end",
         16: "wave0 start", 17: "wave0 h staged", 22: "wave0 first row", 18: "wave0 final summary",
         19: "wave0 scan start", 20: "wave0 scan end", 21: "wave0 planned",
         24: "wave1 start", 25: "wave1 staged", 30: "wave1 first row", 26: "wave1 final", 27: "wave1 scan start",
         28: "wave1 scan end", 29: "wave1 planned"}
for i, h in enumerate(q):
    buf = np.zeros(64, dtype=np.uint64)
    import ctypes as C_
    lib.csvd_l2_flush(ctx._ctx, None)
    out = ctx.step(h, ctx.make_config(cfg))
    lib.csvd_debug_timestamps(ctx._ctx, buf.ctypes.data)
    if i < 2:
        continue
    t0 = int(buf[0])
    print(f"step {i}: clusters={out.stats.clusters_opened} waves={ctx._res.waves}")
    for slot in sorted(names, key=lambda s: int(buf[s]) if buf[s] else 1 << 62):
        if buf[slot]:
            print(f"   {names[slot]:>22s}: {(int(buf[slot]) - t0) / 1000:8.2f} us")
    if i > 4:
        break
