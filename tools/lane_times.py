"""Debug: phase timestamps of batch lane 0's CTA 0 (CSVD_DEBUG_TS=1).
python tools/lane_times.py c5|c4|c3 B"""
import ctypes
import os
import sys

import numpy as np

os.environ["CSVD_DEBUG_TS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_21702_b200 as P  # noqa: E402
from paper_2511_21702_b200 import _lib, workload as wl  # noqa: E402
names = {24: "kernel start", 51: "cert warm-up done", 63: "seg certifier used (+2)", 25: "h staged", 26: "cta0 bounds done", 27: "barrier passed", 28: "head done (cta0)",
         29: "cta0: head rows complete", 31: "cta0: certified", 30: "decision published", 32: "stage_bounds", 33: "order: top cluster", 34: "order: membership", 35: "order: rest + rank", 55: "cert: T (k-th segment max)", 56: "cert: candidates gathered", 58: "cert: k-th selected", 52: "cert: staged + max", 53: "cert: clusters + top-k", 54: "cert: prefixes", 40: "scan: min/max prefix", 41: "scan: log Z prefix",
         42: "scan: 64-merge recompute", 43: "scan: k-th merges", 44: "scan: rho/delta", 45: "scan: ballot+merge",
         46: "scan: state machine", 48: "summary: min/max", 49: "summary: warp min/max", 50: "summary: lse",
         51: "summary: sort"}

which, B = sys.argv[1], int(sys.argv[2])
V, d, C, g, dt = {"c4": (128256, 8192, 1024, 16, "f32"), "c5": (256000, 3584, 3840, 16, "bf16"),
                  "c2": (128256, 4096, 1024, 16, "f32")}[which]
T = wl.synth_vocab(V, d, C // g, 0.3, 1, dtype=dt)
ix = wl.fast_index(T, C // g, g)
ctx = P.prepare(T, ix)
lib = _lib.load()
lib.csvd_debug_timestamps.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
cfg = P.DecodeConfig(k=10)
Q = wl.generate_queries(3 * B, d, "contextual", 7, centroids=ix.centroids)
for it in range(3):
    buf = np.zeros(128 + 512, dtype=np.uint64)
    lib.csvd_l2_flush(ctx._ctx, None)
    outs = ctx.step_batch(Q[it * B:(it + 1) * B], ctx.make_config(cfg))
    lib.csvd_debug_timestamps(ctx._ctx, buf.ctypes.data)
    if it == 0:
        continue
    t0 = int(buf[24])
    print(f"iter {it}: lane 0 clusters={outs[0].stats.clusters_opened} sub={outs[0].stats.sub_size}")
    for slot in sorted(names, key=lambda s: int(buf[s]) if buf[s] else 1 << 62):
        if buf[slot] and slot not in (57, 59, 60, 61, 62, 63):
            print(f"   {names[slot]:>28s}: {(int(buf[slot]) - t0) / 1000:8.2f} us")
