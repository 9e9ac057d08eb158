"""Debug: per-phase device timestamps of the head step (CSVD_DEBUG_TS=1)."""
import ctypes
import os
import sys

import numpy as np

os.environ["CSVD_DEBUG_TS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_21702_b200 as P  # noqa: E402
from paper_2511_21702_b200 import _lib, workload as wl  # noqa: E402

V, d, C, g = [int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (128256, 4096, 1024, 16))]
dtype = os.environ.get("DTYPE", "f32")
T = wl.synth_vocab(V, d, C // g, 0.3, 1, dtype=dtype)
ix = wl.fast_index(T, C // g, g)
q = wl.generate_queries(12, d, "contextual", 7, centroids=ix.centroids)
ctx = P.prepare(T, ix)
lib = _lib.load()
lib.csvd_debug_timestamps.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
cfg = P.DecodeConfig(k=10)
names = {24: "kernel start", 51: "cert warm-up done", 63: "seg certifier used (+2)", 25: "h staged", 26: "cta0 bounds done", 27: "barrier passed", 28: "head done (cta0)",
         29: "cta0: head rows complete", 31: "cta0: certified", 30: "decision published", 32: "stage_bounds", 33: "order: top cluster", 34: "order: membership", 35: "order: rest + rank", 55: "cert: T (k-th segment max)", 56: "cert: candidates gathered", 58: "cert: k-th selected", 52: "cert: staged + max", 53: "cert: clusters + top-k", 54: "cert: prefixes", 40: "scan: min/max prefix", 41: "scan: log Z prefix",
         42: "scan: 64-merge recompute", 43: "scan: k-th merges", 44: "scan: rho/delta", 45: "scan: ballot+merge",
         46: "scan: state machine", 48: "summary: min/max", 49: "summary: warp min/max", 50: "summary: lse",
         51: "summary: sort"}
for i, h in enumerate(q):
    buf = np.zeros(128 + 512, dtype=np.uint64)
    if not os.environ.get("NOFLUSH"):
        lib.csvd_l2_flush(ctx._ctx, None)
    out = ctx.step(h, ctx.make_config(cfg))
    lib.csvd_debug_timestamps(ctx._ctx, buf.ctypes.data)
    if i < 2:
        continue
    t0 = int(buf[24])
    nb = ctx.info()["grid_ctas"]
    rd = buf[384:384 + min(nb, 256)].astype(np.int64) - t0
    print(f"step {i}: clusters={out.stats.clusters_opened} waves={ctx._res.waves} kind={out.status.kind} "
          f"fb={out.fallback_used}")
    print(f"   rows done per CTA: first {rd.min() / 1e3:.2f} median {np.median(rd) / 1e3:.2f} "
          f"last {rd.max() / 1e3:.2f} us")
    print(f"   seg result {int(buf[63]) - 2} (1 decided, 0 general, -1 fallback)")

    print(f"   candidates / certify path {int(buf[60])} (1 = block-parallel), fast result {int(buf[59]) - 2} "
          f"(1 decided, 0 general, -1 full certifier), hn {int(buf[61])}, R {int(buf[62])}")
    sd = buf[128:128 + min(nb, 256)].astype(np.int64) - t0
    print(f"   decision seen per CTA: first {sd.min() / 1e3:.2f} median {np.median(sd) / 1e3:.2f} "
          f"last {sd.max() / 1e3:.2f} us")
    for slot in sorted(names, key=lambda s: int(buf[s]) if buf[s] else 1 << 62):
        if buf[slot]:
            print(f"   {names[slot]:>22s}: {(int(buf[slot]) - t0) / 1000:8.2f} us")
    if i > 6:
        break
