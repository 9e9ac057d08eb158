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
q = (wl.generate_queries(12, d, "random", 8) if os.environ.get("QUERIES") == "random"
     else wl.generate_queries(12, d, "contextual", 7, centroids=ix.centroids))
ctx = P.prepare(T, ix)
lib = _lib.load()
lib.csvd_debug_timestamps.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
cfg = P.DecodeConfig(k=10)
names = {36: "dense rows start", 37: "dense rows + barrier done", 0: "kernel start", 1: "h staged", 2: "cta0 bounds done", 3: "barrier1 passed",
         4: "order done (head|full)", 5: "head done", 6: "wave 1 planned", 30: "  U loaded", 31: "  sorted",
         32: "  cum/x done", 33: "  e done", 34: "  lrh done", 35: "  lrh done (RESCALE)",
         40: "  scan: min/max", 41: "  scan: lse prefix", 42: "  scan: 64-merge", 43: "  scan: kth lists",
         44: "  scan: rho/delta", 45: "  scan: ballot/jump", 46: "  scan: run", 47: "  next_wave",
         48: "  sum: loaded", 49: "  sum: min/max", 50: "  sum: exp-sum", 51: "  sum: sorted", 52: "  sum: loads issued", 53: "  sum: loads landed"}
for w in range(4):
    names.update({8 + 4 * w: f"wave{w} rows start", 9 + 4 * w: f"wave{w} barrier passed",
                  10 + 4 * w: f"wave{w} summaries loaded", 11 + 4 * w: f"wave{w} scan+plan done"})
for i, h in enumerate(q):
    buf = np.zeros(128 + 512, dtype=np.uint64)
    import ctypes as C_
    if not os.environ.get("NOFLUSH"):
        lib.csvd_l2_flush(ctx._ctx, None)
    out = ctx.step(h, ctx.make_config(cfg))
    lib.csvd_debug_timestamps(ctx._ctx, buf.ctypes.data)
    if i < 2:
        continue
    t0 = int(buf[0])
    nb = ctx.info()["grid_ctas"]
    st_ = buf[128:128 + nb].astype(np.int64)
    en_ = buf[384:384 + nb].astype(np.int64)
    if st_.all() and en_.all():
        t0_ = int(buf[0])
        print(f"CTA starts: first {(st_.min() - t0_) / 1e3:.2f} last {(st_.max() - t0_) / 1e3:.2f} us; "
              f"CTA ends: first {(en_.min() - t0_) / 1e3:.2f} median {(np.median(en_) - t0_) / 1e3:.2f} "
              f"last {(en_.max() - t0_) / 1e3:.2f} us (slowest CTA {int(en_.argmax())})")
    rw = buf[512:640].astype(np.int64)
    if rw.any():
        rw = rw[rw > 0]
        print(f"rows done per CTA: first {(rw.min() - int(buf[0])) / 1e3:.2f} median {(np.median(rw) - int(buf[0])) / 1e3:.2f} last {(rw.max() - int(buf[0])) / 1e3:.2f} us")
    print(f"head n = {int(buf[63])}")
    buf[63] = 0
    print(f"step {i}: clusters={out.stats.clusters_opened} waves={ctx._res.waves} kind={out.status.kind} fb={out.fallback_used}")
    prev = None
    for slot in sorted(names, key=lambda s: int(buf[s]) if buf[s] else 1 << 62):
        if buf[slot]:
            ghz = ""
            if prev is not None and buf[64 + slot] and buf[64 + prev] and int(buf[slot]) > int(buf[prev]):
                dc = int(buf[64 + slot]) - int(buf[64 + prev])
                dt = int(buf[slot]) - int(buf[prev])
                if 0 < dc < 1e9:
                    ghz = f"   {dc / dt:5.2f} cyc/ns over {dc} cyc"
            print(f"   {names[slot]:>22s}: {(int(buf[slot]) - t0) / 1000:8.2f} us{ghz}")
            prev = slot
    if i > 4:
        break
