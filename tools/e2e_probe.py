"""Where the e2e (host API) time goes: Python wrapper vs the C call."""
import ctypes
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2511_21702_b200 as P  # noqa: E402
from paper_2511_21702_b200 import _lib, engine, workload as wl  # noqa: E402

V, d, C, g = 128256, 4096, 1024, 16
T = wl.synth_vocab(V, d, C // g, 0.3, 1)
ix = wl.fast_index(T, C // g, g)
q = wl.generate_queries(300, d, "contextual", 7, centroids=ix.centroids)
cfg = P.DecodeConfig(k=10)
ctx = P.prepare(T, ix)
lib = _lib.load()
for i in range(20):
    P.decode_step(T, ix, q[i], cfg)
acc = {"prepare": 0.0, "make_config": 0.0, "c_call": 0.0, "outcome": 0.0, "total": 0.0}
n = 200
for i in range(n):
    h = q[20 + i]
    t0 = time.perf_counter()
    c = P.prepare(T, ix)
    t1 = time.perf_counter()
    cs = c.make_config(cfg, None, _lib.VARIANT_INCREMENTAL)
    t2 = time.perf_counter()
    hh = np.ascontiguousarray(h, dtype=np.float64)
    rc = lib.csvd_step_host(c._ctx, hh.ctypes.data, ctypes.byref(cs), ctypes.byref(c._res), c._ids.ctypes.data,
                            c._logits.ctypes.data, c.V)
    t3 = time.perf_counter()
    r = c._res
    m = int(r.sub_size)
    out = c._outcome(r, c._ids[:m].copy(), c._logits[:m].copy())
    t4 = time.perf_counter()
    acc["prepare"] += t1 - t0
    acc["make_config"] += t2 - t1
    acc["c_call"] += t3 - t2
    acc["outcome"] += t4 - t3
    acc["total"] += t4 - t0
print({k: f"{1e6 * v / n:.1f} us" for k, v in acc.items()})
t0 = time.perf_counter()
for i in range(n):
    P.decode_step(T, ix, q[20 + i], cfg)
print(f"decode_step: {1e6 * (time.perf_counter() - t0) / n:.1f} us/call")
