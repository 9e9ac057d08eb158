"""Where the batched e2e time goes (c3 shape, B=16)."""
import ctypes
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2511_21702_b200 as P  # noqa: E402
from paper_2511_21702_b200 import _lib, workload as wl  # noqa: E402

V, d, C = 151552, 3584, 2273
T = wl.synth_vocab(V, d, C, 0.3, 1, dtype="bf16")
ix = wl.fast_index(T, C, 1)
B = 16
Q = wl.generate_queries(B * 60, d, "contextual", 7, centroids=ix.centroids)
cfg = P.DecodeConfig(k=10, epsilon=1e-3, targets=("softmax_eps",))
ctx = P.prepare(T, ix)
lib = _lib.load()
cs = ctx.make_config(cfg)
for i in range(5):
    ctx.step_batch(Q[i * B:(i + 1) * B], cs)
res = (_lib.Result * B)()
ids = np.empty((B, V), dtype=np.int64)
lg = np.empty((B, V), dtype=np.float64)
n = 40
tc = to = 0.0
for i in range(5, 5 + n):
    H = np.ascontiguousarray(Q[i * B:(i + 1) * B])
    t0 = time.perf_counter()
    rc = lib.csvd_step_batch_host(ctx._ctx, B, H.ctypes.data, ctypes.byref(cs), res, ids.ctypes.data, lg.ctypes.data, V)
    t1 = time.perf_counter()
    outs = [ctx._outcome(res[b], ids[b, :int(res[b].sub_size)].copy(), lg[b, :int(res[b].sub_size)].copy())
            for b in range(B)]
    t2 = time.perf_counter()
    tc += t1 - t0
    to += t2 - t1
print(f"C call {1e6 * tc / n:.1f} us, python outcomes {1e6 * to / n:.1f} us per batch of {B}")
t0 = time.perf_counter()
for i in range(5, 5 + n):
    P.decode_step_batch(T, ix, Q[i * B:(i + 1) * B], cfg)
print(f"decode_step_batch {1e6 * (time.perf_counter() - t0) / n:.1f} us per batch")
import torch  # noqa: E402
sp = ctypes.c_void_p()
lib.csvd_stream(ctx._ctx, ctypes.byref(sp))
ext = torch.cuda.ExternalStream(sp.value)
Hd = torch.from_numpy(Q).cuda()
torch.cuda.synchronize()
t0 = time.perf_counter()
ev = []
for i in range(5, 5 + n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    lib.csvd_step_batch_device(ctx._ctx, B, Hd[i * B:(i + 1) * B].data_ptr(), ctypes.byref(cs), sp)
    e1.record(ext)
    e1.synchronize()
    ev.append(e0.elapsed_time(e1))
print(f"device graph: wall {1e6 * (time.perf_counter() - t0) / n:.1f} us per batch (sync each), events {1e3 * np.median(ev):.1f} us")
