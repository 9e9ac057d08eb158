"""Where the host-API step's time goes (c2): decode_step vs ctx.step vs the
raw C call, plus the C entry point's own launch / wait split."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2511_21702_b200 as P  # noqa: E402
from paper_2511_21702_b200 import _lib, workload as wl  # noqa: E402

T = wl.synth_vocab(128256, 4096, 64, 0.3, 1)
ix = wl.fast_index(T, 64, 16)
q = wl.generate_queries(400, 4096, "contextual", 7, centroids=ix.centroids)
cfg = P.DecodeConfig(k=10)
ctx = P.prepare(T, ix)
lib = _lib.load()
cc = ctx.make_config(cfg)
for i in range(20):
    P.decode_step(T, ix, q[i], cfg)


def timeit(fn, n=300):
    t = time.perf_counter()
    for i in range(n):
        fn(q[i % 400])
    return (time.perf_counter() - t) / n * 1e6


res = _lib.Result()
ids = np.empty(128256, dtype=np.int64)
lg = np.empty(128256)
print(f"decode_step:      {timeit(lambda h: P.decode_step(T, ix, h, cfg)):7.1f} us")
print(f"ctx.step(cfg):    {timeit(lambda h: ctx.step(h, cc)):7.1f} us")
print(f"raw C call:       {timeit(lambda h: lib.csvd_step_host(ctx._ctx, h.ctypes.data, ctypes.byref(cc), ctypes.byref(res), ids.ctypes.data, lg.ctypes.data, 128256)):7.1f} us")
sp = ctypes.c_void_p()
lib.csvd_stream(ctx._ctx, ctypes.byref(sp))
hd = torch.from_numpy(q).cuda()
t = time.perf_counter()
for i in range(300):
    lib.csvd_step_device(ctx._ctx, hd[i % 400].data_ptr(), ctypes.byref(cc), sp)
    torch.cuda.synchronize()
print(f"device step + sync: {(time.perf_counter() - t) / 300 * 1e6:7.1f} us")
