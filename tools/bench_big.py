"""c4 / c5 batched timings (device-timed graph replays, L2 flushed):
python tools/bench_big.py c4|c5 B..."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2511_21702_b200 as P  # noqa: E402
from paper_2511_21702_b200 import _lib, workload as wl  # noqa: E402

which = sys.argv[1]
V, d, C, g, dt = (128256, 8192, 1024, 16, "f32") if which == "c4" else (256000, 3584, 3840, 16, "bf16")
T = wl.synth_vocab(V, d, C // g, 0.3, 1, dtype=dt)
ix = wl.fast_index(T, C // g, g)
ctx = P.prepare(T, ix)
lib = _lib.load()
sp = ctypes.c_void_p()
lib.csvd_stream(ctx._ctx, ctypes.byref(sp))
ext = torch.cuda.ExternalStream(sp.value)
cfg = P.DecodeConfig(k=10)
ccfg = ctx.make_config(cfg)
Q = wl.generate_queries(128 * 4, d, "contextual", 7, centroids=ix.centroids)
Hd = torch.from_numpy(Q).cuda()
for B in [int(x) for x in sys.argv[2:]]:
    ts = []
    for it in range(6):
        lib.csvd_l2_flush(ctx._ctx, sp)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        rc = lib.csvd_step_batch_device(ctx._ctx, B, Hd[(it % 4) * B:(it % 4) * B + B].data_ptr(), ctypes.byref(ccfg), sp)
        e1.record(ext)
        assert rc == 0, lib.csvd_strerror(ctx._ctx)
        torch.cuda.synchronize()
        if it >= 2:
            ts.append(e0.elapsed_time(e1))
    print(f"{which} B={B}: {np.median(ts) * 1e3:.1f} us/batch", flush=True)
