"""Batched-decode throughput probe (c3-like shapes): device-timed graph replays
of csvd_step_batch_device, L2 flushed between replays, B sweep."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2511_21702_b200 as P  # noqa: E402
from paper_2511_21702_b200 import _lib, workload as wl  # noqa: E402

V, d, n_modes, g = 151552, 3584, 2273, 1
dtype = "bf16"
if len(sys.argv) > 1 and sys.argv[1] == "c2":  # V=128256 d=4096 C=1024 shape
    V, d, n_modes, g, dtype = 128256, 4096, 64, 16, "f32"
    sys.argv.pop(1)
t0 = time.time()
T = wl.synth_vocab(V, d, n_modes, 0.3, 1, dtype=dtype)
ix = wl.fast_index(T, n_modes, g)
print(f"setup {time.time() - t0:.1f}s C={ix.n_clusters}", flush=True)
ctx = P.prepare(T, ix)
lib = _lib.load()
sp = ctypes.c_void_p()
lib.csvd_stream(ctx._ctx, ctypes.byref(sp))
ext = torch.cuda.ExternalStream(sp.value)
cfg = P.DecodeConfig(k=10, epsilon=1e-3, targets=("softmax_eps",))
ccfg = ctx.make_config(cfg)
Q = wl.generate_queries(128 * 6, d, "contextual", 7, centroids=ix.centroids)
Hd = torch.from_numpy(Q).cuda()
outs = ctx.step_batch(Q[:16], ccfg)
print("opened per query:", [o.stats.clusters_opened for o in outs], "fb:", [o.fallback_used for o in outs][:8],
      "sub:", int(np.mean([o.stats.sub_size for o in outs])), flush=True)
for B in [int(x) for x in (sys.argv[1:] or ["1", "4", "8", "16", "32", "64"])]:
    times = []
    for it in range(12):
        lib.csvd_l2_flush(ctx._ctx, sp)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        Hb = Hd[(it % 6) * B:(it % 6) * B + B] if (it % 6) * B + B <= Hd.shape[0] else Hd[:B]
        e0.record(ext)
        rc = lib.csvd_step_batch_device(ctx._ctx, B, Hb.data_ptr(), ctypes.byref(ccfg), sp)
        e1.record(ext)
        assert rc == 0, lib.csvd_strerror(ctx._ctx)
        torch.cuda.synchronize()
        if it >= 2:
            times.append(e0.elapsed_time(e1))
    lanes, grid = ctypes.c_int32(), ctypes.c_int32()
    lib.csvd_batch_lanes(ctx._ctx, ctypes.byref(lanes), ctypes.byref(grid))
    ms = float(np.median(times))
    print(f"B={B:4d} lanes={lanes.value} ctas/lane={grid.value}: {ms * 1e3:8.1f} us/batch  "
          f"{B / ms * 1e3:10.0f} query-steps/s", flush=True)
# single-query reference point
times = []
for it in range(12):
    lib.csvd_l2_flush(ctx._ctx, sp)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    lib.csvd_step_device(ctx._ctx, Hd[it].data_ptr(), ctypes.byref(ccfg), sp)
    e1.record(ext)
    torch.cuda.synchronize()
    if it >= 2:
        times.append(e0.elapsed_time(e1))
print(f"single-query step: {np.median(times) * 1e3:.1f} us")
