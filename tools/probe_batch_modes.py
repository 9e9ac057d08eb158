"""Host-API vs device-resident batch graphs, each after an L2 flush (for ncu)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2511_21702_b200 as P  # noqa: E402
from paper_2511_21702_b200 import _lib, workload as wl  # noqa: E402

V, d, C = 151552, 3584, 2273
T = wl.synth_vocab(V, d, C, 0.3, 1, dtype="bf16")
ix = wl.fast_index(T, C, 1)
B = 16
Q = wl.generate_queries(B * 8, d, "contextual", 7, centroids=ix.centroids)
cfg = P.DecodeConfig(k=10, epsilon=1e-3, targets=("softmax_eps",))
ctx = P.prepare(T, ix)
lib = _lib.load()
cs = ctx.make_config(cfg)
sp = ctypes.c_void_p()
lib.csvd_stream(ctx._ctx, ctypes.byref(sp))
Hd = torch.from_numpy(Q).cuda()
res = (_lib.Result * B)()
ids = np.empty((B, V), dtype=np.int64)
lg = np.empty((B, V))
for i in range(4):  # host mode
    lib.csvd_l2_flush(ctx._ctx, sp)
    torch.cuda.synchronize()
    lib.csvd_step_batch_host(ctx._ctx, B, np.ascontiguousarray(Q[i * B:(i + 1) * B]).ctypes.data, ctypes.byref(cs),
                             res, ids.ctypes.data, lg.ctypes.data, V)
for i in range(4):  # device mode
    lib.csvd_l2_flush(ctx._ctx, sp)
    lib.csvd_step_batch_device(ctx._ctx, B, Hd[i * B:(i + 1) * B].data_ptr(), ctypes.byref(cs), sp)
    torch.cuda.synchronize()
print("done")
