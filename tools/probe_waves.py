import ctypes, sys
import numpy as np
sys.path.insert(0, ".")
import paper_2511_21702_b200 as P
from paper_2511_21702_b200 import _lib, workload as wl
V, d, C = 151552, 3584, 2273
T = wl.synth_vocab(V, d, C, 0.3, 1, dtype="bf16")
ix = wl.fast_index(T, C, 1)
B = 16
Q = wl.generate_queries(B * 3, d, "contextual", 7, centroids=ix.centroids)
cfg = P.DecodeConfig(k=10, epsilon=1e-3, targets=("softmax_eps",))
ctx = P.prepare(T, ix)
lib = _lib.load()
cs = ctx.make_config(cfg)
res = (_lib.Result * B)()
ids = np.empty((B, V), dtype=np.int64); lg = np.empty((B, V))
for i in range(2):
    rc = lib.csvd_step_batch_host(ctx._ctx, B, np.ascontiguousarray(Q[i*B:(i+1)*B]).ctypes.data, ctypes.byref(cs), res, ids.ctypes.data, lg.ctypes.data, V)
    print(rc, [(res[b].kind, res[b].fallback, res[b].waves, res[b].sub_size) for b in range(4)])
o = ctx.step(Q[0], cs)
print("single:", o.status.kind, o.fallback_used, ctx._res.waves, o.stats.sub_size)
