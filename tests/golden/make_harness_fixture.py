"""Step 2 of the reference-harness fixture (run on a B200): the device
outcomes of the reference's default bench workload (BenchSpec defaults:
V=5000 d=64, the reference's own k-means index from harness_index.csvi,
contextual queries seed 7, the AdaptiveBudget k_max trajectory), recorded
step by step into tests/golden/harness_outcomes.npz.
tests/test_harness_integration.py replays them through the UNMODIFIED
reference harness (csvd.bench.run_benchmark with the INTEGRATION.md
rebinding), whose _validate_step checks each one against the dense oracle.

usage (GPU box): python tests/golden/make_harness_fixture.py [out.npz]
(gpurun merges only gpurun_out/ back: write there, then copy into tests/golden/)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import paper_2511_21702_b200 as P  # noqa: E402
from paper_2511_21702_b200 import budget, formats, workload as wl  # noqa: E402

N_STEPS = 300
KIND = {"topk_exact": 0, "softmax_eps": 1, "topp_mass": 2}
FB = {None: -1, "partial_expand": 0, "relax_eps": 1, "full_vocab": 2}

table = wl.synth_vocab(5000, 64, 50, 0.05, 1)
index = formats.load_index(os.path.join(HERE, "harness_index.csvi"))
cfg = P.DecodeConfig(k=10, epsilon=0.05)
queries = wl.generate_queries(N_STEPS, 64, "contextual", 7, centroids=index.centroids, noise=0.3,
                              zipf_exponent=1.1)
bud = budget.AdaptiveBudget(cfg, index.vocab_size)
ids, logits, off, scal, ints = [], [], [0], [], []
for t in range(N_STEPS):
    k_eff = bud.effective_k_max(t)
    o = P.decode_step(table, index, queries[t], cfg, k_max=k_eff)
    bud.observe(o.fallback_used is not None)
    ids.append(o.token_ids)
    logits.append(o.logits)
    off.append(off[-1] + len(o.token_ids))
    s = o.status
    scal.append([s.epsilon_achieved, s.u_max, s.topk_min, o.stats.xi, o.stats.rho])
    ints.append([KIND[s.kind], FB[o.fallback_used], o.stats.sub_size, o.stats.clusters_opened,
                 o.stats.heap_pops, o.stats.flops_sparse, o.stats.flops_bounds, k_eff])
OUT = sys.argv[1] if len(sys.argv) > 1 else os.path.join(HERE, "harness_outcomes.npz")
np.savez_compressed(OUT, ids=np.concatenate(ids),
                    logits=np.concatenate(logits), off=np.array(off), scal=np.array(scal), ints=np.array(ints),
                    queries_sha=np.frombuffer(__import__("hashlib").sha256(queries.tobytes()).digest(), np.uint8))
print("steps", N_STEPS, "tokens", off[-1], "fallbacks", sum(i[1] >= 0 for i in ints))
