"""Step 1 of the reference-harness fixture (run HERE, where /root/reference
exists): the reference's own default bench workload (BenchSpec defaults,
/root/reference/pkg/src/csvd/bench.py:100-131), its k-means index written
with the reference's writer (cluster_index.py:398-431) to
tests/golden/harness_index.csvi.  Step 2 (make_harness_fixture.py) runs on a
B200 and records the device outcomes of that workload's query stream.

usage: PYTHONPATH=/root/reference/pkg/src python tests/golden/make_harness_index.py
"""
import os

import csvd
from csvd.bench import BenchSpec
from csvd.cluster_index import build_index, save_index

HERE = os.path.dirname(os.path.abspath(__file__))

spec = BenchSpec()
table = csvd.synth_vocab(spec.vocab_size, spec.hidden_dim, spec.n_modes, spec.spread, spec.table_seed)
index = build_index(table, spec.resolved_clusters(), mode=spec.mode, iters=spec.iters, m=spec.bias_depth,
                    seed=spec.index_seed)
save_index(index, os.path.join(HERE, "harness_index.csvi"))
print("C =", index.n_clusters)
