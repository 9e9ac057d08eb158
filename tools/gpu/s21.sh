timeout 300 python tools/head_times.py > gpurun_out/s21_head_times.txt 2>&1
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-batch > gpurun_out/s21_bench.json 2> gpurun_out/s21_bench.err
CSVD_DEBUG_TS=1 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, paper_2511_21702_b200 as P
from paper_2511_21702_b200 import workload as wl
T=wl.synth_vocab(128256,4096,64,0.3,1); ix=wl.fast_index(T,64,16)
q=wl.generate_queries(4,4096,'random',8)
import time
for h in q:
    t=time.perf_counter(); o=P.decode_step(T,ix,h,P.DecodeConfig(k=10)); print(o.fallback_used, o.stats.clusters_opened, time.perf_counter()-t)
" > gpurun_out/s21_fallback.txt 2>&1
timeout 900 python tests/golden/make_harness_fixture.py > gpurun_out/s21_harness.txt 2>&1
