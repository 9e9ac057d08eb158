timeout 300 python tools/head_times.py > gpurun_out/r2_head2_times.txt 2>&1
NOFLUSH=1 timeout 300 python tools/head_times.py > gpurun_out/r2_head2_times_noflush.txt 2>&1
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-batch > gpurun_out/r2_head2_bench.json 2> gpurun_out/r2_head2_bench.err
CSVD_NO_HEAD=1 timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-batch > gpurun_out/r2_head2_bench_nohead.json 2>> gpurun_out/r2_head2_bench.err
