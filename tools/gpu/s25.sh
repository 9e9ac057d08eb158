timeout 300 python tools/head_times.py > gpurun_out/s25_head_times.txt 2>&1
timeout 1500 python bench.py > gpurun_out/s25_bench_full.json 2> gpurun_out/s25_bench_full.err
