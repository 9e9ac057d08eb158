timeout 2000 python bench.py > gpurun_out/s31_bench_full.json 2> gpurun_out/s31_bench_full.err
