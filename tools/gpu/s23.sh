timeout 300 python tools/head_times.py > gpurun_out/s23_head_times.txt 2>&1
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-batch > gpurun_out/s23_bench.json 2> gpurun_out/s23_bench.err
timeout 600 python tools/bench_batch.py 16 64 > gpurun_out/s23_bench_batch.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/s23_pytest.txt
