timeout 300 python tools/head_times.py > gpurun_out/s28_head_times.txt 2>&1
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-batch > gpurun_out/s28_bench.json 2> gpurun_out/s28_bench.err
DTYPE=bf16 timeout 300 python tools/head_times.py > gpurun_out/s28_head_times_bf16.txt 2>&1
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-batch --dtype bf16 > gpurun_out/s28_bench_bf16.json 2> gpurun_out/s28_bench_bf16.err
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/s28_pytest.txt
