timeout 300 python tools/head_times.py > gpurun_out/s11_head_times.txt 2>&1
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-batch > gpurun_out/s11_bench.json 2> gpurun_out/s11_bench.err
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/s11_pytest.txt
