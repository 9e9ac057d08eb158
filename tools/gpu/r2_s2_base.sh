set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/s2_pytest.txt
timeout 300 python tools/head_times.py > gpurun_out/s2_head_times.txt 2>&1
timeout 600 python bench.py > gpurun_out/s2_bench_default.json 2> gpurun_out/s2_bench_default.err
