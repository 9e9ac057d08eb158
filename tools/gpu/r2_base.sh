set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2_base_pytest.txt
timeout 300 python tools/phase_times.py > gpurun_out/r2_base_phases.txt 2>&1
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --batch-steps 10 > gpurun_out/r2_base_bench.json 2> gpurun_out/r2_base_bench.err
