QUERIES=random CSVD_NO_HEAD=1 timeout 300 python tools/phase_times.py > gpurun_out/s26_phase_random.txt 2>&1
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-batch > gpurun_out/s26_bench.json 2> gpurun_out/s26_bench.err
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/s26_pytest.txt
