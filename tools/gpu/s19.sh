timeout 300 python tools/head_times.py > gpurun_out/s19_head_times.txt 2>&1
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-batch > gpurun_out/s19_bench.json 2> gpurun_out/s19_bench.err
timeout 600 python tools/bench_batch.py 1 16 64 > gpurun_out/s19_bench_batch.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s19_batch_launches.csv python tools/bench_batch.py 16 64 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_kat.py tests/test_gpu_parity.py -q -x 2>&1 | tail -15 > gpurun_out/s19_pytest.txt
