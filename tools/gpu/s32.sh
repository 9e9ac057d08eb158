timeout 600 python tools/bench_batch.py 16 64 > gpurun_out/s32_bench_batch.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s32_batch_launches.csv python tools/bench_batch.py 16 64 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_batch.py -q -x 2>&1 | tail -5 > gpurun_out/s32_pytest.txt
