timeout 300 python tools/head_times.py > gpurun_out/s16_head_times.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -15 > gpurun_out/s16_pytest.txt
timeout 600 python tools/bench_batch.py 1 16 64 > gpurun_out/s16_bench_batch.txt 2>&1
