timeout 600 python tools/bench_big.py c5 16 64 128 > gpurun_out/s33_c5.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s33_c5_launches.csv python tools/bench_big.py c5 128 > /dev/null 2>&1
timeout 600 python tools/bench_big.py c4 64 > gpurun_out/s33_c4.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -5 > gpurun_out/s33_pytest.txt
