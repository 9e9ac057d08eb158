timeout 600 python tools/bench_batch.py 16 64 > gpurun_out/s39_c3_pair.txt 2>&1
CSVD_KBB_PAIR=0 timeout 600 python tools/bench_batch.py 16 64 > gpurun_out/s39_c3_single.txt 2>&1
timeout 600 python tools/bench_big.py c5 64 128 > gpurun_out/s39_c5_pair.txt 2>&1
CSVD_KBB_PAIR=0 timeout 600 python tools/bench_big.py c5 64 128 > gpurun_out/s39_c5_single.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_batch.py -q -x 2>&1 | tail -3 > gpurun_out/s39_pytest.txt
