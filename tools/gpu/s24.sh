timeout 300 python tools/head_times.py > gpurun_out/s24_head_times.txt 2>&1
QUERIES=random CSVD_NO_HEAD=1 timeout 300 python tools/phase_times.py > gpurun_out/s24_phase_random.txt 2>&1
