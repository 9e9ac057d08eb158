timeout 300 python tools/head_times.py > gpurun_out/s10_head_times.txt 2>&1
NOFLUSH=1 timeout 300 python tools/head_times.py > gpurun_out/s10_head_times_noflush.txt 2>&1
