set -x
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:k_head --launch-skip 8 --launch-count 1 -o gpurun_out/s7_head python bench.py --steps 10 --warmup 5 --no-cpu-baseline --no-batch > gpurun_out/s7_ncu.log 2>&1
ls -la gpurun_out/
