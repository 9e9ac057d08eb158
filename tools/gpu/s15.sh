timeout 300 python tools/head_times.py > gpurun_out/s15_head_times.txt 2>&1
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-batch > gpurun_out/s15_bench.json 2> gpurun_out/s15_bench.err
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:k_head --launch-skip 8 --launch-count 1 -o gpurun_out/s15_head python bench.py --steps 10 --warmup 5 --no-cpu-baseline --no-batch > gpurun_out/s15_ncu.log 2>&1
timeout 600 python tools/bench_batch.py 1 16 64 > gpurun_out/s15_bench_batch.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/s15_pytest.txt
