timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/r2_head1_pytest.txt
timeout 300 python tools/head_times.py > gpurun_out/r2_head1_times.txt 2>&1
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-batch > gpurun_out/r2_head1_bench.json 2> gpurun_out/r2_head1_bench.err
CSVD_NO_HEAD=1 timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-batch > gpurun_out/r2_head1_bench_nohead.json 2>> gpurun_out/r2_head1_bench.err
