timeout 600 python bench.py --steps 500 --warmup 10 --no-cpu-baseline --no-batch > gpurun_out/s37_bench_zc.json 2> gpurun_out/s37_bench_zc.err
CSVD_H_COPY=1 timeout 600 python bench.py --steps 500 --warmup 10 --no-cpu-baseline --no-batch > gpurun_out/s37_bench_copy.json 2> gpurun_out/s37_bench_copy.err
timeout 600 python tools/e2e_host_probe.py > gpurun_out/s37_e2e.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/s37_pytest.txt
