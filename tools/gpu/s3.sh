set -x
timeout 300 compute-sanitizer --print-limit 5 python tools/repro_single.py > gpurun_out/s3_sanitizer.txt 2>&1
timeout 60 ./tools/code_addr_probe > gpurun_out/s3_code_addr_probe.txt 2>&1
timeout 120 ./tools/latency_probe > gpurun_out/s3_latency_probe.txt 2>&1
timeout 60 ./tools/icache_probe > gpurun_out/s3_icache_probe.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/s3_launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-batch > gpurun_out/s3_ncu_bench.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q --deselect "tests/test_kat.py::test_singleton_bound_is_exact_logit[gpu]" 2>&1 | tail -15 > gpurun_out/s3_pytest.txt
