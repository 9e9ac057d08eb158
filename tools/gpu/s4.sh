set -x
timeout 300 compute-sanitizer --print-limit 5 python tools/repro_single.py > gpurun_out/s4_sanitizer.txt 2>&1
for v in default NO_HEAD HEAD_NOCOND; do
  if [ $v = default ]; then E=""; else E="CSVD_$v=1"; fi
  env $E timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-batch > gpurun_out/s4_bench_$v.json 2> gpurun_out/s4_bench_$v.err
done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/s4_pytest.txt
timeout 900 python bench.py --steps 200 --no-cpu-baseline > gpurun_out/s4_bench_full.json 2> gpurun_out/s4_bench_full.err
