set -x
timeout 300 python tools/head_times.py > gpurun_out/s5_head_times.txt 2>&1
for v in default NO_HEAD HEAD_NOCOND; do
  if [ $v = default ]; then E=""; else E="CSVD_$v=1"; fi
  env $E timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-batch > gpurun_out/s5_bench_$v.json 2> gpurun_out/s5_bench_$v.err
done
CSVD_NO_HEAD=1 timeout 300 python tools/phase_times.py > gpurun_out/s5_phase_times_nohead.txt 2>&1
timeout 600 python tools/bench_batch.py 1 16 > gpurun_out/s5_bench_batch.txt 2>&1
