set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2_launches_c2.csv python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-batch > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:k_head --launch-skip 8 --launch-count 1 -o gpurun_out/r2_head_c2 python bench.py --steps 10 --warmup 5 --no-cpu-baseline --no-batch > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --kernel-name regex:k_dense_gemv --launch-count 1 -o gpurun_out/r2_dense_c2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-batch > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --kernel-name regex:k_head --launch-skip 2 --launch-count 1 -o gpurun_out/r2_fallback_c2 python tools/fallback_probe.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --kernel-name regex:"k_bounds_batch|k_head_lanes" --launch-skip 4 --launch-count 2 -o gpurun_out/r2_batch_c3 python tools/bench_batch.py 16 > /dev/null 2>&1
ls -la gpurun_out
