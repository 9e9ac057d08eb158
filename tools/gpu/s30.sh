set -x
mkdir -p gpurun_out/r2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2/launches_c2.csv python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-batch > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:k_head --launch-skip 8 --launch-count 1 -o /tmp/r2_head_c2 python bench.py --steps 10 --warmup 5 --no-cpu-baseline --no-batch > /dev/null 2>&1
python tools/ncu_summary.py /tmp/r2_head_c2.ncu-rep sparse_step_c2 > gpurun_out/r2/ncu_head_c2.json
ncu -i /tmp/r2_head_c2.ncu-rep --page source --csv --print-source sass > /tmp/src.csv 2>/dev/null; python tools/ncu_lines.py /tmp/src.csv paper_2511_21702_b200/_build/obj/k_float_8_1.o _Z6k_headIfLi1EEv3Dev 40 > gpurun_out/r2/ncu_head_c2_lines.txt 2>&1
timeout 900 ncu --set full --clock-control none --kernel-name regex:k_dense_gemv --launch-count 1 -o /tmp/r2_dense_c2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-batch > /dev/null 2>&1
python tools/ncu_summary.py /tmp/r2_dense_c2.ncu-rep dense_gemv_c2 > gpurun_out/r2/ncu_dense_c2.json
timeout 900 ncu --set full --clock-control none --kernel-name regex:k_head --launch-skip 2 --launch-count 1 -o /tmp/r2_fallback_c2 python tools/fallback_probe.py > /dev/null 2>&1
python tools/ncu_summary.py /tmp/r2_fallback_c2.ncu-rep fallback_step_c2 > gpurun_out/r2/ncu_fallback_c2.json
timeout 900 ncu --set full --clock-control none --kernel-name regex:"k_bounds_batch|k_head_lanes" --launch-skip 4 --launch-count 2 -o /tmp/r2_batch_c3 python tools/bench_batch.py 16 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/r2_batch_c3.ncu-rep batched_bounds_c3_b16 head_lanes_c3_b16 > gpurun_out/r2/ncu_batch_c3.json
timeout 600 python tools/bench_batch.py 16 64 128 > gpurun_out/r2/bench_batch_c3.txt 2>&1
ls -la gpurun_out/r2
