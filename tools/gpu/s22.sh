timeout 300 python tools/head_times.py > gpurun_out/s22_head_times.txt 2>&1
timeout 900 python tests/golden/make_harness_fixture.py gpurun_out/harness_outcomes.npz > gpurun_out/s22_harness.txt 2>&1
