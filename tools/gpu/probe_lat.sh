timeout 120 ./tools/latency_probe > gpurun_out/latency_probe.txt 2>&1
