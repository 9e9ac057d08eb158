timeout 60 ./tools/code_addr_probe > gpurun_out/code_addr_probe.txt 2>&1
timeout 60 ./tools/icache_probe > gpurun_out/icache_probe.txt 2>&1
