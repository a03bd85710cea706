mkdir -p gpurun_out/s2
timeout 120 ./tools/umma_probe > gpurun_out/s2/umma_probe.txt 2>&1
