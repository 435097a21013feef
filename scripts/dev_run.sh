mkdir -p gpurun_out/abl
timeout 60 scripts/mma_rate_probe > gpurun_out/abl/mma_rate2.txt 2>&1
