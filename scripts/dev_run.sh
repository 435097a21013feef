mkdir -p gpurun_out/abl
export PYTHONUNBUFFERED=1
timeout 60 scripts/mma_rate_probe > gpurun_out/abl/mma_rate.txt 2>&1
timeout 100 python scripts/decode_bench.py 30 8192x16,8192x32,4096x16,11008x16,4096x16x11008,4096x64 > gpurun_out/abl/k6_w1rel.txt 2>&1
