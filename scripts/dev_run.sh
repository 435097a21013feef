mkdir -p gpurun_out/abl
export PYTHONUNBUFFERED=1
for v in "" _s3 _s4; do echo "== stages lib$v"; APMM_LIB=$PWD/abtest/libapmm_b200_dev$v.so timeout 120 python scripts/decode_bench.py 30 8192x1,8192x8,8192x16,4096x1,11008x1,4096x1x11008,4096x16; done > gpurun_out/abl/decode_stages.txt 2>&1
