mkdir -p gpurun_out/abl
export PYTHONUNBUFFERED=1
for v in rel bst8; do echo "== $v"; APMM_LIB=$PWD/abtest/lib_$v.so timeout 100 python scripts/decode_bench.py 40 8192x16,8192x32,4096x16,11008x16,4096x16x11008; done > gpurun_out/abl/k6_bst8.txt 2>&1
