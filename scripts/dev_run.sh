mkdir -p gpurun_out/abl
export PYTHONUNBUFFERED=1
APMM_LIB=$PWD/abtest/lib_bst6.so timeout 100 python -m pytest tests/test_gpu_parity.py -q -x -k "stream_tensor" > gpurun_out/abl/k6_tests.txt 2>&1; echo rc=$? >> gpurun_out/abl/k6_tests.txt
for v in prev bst4 bst6; do echo "== $v"; APMM_LIB=$PWD/abtest/lib_$v.so timeout 100 python scripts/decode_bench.py 40 8192x16,8192x32,4096x16,11008x16,4096x16x11008; done > gpurun_out/abl/k6_bst.txt 2>&1
for v in prev bst6; do echo "== $v"; APMM_LIB=$PWD/abtest/lib_$v.so timeout 100 python scripts/route_sweep.py 4096 4096 2 4 64,128; done >> gpurun_out/abl/k6_bst.txt 2>&1
