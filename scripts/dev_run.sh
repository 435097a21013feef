mkdir -p gpurun_out/abl
export PYTHONUNBUFFERED=1
APMM_LIB=$PWD/abtest/lib_ooo.so timeout 120 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -q -x -k "stream_tensor or graph" > gpurun_out/abl/ooo_tests.txt 2>&1; echo rc=$? >> gpurun_out/abl/ooo_tests.txt
grep -q "rc=0" gpurun_out/abl/ooo_tests.txt && for v in rel ooo; do echo "== $v"; APMM_LIB=$PWD/abtest/lib_$v.so timeout 100 python scripts/decode_bench.py 40 8192x16,8192x32,4096x16,11008x16,4096x16x11008; done > gpurun_out/abl/ooo.txt 2>&1
grep -q "rc=0" gpurun_out/abl/ooo_tests.txt && for v in rel ooo; do echo "== $v"; APMM_LIB=$PWD/abtest/lib_$v.so timeout 100 python scripts/route_sweep.py 4096 4096 2 4 64,128; done >> gpurun_out/abl/ooo.txt 2>&1
