mkdir -p gpurun_out/abl
export PYTHONUNBUFFERED=1
timeout 100 python -m pytest tests/test_gpu_parity.py -q -x -k "skinny or decode or config4 or ragged" > gpurun_out/abl/k5_tests.txt 2>&1; echo rc=$? >> gpurun_out/abl/k5_tests.txt
export APMM_LIB=$PWD/abtest/libapmm_b200_dev.so
for ip in 0 1; do echo "== inprep $ip"; APMM_SK_INPREP=$ip timeout 100 python scripts/decode_bench.py 30 8192x1,8192x8,4096x8,11008x8,4096x1; done > gpurun_out/abl/k5_inprep2.txt 2>&1
