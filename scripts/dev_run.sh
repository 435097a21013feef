mkdir -p gpurun_out/abl
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "skinny or decode or config4 or ragged" > gpurun_out/abl/k5b4_tests.txt 2>&1; echo rc=$? >> gpurun_out/abl/k5b4_tests.txt
for r in 1 2; do for v in prev rel; do echo "== $v"; L=$PWD/abtest/lib_$v.so; [ $v = rel ] && L=$PWD/paper_2409_17870_b200/libapmm_b200.so; APMM_LIB=$L timeout 100 python scripts/decode_bench.py 40 8192x1,8192x8,4096x8,11008x8,4096x1,4096x1x11008; done; done > gpurun_out/abl/k5b4.txt 2>&1
