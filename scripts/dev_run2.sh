mkdir -p gpurun_out/abl
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/ -q -x -m gpu -k "stream_tensor or skinny or graph or every_route" > gpurun_out/abl/pf_tests.txt 2>&1; echo rc=$? >> gpurun_out/abl/pf_tests.txt
for v in prev rel prev rel; do echo "== $v"; L=$PWD/abtest/lib_$v.so; [ $v = rel ] && L=$PWD/paper_2409_17870_b200/libapmm_b200.so; APMM_LIB=$L timeout 100 python scripts/decode_bench.py 40 8192x1,8192x8,4096x1,4096x8,8192x16,4096x16,11008x16; done > gpurun_out/abl/pf.txt 2>&1
