mkdir -p gpurun_out/abl
export PYTHONUNBUFFERED=1
timeout 400 python -m pytest tests/ -q -x -m gpu > gpurun_out/abl/rg_tests.txt 2>&1; echo rc=$? >> gpurun_out/abl/rg_tests.txt
grep -q "rc=0" gpurun_out/abl/rg_tests.txt && for v in prev rel; do echo "== $v"; L=$PWD/abtest/lib_$v.so; [ $v = rel ] && L=$PWD/paper_2409_17870_b200/libapmm_b200.so; APMM_LIB=$L timeout 100 python scripts/decode_bench.py 40 8192x63,4096x63,8192x16,4096x17,4096x125; done > gpurun_out/abl/rg.txt 2>&1
