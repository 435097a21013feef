mkdir -p gpurun_out/abl
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/ -q -x -m gpu -k "stream_tensor or graph or every_route" > gpurun_out/abl/cr_tests.txt 2>&1; echo rc=$? >> gpurun_out/abl/cr_tests.txt
grep -q "rc=0" gpurun_out/abl/cr_tests.txt && for v in prev rel; do echo "== $v"; L=$PWD/abtest/lib_$v.so; [ $v = rel ] && L=$PWD/paper_2409_17870_b200/libapmm_b200.so; APMM_LIB=$L timeout 100 python scripts/decode_bench.py 40 8192x16,8192x32,4096x16,11008x16,4096x16x11008,8192x64; done > gpurun_out/abl/cr.txt 2>&1
grep -q "rc=0" gpurun_out/abl/cr_tests.txt && for v in prev rel; do echo "== $v"; L=$PWD/abtest/lib_$v.so; [ $v = rel ] && L=$PWD/paper_2409_17870_b200/libapmm_b200.so; APMM_LIB=$L timeout 100 python scripts/route_sweep.py 4096 4096 2 4 32,64,96,128; APMM_LIB=$L timeout 100 python scripts/route_sweep.py 11008 4096 2 4 64,128;  done >> gpurun_out/abl/cr.txt 2>&1
