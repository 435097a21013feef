mkdir -p gpurun_out/abl
export PYTHONUNBUFFERED=1
timeout 100 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -q -x -k "stream_tensor or graph or every_route" > gpurun_out/abl/k6_tests.txt 2>&1; echo rc=$? >> gpurun_out/abl/k6_tests.txt
timeout 100 python scripts/decode_bench.py 30 8192x16,8192x32,4096x16,11008x16,4096x16x11008 > gpurun_out/abl/k6_1launch.txt 2>&1
timeout 100 python scripts/route_sweep.py 4096 4096 2 4 16,32,64 >> gpurun_out/abl/k6_1launch.txt 2>&1
