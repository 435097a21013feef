mkdir -p gpurun_out/abl
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "stream_tensor" > gpurun_out/abl/k6_tests.txt 2>&1
echo rc=$? >> gpurun_out/abl/k6_tests.txt
( timeout 200 python scripts/route_sweep.py 8192 8192 3 8 8,16,32,48,64
  timeout 200 python scripts/route_sweep.py 4096 4096 2 4 8,16,32,64 ) > gpurun_out/abl/route_sweep_k6.txt 2>&1
