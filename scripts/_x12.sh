mkdir -p gpurun_out/x12
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "mid_size or fused" > gpurun_out/x12/pytest_mid.log 2>&1; echo rc=$? >> gpurun_out/x12/pytest_mid.log
APMM_MID=1 timeout 200 python scripts/msweep.py 4096 4096 2 4 > gpurun_out/x12/m.txt 2>&1
APMM_MID=1 timeout 200 python scripts/msweep.py 11008 4096 2 4 >> gpurun_out/x12/m.txt 2>&1
