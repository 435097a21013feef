mkdir -p gpurun_out/x10
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "mid_size" > gpurun_out/x10/pytest_mid.log 2>&1; echo rc=$? >> gpurun_out/x10/pytest_mid.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/x10/pytest.log 2>&1; echo rc=$? >> gpurun_out/x10/pytest.log
APMM_DEBUG_PLAN=1 timeout 200 python scripts/msweep.py 4096 4096 2 4 > gpurun_out/x10/m.txt 2>&1
timeout 200 python scripts/msweep.py 11008 4096 2 4 >> gpurun_out/x10/m.txt 2>&1
