mkdir -p gpurun_out/abl
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -q -x -m gpu > gpurun_out/abl/pytest_gpu.txt 2>&1; echo rc=$? >> gpurun_out/abl/pytest_gpu.txt
