mkdir -p gpurun_out/abl
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -q -x -m gpu > gpurun_out/abl/pytest_gpu.txt 2>&1; echo rc=$? >> gpurun_out/abl/pytest_gpu.txt
timeout 300 python bench.py --workload llama7b_mid > gpurun_out/abl/bench_mid.log 2>&1
