mkdir -p gpurun_out/abl
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -q -x -m gpu > gpurun_out/abl/pytest_gpu.txt 2>&1; echo rc=$? >> gpurun_out/abl/pytest_gpu.txt
for w in llama7b_mid llama7b_small decode; do timeout 300 python bench.py --workload $w > gpurun_out/abl/bench_$w.log 2>&1; done
