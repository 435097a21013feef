mkdir -p gpurun_out/c23
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/c23/pytest.log 2>&1; echo rc=$? >> gpurun_out/c23/pytest.log
for w in sweep4096 decode; do timeout 300 python bench.py --workload $w > gpurun_out/c23/bench_$w.log 2>&1; done
