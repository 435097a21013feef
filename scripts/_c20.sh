mkdir -p gpurun_out/c20
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/c20/pytest.log 2>&1; echo rc=$? >> gpurun_out/c20/pytest.log
timeout 100 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c20/smoke.log 2>&1
for w in sweep4096 decode; do timeout 300 python bench.py --workload $w > gpurun_out/c20/bench_$w.log 2>&1; done
