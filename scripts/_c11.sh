mkdir -p gpurun_out/c11
export PYTHONUNBUFFERED=1
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/c11/pytest.log 2>&1; echo rc=$? >> gpurun_out/c11/pytest.log
timeout 100 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c11/smoke.log 2>&1
