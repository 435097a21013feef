mkdir -p gpurun_out/c14
export PYTHONUNBUFFERED=1
timeout 200 python -m pytest tests/test_gpu_parity.py -x -q -k "skinny or config4" > gpurun_out/c14/pytest.log 2>&1; echo rc=$? >> gpurun_out/c14/pytest.log
APMM_SK_INPREP=1 timeout 200 python -m pytest tests/test_gpu_parity.py -x -q -k "skinny or config4" > gpurun_out/c14/pytest_inprep.log 2>&1; echo rc=$? >> gpurun_out/c14/pytest_inprep.log
for ip in 0 1; do for st in 0 2 3 4; do
echo "== inprep $ip stages $st" >> gpurun_out/c14/grid.txt
APMM_SK_INPREP=$ip APMM_SK_STAGES=$st timeout 100 python scripts/decode_bench.py 30 8192x1,8192x8,8192x16,4096x1,11008x16 >> gpurun_out/c14/grid.txt 2>&1
done; done
