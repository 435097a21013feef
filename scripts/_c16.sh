mkdir -p gpurun_out/c16
export PYTHONUNBUFFERED=1
timeout 200 python -m pytest tests/test_gpu_parity.py -x -q -k "skinny or config4" > gpurun_out/c16/pytest.log 2>&1; echo rc=$? >> gpurun_out/c16/pytest.log
for st in 2 3 4; do
echo "== stages $st" >> gpurun_out/c16/grid.txt
APMM_SK_STAGES=$st timeout 100 python scripts/decode_bench.py 30 >> gpurun_out/c16/grid.txt 2>&1
done
