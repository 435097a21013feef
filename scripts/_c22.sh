mkdir -p gpurun_out/c22
export PYTHONUNBUFFERED=1
timeout 200 python -m pytest tests/test_gpu_parity.py -x -q -k "skinny or config4" > gpurun_out/c22/pytest.log 2>&1; echo rc=$? >> gpurun_out/c22/pytest.log
for pf in 0 4 8 16 64; do for st in 2 3; do
echo "== prefetch $pf stages $st" >> gpurun_out/c22/grid.txt
APMM_SK_PREFETCH=$pf APMM_SK_STAGES=$st timeout 100 python scripts/decode_bench.py 30 8192x1,8192x8,8192x16,4096x1,11008x16 >> gpurun_out/c22/grid.txt 2>&1
done; done
