mkdir -p gpurun_out/c7
export PYTHONUNBUFFERED=1
for s in "4096 4096 4096 2 4" "2305 2561 4200 2 4" "4096 4096 4096 4 8"; do
APMM_DEBUG_WAITS=1 APMM_DEBUG_PLAN=1 timeout 60 python scripts/fused_check.py $s 20 >> gpurun_out/c7/fc.txt 2>&1 || { echo FAIL $s >> gpurun_out/c7/fc.txt; break; }
done
