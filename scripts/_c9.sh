mkdir -p gpurun_out/c9
export PYTHONUNBUFFERED=1
for s in "4096 4096 4096 2 4" "2305 2561 4200 2 4" "4096 4096 4096 4 8" "4096 4096 4096 1 2" "4096 4096 4096 8 8" "2304 2560 4096 5 3" "2304 2560 4224 3 8"; do
APMM_DEBUG_WAITS=1 timeout 60 python scripts/fused_check.py $s 20 >> gpurun_out/c9/fc.txt 2>&1 || { echo FAIL $s >> gpurun_out/c9/fc.txt; break; }
done
echo "== ablate 3" >> gpurun_out/c9/fc.txt
APMM_FUSED_ABLATE=3 APMM_DEBUG_WAITS=1 timeout 60 python scripts/fused_check.py 4096 4096 4096 2 4 20 >> gpurun_out/c9/fc.txt 2>&1
