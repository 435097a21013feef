mkdir -p gpurun_out/c8
export PYTHONUNBUFFERED=1
for a in 0 1 2 3; do
echo "== ablate $a" >> gpurun_out/c8/fc.txt
APMM_FUSED_ABLATE=$a APMM_DEBUG_WAITS=1 timeout 60 python scripts/fused_check.py 4096 4096 4096 2 4 20 >> gpurun_out/c8/fc.txt 2>&1
done
