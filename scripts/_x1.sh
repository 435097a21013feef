mkdir -p gpurun_out/x1
export PYTHONUNBUFFERED=1
for cl in 2 4; do
echo "== cluster $cl" >> gpurun_out/x1/fc.txt
for s in "4096 4096 4096 2 4" "8192 8192 8192 2 4" "28672 4096 8192 2 4"; do
APMM_PAIR_CLUSTER=$cl APMM_DEBUG_PLAN=1 timeout 60 python scripts/skinny_probe.py $s 20 >> gpurun_out/x1/fc.txt 2>&1
done; done
