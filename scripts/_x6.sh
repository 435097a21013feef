mkdir -p gpurun_out/x6
export PYTHONUNBUFFERED=1
for b in 148 111 74 37; do
echo "== expand blocks $b" >> gpurun_out/x6/r.txt
APMM_EXPAND_BLOCKS=$b timeout 300 python bench.py --workload sweep4096 --no-cpu-baseline --steps 20 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['expand_us_avg'], d['clocks'])" >> gpurun_out/x6/r.txt 2>&1
done
