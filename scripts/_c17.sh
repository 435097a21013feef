mkdir -p gpurun_out/c17
export PYTHONUNBUFFERED=1
for w in decode sweep4096 llama7b_small; do timeout 300 python bench.py --workload $w > gpurun_out/c17/bench_$w.log 2>&1; done
