mkdir -p gpurun_out/c21
for w in decode sweep4096; do timeout 300 python bench.py --workload $w > gpurun_out/c21/bench_$w.log 2>&1; done
