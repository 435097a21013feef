mkdir -p gpurun_out/x2
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/x2/pytest.log 2>&1; echo rc=$? >> gpurun_out/x2/pytest.log
for s in "4096 4096 4096 2 4" "8192 8192 8192 2 4" "28672 4096 8192 2 4" "11008 2048 4096 2 4"; do
timeout 60 python scripts/skinny_probe.py $s 20 >> gpurun_out/x2/fc.txt 2>&1
done
for w in ffn70b sweep4096 llama7b; do timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/x2/bench_$w.log 2>&1; done
