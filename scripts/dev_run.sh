mkdir -p gpurun_out/abl
export PYTHONUNBUFFERED=1
APMM_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/abl/bench_2rank.log 2>&1; echo rc=$? >> gpurun_out/abl/bench_2rank.log
