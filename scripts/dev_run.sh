# dev A/B run for the decode kernel; outputs under gpurun_out/abl
mkdir -p gpurun_out/abl
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -q -x -m gpu > gpurun_out/abl/pytest_gpu.txt 2>&1
for ip in -1 1; do echo "== inprep $ip"; APMM_LIB=$PWD/abtest/libapmm_b200_dev.so APMM_SK_INPREP=$ip timeout 120 python scripts/decode_bench.py 30; done > gpurun_out/abl/decode_inprep.txt 2>&1
