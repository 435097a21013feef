mkdir -p gpurun_out/abl
export PYTHONUNBUFFERED=1
export APMM_LIB=$PWD/abtest/libapmm_b200_dev.so
for sh in "8192 16 8192 3 8" "4096 16 4096 2 4"; do APMM_TC_TS_MODE=5 APMM_TRACE=16 timeout 60 python scripts/trace_k6_steps.py $sh; done > gpurun_out/abl/k6_steps5.txt 2>&1
