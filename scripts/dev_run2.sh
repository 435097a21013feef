mkdir -p gpurun_out/abl
export PYTHONUNBUFFERED=1 APMM_LIB=$PWD/abtest/libapmm_b200_dev.so APMM_TRACE=16 ROUTE=STREAM_TC
for s in "4096 16 4096 2 4" "4096 64 4096 2 4"; do timeout 60 python scripts/trace_timeline.py $s 4; done > gpurun_out/abl/k6_tl2.txt 2>&1
