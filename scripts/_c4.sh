mkdir -p gpurun_out/c4
export PYTHONUNBUFFERED=1
APMM_DEBUG_PLAN=1 timeout 60 python scripts/fused_check.py 4096 4096 4096 2 4 20 > gpurun_out/c4/fc.txt 2>&1; echo rc=$? >> gpurun_out/c4/fc.txt
nvidia-smi --query-gpu=name,utilization.gpu --format=csv >> gpurun_out/c4/fc.txt
