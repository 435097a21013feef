mkdir -p gpurun_out/c6
export PYTHONUNBUFFERED=1
timeout 120 ncu --set full --import-source on --clock-control none -k regex:wplanes --launch-skip 3 -c 1 -o gpurun_out/c6/fused_w2a4 python scripts/fused_check.py 4096 4096 4096 2 4 5 > gpurun_out/c6/ncu.log 2>&1
