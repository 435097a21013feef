# Scratch script for one-off GPU A/B runs through gpurun (dev): edit, then
#   /usr/local/graft/bin/gpurun --timeout 900 -- 'bash scripts/dev_run.sh'
# Results land under gpurun_out/abl (scratch); copy what is worth keeping into profiles/.
mkdir -p gpurun_out/abl
export PYTHONUNBUFFERED=1
timeout 100 python scripts/decode_bench.py 30 > gpurun_out/abl/decode.txt 2>&1
