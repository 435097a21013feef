mkdir -p gpurun_out/c15
export PYTHONUNBUFFERED=1
for s in "8192 1 8192 3 8" "8192 16 8192 3 8"; do
  echo "== $s" >> gpurun_out/c15/ts.txt
  timeout 60 python scripts/skinny_ts.py $s >> gpurun_out/c15/ts.txt 2>&1
done
timeout 200 ncu --set full --import-source on --clock-control none -k regex:skinny --launch-skip 10 -c 1 -o gpurun_out/c15/sk16 python scripts/skinny_probe.py 8192 16 8192 3 8 20 > gpurun_out/c15/ncu16.log 2>&1
