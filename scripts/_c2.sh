set -x
mkdir -p gpurun_out/c2
for s in "8192 1 8192 3 8" "8192 8 8192 3 8" "8192 16 8192 3 8" "4096 1 4096 2 4" "4096 16 4096 2 4" "11008 1 4096 2 4" "11008 16 4096 2 4" "4096 1 11008 2 4" "4096 16 11008 2 4" "8192 32 8192 3 8" "8192 63 8192 3 8"; do
  timeout 60 python scripts/skinny_probe.py $s 200 >> gpurun_out/c2/probe.txt 2>&1
  APMM_DEBUG_PLAN=1 timeout 60 python scripts/skinny_probe.py $s 5 2>&1 | grep plan | head -1 >> gpurun_out/c2/plan.txt
done
for s in "8192 1 8192 3 8" "8192 16 8192 3 8"; do
  echo "== $s" >> gpurun_out/c2/ts.txt
  timeout 60 python scripts/skinny_ts.py $s >> gpurun_out/c2/ts.txt 2>&1
done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:skinny --launch-skip 10 -c 1 -o gpurun_out/c2/skinny16 python scripts/skinny_probe.py 8192 16 8192 3 8 20 > gpurun_out/c2/ncu16.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:skinny --launch-skip 10 -c 1 -o gpurun_out/c2/skinny1 python scripts/skinny_probe.py 8192 1 8192 3 8 20 > gpurun_out/c2/ncu1.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_u8_pair --launch-skip 5 -c 1 -o gpurun_out/c2/pair_w2a4 python scripts/skinny_probe.py 4096 4096 4096 2 4 10 > gpurun_out/c2/ncupair.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:expand --launch-skip 5 -c 1 -o gpurun_out/c2/expand_w2a4 python scripts/skinny_probe.py 4096 4096 4096 2 4 10 > gpurun_out/c2/ncuexp.log 2>&1
