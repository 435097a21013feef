mkdir -p gpurun_out/c3
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or config2 or config1 or config3" > gpurun_out/c3/pytest.log 2>&1; echo rc=$? >> gpurun_out/c3/pytest.log
for s in "4096 4096 4096 2 4" "4096 4096 4096 1 2" "4096 4096 4096 4 8" "4096 4096 4096 8 8"; do
  timeout 60 python scripts/skinny_probe.py $s 50 >> gpurun_out/c3/probe.txt 2>&1
  APMM_NO_FUSED=1 timeout 60 python scripts/skinny_probe.py $s 50 >> gpurun_out/c3/probe.txt 2>&1
done
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/c3/bench_sweep.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/c3/launches.csv python bench.py --steps 2 --warmup 3 --profile --no-graph > gpurun_out/c3/ncu_launch.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:wplanes --launch-skip 5 -c 1 -o gpurun_out/c3/fused_w2a4 python scripts/skinny_probe.py 4096 4096 4096 2 4 10 > gpurun_out/c3/ncu.log 2>&1
