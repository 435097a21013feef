# round-end evidence: tests, every bench workload, reference arm, ncu launch list + full captures
mkdir -p gpurun_out/fin
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/fin/smi.txt
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/fin/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/fin/pytest_gpu.log
timeout 100 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1
for w in sweep4096 llama7b decode llama7b_small ffn70b; do timeout 300 python bench.py --workload $w > gpurun_out/fin/bench_$w.log 2>&1; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin/bench_ref.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin/launches_sweep.csv python bench.py --steps 2 --warmup 3 --profile --no-graph --no-cpu-baseline > gpurun_out/fin/ncu_launch.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin/launches_decode.csv python bench.py --workload decode --steps 2 --warmup 3 --profile --no-graph --no-cpu-baseline > gpurun_out/fin/ncu_launch_dec.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_u8_pair --launch-skip 5 -c 1 -o gpurun_out/fin/pair_w2a4 python scripts/skinny_probe.py 4096 4096 4096 2 4 10 > gpurun_out/fin/ncu_pair.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:skinny --launch-skip 10 -c 1 -o gpurun_out/fin/skinny_m1 python scripts/skinny_probe.py 8192 1 8192 3 8 20 > gpurun_out/fin/ncu_sk1.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:skinny --launch-skip 10 -c 1 -o gpurun_out/fin/skinny_m16 python scripts/skinny_probe.py 8192 16 8192 3 8 20 > gpurun_out/fin/ncu_sk16.log 2>&1
