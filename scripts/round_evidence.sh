# round-end evidence: tests, every bench workload, reference arm, ncu launch lists + full captures
O=gpurun_out/fin
mkdir -p $O
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/smi.txt
timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
timeout 100 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
for w in ffn70b sweep4096 llama7b decode llama7b_small llama7b_mid; do timeout 300 python bench.py --workload $w > $O/bench_$w.log 2>&1; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2>&1
timeout 200 python scripts/decode_bench.py 30 > $O/decode_bench.txt 2>&1
( timeout 200 python scripts/route_sweep.py 8192 8192 3 8 1,8,16,32,64
  timeout 200 python scripts/route_sweep.py 4096 4096 2 4 8,16,32,64,128,256,512 ) > $O/route_sweep.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_decode.csv python bench.py --workload decode --steps 2 --warmup 3 --profile --no-graph --no-cpu-baseline > $O/ncu_launch_dec.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_mid.csv python bench.py --workload llama7b_mid --steps 2 --warmup 3 --profile --no-graph --no-cpu-baseline > $O/ncu_launch_mid.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:skinny_kernel --launch-skip 10 -c 1 -o $O/skinny_m1 python scripts/skinny_probe.py 8192 1 8192 3 8 20 > $O/ncu_sk1.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:stream_tc_kernel --launch-skip 10 -c 1 -o $O/stream_tc_m16 python scripts/skinny_probe.py 8192 16 8192 3 8 20 > $O/ncu_tc16.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:stream_tc_kernel --launch-skip 10 -c 1 -o $O/stream_tc_m64 python scripts/skinny_probe.py 4096 64 4096 2 4 20 > $O/ncu_tc64.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_pair_wplanes_kernel --launch-skip 10 -c 1 -o $O/k3f_m256 python scripts/skinny_probe.py 4096 256 4096 2 4 20 > $O/ncu_k3f256.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_pair_wplanes_kernel --launch-skip 10 -c 1 -o $O/k3f_m512 python scripts/skinny_probe.py 4096 512 4096 2 4 20 > $O/ncu_k3f512.log 2>&1
