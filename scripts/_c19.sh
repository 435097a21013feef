mkdir -p gpurun_out/c19
for s in "8192 1 8192 3 8" "8192 16 8192 3 8"; do
  echo "== $s" >> gpurun_out/c19/ts.txt
  timeout 60 python scripts/skinny_ts.py $s 2>&1 | tail -8 >> gpurun_out/c19/ts.txt
done
timeout 200 python -m pytest tests/test_gpu_parity.py -x -q -k "skinny or config4" > gpurun_out/c19/pytest.log 2>&1; echo rc=$? >> gpurun_out/c19/pytest.log
timeout 100 python scripts/decode_bench.py 30 > gpurun_out/c19/decode.txt 2>&1
