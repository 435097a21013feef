mkdir -p gpurun_out/c18
for s in "8192 1 8192 3 8" "8192 16 8192 3 8"; do
  echo "== $s" >> gpurun_out/c18/ts.txt
  timeout 60 python scripts/skinny_ts.py $s 2>&1 | tail -8 >> gpurun_out/c18/ts.txt
done
