#!/bin/bash
# A/B of K1's store policy (dev build, APMM_K1_CS: bit0 = weight codes evict-first, bit1 = feature codes)
for wl in ffn70b sweep4096 llama7b; do
  for cs in 0 1 3; do
    r=$(APMM_LIB=abtest/libapmm_b200_dev.so APMM_K1_CS=$cs timeout 300 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1)
    python - "$wl" "$cs" "$r" <<'PY'
import json, sys
wl, cs, line = sys.argv[1], sys.argv[2], sys.argv[3]
try:
    d = json.loads(line)
    r = d["roofline"]
    print(f"{wl:10s} cs={cs}: {d['value']:7.1f} TOPS  step {d['ms_per_step']*1e3:7.1f} us  gemm {r['gemm_us_avg']:6.1f} us  expand {r['expand_us_avg']:6.1f} us  parity={d['parity'][:2]}")
except Exception as e:
    print(wl, cs, "FAILED", line[:300])
PY
  done
done
