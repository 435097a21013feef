#!/bin/bash
# bench summary lines for several workloads with the current library (APMM_LIB may override)
for wl in "$@"; do
  r=$(timeout 300 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1)
  python - "$wl" "$r" <<'PY'
import json, sys
wl, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line)
    r = d["roofline"]
    print(f"{wl:13s}: {d['value']:7.1f} TOPS  step {d['ms_per_step']*1e3:7.1f} us  gemm {r['gemm_us_avg']:6.1f} us  expand {r['expand_us_avg']:6.1f} us  frac {r['frac']:.3f} ({r['bound']})  sm {d['clocks']['sm_mhz']}  parity={str(d['parity'])[:2]}")
except Exception as e:
    print(wl, "FAILED", line[:400])
PY
done
