"""Measured tcgen05 kind::i8 ceiling of the pair GEMM (roofline denominator for bench.py).

Runs the CTA-pair kernel with APMM_PEAK_PROBE=1: after one fill of the operand ring the
stages are re-used without TMA loads, so the timed loop is the tensor pipe + MMA issue +
TMEM epilogue of the real kernel and schedule (results are wrong by design). Device time
per GEMM from CUDA events over back-to-back launches, after 1 s of heat. Writes JSON:
    APMM_PEAK_PROBE=1 python scripts/i8_mma_peak.py out.json"""
import json
import os
import subprocess
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
assert os.environ.get("APMM_PEAK_PROBE") == "1", "run with APMM_PEAK_PROBE=1"
import paper_2409_17870_b200 as ap  # noqa: E402

dev = torch.device("cuda", 0)
ctx = ap.Context(0)
out = {"how": __doc__.split("\n")[2].strip(), "shapes": {}}
for n in (4096, 8192):
    wpr = n // 32
    wp = torch.randint(-2**31, 2**31 - 1, (2 * n * wpr,), dtype=torch.int32, device=dev)
    xp = torch.randint(-2**31, 2**31 - 1, (4 * n * wpr,), dtype=torch.int32, device=dev)
    y = torch.empty((n, n), dtype=torch.int32, device=dev)
    t_end = time.time() + 1.0
    while time.time() < t_end:
        ap.cu_matmul_ap(wp, n, 2, xp, n, 4, n, y, ctx)
        torch.cuda.synchronize()
    ctx.enable_timing(True)
    reps = 20
    for _ in range(reps):
        ap.cu_matmul_ap(wp, n, 2, xp, n, 4, n, y, ctx)
    torch.cuda.synchronize()
    ms, cnt = ctx.kernel_time(0)
    ctx.enable_timing(False)
    us = 1e3 * ms / cnt
    tops = 2.0 * n ** 3 / (us * 1e-6) / 1e12
    clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                         capture_output=True, text=True).stdout.strip()
    out["shapes"][f"{n}^3"] = {"us_per_gemm": us, "tops": tops, "sm_mhz_after": clk}
    print(n, f"{us:.1f} us  {tops:.0f} TOPS", flush=True)
out["i8_tops"] = max(v["tops"] for v in out["shapes"].values())
json.dump(out, open(sys.argv[1], "w"), indent=1)
