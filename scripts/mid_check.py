"""Dev: one mid-size call repeated (device time) with APMM_DEBUG_WAITS breakdown printed at
context close.   python scripts/mid_check.py rows_w rows_x k n_w n_x [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_17870_b200 as ap  # noqa: E402

rows_w, rows_x, k, nw, nx, reps = ([int(a) for a in sys.argv[1:]] + [20])[:6]
dev = torch.device("cuda", 0)
ctx = ap.Context(0)
wpr = (k + 31) // 32
wp = torch.randint(-2**31, 2**31 - 1, (nw * rows_w * wpr,), dtype=torch.int32, device=dev)
xp = torch.randint(-2**31, 2**31 - 1, (nx * rows_x * wpr,), dtype=torch.int32, device=dev)
y = torch.empty((rows_w, rows_x), dtype=torch.int32, device=dev)
for _ in range(3):
    ap.cu_matmul_ap(wp, rows_w, nw, xp, rows_x, nx, k, y, ctx)
torch.cuda.synchronize()
ctx.enable_timing(True)
for _ in range(reps):
    ap.cu_matmul_ap(wp, rows_w, nw, xp, rows_x, nx, k, y, ctx)
torch.cuda.synchronize()
g_ms, g_n = ctx.kernel_time(0)
e_ms, e_n = ctx.kernel_time(1)
ctx.enable_timing(False)
print(f"{rows_w}x{rows_x}x{k} W{nw}A{nx}: gemm {1e3 * g_ms / max(g_n, 1):.1f} us, "
      f"expand {1e3 * e_ms / max(e_n, 1):.1f} us per call", flush=True)
ctx.close()
