"""Dev: cycle stamps of the K3f epilogue's first two chunks on each CTA's last unit
(APMM_TRACE=<slots> APMM_TRACE_CLOCK=1, dev library).
    python scripts/trace_cycles_k3f.py n_out m k n_w n_x [calls]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_17870_b200 as ap  # noqa: E402

n_out, m, k, nw, nx = [int(a) for a in sys.argv[1:6]]
calls = int(sys.argv[6]) if len(sys.argv) > 6 else 4
slots = int(os.environ["APMM_TRACE"])
dev = torch.device("cuda", 0)
ctx = ap.Context(0)
ctx.set_route(ap.Route.MID_SPLITK)
fn = ctx.lib.apmm_dev_trace_read
fn.restype, fn.argtypes = C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
wpr = (k + 31) // 32
w = torch.randint(-2**31, 2**31 - 1, (nw * n_out * wpr,), dtype=torch.int32, device=dev)
xp = torch.randint(-2**31, 2**31 - 1, (nx * m * wpr,), dtype=torch.int32, device=dev)
y = torch.empty((n_out, m), dtype=torch.int32, device=dev)
buf = np.zeros(slots * 1024 * 8, dtype=np.uint64)
kinds = np.zeros(slots, dtype=np.int32)
for i in range(calls):
    ap.cu_matmul_ap(w, n_out, nw, xp, m, nx, k, y, ctx, stream=s)
torch.cuda.synchronize()
fn(ctx.h, buf.ctypes.data, kinds.ctypes.data)
for i in range(calls):
    ap.cu_matmul_ap(w, n_out, nw, xp, m, nx, k, y, ctx, stream=s)
torch.cuda.synchronize()
fn(ctx.h, buf.ctypes.data, kinds.ctypes.data)
t = buf.reshape(slots, 1024, 8).astype(np.int64)
names = ["-", "c0 ld", "c0 math", "c0 issued", "c1 ld", "c1 math", "c1 issued", "all issued"]
print(f"{n_out}x{m}x{k} W{nw}A{nx} mid route: epilogue cycles from the accumulator-ready point (median / p90)")
for i in range(slots):
    if kinds[i] != 3:
        continue
    rows = t[i][t[i][:, 7] > 0]
    if rows.size == 0:
        continue
    print(f"  slot {i:2d}: " + " | ".join(f"{names[c]} {int(np.median(rows[:, c]))}/{int(np.percentile(rows[:, c], 90))}" for c in range(1, 8)))
