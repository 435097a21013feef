"""Dev: per-CTA cycle deltas of the skinny kernel's phases (APMM_TRACE=<slots>
APMM_TRACE_CLOCK=1, dev library): clock64 at each stamp minus the CTA's own start, so
sub-microsecond prologue steps are visible (globaltimer ticks in 256 ns).
    python scripts/trace_cycles.py n_out m k n_w n_x [calls]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_17870_b200 as ap  # noqa: E402

n_out, m, k, nw, nx = [int(a) for a in sys.argv[1:6]]
calls = int(sys.argv[6]) if len(sys.argv) > 6 else 6
slots = int(os.environ["APMM_TRACE"])
dev = torch.device("cuda", 0)
ctx = ap.Context(0)
fn = ctx.lib.apmm_dev_trace_read
fn.restype, fn.argtypes = C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
wpr = (k + 31) // 32
ws = [torch.randint(-2**31, 2**31 - 1, (nw * n_out * wpr,), dtype=torch.int32, device=dev) for _ in range(calls)]
xp = torch.randint(-2**31, 2**31 - 1, (nx * m * wpr,), dtype=torch.int32, device=dev)
y = torch.empty((n_out, m), dtype=torch.int32, device=dev)
for i in range(3):
    ap.cu_matmul_ap(ws[i], n_out, nw, xp, m, nx, k, y, ctx, stream=s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for i in range(calls):
        ap.cu_matmul_ap(ws[i], n_out, nw, xp, m, nx, k, y, ctx, stream=s)
buf = np.zeros(slots * 1024 * 8, dtype=np.uint64)
kinds = np.zeros(slots, dtype=np.int32)
g.replay()
torch.cuda.synchronize()
fn(ctx.h, buf.ctypes.data, kinds.ctypes.data)
g.replay()
torch.cuda.synchronize()
fn(ctx.h, buf.ctypes.data, kinds.ctypes.data)
t = buf.reshape(slots, 1024, 8).astype(np.int64)
names = ["start", "pdl_wait", "x_ready", "item0", "tile0", "end", "inited", "issued"]
order = [6, 7, 1, 2, 3, 4, 5]
print(f"{n_out}x{m}x{k} W{nw}A{nx}: cycles from each CTA's own start (median / p90 over CTAs)")
for i in range(slots):
    if kinds[i] != 5:
        continue
    rows = t[i][t[i][:, 0] > 0]
    if rows.size == 0:
        continue
    d = rows - rows[:, :1]
    print(f"  slot {i:2d}: " + " | ".join(f"{names[c]} {int(np.median(d[:, c]))}/{int(np.percentile(d[:, c], 90))}" for c in order))
