"""Dev: per-step clock64 events of K6 (dev library, APMM_TC_TS_MODE=5 APMM_TRACE=<slots>): for
the CTA-relative steps 0..3, cycles from CTA start (median over CTAs) of: the owning warp's
A-buffer wait done, its weight item in, its A stored (afull arrive); the MMA warp's operands
ready, MMAs issued, B refill wait done; and the first segment's dfull.
    python scripts/trace_k6_steps.py n_out m k n_w n_x"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_17870_b200 as ap  # noqa: E402

n_out, m, k, nw, nx = [int(a) for a in sys.argv[1:6]]
calls = 4
slots = int(os.environ["APMM_TRACE"])
dev = torch.device("cuda", 0)
ctx = ap.Context(0)
ctx.set_route(ap.Route.STREAM_TC)
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
names = [("A-wait done", 0, 0), ("W item in", 0, 4), ("A stored", 1, 0), ("MMA ready", 1, 4),
         ("MMA issued", 2, 0), ("B refill ok", 2, 4)]
print(f"{n_out}x{m}x{k} W{nw}A{nx}: cycles from CTA start, median over CTAs, steps 0..3")
for si in range(slots):
    if kinds[si] != 6:
        continue
    tt = t[si]
    grid = int((tt[:256, :] != 0).any(axis=1).sum())
    start = tt[768:768 + grid, 0]
    ok = start > 0
    if not ok.any():
        continue
    pro = [int(np.median(tt[768:768 + grid, c][ok] - start[ok])) for c in (2, 3, 4, 1)]
    print(f" slot {si}: CTAs {grid}, barriers init {pro[0]}, TMEM alloc + sync {pro[1]}, "
          f"first W issued {pro[2]}, first dfull {pro[3]}")
    for nm, pg, k0 in names:
        vals = []
        for st in range(4):
            v = tt[256 * pg:256 * pg + grid, k0 + st]
            sel = ok & (v > 0)
            vals.append(int(np.median(v[sel] - start[sel])) if sel.any() else -1)
        print(f"   {nm:12s} " + " ".join(f"{x:7d}" for x in vals))
    break
