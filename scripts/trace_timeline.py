"""Per-launch timeline of a CUDA-graph replay of back-to-back matmul_ap calls (dev build:
APMM_LIB=abtest/libapmm_b200_dev.so APMM_TRACE=64). For every launch in one replay: kernel
kind, and min / max over CTAs of each globaltimer stamp, in us from the first launch's
first CTA start. Shows where consecutive calls overlap (PDL) and what is exposed.
    python scripts/trace_timeline.py n_out m_tok k n_w n_x [calls]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_17870_b200 as ap  # noqa: E402

n_out, m, k, nw, nx = [int(a) for a in sys.argv[1:6]]
calls = int(sys.argv[6]) if len(sys.argv) > 6 else 6
slots = int(os.environ.get("APMM_TRACE", "0"))
assert slots >= 2 * calls, "run with APMM_TRACE >= 2 x calls and the dev library"
dev = torch.device("cuda", 0)
ctx = ap.Context(0)
if os.environ.get("ROUTE"):  # e.g. ROUTE=STREAM_TC
    ctx.set_route(ap.Route[os.environ["ROUTE"]])
lib = ctx.lib
fn = lib.apmm_dev_trace_read
fn.restype, fn.argtypes = C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]
s = torch.cuda.Stream()
wpr = (k + 31) // 32
nbuf = max(2, int(300e6 // (4 * nw * n_out * wpr)) + 1)
ws = [torch.randint(-2**31, 2**31 - 1, (nw * n_out * wpr,), dtype=torch.int32, device=dev)
      for _ in range(min(nbuf, calls))]
xp = torch.randint(-2**31, 2**31 - 1, (nx * m * wpr,), dtype=torch.int32, device=dev)
y = torch.empty((n_out, m), dtype=torch.int32, device=dev)
for i in range(3):
    ap.cu_matmul_ap(ws[i % len(ws)], n_out, nw, xp, m, nx, k, y, ctx, stream=s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for i in range(calls):
        ap.cu_matmul_ap(ws[i % len(ws)], n_out, nw, xp, m, nx, k, y, ctx, stream=s)
buf = np.zeros(slots * 1024 * 8, dtype=np.uint64)
kinds = np.zeros(slots, dtype=np.int32)
g.replay()
torch.cuda.synchronize()
fn(ctx.h, buf.ctypes.data, kinds.ctypes.data)  # clear
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
g.replay()
e1.record(s)
torch.cuda.synchronize()
n = fn(ctx.h, buf.ctypes.data, kinds.ctypes.data)
t = buf.reshape(slots, 1024, 8).astype(np.float64)
names = {1: ("expand", ["start", "w_done", "waited", "end"]),
         2: ("pair", ["start", "pdl_wait", "first_full", "last_issue", "end"]),
         3: ("wplanes", ["start", "pdl_wait", "first_full", "last_issue", "end", "epi_done",
                         "acc_ready", "chunks_out"]),
         5: ("skinny", ["start", "pdl_wait", "x_ready", "item0", "tile0", "end", "inited", "issued"]),
         6: ("stream_tc", ["start", "pdl_wait", "w0_in", "a0_st", "mma0", "mma_last", "epi0", "end"]),
         7: ("tc_prep", ["start", "pdl_wait", "end"])}
t0 = min(t[i][t[i] > 0].min() for i in range(slots) if (t[i] > 0).any())
print(f"{n_out}x{m}x{k} W{nw}A{nx}: {calls} calls, {1e3 * e0.elapsed_time(e1) / calls:.2f} us/call (graph)")
for i in range(slots):
    if kinds[i] == 0 or not (t[i] > 0).any():
        continue
    nm, cols = names.get(int(kinds[i]), (str(kinds[i]), [str(c) for c in range(8)]))
    parts = []
    for c, cn in enumerate(cols):
        v = t[i][:, c]
        v = v[v > 0]
        if cn == "-" or v.size == 0:
            continue
        parts.append(f"{cn} {(v.min() - t0) / 1e3:7.2f}..{(v.max() - t0) / 1e3:7.2f}")
    print(f"  slot {i:2d} {nm:8s} " + " | ".join(parts))
