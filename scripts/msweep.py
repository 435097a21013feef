"""Effective TOPS across the token count M for one weight shape (graph replay, device time):
    python scripts/msweep.py n_out k n_w n_x"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_17870_b200 as ap  # noqa: E402

n_out, k, nw, nx = [int(a) for a in sys.argv[1:5]]
dev = torch.device("cuda", 0)
ctx = ap.Context(0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
wpr = (k + 31) // 32
ws = [torch.randint(-2**31, 2**31 - 1, (nw * n_out * wpr,), dtype=torch.int32, device=dev)
      for _ in range(max(2, int(300e6 // (4 * nw * n_out * wpr)) + 1))]
ms = [int(v) for v in os.environ.get('MSWEEP', '1,16,32,63,64,96,128,192,256,384,512,768,1024,2048,4096').split(',')]
for m in ms:
    xp = torch.randint(-2**31, 2**31 - 1, (nx * m * wpr,), dtype=torch.int32, device=dev)
    y = torch.empty((n_out, m), dtype=torch.int32, device=dev)
    reps = 20
    for i in range(3):
        ap.cu_matmul_ap(ws[i % len(ws)], n_out, nw, xp, m, nx, k, y, ctx, stream=s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(reps):
            ap.cu_matmul_ap(ws[i % len(ws)], n_out, nw, xp, m, nx, k, y, ctx, stream=s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    us = 1e3 * e0.elapsed_time(e1) / reps
    print(f"{n_out}x{m}x{k} W{nw}A{nx}: {us:8.2f} us  {2 * n_out * m * k / us / 1e6:7.1f} TOPS", flush=True)
