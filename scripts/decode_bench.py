"""Device time per call of small-M matmul_ap shapes, host overhead removed by replaying a
CUDA graph of `reps` back-to-back calls (the serving pattern). Weight buffers rotate over
`nbuf` copies so the working set exceeds L2.
    python scripts/decode_bench.py [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_17870_b200 as ap  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
only = sys.argv[2].split(",") if len(sys.argv) > 2 else None  # e.g. "8192x1,8192x16"
shapes = [(8192, 1, 8192, 3, 8), (8192, 8, 8192, 3, 8), (8192, 16, 8192, 3, 8),
          (4096, 1, 4096, 2, 4), (4096, 8, 4096, 2, 4), (4096, 16, 4096, 2, 4), (11008, 8, 4096, 2, 4), (11008, 1, 4096, 2, 4),
          (11008, 16, 4096, 2, 4), (4096, 1, 11008, 2, 4), (4096, 16, 11008, 2, 4),
          (8192, 32, 8192, 3, 8), (8192, 63, 8192, 3, 8)]
dev = torch.device("cuda", 0)
ctx = ap.Context(0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
peak = 6544.0
for (rw, m, k, nw, nx) in shapes:
    if only and f"{rw}x{m}" not in only and f"{rw}x{m}x{k}" not in only:
        continue
    wpr = (k + 31) // 32
    nbuf = max(2, int(300e6 // (4 * nw * rw * wpr)) + 1)
    ws = [torch.randint(-2**31, 2**31 - 1, (nw * rw * wpr,), dtype=torch.int32, device=dev)
          for _ in range(nbuf)]
    if k % 32:
        raise SystemExit("K % 32 != 0 needs zero padding")
    xp = torch.randint(-2**31, 2**31 - 1, (nx * m * wpr,), dtype=torch.int32, device=dev)
    y = torch.empty((rw, m), dtype=torch.int32, device=dev)
    for i in range(3):
        ap.cu_matmul_ap(ws[i % nbuf], rw, nw, xp, m, nx, k, y, ctx, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(reps):
            ap.cu_matmul_ap(ws[i % nbuf], rw, nw, xp, m, nx, k, y, ctx, stream=s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(5):
        g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    us = 1e3 * e0.elapsed_time(e1) / (5 * reps)
    byts = 4 * wpr * (nw * rw + nx * m) + 4 * rw * m
    print(f"{rw}x{m}x{k} W{nw}A{nx}: {us:7.2f} us/call  {byts / us / 1e3:6.0f} GB/s "
          f"({byts / us / 1e3 / peak:.2f} of {peak:.0f})  {2 * rw * m * k / us / 1e6:6.1f} TOPS",
          flush=True)
    del ws, xp, y, g
