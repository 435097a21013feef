"""Per-call device time of every kernel route that can serve a shape, over the token count M
(graph replay of back-to-back calls, weights rotated past L2). Evidence for the AUTO route
choice:
    python scripts/route_sweep.py n_out k n_w n_x [M,M,...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_17870_b200 as ap  # noqa: E402

n_out, k, nw, nx = [int(a) for a in sys.argv[1:5]]
ms = [int(v) for v in (sys.argv[5] if len(sys.argv) > 5 else "16,32,48,64,96,128,192,256,384,512,768,1024").split(",")]
dev = torch.device("cuda", 0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)  # graph replays and the timing events run on s
wpr = (k + 31) // 32
ws = [torch.randint(-2**31, 2**31 - 1, (nw * n_out * wpr,), dtype=torch.int32, device=dev)
      for _ in range(max(2, int(300e6 // (4 * nw * n_out * wpr)) + 1))]
routes = [ap.Route.AUTO, ap.Route.SKINNY, ap.Route.STREAM_TC, ap.Route.MID_SPLITK, ap.Route.SINGLE_SM,
          ap.Route.PAIR_SPLITK, ap.Route.PAIR, ap.Route.PAIR_WPLANES]
print(f"{n_out} x M x {k} W{nw}A{nx}: us per call (graph replay); roofline = max(bytes/6544 GB/s, ops/3219 TOPS)")
print("     M  roofline " + " ".join(f"{r.name:>12s}" for r in routes))
for m in ms:
    xp = torch.randint(-2**31, 2**31 - 1, (nx * m * wpr,), dtype=torch.int32, device=dev)
    y = torch.empty((n_out, m), dtype=torch.int32, device=dev)
    byts = 4 * wpr * (nw * n_out + nx * m) + 4 * n_out * m
    roof = max(byts / 6544e3, 2 * n_out * m * k / 3219e6)
    row = []
    for r in routes:
        ctx = ap.Context(0)
        ctx.set_route(r)
        try:
            for i in range(3):
                ap.cu_matmul_ap(ws[i % len(ws)], n_out, nw, xp, m, nx, k, y, ctx, stream=s)
        except ap.InvalidArgument:
            row.append(f"{'-':>12s}")
            continue
        reps = 20
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(reps):
                ap.cu_matmul_ap(ws[i % len(ws)], n_out, nw, xp, m, nx, k, y, ctx, stream=s)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        g.replay()
        e1.record(s)
        torch.cuda.synchronize()
        us = 1e3 * e0.elapsed_time(e1) / (2 * reps)
        row.append(f"{us:6.2f} ({roof / us:.2f})".rjust(12))
        del g
    print(f"{m:6d} {roof:8.2f} " + " ".join(row), flush=True)
