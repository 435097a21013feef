"""A few dequant calls of one shape on one route (ncu captures of the fp64 epilogue):
    python scripts/one_call_dequant.py n_out m k n_w n_x [ROUTE] [calls]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_17870_b200 as ap  # noqa: E402

n_out, m, k, nw, nx = [int(a) for a in sys.argv[1:6]]
route = getattr(ap.Route, sys.argv[6]) if len(sys.argv) > 6 else ap.Route.AUTO
calls = int(sys.argv[7]) if len(sys.argv) > 7 else 3
dev = torch.device("cuda", 0)
wpr = (k + 31) // 32
w = torch.randint(-2**31, 2**31 - 1, (nw * n_out * wpr,), dtype=torch.int32, device=dev)
x = torch.randint(-2**31, 2**31 - 1, (nx * m * wpr,), dtype=torch.int32, device=dev)
sw = torch.rand(n_out, dtype=torch.float64, device=dev) + 0.5
sx = torch.rand(m, dtype=torch.float64, device=dev) + 0.5
yf = torch.empty((n_out, m), dtype=torch.float32, device=dev)
ctx = ap.Context(0)
ctx.set_route(route)
for _ in range(calls):
    ap.cu_matmul_ap_dequant(w, n_out, nw, sw, 1, x, m, nx, sx, 1, k, yf, ctx)
torch.cuda.synchronize()
print("ok", n_out, m, k, nw, nx, route.name)
