"""Dev: wait-cycle breakdown of the K3f roles (APMM_DEBUG_WAITS=1, dev library) for one shape,
printed by the library at context teardown.
    APMM_LIB=abtest/libapmm_b200_dev.so APMM_DEBUG_WAITS=1 python scripts/mid_waits.py n_out m k n_w n_x [route]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_17870_b200 as ap  # noqa: E402

n_out, m, k, nw, nx = [int(a) for a in sys.argv[1:6]]
route = getattr(ap.Route, sys.argv[6]) if len(sys.argv) > 6 else ap.Route.MID_SPLITK
dev = torch.device("cuda", 0)
wpr = (k + 31) // 32
w = torch.randint(-2**31, 2**31 - 1, (nw * n_out * wpr,), dtype=torch.int32, device=dev)
x = torch.randint(-2**31, 2**31 - 1, (nx * m * wpr,), dtype=torch.int32, device=dev)
y = torch.empty((n_out, m), dtype=torch.int32, device=dev)
ctx = ap.Context(0)
ctx.set_route(route)
for _ in range(20):
    ap.cu_matmul_ap(w, n_out, nw, x, m, nx, k, y, ctx)
torch.cuda.synchronize()
print(f"{n_out}x{m}x{k} W{nw}A{nx} route {route.name}", flush=True)
ctx.close()
