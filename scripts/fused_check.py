"""Dev check of the fused weight-plane GEMM (K3f) against the two-kernel path on one shape:
    python scripts/fused_check.py rows_w rows_x k n_w n_x [reps]
Prints equality and us/call of both paths (CUDA events, device-resident planes)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_17870_b200 as ap  # noqa: E402

rows_w, rows_x, k, nw, nx, reps = ([int(a) for a in sys.argv[1:]] + [50])[:6]
dev = torch.device("cuda", 0)
ctx = ap.Context(0)
wpr = (k + 31) // 32
g = torch.Generator(device=dev)
g.manual_seed(1)
wc = torch.randint(0, 1 << nw, (rows_w, k), generator=g, device=dev, dtype=torch.uint8)
xc = torch.randint(0, 1 << nx, (rows_x, k), generator=g, device=dev, dtype=torch.uint8)
wp = torch.empty(nw * rows_w * wpr, dtype=torch.int32, device=dev)
xp = torch.empty(nx * rows_x * wpr, dtype=torch.int32, device=dev)
ap.cu_pack(wc, rows_w, k, nw, wp, ctx)
ap.cu_pack(xc, rows_x, k, nx, xp, ctx)
y = {}
for mode in ("fused", "two-kernel"):
    os.environ["APMM_FUSED"] = "1" if mode == "fused" else "0"
    out = torch.empty((rows_w, rows_x), dtype=torch.int32, device=dev)
    ap.cu_matmul_ap(wp, rows_w, nw, xp, rows_x, nx, k, out, ctx)
    torch.cuda.synchronize()
    y[mode] = out
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        ap.cu_matmul_ap(wp, rows_w, nw, xp, rows_x, nx, k, out, ctx)
    e1.record()
    torch.cuda.synchronize()
    us = 1e3 * e0.elapsed_time(e1) / reps
    print(f"{mode:10s} {rows_w}x{rows_x}x{k} W{nw}A{nx}: {us:8.2f} us/call "
          f"{2 * rows_w * rows_x * k / us / 1e6:7.1f} TOPS", flush=True)
os.environ.pop("APMM_NO_FUSED", None)
ctx.close()  # prints the APMM_DEBUG_WAITS counters
eq = torch.equal(y["fused"], y["two-kernel"])
print("equal:", eq)
if not eq:
    d = (y["fused"] != y["two-kernel"]).nonzero()
    print("mismatches", d.shape[0], "first", d[:8].tolist())
