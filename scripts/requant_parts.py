"""Where the fused requant layer call spends its time (70B FFN shape by default): int32 GEMM,
dequant GEMM, dequant GEMM + fused absmax (split form), requant_pack alone, single call.
    python scripts/requant_parts.py [n_out m k n_w n_x]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_17870_b200 as ap  # noqa: E402

n_out, m, k, nw, nx = [int(a) for a in sys.argv[1:6]] if len(sys.argv) > 5 else (28672, 4096, 8192, 2, 4)
dev = torch.device("cuda", 0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = ap.Context(0)
wpr = (k + 31) // 32
w = torch.randint(-2**31, 2**31 - 1, (nw * n_out * wpr,), dtype=torch.int32, device=dev)
x = torch.randint(-2**31, 2**31 - 1, (nx * m * wpr,), dtype=torch.int32, device=dev)
y = torch.empty((n_out, m), dtype=torch.int32, device=dev)
yf = torch.empty((n_out, m), dtype=torch.float32, device=dev)
sw = torch.rand(n_out, dtype=torch.float64, device=dev) + 0.5
sx = torch.rand(m, dtype=torch.float64, device=dev) + 0.5
planes = torch.empty(4 * m * ((n_out + 31) // 32), dtype=torch.int32, device=dev)
scales = torch.empty(m, dtype=torch.float64, device=dev)
amax = torch.empty(m, dtype=torch.float64, device=dev)


def timed(name, fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    print(f"{name:45s} {e0.elapsed_time(e1) / reps * 1e3:9.1f} us", flush=True)


timed("int32 GEMM (cu_matmul_ap)", lambda: ap.cu_matmul_ap(w, n_out, nw, x, m, nx, k, y, ctx, stream=s))
timed("dequant GEMM (cu_matmul_ap_dequant)",
      lambda: ap.cu_matmul_ap_dequant(w, n_out, nw, sw, 1, x, m, nx, sx, 1, k, yf, ctx, stream=s))
timed("dequant GEMM + fused absmax (split form)",
      lambda: ap.cu_matmul_ap_requant(w, n_out, nw, sw, 1, x, m, nx, sx, 1, k, 4, 1, yf, absmax=amax,
                                      ctx=ctx, stream=s))
timed("requant_pack alone (+ NonFinite sync)",
      lambda: ap.cu_requant_pack(yf, n_out, m, amax, 4, 1, planes, scales, ctx=ctx, stream=s))
timed("single call (GEMM + absmax + requant + sync)",
      lambda: ap.cu_matmul_ap_requant(w, n_out, nw, sw, 1, x, m, nx, sx, 1, k, 4, 1, yf, planes, scales,
                                      ctx=ctx, stream=s))
