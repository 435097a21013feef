"""The reference's LLM-layer flow quantize(X) -> pack -> matmul_ap -> dequant (apmm.cpp:275-340)
on Llama-2-7B shapes (W2A4, M=2048, per-token X scales, fp64 X as the reference's RealMatrix),
two ways: (a) apmm_cu_quantize_pack + apmm_cu_matmul_ap_dequant, (b) the fused
apmm_cu_quantize_matmul_ap_dequant (quantizer writes the GEMM operand; no X planes / X
expansion). Eager launches (both entry points synchronise once on the quantizer's flag),
CUDA-event device time per call, W rotated past L2.
    python scripts/quant_flow_bench.py [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_17870_b200 as ap  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
dev = torch.device("cuda", 0)
ctx = ap.Context(0)
for (n_out, k) in ((4096, 4096), (11008, 4096), (4096, 11008)):
    m, nw, nx = 2048, 2, 4
    wpr = (k + 31) // 32
    ws = []
    for _ in range(3):
        wc = torch.randint(0, 1 << nw, (n_out, k), device=dev, dtype=torch.uint8)
        wp = torch.empty(nw * n_out * wpr, dtype=torch.int32, device=dev)
        ap.cu_pack(wc, n_out, k, nw, wp, ctx)
        ws.append(wp)
    sw = torch.rand(n_out, dtype=torch.float64, device=dev)
    xv = torch.randn((m, k), dtype=torch.float64, device=dev)
    sx = torch.empty(m, dtype=torch.float64, device=dev)
    xp = torch.empty(nx * m * wpr, dtype=torch.int32, device=dev)
    out = torch.empty((n_out, m), dtype=torch.float32, device=dev)

    def two_calls(i):
        ap.cu_quantize_pack(xv, m, k, nx, 1, xp, sx, ctx=ctx)
        ap.cu_matmul_ap_dequant(ws[i % 3], n_out, nw, sw, 1, xp, m, nx, sx, 1, k, out, ctx)

    def fused(i):
        ap.cu_quantize_matmul_ap_dequant(ws[i % 3], n_out, nw, sw, 1, xv, m, k, nx, 1, sx, out, ctx)

    res = {}
    for name, fn in (("quantize_pack + matmul_ap_dequant", two_calls), ("fused K2->K3", fused)):
        for i in range(3):
            fn(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(reps):
            fn(i)
        e1.record()
        torch.cuda.synchronize()
        res[name] = 1e3 * e0.elapsed_time(e1) / reps
    ops = 2.0 * n_out * m * k
    print(f"{n_out}x{m}x{k} W{nw}A{nx}: " + "; ".join(
        f"{k_}: {v:.1f} us ({ops / v / 1e6:.0f} TOPS)" for k_, v in res.items()), flush=True)
