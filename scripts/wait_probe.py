"""Dev probe: run the 4096^3 W2A4 GEMM N times with APMM_DEBUG_WAITS=1 and print the
MMA-issuer wait breakdown (printed by the library when the context is destroyed)."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2409_17870_b200 as ap
n_out = m_tok = k = int(os.environ.get("N", "4096")); nw, nx = 2, 4
dev = torch.device("cuda")
ctx = ap.Context(0)
wc = torch.randint(0, 1 << nw, (n_out, k), device=dev, dtype=torch.uint8)
xc = torch.randint(0, 1 << nx, (m_tok, k), device=dev, dtype=torch.uint8)
wpr = (k + 31) // 32
wp = torch.empty(nw * n_out * wpr, dtype=torch.int32, device=dev); xp = torch.empty(nx * m_tok * wpr, dtype=torch.int32, device=dev)
ap.cu_pack(wc, n_out, k, nw, wp, ctx); ap.cu_pack(xc, m_tok, k, nx, xp, ctx)
y = torch.empty((n_out, m_tok), dtype=torch.int32, device=dev)
for _ in range(5):
    ap.cu_matmul_ap(wp, n_out, nw, xp, m_tok, nx, k, y, ctx)
torch.cuda.synchronize()
ctx.enable_timing(True)
for _ in range(20):
    ap.cu_matmul_ap(wp, n_out, nw, xp, m_tok, nx, k, y, ctx)
torch.cuda.synchronize()
ms, n = ctx.kernel_time(0)
print(f"N={n_out}: gemm {1e3*ms/n:.1f} us/launch  {2*n_out*m_tok*k/(ms/n*1e-3)/1e12:.0f} TOPS", flush=True)
ctx.close()
