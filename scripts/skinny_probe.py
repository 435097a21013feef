"""Time the skinny (small-M) path on one shape, CUDA events, device-resident planes.

    python scripts/skinny_probe.py [rows_w] [m_tok] [k] [n_w] [n_x] [reps]
Prints us per call and effective GB/s of packed weight planes (dev/measurement tool)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_17870_b200 as ap  # noqa: E402

args = [int(a) for a in sys.argv[1:]]
rows_w, m_tok, k, nw, nx, reps = (args + [8192, 1, 8192, 3, 8, 50][len(args):])[:6]
dev = torch.device("cuda", 0)
ctx = ap.Context(0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
wpr = (k + 31) // 32
g = torch.Generator(device=dev)
g.manual_seed(1)
wc = torch.randint(0, 1 << nw, (rows_w, k), generator=g, device=dev, dtype=torch.uint8)
xc = torch.randint(0, 1 << nx, (m_tok, k), generator=g, device=dev, dtype=torch.uint8)
wp = torch.empty(nw * rows_w * wpr, dtype=torch.int32, device=dev)
xp = torch.empty(nx * m_tok * wpr, dtype=torch.int32, device=dev)
ap.cu_pack(wc, rows_w, k, nw, wp, ctx)
ap.cu_pack(xc, m_tok, k, nx, xp, ctx)
del wc, xc
y = torch.empty((rows_w, m_tok), dtype=torch.int32, device=dev)
for _ in range(5):
    ap.cu_matmul_ap(wp, rows_w, nw, xp, m_tok, nx, k, y, ctx)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(reps):
    ap.cu_matmul_ap(wp, rows_w, nw, xp, m_tok, nx, k, y, ctx)
e1.record(s)
torch.cuda.synchronize()
us = 1e3 * e0.elapsed_time(e1) / reps
byts = 4 * wpr * (nw * rows_w + nx * m_tok) + 4 * rows_w * m_tok
print(f"{rows_w}x{m_tok}x{k} W{nw}A{nx} dbg={os.environ.get('APMM_SKINNY_DBG', '0')}: "
      f"{us:.2f} us/call  {byts / us / 1e3:.0f} GB/s  {2 * rows_w * m_tok * k / us / 1e6:.1f} TOPS")
