"""Per-CTA phase timeline of the pair GEMM (APMM_PAIR_TS=1, dev only): a few calls of one
shape, each synchronised; the library prints the phases of every call.
    APMM_PAIR_TS=1 python scripts/pair_ts.py rows_w rows_x k n_w n_x"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_17870_b200 as ap  # noqa: E402

rows_w, m_tok, k, nw, nx = [int(a) for a in sys.argv[1:6]]
dev = torch.device("cuda", 0)
ctx = ap.Context(0)
wpr = (k + 31) // 32
wp = torch.randint(-2**31, 2**31 - 1, (nw * rows_w * wpr,), dtype=torch.int32, device=dev)
xp = torch.randint(-2**31, 2**31 - 1, (nx * m_tok * wpr,), dtype=torch.int32, device=dev)
y = torch.empty((rows_w, m_tok), dtype=torch.int32, device=dev)
for _ in range(3):
    ap.cu_matmul_ap(wp, rows_w, nw, xp, m_tok, nx, k, y, ctx)
    torch.cuda.synchronize()
