"""Per-CTA phase timeline of the skinny kernel (APMM_SKINNY_TS=1, dev only): runs a few
calls of one shape and lets the library print phase timestamps of the last call."""
import os
import sys

os.environ["APMM_SKINNY_TS"] = "1"
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_17870_b200 as ap  # noqa: E402

rows_w, m_tok, k, nw, nx = [int(a) for a in sys.argv[1:6]]
dev = torch.device("cuda", 0)
ctx = ap.Context(0)
wpr = (k + 31) // 32
wp = torch.randint(-2**31, 2**31 - 1, (nw * rows_w * wpr,), dtype=torch.int32, device=dev)
xp = torch.randint(-2**31, 2**31 - 1, (nx * m_tok * wpr,), dtype=torch.int32, device=dev)
if k % 32:
    raise SystemExit("use K % 32 == 0 (random words have no zero padding)")
y = torch.empty((rows_w, m_tok), dtype=torch.int32, device=dev)
for _ in range(3):
    ap.cu_matmul_ap(wp, rows_w, nw, xp, m_tok, nx, k, y, ctx)
    torch.cuda.synchronize()
