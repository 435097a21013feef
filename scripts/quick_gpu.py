import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_2409_17870_b200 as ap
from oracle import Oracle
o = Oracle()
rng = o.rng(1)
bad = 0
for (m, n, k, nw, nx) in [(1,1,1,1,1),(5,7,40,3,2),(128,256,128,2,2),(130,300,300,4,8),(300,700,1000,2,4),(1024,1024,1024,2,2),(1,1,33025,8,8)]:
    wc = rng.random_codes(m, k, nw); xc = rng.random_codes(n, k, nx)
    wp = o.pack(wc, nw); xp = o.pack(xc, nx)
    want = o.matmul_ap(wp, m, nw, xp, n, nx, k)
    try:
        got = ap.matmul_ap(ap.PackedBitPlanes(m, k, ap.BitWidth(nw), wp), ap.PackedBitPlanes(n, k, ap.BitWidth(nx), xp))
        ok = np.array_equal(got, want)
    except Exception as e:
        ok = False; got = None; print('EXC', e)
    print((m,n,k,nw,nx), 'OK' if ok else 'MISMATCH', flush=True)
    if not ok and got is not None:
        d = np.argwhere(got != want); print(' first diffs', d[:5].tolist(), got[tuple(d[0])], want[tuple(d[0])], 'count', len(d))
