"""GPU checks of the boundary additions of round 2: dot_1bit_xor and the host
matmul_plane_pair (kernel.hpp:61-69), the fused next-layer requantization (SURVEY.md 8(f)
row 3), workspace reservation for CUDA-graph capture, and the one-stream-per-context rule."""
import os

import numpy as np
import pytest

from oracle import PER_ROW, PER_TENSOR

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------- dot_1bit_xor
def test_dot_1bit_xor_known_answers_and_errors(gpu, oracle):
    # test_kernel.cpp:22-56, and the reference's error classes (kernel.cpp:117-121)
    ap, ctx = gpu
    a = np.array([0xA5A5A5A5], np.uint32)
    assert ap.dot_1bit_xor(a, a, 32, ctx) == 32
    assert ap.dot_1bit_xor(np.array([0xFFFFFFFF], np.uint32), np.array([0], np.uint32), 32, ctx) == -32
    assert ap.dot_1bit_xor(np.array([0b1100], np.uint32), np.array([0b1010], np.uint32), 4, ctx) == 0
    a = np.array([0xFFFFFFFF] * 3 + [0xF], np.uint32)
    b = a.copy()
    assert ap.dot_1bit_xor(a, b, 100, ctx) == 100
    b[1] = 0
    assert ap.dot_1bit_xor(a, b, 100, ctx) == 100 - 64
    with pytest.raises(ap.LengthMismatch):
        ap.dot_1bit_xor(np.zeros(1, np.uint32), np.zeros(2, np.uint32), 32, ctx)
    with pytest.raises(ap.OutOfRange):
        ap.dot_1bit_xor(np.zeros(1, np.uint32), np.zeros(1, np.uint32), 0, ctx)
    rng = np.random.default_rng(5)
    for k in (1, 31, 32, 33, 1000, 70001):
        w = (k + 31) // 32
        x, y = (rng.integers(0, 2**32, size=w, dtype=np.uint64).astype(np.uint32) for _ in range(2))
        assert ap.dot_1bit_xor(x, y, k, ctx) == oracle.dot_1bit_xor(x, y, k)


def test_cu_dot_1bit_xor(gpu, oracle):
    import torch
    ap, _ = gpu
    rng = np.random.default_rng(6)
    x, y = (rng.integers(0, 2**32, size=40, dtype=np.uint64).astype(np.uint32) for _ in range(2))
    dev = torch.device("cuda", 0)
    out = torch.empty(1, dtype=torch.int64, device=dev)
    ap.cu_dot_1bit_xor(torch.from_numpy(x.view(np.int32)).to(dev),
                       torch.from_numpy(y.view(np.int32)).to(dev), 1270, out)
    assert int(out.item()) == oracle.dot_1bit_xor(x, y, 1270)


def test_host_matmul_plane_pair_matches_reference(gpu, oracle):
    ap, ctx = gpu
    rng = oracle.rng(77)
    m, n, k, nw, nx = 37, 29, 333, 3, 4
    wc, xc = rng.random_codes(m, k, nw), rng.random_codes(n, k, nx)
    w = ap.PackedBitPlanes(m, k, ap.BitWidth(nw), oracle.pack(wc, nw))
    x = ap.PackedBitPlanes(n, k, ap.BitWidth(nx), oracle.pack(xc, nx))
    stack = oracle.plane_products(w.words(), m, nw, x.words(), n, nx, k)
    for i in range(nw):
        for j in range(nx):
            assert np.array_equal(ap.matmul_plane_pair(w, i, x, j, ctx), stack[i, j])
    with pytest.raises(ap.IndexOutOfBounds):
        ap.matmul_plane_pair(w, nw, x, 0, ctx)


# ---------------------------------------------------------------- requant (8(f) row 3)
def _requant_case(ap, ctx, n_out, m_tok, k, nw, nx, n_next, gran, route, seed):
    """matmul_ap_requant vs apmm_cu_quantize_pack((double) dequant(Y)^T) on the same device
    data: planes and scales bit-identical, yf bit-identical to the dequant call."""
    import torch
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    wc = torch.randint(0, 1 << nw, (n_out, k), generator=g, device=dev, dtype=torch.uint8)
    xc = torch.randint(0, 1 << nx, (m_tok, k), generator=g, device=dev, dtype=torch.uint8)
    wpr = (k + 31) // 32
    wp = torch.empty(nw * n_out * wpr, dtype=torch.int32, device=dev)
    xp = torch.empty(nx * m_tok * wpr, dtype=torch.int32, device=dev)
    ap.cu_pack(wc, n_out, k, nw, wp, ctx)
    ap.cu_pack(xc, m_tok, k, nx, xp, ctx)
    sw = torch.rand(n_out, dtype=torch.float64, device=dev, generator=g) + 0.01
    sx = torch.rand(m_tok, dtype=torch.float64, device=dev, generator=g) + 0.01
    yf = torch.empty((n_out, m_tok), dtype=torch.float32, device=dev)
    wpr2 = (n_out + 31) // 32
    planes = torch.empty(n_next * m_tok * wpr2, dtype=torch.int32, device=dev)
    scales = torch.empty(m_tok if gran == PER_ROW else 1, dtype=torch.float64, device=dev)
    old = ctx.route()
    ctx.set_route(route)
    try:
        ap.cu_matmul_ap_requant(wp, n_out, nw, sw, 1, xp, m_tok, nx, sx, 1, k, n_next, gran, yf,
                                planes, scales, ctx=ctx)
        ref_yf = torch.empty_like(yf)
        ap.cu_matmul_ap_dequant(wp, n_out, nw, sw, 1, xp, m_tok, nx, sx, 1, k, ref_yf, ctx)
    finally:
        ctx.set_route(old)
    xt = ref_yf.double().t().contiguous()
    ref_planes = torch.empty_like(planes)
    ref_scales = torch.empty_like(scales)
    ap.cu_quantize_pack(xt, m_tok, n_out, n_next, gran, ref_planes, ref_scales, ctx=ctx)
    torch.cuda.synchronize()
    assert torch.equal(yf, ref_yf)
    assert torch.equal(scales, ref_scales)
    assert torch.equal(planes, ref_planes)
    return yf, planes, scales


@pytest.mark.parametrize("n_out,m_tok,k,nw,nx,n_next,gran,route", [
    (2304, 2560, 4096, 2, 4, 4, PER_ROW, "PAIR"),
    (2305, 300, 1000, 3, 8, 2, PER_TENSOR, "SINGLE_SM"),
    (4096, 16, 4096, 3, 8, 8, PER_ROW, "SKINNY"),
    (1000, 37, 999, 2, 4, 3, PER_TENSOR, "AUTO"),
    (2304, 2560, 4096, 2, 2, 4, PER_ROW, "PAIR_WPLANES"),
    (100, 5, 64, 1, 1, 1, PER_ROW, "AUTO")])
def test_requant_bit_identical_to_quantize_of_dequant(gpu, n_out, m_tok, k, nw, nx, n_next,
                                                      gran, route):
    ap, ctx = gpu
    _requant_case(ap, ctx, n_out, m_tok, k, nw, nx, n_next, gran, getattr(ap.Route, route),
                  n_out + m_tok)


def test_requant_split_form_equals_fused(gpu):
    """The N-sharded form: absmax out of the GEMM, reduced (here: one shard), then
    apmm_cu_requant_pack -- same bits as the single-call form."""
    import torch
    ap, ctx = gpu
    yf, planes, scales = _requant_case(ap, ctx, 2048, 512, 2048, 2, 4, 4, PER_ROW, ap.Route.AUTO, 9)
    dev = yf.device
    amax = yf.abs().amax(dim=0).double()
    p2, s2 = torch.empty_like(planes), torch.empty_like(scales)
    ap.cu_requant_pack(yf, 2048, 512, amax, 4, PER_ROW, p2, s2, ctx=ctx)
    torch.cuda.synchronize()
    assert torch.equal(p2, planes) and torch.equal(s2, scales)


def test_requant_nonfinite(gpu):
    import torch
    ap, ctx = gpu
    dev = torch.device("cuda", 0)
    yf = torch.zeros((64, 8), dtype=torch.float32, device=dev)
    yf[3, 5] = float("inf")
    amax = yf.abs().amax(dim=0).double()
    p = torch.empty(4 * 8 * 2, dtype=torch.int32, device=dev)
    s = torch.empty(8, dtype=torch.float64, device=dev)
    with pytest.raises(ap.NonFinite):
        ap.cu_requant_pack(yf, 64, 8, amax, 4, PER_ROW, p, s, ctx=ctx)


# ---------------------------------------------------------------- graphs and streams
def test_graph_capture_needs_reserve(gpu):
    """No hot call synchronises or allocates: a first call at a larger shape inside a CUDA
    graph capture is refused (InvalidArgument) instead of breaking the capture, and after
    apmm_ctx_reserve the same call captures and replays bit-exactly."""
    import torch
    ap, _ = gpu
    ctx = ap.Context(0)
    dev = torch.device("cuda", 0)
    n_out, m_tok, k, nw, nx = 4096, 2048, 4096, 2, 4
    wpr = k // 32
    wp = torch.randint(-2**31, 2**31 - 1, (nw * n_out * wpr,), dtype=torch.int32, device=dev)
    xp = torch.randint(-2**31, 2**31 - 1, (nx * m_tok * wpr,), dtype=torch.int32, device=dev)
    y = torch.empty((n_out, m_tok), dtype=torch.int32, device=dev)
    s = torch.cuda.Stream()
    ctx.set_stream(s)
    g = torch.cuda.CUDAGraph()
    err = None
    with torch.cuda.graph(g, stream=s):
        try:
            ap.cu_matmul_ap(wp, n_out, nw, xp, m_tok, nx, k, y, ctx, stream=s)
        except ap.InvalidArgument as e:
            err = e
    assert err is not None and "apmm_ctx_reserve" in str(err)
    ctx.reserve(n_out, m_tok, k, nw)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ap.cu_matmul_ap(wp, n_out, nw, xp, m_tok, nx, k, y, ctx, stream=s)
    y.zero_()
    g.replay()
    torch.cuda.synchronize()
    want = torch.empty_like(y)
    ap.cu_matmul_ap(wp, n_out, nw, xp, m_tok, nx, k, want, ap.Context(0))
    torch.cuda.synchronize()
    assert torch.equal(y, want)


def test_context_is_bound_to_one_stream(gpu):
    import torch
    ap, _ = gpu
    ctx = ap.Context(0)
    dev = torch.device("cuda", 0)
    wp = torch.zeros(2 * 64 * 4, dtype=torch.int32, device=dev)
    y = torch.empty((64, 64), dtype=torch.int32, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ap.cu_matmul_ap(wp, 64, 2, wp, 64, 2, 128, y, ctx, stream=s1)
    with pytest.raises(ap.InvalidArgument):
        ap.cu_matmul_ap(wp, 64, 2, wp, 64, 2, 128, y, ctx, stream=s2)
    s1.synchronize()
    ctx.set_stream(s2)
    ap.cu_matmul_ap(wp, 64, 2, wp, 64, 2, 128, y, ctx, stream=s2)
    torch.cuda.synchronize()
    # the default wrappers key their context by (device, stream): no error, no race
    ap.cu_matmul_ap(wp, 64, 2, wp, 64, 2, 128, y, stream=s1)
    ap.cu_matmul_ap(wp, 64, 2, wp, 64, 2, 128, y, stream=s2)
    torch.cuda.synchronize()


def test_early_read_options_are_bit_identical(gpu, oracle):
    """APMM_OPT_EARLY_WEIGHT_READ = 0 (every operand read after the previous kernel) and
    APMM_OPT_EARLY_FEATURE_READ = 1 (features read early too) give the same bits on the
    expand + GEMM and skinny routes."""
    import torch
    ap, _ = gpu
    ctx = ap.Context(0)
    dev = torch.device("cuda", 0)
    for (n_out, m_tok, k) in [(2304, 2560, 4096), (4096, 8, 4096)]:
        wp = torch.randint(-2**31, 2**31 - 1, (2 * n_out * k // 32,), dtype=torch.int32, device=dev)
        xp = torch.randint(-2**31, 2**31 - 1, (4 * m_tok * k // 32,), dtype=torch.int32, device=dev)
        y1 = torch.empty((n_out, m_tok), dtype=torch.int32, device=dev)
        y2 = torch.empty_like(y1)
        ap.cu_matmul_ap(wp, n_out, 2, xp, m_tok, 4, k, y1, ctx)
        ctx.set_early_weight_read(False)
        ap.cu_matmul_ap(wp, n_out, 2, xp, m_tok, 4, k, y2, ctx)
        ctx.set_early_weight_read(True)
        y3 = torch.empty_like(y1)
        ctx.set_early_feature_read(True)
        ap.cu_matmul_ap(wp, n_out, 2, xp, m_tok, 4, k, y3, ctx)
        ap.cu_matmul_ap(wp, n_out, 2, xp, m_tok, 4, k, y3, ctx)
        ctx.set_early_feature_read(False)
        torch.cuda.synchronize()
        assert torch.equal(y1, y2) and torch.equal(y1, y3)


def test_graph_replays_of_every_route(gpu):
    """Back-to-back calls captured once and replayed several times (the serving pattern):
    the PDL chain between calls, the ping-pong workspace halves, K6's feature prep + stream-K
    reduce-adds (M = 16, 128) and the mid route's in-kernel grid barrier (count + generation,
    reused across replays; M = 256) give the eager results on every replay."""
    import torch
    ap, _ = gpu
    dev = torch.device("cuda", 0)
    s = torch.cuda.Stream()
    shapes = [(4096, 8, 4096, 3, 8), (4096, 128, 4096, 2, 4), (2304, 2560, 4096, 2, 4),
              (4096, 512, 4096, 2, 4), (8192, 16, 8192, 3, 8), (4096, 256, 4096, 2, 4),
              (8192, 63, 8192, 3, 8)]
    for (n_out, m, k, nw, nx) in shapes:
        ctx = ap.Context(0)
        ctx.set_stream(s)
        ctx.reserve(n_out, m, k, nw)
        wpr = k // 32
        ws = [torch.randint(-2**31, 2**31 - 1, (nw * n_out * wpr,), dtype=torch.int32, device=dev)
              for _ in range(3)]
        xs = [torch.randint(-2**31, 2**31 - 1, (nx * m * wpr,), dtype=torch.int32, device=dev)
              for _ in range(3)]
        ys = [torch.empty((n_out, m), dtype=torch.int32, device=dev) for _ in range(3)]
        want = []
        ref_ctx = ap.Context(0)
        for i in range(3):
            y = torch.empty_like(ys[i])
            ap.cu_matmul_ap(ws[i], n_out, nw, xs[i], m, nx, k, y, ref_ctx)
            want.append(y)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(3):
                ap.cu_matmul_ap(ws[i], n_out, nw, xs[i], m, nx, k, ys[i], ctx, stream=s)
        for rep in range(3):
            for y in ys:
                y.fill_(-1)
            g.replay()
            torch.cuda.synchronize()
            for i in range(3):
                assert torch.equal(ys[i], want[i]), (n_out, m, k, rep, i)
