"""GPU parity: the B200 path (through the C ABI) against the oracle / reference, bit for
bit on integers, on the same seeded inputs. Mirrors the reference's own tests
(proj/tests/test_kernel.cpp, test_bitplane.cpp, test_bipolar.cpp, acceptance.cpp) and
extends them to BASELINE.json's full sizes via exact row-sampled checks."""
import os
import subprocess

import numpy as np
import pytest

from oracle import PER_ROW, PER_TENSOR

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def planes(ap, oracle, codes, n):
    rows, cols = codes.shape
    return ap.PackedBitPlanes(rows, cols, ap.BitWidth(n), oracle.pack(codes, n))


def gpu_matmul(ap, ctx, oracle, wc, nw, xc, nx, cfg=None):
    w, x = planes(ap, oracle, wc, nw), planes(ap, oracle, xc, nx)
    return ap.matmul_ap(w, x, cfg or ap.TileConfig(), ctx)


# ---------------------------------------------------------------- known answers
def test_worked_two_bit_example(gpu, oracle):
    ap, ctx = gpu
    # test_kernel.cpp:125-136: W=[3,1], X=[-1,3] -> 0
    wc = np.array([[0b11, 0b10]], np.uint8)
    xc = np.array([[0b01, 0b11]], np.uint8)
    assert gpu_matmul(ap, ctx, oracle, wc, 2, xc, 2).tolist() == [[0]]
    # 1-bit worked row (test_kernel.cpp:58-66): [+1,+1].[-1,+1] = 0
    assert gpu_matmul(ap, ctx, oracle, np.array([[1, 1]], np.uint8), 1,
                      np.array([[0, 1]], np.uint8), 1).tolist() == [[0]]


def test_k1_plane_products_are_signs(gpu, oracle):
    ap, ctx = gpu
    rng = oracle.rng(3)
    for _ in range(20):
        wc, xc = rng.random_codes(3, 1, 2), rng.random_codes(4, 1, 2)
        assert np.array_equal(gpu_matmul(ap, ctx, oracle, wc, 2, xc, 2),
                              oracle.decoded_matmul(wc, 2, xc, 2))


def test_ragged_k40(gpu, oracle):
    ap, ctx = gpu
    rng = oracle.rng(27)  # test_kernel.cpp:226-231
    wc, xc = rng.random_codes(6, 40, 3), rng.random_codes(5, 40, 2)
    assert np.array_equal(gpu_matmul(ap, ctx, oracle, wc, 3, xc, 2),
                          oracle.decoded_matmul(wc, 3, xc, 2))


def test_golden_vectors_from_reference(gpu, golden):
    ap, ctx = gpu
    for c in golden["matmul"]:
        w = ap.PackedBitPlanes(c["rows_w"], c["k"], ap.BitWidth(c["n_w"]),
                               np.array(c["w_words"], np.uint32))
        x = ap.PackedBitPlanes(c["rows_x"], c["k"], ap.BitWidth(c["n_x"]),
                               np.array(c["x_words"], np.uint32))
        assert ap.matmul_ap(w, x, ctx=ctx).reshape(-1).tolist() == c["y"]


# ---------------------------------------------------------------- randomized corpora
def test_randomized_corpus_200(gpu, oracle):
    ap, ctx = gpu
    rng = oracle.rng(31)  # test_kernel.cpp:233-245
    for _ in range(200):
        m, n, k = rng.range(1, 32), rng.range(1, 32), rng.range(1, 200)
        nw, nx = rng.range(1, 8), rng.range(1, 8)
        wc, xc = rng.random_codes(m, k, nw), rng.random_codes(n, k, nx)
        assert np.array_equal(gpu_matmul(ap, ctx, oracle, wc, nw, xc, nx),
                              oracle.decoded_matmul(wc, nw, xc, nx)), (m, n, k, nw, nx)


def test_acceptance_oracle_equivalence_1000(gpu, oracle):
    ap, ctx = gpu
    rng = oracle.rng(101)  # acceptance.cpp:56-77
    for _ in range(1000):
        m, n, k = rng.range(1, 32), rng.range(1, 32), rng.range(1, 200)
        nw, nx = rng.range(1, 8), rng.range(1, 8)
        wc, xc = rng.random_codes(m, k, nw), rng.random_codes(n, k, nx)
        assert np.array_equal(gpu_matmul(ap, ctx, oracle, wc, nw, xc, nx),
                              oracle.decoded_matmul(wc, nw, xc, nx))


def test_tile_shapes_and_edges(gpu, oracle):
    """Shapes straddling the 128x256x128 tile grid, ragged in every dimension."""
    ap, ctx = gpu
    rng = oracle.rng(77)
    for (m, n, k) in [(127, 255, 127), (128, 256, 128), (129, 257, 129), (300, 513, 1000),
                      (1, 600, 300), (700, 1, 300), (257, 3, 4097), (5, 260, 33)]:
        nw, nx = rng.range(1, 8), rng.range(1, 8)
        while oracle.overflow_bound(nw, nx, k) > 2**31 - 1:
            nx -= 1
        wc, xc = rng.random_codes(m, k, nw), rng.random_codes(n, k, nx)
        wp, xp = oracle.pack(wc, nw), oracle.pack(xc, nx)
        want = oracle.matmul_ap_mt(wp, m, nw, xp, n, nx, k, 8)
        assert np.array_equal(gpu_matmul(ap, ctx, oracle, wc, nw, xc, nx), want), (m, n, k)


@pytest.fixture(scope="module")
def gpu_tc(gpu):
    """A second context pinned to the tensor-core (expand + tcgen05) routes for every shape
    (APMM_ROUTE_TENSOR_CORE: AUTO without K5), so small shapes also exercise them."""
    ap, _ = gpu
    ctx = ap.Context(0)
    ctx.set_route(ap.Route.TENSOR_CORE)
    return ap, ctx


class _route:
    """Pin a context's kernel route for a block (apmm_ctx_set_option APMM_OPT_ROUTE)."""

    def __init__(self, ctx, route):
        self.ctx, self.route = ctx, route

    def __enter__(self):
        self.old = self.ctx.route()
        self.ctx.set_route(self.route)

    def __exit__(self, *exc):
        self.ctx.set_route(self.old)


def test_randomized_corpus_tensor_core_path(gpu_tc, oracle):
    ap, ctx = gpu_tc
    rng = oracle.rng(31)
    for _ in range(200):
        m, n, k = rng.range(1, 40), rng.range(1, 80), rng.range(1, 300)
        nw, nx = rng.range(1, 8), rng.range(1, 8)
        wc, xc = rng.random_codes(m, k, nw), rng.random_codes(n, k, nx)
        assert np.array_equal(gpu_matmul(ap, ctx, oracle, wc, nw, xc, nx),
                              oracle.decoded_matmul(wc, nw, xc, nx)), (m, n, k, nw, nx)


@pytest.mark.parametrize("m_tok", [1, 2, 7, 8, 9, 16, 17, 31, 33, 64])
def test_skinny_path_shapes(gpu, gpu_tc, oracle, m_tok):
    """Few feature rows (K5: weight planes streamed into mma.sync): ragged rows, ragged K,
    the unaligned (scalar-load) path, every weight width, and the single-accumulator variant
    (K*(2^n_w-1)*(2^n_x-1) >= 2^28). Checked against the oracle and the tensor-core path."""
    ap, ctx = gpu
    _, ctx_tc = gpu_tc
    rng = oracle.rng(500 + m_tok)
    for (n_out, k, nw, nx) in [(300, 1000, 3, 8), (129, 4096, 2, 4), (1000, 777, 8, 8),
                               (257, 8232, 4, 8), (40, 70200, 4, 8), (33, 40, 1, 1),
                               (130, 100, 5, 3), (128, 2048, 1, 2), (17, 33025, 8, 8)]:
        wc, xc = rng.random_codes(n_out, k, nw), rng.random_codes(m_tok, k, nx)
        wp, xp = oracle.pack(wc, nw), oracle.pack(xc, nx)
        want = oracle.matmul_ap_mt(wp, n_out, nw, xp, m_tok, nx, k, os.cpu_count() or 4)
        w = ap.PackedBitPlanes(n_out, k, ap.BitWidth(nw), wp)
        x = ap.PackedBitPlanes(m_tok, k, ap.BitWidth(nx), xp)
        assert np.array_equal(ap.matmul_ap(w, x, ctx=ctx), want), (n_out, m_tok, k, nw, nx)
        assert np.array_equal(ap.matmul_ap(w, x, ctx=ctx_tc), want), (n_out, m_tok, k, nw, nx)


def test_schedule_independence(gpu, oracle):
    ap, ctx = gpu
    rng = oracle.rng(707)  # acceptance.cpp:268-294: 100x100x300 W3A4, 9 configs
    wc, xc = rng.random_codes(100, 300, 3), rng.random_codes(100, 300, 4)
    ref = gpu_matmul(ap, ctx, oracle, wc, 3, xc, 4)
    assert np.array_equal(ref, oracle.decoded_matmul(wc, 3, xc, 4))
    for cfg in [(1, 1, 32), (1, 100, 32), (100, 1, 96), (100, 100, 320), (128, 128, 4096),
                (7, 13, 64), (33, 17, 160), (3, 97, 2048), (64, 64, 512)]:
        assert np.array_equal(gpu_matmul(ap, ctx, oracle, wc, 3, xc, 4, ap.TileConfig(*cfg)), ref)


def test_determinism(gpu, oracle):
    ap, ctx = gpu
    rng = oracle.rng(5)
    wc, xc = rng.random_codes(333, 777, 4), rng.random_codes(444, 777, 8)
    a = gpu_matmul(ap, ctx, oracle, wc, 4, xc, 8)
    b = gpu_matmul(ap, ctx, oracle, wc, 4, xc, 8)
    assert np.array_equal(a, b)


# ---------------------------------------------------------------- overflow contract
def test_overflow_guard(gpu, oracle):
    ap, ctx = gpu
    rng = oracle.rng(99)  # verify.cpp:373-409
    wc, xc = rng.random_codes(1, 33026, 8), rng.random_codes(1, 33026, 8)
    with pytest.raises(ap.OverflowBound):
        gpu_matmul(ap, ctx, oracle, wc, 8, xc, 8)
    wc, xc = rng.random_codes(3, 33025, 8), rng.random_codes(2, 33025, 8)
    assert np.array_equal(gpu_matmul(ap, ctx, oracle, wc, 8, xc, 8),
                          oracle.decoded_matmul(wc, 8, xc, 8))
    # extreme codes: all-max and all-min at the admissible edge (|Y| = bound)
    for cw, cx in [(255, 255), (0, 255), (0, 0)]:
        wc = np.full((2, 33025), cw, np.uint8)
        xc = np.full((3, 33025), cx, np.uint8)
        got = gpu_matmul(ap, ctx, oracle, wc, 8, xc, 8)
        assert np.array_equal(got, oracle.decoded_matmul(wc, 8, xc, 8))
        assert abs(int(got[0, 0])) == 33025 * 255 * 255


def test_dimension_mismatch(gpu, oracle):
    ap, ctx = gpu
    w = planes(ap, oracle, np.ones((1, 2), np.uint8), 1)
    x = planes(ap, oracle, np.ones((1, 3), np.uint8), 1)
    with pytest.raises(ap.DimensionMismatch):
        ap.matmul_ap(w, x, ctx=ctx)


# ---------------------------------------------------------------- full BASELINE sizes
def _sample_rows(n_out, seed, sample=None):
    """Two random W rows from every 256-row tile (the pair GEMM's M tile) plus the first and
    last row; or, with `sample`, that many random rows."""
    rng = np.random.default_rng(seed)
    if sample is not None:
        extra = rng.integers(0, n_out, size=sample)
    else:
        extra = np.concatenate([t0 + rng.integers(0, min(256, n_out - t0), size=2)
                                for t0 in range(0, n_out, 256)])
    return np.unique(np.concatenate([np.array([0, n_out - 1]), extra]))


def _reference_rows(oracle, w_rows_planes, rows, nw, x_planes, m_tok, nx, k):
    """matmul_ap of the sampled W rows by the reference library itself when it is built
    (oracle/_ref), else by the C restatement; row-sliced over the host threads."""
    from oracle import Reference
    threads = os.cpu_count() or 4
    if Reference.available():
        job = Reference().job(w_rows_planes, rows, nw, x_planes, m_tok, nx, k, threads)
        job.run()
        return job.result()
    return oracle.matmul_ap_mt(w_rows_planes, rows, nw, x_planes, m_tok, nx, k, threads)


def _device_operands(ap, ctx, n_out, m_tok, k, nw, nx, seed):
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
    return wc, xc, wp, xp


def _check_rows(oracle, y, wc, xc, wp, xp, n_out, m_tok, k, nw, nx, rows):
    """y[rows] (device) == reference matmul_ap on those W rows; the device packs of the
    sampled rows and of X are themselves checked against the oracle's pack."""
    import torch
    wpr = (k + 31) // 32
    idx = torch.as_tensor(rows, device=wp.device, dtype=torch.long)
    wc_h = wc.index_select(0, idx).cpu().numpy()
    xc_h = xc.cpu().numpy()
    xp_h = xp.cpu().numpy().view(np.uint32)
    wp_rows = wp.view(nw, n_out, wpr).index_select(1, idx).contiguous().cpu().numpy().view(np.uint32)
    assert np.array_equal(xp_h, oracle.pack(xc_h, nx))
    assert np.array_equal(wp_rows.reshape(-1), oracle.pack(wc_h, nw))
    want = _reference_rows(oracle, wp_rows.reshape(-1), len(rows), nw, xp_h, m_tok, nx, k)
    got = y.index_select(0, idx).cpu().numpy()
    assert np.array_equal(got, want), (n_out, m_tok, k, nw, nx, int((got != want).sum()))


def _row_sample_check(ap, ctx, oracle, n_out, m_tok, k, nw, nx, seed, sample=None):
    """Exact check of sampled output rows (two per 256-row tile unless `sample` is given;
    all columns) against the reference computed on just those weight rows."""
    import torch
    dev = torch.device("cuda", 0)
    wc, xc, wp, xp = _device_operands(ap, ctx, n_out, m_tok, k, nw, nx, seed)
    y = torch.empty((n_out, m_tok), dtype=torch.int32, device=dev)
    ap.cu_matmul_ap(wp, n_out, nw, xp, m_tok, nx, k, y, ctx)
    torch.cuda.synchronize()
    _check_rows(oracle, y, wc, xc, wp, xp, n_out, m_tok, k, nw, nx, _sample_rows(n_out, seed, sample))
    return y


def _route_vs_route(ap, ctx, oracle, n_out, m_tok, k, nw, nx, seed, route, other):
    """`route` against the oracle on sampled rows, then bit-equal to `other` on every entry."""
    import torch
    with _route(ctx, route):
        y = _row_sample_check(ap, ctx, oracle, n_out, m_tok, k, nw, nx, seed=seed, sample=24)
    wc, xc, wp, xp = _device_operands(ap, ctx, n_out, m_tok, k, nw, nx, seed)
    y2 = torch.empty((n_out, m_tok), dtype=torch.int32, device=wp.device)
    with _route(ctx, other):
        ap.cu_matmul_ap(wp, n_out, nw, xp, m_tok, nx, k, y2, ctx)
    torch.cuda.synchronize()
    assert torch.equal(y, y2), (n_out, m_tok, k, nw, nx, route, other)
    return wp, xp, y2


@pytest.mark.parametrize("nw,nx,n_out,m_tok,k", [
    (1, 2, 2304, 2560, 4096), (2, 4, 2305, 2561, 4200), (3, 8, 2304, 2560, 4224),
    (4, 4, 2560, 2304, 4096), (5, 3, 2304, 2560, 4096), (6, 2, 2304, 2304, 2048),
    (7, 7, 2304, 2560, 4096), (8, 8, 2304, 2560, 4096)])
def test_fused_weight_plane_gemm(gpu, oracle, nw, nx, n_out, m_tok, k):
    """K3f (APMM_ROUTE_PAIR_WPLANES: weight planes expanded on chip by transform warps)
    against the oracle on sampled rows and, on the full output, against K1 + K3
    (APMM_ROUTE_PAIR). The shapes fill >= 74 CTA pairs and cover every weight width, ragged
    rows, the half-width last-wave tiles and a tail word (K % 32 != 0 with ceil(K/32) % 4 ==
    0); also the fp64 dequant epilogue through K3f."""
    import torch
    ap, ctx = gpu
    wp, xp, y2 = _route_vs_route(ap, ctx, oracle, n_out, m_tok, k, nw, nx, nw * 100 + nx,
                                 ap.Route.PAIR_WPLANES, ap.Route.PAIR)
    dev = wp.device
    sw = torch.rand(n_out, dtype=torch.float64, device=dev)
    sx = torch.rand(m_tok, dtype=torch.float64, device=dev)
    f1 = torch.empty((n_out, m_tok), dtype=torch.float32, device=dev)
    with _route(ctx, ap.Route.PAIR_WPLANES):
        ap.cu_matmul_ap_dequant(wp, n_out, nw, sw, 1, xp, m_tok, nx, sx, 1, k, f1, ctx)
    want = ((y2.double() * sw[:, None]) * sx[None, :]).float()
    torch.cuda.synchronize()
    assert torch.equal(f1, want)


def test_forced_route_that_cannot_serve_fails_loudly(gpu):
    """A forced route that cannot serve a call is an InvalidArgument, never a silent
    fallback: K3f needs a 16-byte weight row pitch (ceil(K/32) % 4 == 0), K5 <= 63 rows."""
    import torch
    ap, ctx = gpu
    dev = torch.device("cuda", 0)
    n_out, m_tok, k = 512, 300, 4100  # 129 words per row
    wp = torch.zeros(2 * n_out * 129, dtype=torch.int32, device=dev)
    xp = torch.zeros(2 * m_tok * 129, dtype=torch.int32, device=dev)
    y = torch.empty((n_out, m_tok), dtype=torch.int32, device=dev)
    for route in (ap.Route.PAIR_WPLANES, ap.Route.MID_SPLITK, ap.Route.SKINNY):
        with _route(ctx, route):
            with pytest.raises(ap.InvalidArgument):
                ap.cu_matmul_ap(wp, n_out, 2, xp, m_tok, 2, k, y, ctx)


@pytest.mark.parametrize("n_out,m_tok,k,nw,nx", [
    (4096, 128, 4096, 2, 4), (4096, 512, 4096, 3, 8), (2305, 68, 4200, 1, 2),
    (4096, 1024, 11008, 2, 4), (300, 260, 4224, 8, 8), (11008, 256, 4096, 4, 4),
    (1000, 96, 128, 5, 3)])
def test_mid_size_split_k_path(gpu, oracle, n_out, m_tok, k, nw, nx):
    """Mid-size calls (APMM_ROUTE_MID_SPLITK; AUTO for M_tok <= 256 with few tiles): weight
    planes expanded on chip, rowsum(U_w) in the transform warps, K split over CTA pairs, int32
    partials TMA reduce-added into a Y zeroed by K1. Against the oracle on sampled rows and
    against the 1-SM route on every entry."""
    ap, ctx = gpu
    _route_vs_route(ap, ctx, oracle, n_out, m_tok, k, nw, nx, n_out * 7 + m_tok,
                    ap.Route.MID_SPLITK, ap.Route.SINGLE_SM)


@pytest.mark.parametrize("n_out,m_tok,k,nw,nx", [
    (4096, 64, 4096, 2, 4), (8192, 16, 8192, 3, 8), (4096, 8, 4096, 2, 4), (11008, 32, 4096, 4, 4),
    (4096, 64, 11008, 1, 2), (1000, 4, 4224, 3, 5), (2305, 60, 4200, 2, 8), (300, 12, 128, 4, 1),
    (8192, 48, 8192, 3, 8), (129, 64, 640, 2, 3), (4096, 128, 4096, 2, 4), (1000, 100, 4224, 4, 8),
    (4096, 96, 11008, 3, 4), (2048, 124, 4096, 4, 8), (2051, 128, 1152, 1, 1),
    (8192, 63, 8192, 3, 8), (1000, 17, 4224, 2, 4), (2051, 125, 1152, 1, 1), (300, 30, 640, 4, 2)])
def test_stream_tensor_memory_path(gpu, oracle, n_out, m_tok, k, nw, nx):
    """K6 (APMM_ROUTE_STREAM_TC): weight planes streamed per warp, expanded in registers into
    TMEM as the MMA's A operand, K split over every SM (stream-K ranges, partial tiles TMA
    reduce-added into a Y zeroed by the feature prep), rowsum(U_w) from an all-ones feature row.
    Against the oracle on sampled rows and bit-equal to the 1-SM route on every entry; ragged
    row tiles, a tail word (K % 32 != 0), one-step K, segments that start mid-tile, and feature
    counts that are not a multiple of 4 (a padded Y in the workspace, then an unpad copy)."""
    ap, ctx = gpu
    _route_vs_route(ap, ctx, oracle, n_out, m_tok, k, nw, nx, n_out * 3 + m_tok,
                    ap.Route.STREAM_TC, ap.Route.SINGLE_SM)


@pytest.mark.parametrize("n_out,m_tok,k,nw,nx", [
    (4096, 512, 4096, 2, 4), (2305, 300, 4200, 3, 8), (4096, 1024, 11008, 4, 4),
    (1000, 96, 128, 5, 3)])
def test_pair_split_k_path(gpu, oracle, n_out, m_tok, k, nw, nx):
    """The u8-code pair GEMM with K split over the pairs (APMM_ROUTE_PAIR_SPLITK) == oracle
    on sampled rows and == the AUTO route on every entry."""
    ap, ctx = gpu
    _route_vs_route(ap, ctx, oracle, n_out, m_tok, k, nw, nx, n_out + 3 * m_tok,
                    ap.Route.PAIR_SPLITK, ap.Route.AUTO)


@pytest.mark.parametrize("n_out,m_tok,k,nw,nx", [
    (2304, 2560, 4096, 2, 4), (4096, 128, 4096, 3, 8), (1000, 40, 4096, 2, 4),
    (257, 16, 8232, 4, 8), (4096, 1, 4096, 2, 4)])
def test_every_route_agrees(gpu, oracle, n_out, m_tok, k, nw, nx):
    """Routes are schedules only (like TileConfig): every route that can serve a
    call returns the same bits as the oracle-checked AUTO route."""
    import torch
    ap, ctx = gpu
    y = _row_sample_check(ap, ctx, oracle, n_out, m_tok, k, nw, nx, seed=m_tok + 5)
    wc, xc, wp, xp = _device_operands(ap, ctx, n_out, m_tok, k, nw, nx, m_tok + 5)
    served = 0
    for route in ap.Route:
        y2 = torch.full((n_out, m_tok), -7, dtype=torch.int32, device=wp.device)
        with _route(ctx, route):
            try:
                ap.cu_matmul_ap(wp, n_out, nw, xp, m_tok, nx, k, y2, ctx)
            except ap.InvalidArgument:
                continue
        torch.cuda.synchronize()
        assert torch.equal(y, y2), route
        served += 1
    assert served >= 4


SWEEP = [(nw, nx) for nw in (1, 2, 3, 4) for nx in (2, 4, 8)]


@pytest.mark.parametrize("nw,nx", SWEEP)
def test_config2_4096_cubed_row_sampled(gpu, oracle, nw, nx):
    """BASELINE configs[1]: all 12 sweep precisions at 4096^3 (the bench's sweep4096)."""
    ap, ctx = gpu
    _row_sample_check(ap, ctx, oracle, 4096, 4096, 4096, nw, nx, seed=nw * 10 + nx)


def test_config5_ffn70b_and_shards(gpu, oracle):
    """BASELINE configs[4] -- exactly the bench's default workload: W[28672 x 8192] W2A4 x
    X[4096 x 8192] A4, two rows of every 256-row tile vs the reference's matmul_ap; then
    every shard of the P = 2/4/8 N-sharding (shard.slice_plane_rows + the kernel on the
    shard alone, the per-rank GEMM of bench.py --gpus P) equals its row block of the full Y
    bit for bit, and is itself row-sampled against the reference."""
    import torch
    from paper_2409_17870_b200.shard import shard_bounds, slice_plane_rows
    ap, ctx = gpu
    n_out, m_tok, k, nw, nx = 28672, 4096, 8192, 2, 4
    wc, xc, wp, xp = _device_operands(ap, ctx, n_out, m_tok, k, nw, nx, seed=70)
    y = torch.empty((n_out, m_tok), dtype=torch.int32, device=wp.device)
    ap.cu_matmul_ap(wp, n_out, nw, xp, m_tok, nx, k, y, ctx)
    torch.cuda.synchronize()
    _check_rows(oracle, y, wc, xc, wp, xp, n_out, m_tok, k, nw, nx, _sample_rows(n_out, 70))
    for world in (2, 4, 8):
        for rank in range(world):
            r0, r1 = shard_bounds(n_out, world, rank)
            ws = slice_plane_rows(wp, n_out, k, nw, r0, r1)
            ys = torch.empty((r1 - r0, m_tok), dtype=torch.int32, device=wp.device)
            ap.cu_matmul_ap(ws, r1 - r0, nw, xp, m_tok, nx, k, ys, ctx)
            torch.cuda.synchronize()
            assert torch.equal(ys, y[r0:r1]), (world, rank)
            if rank == world - 1:
                _check_rows(oracle, ys, wc[r0:r1], xc, ws, xp, r1 - r0, m_tok, k, nw, nx,
                            _sample_rows(r1 - r0, world))
    del y


def test_config1_1024_cubed_full_bit_exact(gpu, oracle):
    ap, ctx = gpu
    rng = oracle.rng(1)  # apmm.cpp:150,161-162: seed 1, W then X
    wc, xc = rng.random_codes(1024, 1024, 2), rng.random_codes(1024, 1024, 2)
    wp, xp = oracle.pack(wc, 2), oracle.pack(xc, 2)
    want = oracle.matmul_ap_mt(wp, 1024, 2, xp, 1024, 2, 1024, os.cpu_count() or 4)
    assert np.array_equal(gpu_matmul(ap, ctx, oracle, wc, 2, xc, 2), want)


@pytest.mark.parametrize("n_out,k,m_tok", [(4096, 4096, 2048), (11008, 4096, 512),
                                           (4096, 11008, 128), (4096, 4096, 1)])
def test_config3_llama7b_row_sampled(gpu, oracle, n_out, k, m_tok):
    ap, ctx = gpu
    _row_sample_check(ap, ctx, oracle, n_out, m_tok, k, 2, 4, seed=n_out + k + m_tok)


@pytest.mark.parametrize("m_tok", [1, 8, 16])
def test_config4_decode_w3a8(gpu, oracle, m_tok):
    ap, ctx = gpu
    _row_sample_check(ap, ctx, oracle, 8192, m_tok, 8192, 3, 8, seed=m_tok)


# ---------------------------------------------------------------- pack / unpack / quantize
def test_pack_unpack_match_oracle(gpu, oracle, golden):
    ap, ctx = gpu
    for case in golden["pack"]:
        codes = np.array(case["codes"], np.uint8).reshape(case["rows"], case["cols"])
        p = ap.decompose_and_pack(codes, ap.BitWidth(case["n"]), ctx)
        assert p.words().tolist() == case["words"]
        assert np.array_equal(ap.unpack(p, ctx), codes)
    rng = oracle.rng(7)  # test_bitplane.cpp:68-78: 500 round trips
    for _ in range(100):
        rows, cols, n = rng.range(1, 70), rng.range(1, 70), rng.range(1, 8)
        codes = rng.random_codes(rows, cols, n)
        p = ap.decompose_and_pack(codes, ap.BitWidth(n), ctx)
        assert np.array_equal(p.words(), oracle.pack(codes, n))
        assert np.array_equal(ap.unpack(p, ctx), codes)
    with pytest.raises(ap.OutOfRange):  # CodeMatrix ctor (bipolar.cpp:33-36)
        ap.decompose_and_pack(np.array([[4]], np.uint8), ap.BitWidth(2), ctx)


def test_quantize_bit_exact(gpu, oracle, golden):
    ap, ctx = gpu
    for case in golden["quantize"]:
        x = np.array([float.fromhex(h) for h in case["x"]]).reshape(case["rows"], case["cols"])
        q = ap.quantize(x, ap.BitWidth(case["n"]), ap.Granularity(case["gran"]), ctx)
        assert q.codes.reshape(-1).tolist() == case["codes"]
        assert [float(v).hex() for v in q.scales] == case["scales"]
        assert np.array_equal(q.packed.words(), oracle.pack(q.codes, case["n"]))
    rng = np.random.default_rng(606)  # acceptance.cpp:236-263 style inputs
    for t in range(40):
        rows, cols, n = int(rng.integers(1, 80)), int(rng.integers(1, 300)), int(rng.integers(1, 9))
        x = rng.uniform(-100, 100, size=(rows, cols))
        x[rng.random(size=x.shape) < 0.1] = 0.0
        if t % 5 == 0:
            x[0] = 0.0
        for gran in (PER_TENSOR, PER_ROW):
            q = ap.quantize(x, ap.BitWidth(n), ap.Granularity(gran), ctx)
            c, s = oracle.quantize(x, n, gran)
            assert np.array_equal(q.codes, c) and np.array_equal(q.scales, s)
    # grid-boundary inputs: values at and within a few ulps of every multiple of the scale
    # (where floor(x / (2s)) flips), exact zeros, tiny and huge magnitudes -- the quantizer's
    # reciprocal fast path must hand every such element to the exact division
    for n in (1, 2, 3, 4, 8):
        maxv = (1 << n) - 1
        for amax in (float(maxv), 1.0, 3.0e-300, 7.25e250, 0.1):
            sc = amax / maxv
            ks = np.arange(-maxv - 1, maxv + 2, dtype=np.float64)
            base = ks * sc
            x = np.concatenate([base, np.nextafter(base, np.inf), np.nextafter(base, -np.inf),
                                np.nextafter(np.nextafter(base, np.inf), np.inf),
                                np.nextafter(np.nextafter(base, -np.inf), -np.inf), [0.0, -0.0]])
            x = np.clip(x, -amax, amax)
            x[0] = amax  # the absmax (and so the scale) is exactly `amax`
            x = np.ascontiguousarray(np.tile(x, (3, 1)))
            for gran in (PER_TENSOR, PER_ROW):
                q = ap.quantize(x, ap.BitWidth(n), ap.Granularity(gran), ctx)
                c, sref = oracle.quantize(x, n, gran)
                assert np.array_equal(q.codes, c) and np.array_equal(q.scales, sref), (n, amax)
    with pytest.raises(ap.NonFinite):
        ap.quantize(np.array([[1.0, np.nan]]), ap.BitWidth(2), ap.Granularity.PerTensor, ctx)
    with pytest.raises(ap.NonFinite):
        ap.quantize(np.array([[1.0], [np.inf]]), ap.BitWidth(2), ap.Granularity.PerRow, ctx)


def test_dequant_epilogue(gpu, oracle):
    """Fused dequant vs the CLI epilogue (apmm.cpp:329-340) computed by the oracle in fp64:
    north-star tolerance 1e-3 relative; the device does the same fp64 ops, so it is exact."""
    ap, ctx = gpu
    rng = np.random.default_rng(11)
    # (n = 8 and 16 feature rows take K5's popcount-rowsum variant)
    for (m, n, k, nw, nx, gw, gx) in [(1, 1, 2, 2, 2, 0, 0), (64, 48, 300, 2, 4, 1, 1),
                                      (300, 257, 1000, 3, 8, 1, 0), (129, 1, 4096, 4, 8, 0, 1),
                                      (500, 8, 4096, 3, 8, 1, 1), (257, 16, 2048, 2, 4, 0, 1)]:
        wv, xv = rng.uniform(-1, 1, (m, k)), rng.uniform(-1, 1, (n, k))
        wc, ws = oracle.quantize(wv, nw, gw)
        xc, xs = oracle.quantize(xv, nx, gx)
        w, x = planes(ap, oracle, wc, nw), planes(ap, oracle, xc, nx)
        got = ap.matmul_ap_dequant(w, ws, ap.Granularity(gw), x, xs, ap.Granularity(gx), ctx)
        y = oracle.matmul_ap(w.words(), m, nw, x.words(), n, nx, k)
        want = oracle.dequant_epilogue(y, ws, gw, xs, gx)
        np.testing.assert_allclose(got, want, rtol=1e-3, atol=0)
        assert np.array_equal(got, want)
    # CLI worked example (test_cli.cpp:147-181) -> 0
    wc, ws = oracle.quantize(np.array([[3.0, 1.0]]), 2, 0)
    xc, xs = oracle.quantize(np.array([[-1.0, 3.0]]), 2, 0)
    out = ap.matmul_ap_dequant(planes(ap, oracle, wc, 2), ws, ap.Granularity.PerTensor,
                               planes(ap, oracle, xc, 2), xs, ap.Granularity.PerTensor, ctx)
    assert out.tolist() == [[0.0]]


def test_end_to_end_quantize_pack_matmul_dequant(gpu, oracle):
    """The whole north-star path on device: fp64 activations -> quantize+pack (K2) ->
    GEMM (K3) -> dequant, vs the oracle chain."""
    ap, ctx = gpu
    rng = np.random.default_rng(2409)
    wv, xv = rng.uniform(-1, 1, (256, 512)), rng.uniform(-1, 1, (130, 512))
    qw = ap.quantize(wv, ap.BitWidth(2), ap.Granularity.PerRow, ctx)
    qx = ap.quantize(xv, ap.BitWidth(4), ap.Granularity.PerRow, ctx)
    got = ap.matmul_ap_dequant(qw.packed, qw.scales, qw.granularity, qx.packed, qx.scales,
                               qx.granularity, ctx)
    wc, ws = oracle.quantize(wv, 2, PER_ROW)
    xc, xs = oracle.quantize(xv, 4, PER_ROW)
    y = oracle.decoded_matmul(wc, 2, xc, 4)
    assert np.array_equal(got, oracle.dequant_epilogue(y, ws, PER_ROW, xs, PER_ROW))


# ---------------------------------------------------------------- the reference's own suite
def test_reference_run_verify_with_gpu_kernel():
    """apmm::run_verify (verify.cpp:413-463) with the B200 kernel in its KernelFn seam,
    via include/apmm_b200.hpp; plus the mutation check (test_verify.cpp:47-86)."""
    exe = os.path.join(ROOT, "oracle", "_ref", "verify_gpu")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/verify_gpu not built")
    for seed in ("1", "2"):
        r = subprocess.run([exe, seed, "1000"], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout + r.stderr
        assert r.stdout.count("PASS") == 12 and "mutant kernel caught" in r.stdout
        assert "PASS compute_plane_products + recover on the device" in r.stdout
        assert "PASS xor_identity / dot_1bit_xor / matmul_plane_pair through the drop-in" in r.stdout


def test_host_api_row_block_pipeline(gpu, oracle):
    """The synchronous host entry points pipeline large calls over row blocks of W / Y
    (H2D, GEMM and D2H on three streams): outputs > 16 MB, ragged last block, int32 and
    dequant, against the oracle on sampled rows and the device entry point on all rows."""
    import torch
    ap, ctx = gpu
    rng = np.random.default_rng(5)
    for (m, n, k, nw, nx) in [(4173, 1100, 256, 3, 4), (2300, 2049, 96, 2, 2), (700, 40, 4000, 4, 8),
                              (45000, 100, 256, 2, 4), (300, 44, 4096, 1, 8)]:
        wc = rng.integers(0, 1 << nw, size=(m, k), dtype=np.uint8)
        xc = rng.integers(0, 1 << nx, size=(n, k), dtype=np.uint8)
        wp, xp = oracle.pack(wc, nw), oracle.pack(xc, nx)
        w = ap.PackedBitPlanes(m, k, ap.BitWidth(nw), wp)
        x = ap.PackedBitPlanes(n, k, ap.BitWidth(nx), xp)
        got = ap.matmul_ap(w, x, ctx=ctx)
        rows = np.unique(np.concatenate([[0, m - 1], rng.integers(0, m, 24)]))
        want = oracle.matmul_ap_mt(oracle.pack(wc[rows], nw), len(rows), nw, xp, n, nx, k, 8)
        assert np.array_equal(got[rows], want), (m, n, k)
        dev = torch.device("cuda", 0)
        yd = torch.empty((m, n), dtype=torch.int32, device=dev)
        ap.cu_matmul_ap(torch.from_numpy(wp.view(np.int32)).to(dev), m, nw,
                        torch.from_numpy(xp.view(np.int32)).to(dev), n, nx, k, yd, ctx)
        torch.cuda.synchronize()
        assert np.array_equal(got, yd.cpu().numpy()), (m, n, k)
        sw, sx = rng.random(m), rng.random(n)
        deq = ap.matmul_ap_dequant(w, sw, ap.Granularity.PerRow, x, sx, ap.Granularity.PerRow, ctx)
        assert np.array_equal(deq, oracle.dequant_epilogue(got, sw, 1, sx, 1))


@pytest.mark.parametrize("rows_w,rows_x,k,nw,nx,gx", [
    (300, 260, 1000, 3, 4, 1), (2305, 2561, 4200, 2, 4, 0), (513, 700, 33, 4, 8, 1),
    (4096, 2048, 4096, 2, 4, 1), (300, 16, 1000, 3, 8, 0), (129, 1, 4096, 2, 4, 1)])
def test_fused_quantize_matmul_dequant(gpu, oracle, rows_w, rows_x, k, nw, nx, gx):
    """K2 -> K3 (quantizer writes the GEMM operand) == quantize_pack +
    matmul_ap_dequant, bit for bit, including X's scales; skinny shapes go through planes."""
    import torch
    ap, ctx = gpu
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(rows_w + rows_x + k)
    wc = torch.randint(0, 1 << nw, (rows_w, k), generator=g, device=dev, dtype=torch.uint8)
    wpr = (k + 31) // 32
    wp = torch.empty(nw * rows_w * wpr, dtype=torch.int32, device=dev)
    ap.cu_pack(wc, rows_w, k, nw, wp, ctx)
    sw = torch.rand(rows_w, dtype=torch.float64, device=dev, generator=g)
    xv = (torch.rand((rows_x, k), dtype=torch.float64, device=dev, generator=g) - 0.5) * 200
    xv[xv.abs() < 10] = 0.0  # zeros, as the acceptance test's inputs (acceptance.cpp:247)
    n_sx = rows_x if gx else 1
    sx1 = torch.empty(n_sx, dtype=torch.float64, device=dev)
    out1 = torch.empty((rows_w, rows_x), dtype=torch.float32, device=dev)
    ap.cu_quantize_matmul_ap_dequant(wp, rows_w, nw, sw, 1, xv, rows_x, k, nx, gx, sx1, out1, ctx)
    xp = torch.empty(nx * rows_x * wpr, dtype=torch.int32, device=dev)
    sx2 = torch.empty(n_sx, dtype=torch.float64, device=dev)
    ap.cu_quantize_pack(xv, rows_x, k, nx, gx, xp, sx2, ctx=ctx)
    out2 = torch.empty((rows_w, rows_x), dtype=torch.float32, device=dev)
    ap.cu_matmul_ap_dequant(wp, rows_w, nw, sw, 1, xp, rows_x, nx, sx2, gx, k, out2, ctx)
    torch.cuda.synchronize()
    assert torch.equal(sx1, sx2)
    assert torch.equal(out1, out2), (out1 - out2).abs().max().item()
    # and against the C restatement on a few rows: quantize, pack, matmul, dequant epilogue
    codes, scales = oracle.quantize(xv.cpu().numpy(), nx, gx)
    assert np.array_equal(scales, sx1.cpu().numpy())
    rows = np.unique(np.array([0, rows_w - 1, rows_w // 2]))
    wc_h = wc.cpu().numpy()[rows]
    y = oracle.matmul_ap(oracle.pack(wc_h, nw), len(rows), nw, oracle.pack(codes, nx), rows_x, nx, k)
    want = oracle.dequant_epilogue(y, sw.cpu().numpy()[rows], 1, scales, gx)
    assert np.array_equal(out1.cpu().numpy()[rows], want)


def test_fused_quantize_matmul_nonfinite(gpu):
    import torch
    ap, ctx = gpu
    dev = torch.device("cuda", 0)
    wp = torch.zeros(2 * 300 * 8, dtype=torch.int32, device=dev)
    sw = torch.ones(300, dtype=torch.float64, device=dev)
    xv = torch.zeros((100, 256), dtype=torch.float64, device=dev)
    xv[3, 7] = float("nan")
    with pytest.raises(ap.NonFinite):
        ap.cu_quantize_matmul_ap_dequant(wp, 300, 2, sw, 1, xv, 100, 256, 4, 1,
                                         torch.empty(100, dtype=torch.float64, device=dev),
                                         torch.empty((300, 100), dtype=torch.float32, device=dev), ctx)


# ---------------------------------------------------------------- plane products / recover
def test_plane_products_and_recover_match_oracle(gpu, oracle):
    """compute_plane_products / matmul_plane_pair / recover (kernel.cpp:125-181) on the GPU
    vs the C restatement, on the reference's seeded corpus shapes plus a tile-sized case."""
    ap, ctx = gpu
    rng = oracle.rng(41)
    cases = [(rng.range(1, 24), rng.range(1, 24), rng.range(1, 300), rng.range(1, 8),
              rng.range(1, 8)) for _ in range(60)] + [(300, 260, 1000, 3, 4), (5, 70, 33025, 1, 1)]
    for (m, n, k, nw, nx) in cases:
        wc, xc = rng.random_codes(m, k, nw), rng.random_codes(n, k, nx)
        wp, xp = oracle.pack(wc, nw), oracle.pack(xc, nx)
        want = oracle.plane_products(wp, m, nw, xp, n, nx, k).reshape(nw, nx, m, n)
        w = ap.PackedBitPlanes(m, k, ap.BitWidth(nw), wp)
        x = ap.PackedBitPlanes(n, k, ap.BitWidth(nx), xp)
        stack = ap.compute_plane_products(w, x, ctx)
        assert np.array_equal(stack.products(), want), (m, n, k, nw, nx)
        i, j = nw - 1, nx - 1
        assert np.array_equal(ap.matmul_plane_pair(w, i, x, j, ctx), want[i, j])
        if oracle.overflow_bound(nw, nx, k) <= 2**31 - 1:
            assert np.array_equal(ap.recover(stack, ctx), oracle.recover(want))


def test_plane_product_and_recover_errors(gpu, oracle):
    ap, ctx = gpu
    wc = np.array([[0b11, 0b10]], np.uint8)
    w = ap.PackedBitPlanes(1, 2, ap.BitWidth(2), oracle.pack(wc, 2))
    with pytest.raises(ap.IndexOutOfBounds):  # plane_row range (bitplane.cpp:40-45)
        ap.matmul_plane_pair(w, 2, w, 0, ctx)
    # worked example (test_kernel.cpp:125-136): planes (0,-2,2,0) recover to 0
    x = ap.PackedBitPlanes(1, 2, ap.BitWidth(2), oracle.pack(np.array([[0b01, 0b11]], np.uint8), 2))
    st = ap.compute_plane_products(w, x, ctx)
    assert st.products().reshape(-1).tolist() == [0, -2, 2, 0] and ap.recover(st, ctx).tolist() == [[0]]
    # recover narrows with a check -> Overflow (kernel.cpp:172-176)
    big = ap.PlaneProductStack(ap.BitWidth(8), ap.BitWidth(8), 40000,
                               np.full((8, 8, 1, 1), 40000, np.int32))
    with pytest.raises(ap.Overflow):
        ap.recover(big, ctx)
    # entries outside [-K, K] are an OutOfRange, as the PlaneProductStack ctor (kernel.cpp:91-101)
    bad = ap.PlaneProductStack(ap.BitWidth(1), ap.BitWidth(1), 3, np.full((1, 1, 2, 2), 4, np.int32))
    with pytest.raises(ap.OutOfRange):
        ap.recover(bad, ctx)
