"""Multi-process (gloo, world_size 2 and 3) checks of the N-sharded path
(paper_2409_17870_b200/shard.py): row-block shards of W, replicated X, independent
per-rank GEMMs, one all-gather of row blocks. The gathered result must equal the unsharded
reference result bit for bit, including uneven splits.

* CPU tests: the per-rank GEMM is the oracle (so the sharding and gather logic run without
  a GPU).
* GPU test (`-m gpu`): the per-rank GEMM is the real kernel (apmm_cu_matmul_ap), both ranks
  sharing cuda:0, the row blocks gathered over gloo."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cases, q, use_gpu=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import Oracle
        from paper_2409_17870_b200.shard import sharded_matmul_ap, shard_bounds
        o = Oracle()
        ok = True
        for (n_out, m_tok, k, nw, nx, seed) in cases:
            rng = o.rng(seed)
            wc, xc = rng.random_codes(n_out, k, nw), rng.random_codes(m_tok, k, nx)
            wp = torch.from_numpy(o.pack(wc, nw).view(np.int32))
            xp = torch.from_numpy(o.pack(xc, nx).view(np.int32))

            def local_gemm(w_shard, rows, x_planes):
                if use_gpu:  # the B200 kernel on this rank's shard, result back on the host
                    from paper_2409_17870_b200 import cu_matmul_ap
                    dev = torch.device("cuda", 0)
                    y = torch.empty((rows, m_tok), dtype=torch.int32, device=dev)
                    cu_matmul_ap(w_shard.to(dev), rows, nw, x_planes.to(dev), m_tok, nx, k, y)
                    torch.cuda.synchronize()
                    return y.cpu()
                y = o.matmul_ap(w_shard.numpy().view(np.uint32), rows, nw,
                                x_planes.numpy().view(np.uint32), m_tok, nx, k)
                return torch.from_numpy(y)

            block = sharded_matmul_ap(wp, n_out, nw, xp, m_tok, nx, k, gather=False,
                                      local_gemm=local_gemm)
            full = sharded_matmul_ap(wp, n_out, nw, xp, m_tok, nx, k, gather=True,
                                     local_gemm=local_gemm)
            want = (o.matmul_ap_mt(wp.numpy().view(np.uint32), n_out, nw,
                                   xp.numpy().view(np.uint32), m_tok, nx, k, 4)
                    if use_gpu else o.decoded_matmul(wc, nw, xc, nx))
            r0, r1 = shard_bounds(n_out, world, rank)
            ok &= np.array_equal(block.numpy(), want[r0:r1])
            ok &= np.array_equal(full.numpy(), want)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def _run(world, cases, use_gpu=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q, use_gpu))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    results = dict(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert all(results[r] for r in range(world)), results


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gather_matches_unsharded(world):
    _run(world, [(64, 9, 100, 2, 4, 1), (37, 5, 33, 3, 8, 2), (5, 3, 70, 1, 1, 3)])


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gather_with_gpu_kernel(world):
    """The real kernel per rank: skinny (M=9), split-K mid (M=128), 1-SM and pair tile
    routes (M=600 / 2048 at 2300 rows), uneven splits, ragged K."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _run(world, [(64, 9, 100, 2, 4, 1), (4099, 128, 4096, 2, 4, 2), (2300, 600, 1000, 3, 8, 3),
                 (4608, 2048, 2048, 2, 4, 4), (37, 5, 33, 1, 1, 5)], use_gpu=True)


def test_shard_bounds_cover_rows_exactly():
    from paper_2409_17870_b200.shard import max_shard, shard_bounds
    for n_out in (1, 7, 28672, 28673):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_bounds(n_out, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n_out
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(r1 - r0 for r0, r1 in spans) == max_shard(n_out, world)


def _requant_worker(rank, world, port, q):
    """N-sharded layer -> next layer's packed activation: per-rank GEMM + dequant + absmax,
    MAX all-reduce, per-rank quantize + pack of its word block, all-gather of packed planes.
    Local ops are the oracle (+ a numpy round_to_grid, bipolar.cpp:63-68); the result must be
    bit-identical to quantize(dequant(Y_full)^T) + pack of the unsharded layer."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import Oracle
        from paper_2409_17870_b200.shard import sharded_matmul_requant
        o = Oracle()
        ok = True
        for (n_out, m_tok, k, nw, nx, n_next, gran, seed) in [(200, 9, 100, 2, 4, 4, 1, 1),
                                                              (96, 5, 70, 3, 8, 2, 0, 2),
                                                              (257, 33, 64, 1, 2, 8, 1, 3)]:
            rng = o.rng(seed)
            wc, xc = rng.random_codes(n_out, k, nw), rng.random_codes(m_tok, k, nx)
            wp = torch.from_numpy(o.pack(wc, nw).view(np.int32))
            xp = torch.from_numpy(o.pack(xc, nx).view(np.int32))
            gen = np.random.default_rng(seed)
            ws = gen.uniform(0.01, 1.0, size=n_out)
            xs = gen.uniform(0.01, 1.0, size=m_tok)
            maxv = (1 << n_next) - 1

            def gemm_absmax(w_shard, rows, ws_shard):
                y = o.matmul_ap(w_shard.numpy().view(np.uint32), rows, nw, xp.numpy().view(np.uint32),
                                m_tok, nx, k)
                yf = o.dequant_epilogue(y, np.asarray(ws_shard), 1, xs, 1).astype(np.float32)
                a = np.abs(yf).max(axis=0) if gran == 1 else np.array([np.abs(yf).max()])
                return yf, torch.from_numpy(a.astype(np.float64))

            def requant_pack(yf, rows, absmax):
                a = absmax.numpy()
                s = np.where(a == 0.0, 1.0, a / maxv)
                xt = yf.T.astype(np.float64)                  # X' rows = tokens
                t = xt / (s[:, None] if gran == 1 else s[0])
                qv = np.clip(2.0 * np.floor(t / 2.0) + 1.0, -maxv, maxv).astype(np.int64)
                codes = ((qv + maxv) // 2).astype(np.uint8)
                return torch.from_numpy(o.pack(codes, n_next).view(np.int32)), torch.from_numpy(s)

            planes, scales = sharded_matmul_requant(
                wp, n_out, nw, torch.from_numpy(ws), 1, xp, m_tok, nx, torch.from_numpy(xs), 1, k,
                n_next, gran, local_ops=(gemm_absmax, requant_pack))
            y = o.matmul_ap(wp.numpy().view(np.uint32), n_out, nw, xp.numpy().view(np.uint32),
                            m_tok, nx, k)
            yf = o.dequant_epilogue(y, ws, 1, xs, 1).astype(np.float32)
            codes, want_s = o.quantize(yf.T.astype(np.float64), n_next, gran)
            ok &= np.array_equal(planes.numpy().view(np.uint32), o.pack(codes, n_next))
            ok &= np.array_equal(scales.numpy(), want_s)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_requant_gather_packed(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_requant_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    results = dict(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert all(results[r] for r in range(world)), results


def test_word_shard_bounds():
    from paper_2409_17870_b200.shard import word_shard_bounds
    for n_out in (32, 257, 28672, 1000):
        for world in (1, 2, 3, 8):
            spans = [word_shard_bounds(n_out, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n_out
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert all(r0 % 32 == 0 for r0, _ in spans)
