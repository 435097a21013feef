"""Multi-process (gloo, world_size 2 and 3, CPU) checks of the N-sharded path
(paper_2409_17870_b200/shard.py): row-block shards of W, replicated X, independent
per-rank GEMMs, one all-gather of row blocks. The per-rank GEMM is the oracle here (the
GPU runs it through apmm_cu_matmul_ap); the gathered result must equal the unsharded
reference result bit for bit, including uneven splits."""
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


def _worker(rank, world, port, cases, q):
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
                y = o.matmul_ap(w_shard.numpy().view(np.uint32), rows, nw,
                                x_planes.numpy().view(np.uint32), m_tok, nx, k)
                return torch.from_numpy(y)

            block = sharded_matmul_ap(wp, n_out, nw, xp, m_tok, nx, k, gather=False,
                                      local_gemm=local_gemm)
            full = sharded_matmul_ap(wp, n_out, nw, xp, m_tok, nx, k, gather=True,
                                     local_gemm=local_gemm)
            want = o.decoded_matmul(wc, nw, xc, nx)
            r0, r1 = shard_bounds(n_out, world, rank)
            ok &= np.array_equal(block.numpy(), want[r0:r1])
            ok &= np.array_equal(full.numpy(), want)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gather_matches_unsharded(world):
    cases = [(64, 9, 100, 2, 4, 1), (37, 5, 33, 3, 8, 2), (5, 3, 70, 1, 1, 3)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    results = dict(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert all(results[r] for r in range(world)), results


def test_shard_bounds_cover_rows_exactly():
    from paper_2409_17870_b200.shard import max_shard, shard_bounds
    for n_out in (1, 7, 28672, 28673):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_bounds(n_out, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n_out
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(r1 - r0 for r0, r1 in spans) == max_shard(n_out, world)
