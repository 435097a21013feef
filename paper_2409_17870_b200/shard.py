"""N-sharded multi-GPU matmul_ap (BASELINE configs[4]: Llama-2-70B FFN across 1/2/4/8 GPUs).

The weights W [N_out x K] are split into P contiguous row blocks, one per rank; the
features X [M_tok x K] are replicated. In the reference orientation
matmul_ap(W, X) -> Y [N_out x M_tok] each rank's result is a contiguous row block of Y, so
the GEMMs are independent (no exchange in the compute phase) and the full output -- only
when the consumer needs it -- is one all-gather of row blocks with no re-layout.

One process per GPU, torch.distributed for the plumbing (NCCL on GPUs; the same code
runs under gloo on CPU tensors for the multi-process tests). Shards are padded to the
largest shard so the all-gather is a single ``all_gather_into_tensor``.
"""
from __future__ import annotations

from typing import Callable


def shard_bounds(n_out: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced row block [r0, r1) of rank `rank` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    base, extra = divmod(n_out, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def max_shard(n_out: int, world: int) -> int:
    return -(-n_out // world)


def slice_plane_rows(planes, rows: int, cols: int, n: int, r0: int, r1: int):
    """Rows [r0, r1) of every plane of a packed buffer (bitplane.hpp:12-18 layout), as a
    new contiguous packed buffer of (r1-r0) rows. Works on torch tensors or numpy arrays."""
    wpr = (cols + 31) // 32
    v = planes.reshape(n, rows, wpr)[:, r0:r1, :]
    try:
        return v.contiguous().reshape(-1)          # torch
    except AttributeError:
        import numpy as np
        return np.ascontiguousarray(v).reshape(-1)  # numpy


def gather_rows(local_y, n_out: int, m_tok: int, group=None):
    """All-gather the per-rank row blocks of Y into the full [n_out, m_tok] result on every
    rank (torch.distributed; NCCL all_gather_into_tensor over NVLink on GPUs)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ms = max_shard(n_out, world)
    r0, r1 = shard_bounds(n_out, world, rank)
    if local_y.shape != (r1 - r0, m_tok):
        raise ValueError(f"local block has shape {tuple(local_y.shape)}, expected {(r1 - r0, m_tok)}")
    send = local_y
    if r1 - r0 != ms:  # uneven split: pad to the common block size
        send = torch.zeros((ms, m_tok), dtype=local_y.dtype, device=local_y.device)
        send[: r1 - r0] = local_y
    out = torch.empty((world * ms, m_tok), dtype=local_y.dtype, device=local_y.device)
    dist.all_gather_into_tensor(out, send.contiguous(), group=group)
    if ms * world == n_out:
        return out
    rows = [out[p * ms: p * ms + (shard_bounds(n_out, world, p)[1] - shard_bounds(n_out, world, p)[0])]
            for p in range(world)]
    return torch.cat(rows, dim=0)


def sharded_matmul_ap(w_planes_full, n_out: int, n_w: int, x_planes, m_tok: int, n_x: int,
                      k: int, gather: bool = True, group=None,
                      local_gemm: Callable | None = None):
    """This rank's row block of matmul_ap(W, X) (and the all-gathered full Y if `gather`).

    `local_gemm(w_shard_planes, rows, x_planes) -> y_block` defaults to the B200 kernel
    (apmm_cu_matmul_ap on this rank's GPU). The multi-process CPU tests pass a CPU GEMM so
    the sharding and gather logic can be exercised under gloo without a GPU.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    r0, r1 = shard_bounds(n_out, world, rank)
    w_shard = slice_plane_rows(w_planes_full, n_out, k, n_w, r0, r1)
    if local_gemm is None:
        from .apmm import cu_matmul_ap
        y = torch.empty((r1 - r0, m_tok), dtype=torch.int32, device=x_planes.device)
        cu_matmul_ap(w_shard, r1 - r0, n_w, x_planes, m_tok, n_x, k, y)
    else:
        y = local_gemm(w_shard, r1 - r0, x_planes)
    if not gather:
        return y
    return gather_rows(y, n_out, m_tok, group)
