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


# ---- next-layer activations: requantize, then gather packed planes
def word_shard_bounds(n_out: int, world: int, rank: int) -> tuple[int, int]:
    """Row block [r0, r1) of rank `rank` with both ends on 32-row (one plane word)
    boundaries, so each rank's block of the next layer's activation X' = Y^T is a block of
    whole plane words in every X' row (the last rank takes the ragged end)."""
    words = -(-n_out // 32)
    w0, w1 = shard_bounds(words, world, rank)
    return min(32 * w0, n_out), min(32 * w1, n_out)


def gather_packed_planes(local_planes, n_next: int, m_tok: int, n_out: int, group=None):
    """All-gather every rank's X' plane block ([n_next][m_tok][words_p] u32, rows of its
    word_shard_bounds block) into the full next-layer activation planes
    [n_next][m_tok][ceil(n_out/32)] (the PackedBitPlanes layout) on every rank: one
    all_gather_into_tensor of padded blocks, then one word-block re-layout."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    spans = [word_shard_bounds(n_out, world, p) for p in range(world)]
    wps = [-(-(r1 - r0) // 32) for r0, r1 in spans]
    wmax = max(wps)
    mine = wps[rank]
    if local_planes.numel() != n_next * m_tok * mine:
        raise ValueError("local plane block has the wrong size")
    send = local_planes.reshape(n_next, m_tok, mine)
    if mine != wmax:
        pad = torch.zeros((n_next, m_tok, wmax), dtype=local_planes.dtype, device=local_planes.device)
        pad[:, :, :mine] = send
        send = pad
    out = torch.empty((world * n_next, m_tok, wmax), dtype=local_planes.dtype,
                      device=local_planes.device)
    dist.all_gather_into_tensor(out, send.contiguous(), group=group)
    out = out.view(world, n_next, m_tok, wmax)
    if all(w == wmax for w in wps):
        return out.permute(1, 2, 0, 3).reshape(n_next, m_tok, world * wmax).reshape(-1)
    blocks = [out[p, :, :, :wps[p]] for p in range(world)]
    return torch.cat(blocks, dim=2).reshape(-1)


def sharded_matmul_requant(w_planes_full, n_out: int, n_w: int, w_scales_full, w_gran: int,
                           x_planes, m_tok: int, n_x: int, x_scales, x_gran: int, k: int,
                           n_next: int, next_gran: int, group=None, local_ops=None):
    """One N-sharded layer whose consumer needs the full output as the NEXT layer's packed
    activation: per rank matmul_ap -> dequant (+ column absmax in the GEMM epilogue), a MAX
    all-reduce of the per-token (or global) absmax, the rank's quantize + pack of its word
    block, then the all-gather of packed planes -- n_next/32 of the int32 gather's bytes.
    Returns (planes [n_next * m_tok * ceil(n_out/32)] int32, scales f64) on every rank,
    bit-identical to quantize_pack(dequant(Y_full)^T).

    `local_ops` = (gemm_absmax, requant_pack) replaces the B200 calls (CPU tests):
    gemm_absmax(w_shard, rows, w_scales_shard) -> (yf [rows, m_tok] f32, absmax f64);
    requant_pack(yf, rows, absmax) -> (planes, scales)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    r0, r1 = word_shard_bounds(n_out, world, rank)
    rows = r1 - r0
    w_shard = slice_plane_rows(w_planes_full, n_out, k, n_w, r0, r1)
    ws = w_scales_full[r0:r1] if w_gran == 1 else w_scales_full
    n_scales = m_tok if next_gran == 1 else 1
    if local_ops is None:
        from .apmm import cu_matmul_ap_requant, cu_requant_pack
        dev = x_planes.device
        yf = torch.empty((rows, m_tok), dtype=torch.float32, device=dev)
        absmax = torch.empty(n_scales, dtype=torch.float64, device=dev)
        cu_matmul_ap_requant(w_shard, rows, n_w, ws.contiguous(), w_gran, x_planes, m_tok, n_x,
                             x_scales, x_gran, k, n_next, next_gran, yf, absmax=absmax)
        dist.all_reduce(absmax, op=dist.ReduceOp.MAX, group=group)
        planes = torch.empty(n_next * m_tok * (-(-rows // 32)), dtype=torch.int32, device=dev)
        scales = torch.empty(n_scales, dtype=torch.float64, device=dev)
        cu_requant_pack(yf, rows, m_tok, absmax, n_next, next_gran, planes, scales)
    else:
        gemm_absmax, requant_pack = local_ops
        yf, absmax = gemm_absmax(w_shard, rows, ws)
        dist.all_reduce(absmax, op=dist.ReduceOp.MAX, group=group)
        planes, scales = requant_pack(yf, rows, absmax)
    return gather_packed_planes(planes, n_next, m_tok, n_out, group), scales
