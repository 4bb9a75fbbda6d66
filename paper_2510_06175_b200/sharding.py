"""Multi-GPU host logic (one process per GPU, torch.distributed over NCCL/NVLink).

Two partitions of the decode-attention work:
  * batch x KV-head sharding (large batch, BASELINE configs[2]): units are independent, each rank
    owns a contiguous slice of sequences -> no collective on the data path ("scaling": weak).
  * sequence sharding (single 196k-token sequence, configs[3]): rank r attends tokens
    [r*N/P, (r+1)*N/P) through vecinfer_attn_decode's tok_begin/tok_end hook, producing a
    normalised partial (o_r, L_r) of 32 x (128 + 1) fp32 per sequence; ONE all-gather exchanges
    the P partials and every rank merges them with vecinfer_merge_lse in rank order, so all
    ranks hold bitwise-identical outputs.
The functions here only compute ranges and move partials; the arithmetic is in the kernels.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_tokens: int, rank: int, world: int, align: int = 32) -> tuple[int, int]:
    """Contiguous token shard of rank `rank`: boundaries rounded to `align` tokens, union = [0, n)."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    per = -(-n_tokens // world)
    per = -(-per // align) * align
    b = min(rank * per, n_tokens)
    e = min(b + per, n_tokens)
    return b, e


def batch_shard(batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous slice of sequences owned by `rank` (batch x KV-head sharding)."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    per = -(-batch // world)
    b = min(rank * per, batch)
    return b, min(b + per, batch)


def gather_partials(o_local: torch.Tensor, lse_local: torch.Tensor, group=None):
    """All-gather the per-rank partials into [P, ...] tensors in rank order (one collective each
    for o and lse; 16.1 KiB + 128 B per rank for B = 1, H_q = 32)."""
    world = dist.get_world_size(group)
    o_all = torch.empty((world,) + tuple(o_local.shape), dtype=o_local.dtype, device=o_local.device)
    l_all = torch.empty((world,) + tuple(lse_local.shape), dtype=lse_local.dtype, device=lse_local.device)
    if o_local.is_cuda:
        dist.all_gather_into_tensor(o_all, o_local.contiguous(), group=group)
        dist.all_gather_into_tensor(l_all, lse_local.contiguous(), group=group)
    else:   # gloo path (host-side tests)
        dist.all_gather(list(o_all.unbind(0)), o_local.contiguous(), group=group)
        dist.all_gather(list(l_all.unbind(0)), lse_local.contiguous(), group=group)
    return o_all, l_all


def gather_partials_packed(o_local: torch.Tensor, lse_local: torch.Tensor, group=None):
    """Same exchange with ONE collective: lse is packed behind o in a single fp32 buffer."""
    world = dist.get_world_size(group)
    flat = torch.cat([o_local.reshape(-1).float(), lse_local.reshape(-1).float()])
    out = torch.empty(world * flat.numel(), dtype=flat.dtype, device=flat.device)
    if flat.is_cuda:
        dist.all_gather_into_tensor(out, flat, group=group)
    else:
        dist.all_gather(list(out.view(world, -1).unbind(0)), flat, group=group)
    out = out.view(world, -1)
    no = o_local.numel()
    return (out[:, :no].reshape((world,) + tuple(o_local.shape)),
            out[:, no:].reshape((world,) + tuple(lse_local.shape)).contiguous())
