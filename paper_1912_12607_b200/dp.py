"""Data-parallel host logic, kept free of CUDA so it can be
tested with the gloo backend on CPU.

The reference trains on one process with one LCG gradient stream
(train.cpp:13) and quantises the *whole* batch gradient of a layer with one
clip (layers.cpp:19-59).  Sharding the batch over R ranks keeps that exact:

* rank r holds the contiguous samples [r*B/R, (r+1)*B/R); its g_z is the
  contiguous slice [r*n, (r+1)*n) of the NCHW-flattened global tensor
  (N is the outermost dimension), so its stochastic draws start at global
  draw offset r*n and the stream advances by R*n for the layer;
* max|g| is combined with MAX, every d_c / eps / g_hat sum (and each DSGC
  candidate's sums) with SUM -- the device kernels expose them as a small
  buffer of doubles between phases (i8t_ctx_set_allreduce);
* the weight gradient is summed as int64 accumulators (exact and
  order-independent: every rank uses the same global scales), then rescaled.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

LCG_MOD = 1 << 32


def shard_draw_offset(rank: int, numel_local: int) -> int:
    """First global LCG draw index consumed by `rank` (mod 2^32)."""
    return (rank * numel_local) % LCG_MOD


def layer_draws(world: int, numel_local: int) -> int:
    """Draws the whole layer consumes (all ranks), i.e. the stream advance."""
    return (world * numel_local) % LCG_MOD


def combine_totals(totals: torch.Tensor, group=None) -> torch.Tensor:
    """Global DSGC totals: [0] max|g| (MAX), [1:] sums (SUM); in place."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return totals
    head = totals[:1].clone()
    dist.all_reduce(head, op=dist.ReduceOp.MAX, group=group)
    if totals.numel() > 1:
        tail = totals[1:].clone()
        dist.all_reduce(tail, op=dist.ReduceOp.SUM, group=group)
        totals[1:] = tail
    totals[:1] = head
    return totals


def combine_totals_gather(totals: torch.Tensor, group=None) -> torch.Tensor:
    """combine_totals with one all_gather instead of two all_reduces (the
    buffers are a few doubles: the collective is latency-bound).  The fold is
    in rank order, so every rank computes identical totals."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return totals
    world = dist.get_world_size(group)
    rows = torch.empty((world, totals.numel()), dtype=totals.dtype, device=totals.device)
    try:
        dist.all_gather_into_tensor(rows, totals.contiguous(), group=group)
    except (RuntimeError, NotImplementedError):  # backends without the fused all-gather
        dist.all_gather(list(rows.unbind(0)), totals.contiguous(), group=group)
    totals[:1] = rows[:, :1].max(dim=0).values
    if totals.numel() > 1:
        acc = rows[0, 1:].clone()
        for r in range(1, world):
            acc += rows[r, 1:]
        totals[1:] = acc
    return totals


def allreduce_int64_(acc: torch.Tensor, group=None, async_op: bool = False):
    """Exact sum of int64 weight-gradient accumulators across ranks (in place).
    async_op: return the collective's work handle (None when there is nothing
    to reduce) instead of waiting."""
    assert acc.dtype == torch.int64
    work = None
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        work = dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
    return work if async_op else acc


def shard_batch(x: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    """Contiguous batch shard of rank `rank` (equal shards required)."""
    if x.shape[0] % world:
        raise ValueError("data parallel: the global batch must divide evenly across ranks")
    b = x.shape[0] // world
    return x[rank * b:(rank + 1) * b]
