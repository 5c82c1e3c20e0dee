"""Data parallelism over the stream index d.

Rank p of P owns the contiguous training range [floor(pD/P), floor((p+1)D/P)), accumulates
its partial mode-1 Gram G_p = sum_{d in shard} A_d A_d^T on its GPU (``sketch_gram``), and
one all-reduce (sum) of the m x m Gram over NCCL / NVLink gives G on every rank.  The
eigensolver then runs redundantly on every rank; it is deterministic, so every rank holds
the same S and no broadcast is needed.  The test stream is sharded by matrix with no
communication (each rank computes the errors of its own test matrices).
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist


def shard_range(D: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous d-range of `rank` among `world` ranks: [floor(rank*D/world), floor((rank+1)*D/world))."""
    if world < 1 or not (0 <= rank < world) or D < 0:
        raise ValueError(f"bad shard request D={D} rank={rank} world={world}")
    return (rank * D) // world, ((rank + 1) * D) // world


def reduce_gram(G64: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the ranks' partial Grams in place (the only collective of the training path)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(G64, op=dist.ReduceOp.SUM, group=group)
    return G64


def gather_errors(err_local: torch.Tensor, B_total: int, group=None) -> torch.Tensor:
    """All ranks' per-matrix test errors in stream order on every rank (the torch.distributed route of
    tsk_allgather_errors): rank p holds matrices shard_range(B_total, p, P); the shards are padded to
    ceil(B/P), all-gathered, and compacted.  The paper's test error is a mean over
    the whole test set, so it needs every rank's errors."""
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    if world == 1:
        return err_local.clone()
    rank = dist.get_rank(group)
    lo, hi = shard_range(B_total, rank, world)
    if err_local.numel() != hi - lo:
        raise ValueError(f"rank {rank} holds {err_local.numel()} errors, its shard has {hi - lo}")
    per = -(-B_total // world)
    pad = torch.zeros(per, dtype=err_local.dtype, device=err_local.device)
    pad[: hi - lo] = err_local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([parts[p][: shard_range(B_total, p, world)[1] - shard_range(B_total, p, world)[0]]
                      for p in range(world)])


def init_native_comm(ctx=None, group=None):
    """Give the library its own NCCL communicator over the ranks of `group` (tsk_comm_init): rank 0
    draws the unique id, torch.distributed broadcasts it.  Afterwards ``sketch_train`` all-reduces the
    Gram of the local shard itself (C ABI path); ``train`` below keeps torch's all-reduce."""
    from . import context, get_unique_id

    ctx = ctx or context()
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    obj = [get_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(obj, src=0, group=group)
    ctx.comm_init(world, rank, obj[0])
    return ctx


def train(A_local: torch.Tensor, k: int, group=None, opts=None, G64: Optional[torch.Tensor] = None,
          gram_fn=None, topk_fn=None):
    """Algorithm 2 lines 1-2 over all ranks of `group`: local Gram of this rank's shard,
    all-reduce, top-k eigenvectors.  Returns (S [k, m], lambda [k], info, status).
    gram_fn / topk_fn default to the library's sketch_gram / sketch_topk (the CPU multi-process tests
    substitute fp64 stand-ins to exercise this control flow without a GPU)."""
    from . import sketch_gram, sketch_topk

    sketch_gram = gram_fn or sketch_gram
    sketch_topk = topk_fn or sketch_topk

    if A_local.shape[0] == 0:  # an empty shard still joins the all-reduce (zero contribution)
        m = A_local.shape[1]
        G64 = torch.zeros((m, m), dtype=torch.float64, device=A_local.device) if G64 is None else G64.zero_()
        ginfo = None
    else:
        G64, ginfo = sketch_gram(A_local, G64=G64, opts=opts)
    reduce_gram(G64, group)
    S, lam, info, st = sketch_topk(G64, k, opts=opts)
    if ginfo is not None:
        info.gram_splits, info.gram_tiles = ginfo.gram_splits, ginfo.gram_tiles
    return S, lam, info, st
