"""Multi-GPU evaluation: one process per GPU, torch.distributed for the plumbing.

The DMK evaluation shards by target leaves: every rank
builds the same tree (bit-exact ids without communication) and the same
upward pass, then forms the downward pass, far fields and near-field
residual only for its own contiguous Morton run of target leaves
(``Context.set_shard``).  Each rank's output holds zeros for other ranks'
targets, so one ``all_reduce(SUM)`` of u assembles the result -- bitwise
equal to the single-GPU evaluation, because every owned target's sums are
formed exactly as on one GPU and the other summands are exact zeros.
"""
from __future__ import annotations

from . import Context, DmkPlan


def evaluate_sharded(ctx: Context, plan: DmkPlan, dim: int, n_src: int, src_ptr: int, n_tgt: int, tgt_ptr: int,
                     str_ptr: int, mode: int, u, group=None, report=None):
    """Evaluate on this rank's shard and all-reduce u (a torch CUDA tensor of
    n_tgt_or_src * dim doubles whose pointer is passed to the library)."""
    import torch.distributed as dist

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    ctx.set_shard(rank, world)
    ctx.evaluate_device(plan, dim, n_src, src_ptr, n_tgt, tgt_ptr, str_ptr, mode, u.data_ptr(), report)
    if world > 1:
        dist.all_reduce(u, op=dist.ReduceOp.SUM, group=group)
    return u
