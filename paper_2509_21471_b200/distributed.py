"""Multi-GPU evaluation: one process per GPU, torch.distributed for the plumbing.

The DMK evaluation shards one system; see
include/sdmk.h sdmk_comm_init.  Every rank builds the same tree (bit-exact
ids without communication).  The upward pass is cut into subtrees of at
most N / (8 nranks) sources dealt to ranks in Morton runs; each rank
anterpolates and merges only its own subtrees, then one NCCL group on the
library's stream exchanges the outgoing expansions every rank reads (the
colleagues of its plane-wave targets: the source halo) plus the cut boxes,
and every rank merges the few boxes above the cut.  The downward pass, far
fields and near-field residual run for the rank's contiguous Morton run of
target leaves, and an NCCL all-reduce assembles u on every rank -- bitwise
equal to the single-GPU evaluation, because every box and every owned
target is formed exactly as on one GPU and the other summands are exact
zeros.

torch.distributed only carries the 128-byte NCCL id; the library's own
communicator does the data path.
"""
from __future__ import annotations

from . import Context, comm_unique_id


def init_comm(ctx: Context, group=None) -> None:
    """Give `ctx` an NCCL communicator over the ranks of `group` (the default
    process group if None); a no-op at world size 1."""
    import torch.distributed as dist

    if not dist.is_initialized():
        return
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if world == 1:
        return
    obj = [comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    ctx.comm_init(rank, world, obj[0])


def evaluate_sharded(ctx: Context, plan, dim: int, n_src: int, src_ptr: int, n_tgt: int, tgt_ptr: int,
                     str_ptr: int, mode: int, u, report=None):
    """Evaluate with device pointers on a context prepared by init_comm; u (a
    torch CUDA tensor of n_tgt_or_src * dim doubles) receives the full result
    on every rank."""
    ctx.evaluate_device(plan, dim, n_src, src_ptr, n_tgt, tgt_ptr, str_ptr, mode, u.data_ptr(), report)
    return u
