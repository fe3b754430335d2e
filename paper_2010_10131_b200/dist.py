"""Host-side helpers for the multi-GPU st-HOSVD (one process per GPU).

The engine (csrc/dist.cu) shards the input along the LAST mode: rank r holds
the contiguous slab [.., lo:hi] of the column-major tensor and the Gram
partial sums of every earlier mode are combined with one NCCL allreduce.  This
module only plans the shards and bootstraps the NCCL communicator over an
existing torch.distributed process group (any backend: the 128-byte unique id
is broadcast as a uint8 tensor).
"""
from __future__ import annotations


def shard_range(n_last: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of the last mode owned by `rank` (balanced, contiguous, ordered)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return n_last * rank // world, n_last * (rank + 1) // world


def init_comm_from_torch(ctx, group=None) -> None:
    """ncclCommInitRank for `ctx` using the ranks of a torch.distributed group."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = ctx.nccl_unique_id() if rank == 0 else bytes(128)
    t = torch.tensor(list(uid), dtype=torch.uint8)
    dist.broadcast(t, 0, group=group)
    ctx.comm_init(bytes(t.tolist()), rank, world)


def init_host_comm_from_torch(ctx, group=None) -> None:
    """atk_comm_init_host over a torch.distributed group (e.g. gloo): the
    collectives are staged through host memory, so ranks may share a GPU."""
    import torch
    import torch.distributed as dist

    def allreduce_f64(a):
        t = torch.from_numpy(a)  # shares memory with the engine's staging buffer
        dist.all_reduce(t, group=group)

    def broadcast(a, root):
        t = torch.from_numpy(a)
        dist.broadcast(t, root, group=group)

    ctx.comm_init_host(allreduce_f64, broadcast, dist.get_rank(group), dist.get_world_size(group))
