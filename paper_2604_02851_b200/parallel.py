"""View sharding for the optimize step.

The reference sums per-view gradients and scales by 1/len(views)
(ref pkg/src/splatstream/optim.py:365-372).  Across GPUs that sum is the
path's only exchange step: views are dealt round-robin to ranks, every rank
accumulates its views into one flat gradient buffer, and a single
all-reduce (sum) of that buffer plus the loss precedes the replicated Adam
update.  NCCL over NVLink on the GPU box; the same functions run with gloo
on CPU tensors in tests/test_parallel_gloo.py.
"""

from __future__ import annotations


def shard_views(views, rank: int, world: int):
    """The views rank `rank` renders: rank, rank+world, ..."""
    return list(views)[rank::world]


def global_view_count(n_local: int, group, device) -> int:
    import torch
    import torch.distributed as dist
    t = torch.tensor([n_local], dtype=torch.int64, device=device)
    dist.all_reduce(t, group=group)
    return int(t.item())


def reduce_gradients(grad, loss, group) -> None:
    """Sum the flat gradient buffer and the loss over the group, in place."""
    import torch.distributed as dist
    dist.all_reduce(grad, group=group)
    dist.all_reduce(loss, group=group)
