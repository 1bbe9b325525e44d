"""Data-parallel plumbing for the cnn_train multi-GPU mode.

The device side -- per-layer NCCL allreduce of the parameter derivatives,
overlapped with backward, then SGD -- lives in libck.so (`ck_trainer`,
engine.cu).  This module is the host logic around it: the bucket plan the
engine follows, batch sharding, and the NCCL unique-id exchange through
torch.distributed (used only as a rendezvous).
"""
from __future__ import annotations

from typing import Callable


def bucket_plan(net):
    """[(layer, [params])] in the order backward finishes them.

    Mirrors ck_trainer_create (engine.cu): a parameter is final after its
    last consumer in backward order, i.e. its first consumer in firing order;
    layers fire in declaration order for the chain networks built here.
    """
    params = {name for name, _, _ in net.params}
    first = {}
    for li, (kind, name, ins, outs, p) in enumerate(net.layers):
        for i in ins:
            if i in params and i not in first:
                first[i] = li
    plan = []
    for li in reversed(range(len(net.layers))):
        ps = [i for i in net.layers[li][2] if first.get(i) == li]
        if ps:
            plan.append((net.layers[li][1], ps))
    return plan


def shard(global_batch: int, rank: int, world: int):
    """Contiguous batch slice [lo, hi) of this rank (sub-batches of equal size)."""
    if global_batch % world:
        raise ValueError(f"global batch {global_batch} not divisible by {world} ranks")
    per = global_batch // world
    return rank * per, (rank + 1) * per


def share_unique_id(make_id: Callable[[], bytes], rank: int) -> bytes:
    """Rank 0 creates the NCCL unique id; everyone receives it."""
    import torch.distributed as dist
    box = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    return box[0]
