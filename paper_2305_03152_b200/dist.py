"""Host-side multi-GPU plumbing (one process per GPU, torch.distributed for
the control plane only; the data plane is CUDA IPC + NVLink inside the gather
kernel).

* `owned_partitions`: partition k lives on GPU k mod N (partitions
  shard naturally; K > N loops partitions per GPU).
* `minibatch_schedule`: the (epoch, partition, batch) sequence a GPU runs --
  round-robin over its partitions, each cell in the reference's order
  (epoch_minibatches chunks, commsim.cpp:45-52), epochs advancing as cells run
  out.
* `exchange_plane_handles`: every GPU exports the CUDA IPC handles of the
  partitions it holds and attaches everyone else's.
* `max_over_ranks`: the bench's timing reduction.
"""
from __future__ import annotations

from typing import Callable, Sequence


def owned_partitions(K: int, world: int, rank: int) -> list:
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return [k for k in range(K) if k % world == rank]


def minibatch_schedule(permutation: Callable[[int, int], Sequence[int]], parts: Sequence[int], b: int,
                       count: int) -> list:
    """[(epoch, k, batch_index, seeds)] of length `count`; permutation(k, e)
    returns partition k's epoch-e train permutation (vipkit::epoch_minibatches)."""
    out, e = [], 0
    while len(out) < count:
        per = {k: permutation(k, e) for k in parts}
        nb = {k: (len(per[k]) + b - 1) // b for k in parts}
        for i in range(max(nb.values())):
            for k in parts:
                if i < nb[k]:
                    out.append((e, k, i, per[k][i * b:(i + 1) * b]))
        e += 1
    return out[:count]


def exchange_plane_handles(plane, owned: Sequence[int], group=None) -> dict:
    """Export owned partitions, all-gather the handles (any host backend, e.g.
    gloo) and attach every partition owned elsewhere. Returns {k: owner_rank}."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    mine = {k: plane.export(k) for k in owned}
    allh = [None] * world
    dist.all_gather_object(allh, mine, group=group)
    owner = {}
    for r, hs in enumerate(allh):
        for k, (handle, rows) in hs.items():
            if k in owner:
                raise RuntimeError(f"partition {k} exported by two ranks")
            owner[k] = r
            if r != rank:
                plane.attach(k, handle, rows)
    dist.barrier(group=group)
    return owner


def max_over_ranks(values: Sequence[float], group=None) -> list:
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return [float(x) for x in t]
