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


class MinibatchStream:
    """`minibatch_schedule`'s sequence produced incrementally, for loops that
    time the schedule with the rest of the step: every partition's train
    members are listed once (PartitionMap::train_members), and each epoch's
    permutations (epoch_minibatches' shuffle, sampling.cpp:54-63) are computed
    on a worker thread one epoch ahead of the consumer (the ctypes calls
    release the GIL), so the host keeps queueing GPU work meanwhile."""

    def __init__(self, vk, roles, part_of, parts: Sequence[int], b: int, seed: int, epoch: int = 0):
        import concurrent.futures as cf
        self._vk, self._parts, self._b, self._seed = vk, list(parts), b, seed
        self._train = {k: vk.train_members(roles, part_of, k) for k in self._parts}
        self._pool = cf.ThreadPoolExecutor(max_workers=1)
        self._epoch = epoch
        self._next = self._pool.submit(self._cells, epoch)
        self._buf, self._pos = [], 0

    def _cells(self, e):
        per = {k: self._vk.epoch_shuffle(self._train[k], k, e, self._seed) for k in self._parts}
        b = self._b
        nb = {k: (len(per[k]) + b - 1) // b for k in self._parts}
        return [(e, k, i, per[k][i * b:(i + 1) * b]) for i in range(max(nb.values()))
                for k in self._parts if i < nb[k]]

    def ready(self):
        """Block until the first epoch's schedule exists (steady state: the
        worker stays one epoch ahead of the consumer)."""
        self._next.result()
        return self

    def take(self, count: int) -> list:
        out = []
        while len(out) < count:
            if self._pos == len(self._buf):
                self._buf, self._pos = self._next.result(), 0
                self._epoch += 1
                self._next = self._pool.submit(self._cells, self._epoch)
            t = min(count - len(out), len(self._buf) - self._pos)
            out.extend(self._buf[self._pos:self._pos + t])
            self._pos += t
        return out

    def close(self):
        self._pool.shutdown(wait=True)


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
