"""CPU, world_size 2 over gloo: the multi-GPU host logic (partition ownership,
minibatch schedule, IPC-handle exchange, max-over-ranks timing) with a fake
feature plane standing in for the device one."""
import os

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT


class FakePlane:
    def __init__(self, rank, K):
        self.rank, self.K, self.attached = rank, K, {}

    def export(self, k):
        return bytes([k, self.rank]) * 32, 1000 + k

    def attach(self, k, handle, rows):
        self.attached[k] = (handle, rows)


def _worker(rank, world, port, K, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_2305_03152_b200 import dist as vd
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = vd.owned_partitions(K, world, rank)
    plane = FakePlane(rank, K)
    owner = vd.exchange_plane_handles(plane, mine)
    t = vd.max_over_ranks([1.0 + rank, 5.0 - rank])
    perm = lambda k, e: np.arange(k * 100, k * 100 + 37) + e  # noqa: E731
    sched = vd.minibatch_schedule(perm, mine, 10, 12)
    q.put((rank, mine, owner, {k: v for k, v in plane.attached.items()}, t,
           [(e, k, i, list(s)) for e, k, i, s in sched]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_host_plumbing():
    world, K = 2, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 300
    procs = [ctx.Process(target=_worker, args=(r, world, port, K, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=120)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    owned = [res[r][1] for r in range(world)]
    assert sorted(sum(owned, [])) == list(range(K))            # disjoint and complete
    assert owned[0] == [0, 2, 4] and owned[1] == [1, 3]
    for r in range(world):
        owner, attached, t, sched = res[r][2], res[r][3], res[r][4], res[r][5]
        assert owner == {k: k % world for k in range(K)}
        assert sorted(attached) == [k for k in range(K) if k % world != r]
        for k, (h, rows) in attached.items():
            assert h == bytes([k, k % world]) * 32 and rows == 1000 + k
        assert t == [2.0, 5.0]                                 # max over ranks
        # round-robin over owned partitions; batches are consecutive chunks
        assert [s[1] for s in sched[:len(owned[r])]] == owned[r]
        for e, k, i, seeds in sched:
            assert seeds == list(range(k * 100 + e + i * 10, k * 100 + e + min(37, (i + 1) * 10)))
