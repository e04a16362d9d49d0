"""Multi-GPU parity worker (run under torchrun, one process per GPU): each rank
owns partitions k = rank (mod N), attaches the others over CUDA IPC, samples
its minibatches and gathers; rows and tallies are checked bit-exact against
the oracle. Used by tests/test_gpu_multigpu.py and the 2-GPU gpurun checks.
Exit code 0 = parity on every rank."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2305_03152_b200 import vipkit as vk

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    P = O.port()
    csr = P.generate("pa", 20000, 6, 11)
    n, K, dim = csr.n, 4, 32
    roles = P.make_roles(n, 0.1, 0, 0, 3)
    labels = (np.arange(n) * 2654435761 % K).astype(np.uint32)
    g = vk.Graph.from_csr(csr.off, csr.tgt, undirected=True, device=local)
    p0 = np.stack([vk.initial_probs(roles, labels, k, 128) for k in range(K)])
    totals = np.stack([s.total for s in vk.propagate(g, [10, 5], p0, with_hops=False)])
    orders = [vk.rank_by_scores(labels, k, totals[k], device=local)[0] for k in range(K)]
    plan = vk.build_cache(orders, 0.2, n)
    oon, ranges = vk.build_reorder(labels, K, totals, device=local)
    plane = vk.FeaturePlane(n, K, dim, labels, oon, ranges, device=local)
    mine = [k for k in range(K) if k % world == rank]
    for k in mine:
        plane.load_partition(k, plan.cached[k], feature_seed=5)
    handles = {k: plane.export(k) for k in mine}
    allh = [None] * world
    dist.all_gather_object(allh, handles)
    for r, hs in enumerate(allh):
        if r != rank:
            for k, (h, rows) in hs.items():
                plane.attach(k, h, rows)
    dist.barrier()
    batches, refs = [], []
    for k in mine:
        perm = vk.epoch_permutation(roles, labels, k, 128, 0, 42)
        for i in range(3):
            batches.append(perm[i * 128:(i + 1) * 128])
            refs.append((0, k, i))
    s = vk.Sampler(g, [10, 5], 128, len(batches), 42)
    s.run(batches, refs)
    view = s.view()
    out, cnt = C.c_void_p(), C.c_void_p()
    vk.check(vk.lib().vk_device_alloc(local, len(batches) * view.all_stride * plane.row_bytes, C.byref(out)))
    vk.check(vk.lib().vk_device_alloc(local, len(batches) * 32, C.byref(cnt)))
    ok = check_wave(vk, P, csr, plane, plan, labels, batches, refs, s, out, cnt, dim, local, rank, world,
                    prefetch=False)
    # the same wave again, exchange prefetched on the aux stream, into fresh buffers
    out2, cnt2 = C.c_void_p(), C.c_void_p()
    vk.check(vk.lib().vk_device_alloc(local, len(batches) * view.all_stride * plane.row_bytes, C.byref(out2)))
    vk.check(vk.lib().vk_device_alloc(local, len(batches) * 32, C.byref(cnt2)))
    s.run(batches, refs)
    ok &= check_wave(vk, P, csr, plane, plan, labels, batches, refs, s, out2, cnt2, dim, local, rank, world,
                     prefetch=True)
    # sparse (bucket) frontiers -- the papers-scale representation, whose
    # gather tiles come from bucket bases -- with the exchange ordered after
    # a caller stream's queued work (vk_plane_prefetch_after)
    sp = vk.Sampler(g, [10, 5], 128, len(batches), 42, frontier="sparse")
    sp.run(batches, refs)
    out3, cnt3 = C.c_void_p(), C.c_void_p()
    vk.check(vk.lib().vk_device_alloc(local, len(batches) * sp.view().all_stride * plane.row_bytes, C.byref(out3)))
    vk.check(vk.lib().vk_device_alloc(local, len(batches) * 32, C.byref(cnt3)))
    side = torch.cuda.Stream()
    ok &= check_wave(vk, P, csr, plane, plan, labels, batches, refs, sp, out3, cnt3, dim, local, rank, world,
                     prefetch="after", stream=side.cuda_stream)
    for b_ in (out, cnt, out2, cnt2, out3, cnt3):
        vk.lib().vk_device_free(b_)
    flag = torch.tensor([1 if ok else 0])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    dist.barrier()
    print(f"rank {rank}: {'ok' if ok else 'FAIL'} ({len(refs)} minibatches x 3)", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if int(flag) == 1 else 1)


def check_wave(vk, P, csr, plane, plan, labels, batches, refs, s, out, cnt, dim, local, rank, world, prefetch,
               stream=None):
    view = s.view()
    if prefetch == "after":
        plane.prefetch_after(s, stream)
    elif prefetch:
        plane.prefetch(s)
    plane.gather(s, out.value, view.all_stride, cnt.value)
    counts = np.zeros(len(batches) * 4, np.uint64)
    vk.check(vk.lib().vk_memcpy(counts.ctypes.data, cnt, counts.nbytes, 2))
    counts = counts.reshape(-1, 4)
    ok, peer_rows = True, 0
    for i, (e, k, bi) in enumerate(refs):
        x = P.expand(csr, batches[i], [10, 5], 42, e, k, bi)
        rows = np.zeros((len(x.all_vertices), dim), np.float32)
        vk.check(vk.lib().vk_memcpy(rows.ctypes.data, out.value + i * view.all_stride * plane.row_bytes,
                                    rows.nbytes, 2))
        exp = P.features(5, dim, x.all_vertices)
        if not np.array_equal(rows.view(np.uint32), exp.view(np.uint32)):
            print(f"rank {rank}: row mismatch in minibatch {i}", flush=True)
            ok = False
        tal = P.classify(x.all_vertices, labels, k, plan.member_bits[k])
        if tuple(int(c) for c in counts[i][:3]) != tal:
            print(f"rank {rank}: tally mismatch {counts[i][:3]} vs {tal}", flush=True)
            ok = False
        # misses owned by partitions on other ranks must have crossed NVLink
        owners = labels[x.all_vertices]
        remote = (owners != k) & (np.array([o % world != rank for o in owners])) & \
            ~np.array([plan.is_cached(k, int(v)) for v in x.all_vertices])
        if int(counts[i][3]) != int(remote.sum()):
            print(f"rank {rank}: peer rows {counts[i][3]} vs {remote.sum()}", flush=True)
            ok = False
        peer_rows += int(counts[i][3])
    print(f"rank {rank}: prefetch={prefetch} {'ok' if ok else 'FAIL'} ({peer_rows} rows over NVLink)", flush=True)
    return ok


if __name__ == "__main__":
    main()
