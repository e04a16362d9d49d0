#!/usr/bin/env python
"""Sample+gather minibatches/s (+ VIP edges/s) on B200, BASELINE.json metric.

One process per GPU (torchrun for N > 1). Default workload `c4`, BASELINE.json
configs[3] (the largest configuration, and it fits one B200): the
ogbn-papers100M-shaped community power-law graph n=111,059,956, d=15
(m ~ 3.33B CSR slots), K=8 partitions (communities), 1.1% train, 128-dim fp16
features, VIP cache alpha=0.32 (sweep 0-32%), fanouts (15,10,5), batch 1024,
SeedSpec{42}. `--config c1|c2|c3` select the smaller configs, `c5` the
VIP-analysis-only sweep.

A "step" is one wave of `--wave` minibatches per GPU through the whole hot
path: sampler (K5/K6 + MFG + relabel) then classify+gather (K9/K10). GPU g
owns partitions k = g (mod N) and processes their minibatches; rows of
partitions owned by other GPUs are read over NVLink by the gather kernel
(CUDA IPC mappings). Per-GPU work is fixed as N grows -> "scaling": "weak".

`value`: inputs (seed ids) already resident in HBM. `e2e`: the same through
the C ABI with the epoch schedule (train members once, each epoch's
permutations on a host worker thread) produced inside the timed region,
pinned HOST seed buffers copied H2D every wave and the per-minibatch tallies
read back to the host. Both timed with CUDA events on the launching stream,
max over ranks.

`--impl reference` times the reference's own CPU implementation (the
unmodified vipkit library compiled in oracle/_ref: epoch_minibatches +
expand + classify, plus a labelled row-gather restatement) on the same config
with all host threads; it never imports the product package.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[0]: synthetic power-law 100K / 2M edges, 64-d fp32, 1 partition
    "c1": dict(workload="C1 synthetic power-law 100K nodes / 2M edges, 64-d fp32, 1 partition",
               n=100_000, d=10, K=1, p_in=1.0, train=0.10, dim=64, dtype=0, alpha=0.0,
               fanouts=(15, 10, 5), b=1024, wave=128),
    # configs[1]: ogbn-arxiv-shaped, 169K nodes, ~1.2M edges (x2 slots), 128-d, 2 partitions, cache 10%
    "c2": dict(workload="C2 ogbn-arxiv-shaped 169K nodes, 128-d fp32, 2 partitions, VIP cache 10%",
               n=169_343, d=7, K=2, p_in=0.8, train=0.537, dim=128, dtype=0, alpha=0.10,
               fanouts=(15, 10, 5), b=1024, wave=128, alpha_sweep=(0.0, 0.05, 0.10, 0.20)),
    # configs[2]: ogbn-products-shaped, 2.45M nodes, 62M edges (x2 slots), 100-d, 8 partitions, cache 20%
    "c3": dict(workload="C3 ogbn-products-shaped 2.45M nodes / 122M CSR slots, 100-d fp32, "
                        "8 partitions, fanout (15,10,5), batch 1024, VIP cache 20%",
               n=2_449_029, d=25, K=8, p_in=0.8, train=0.08, dim=100, dtype=0, alpha=0.20,
               fanouts=(15, 10, 5), b=1024, wave=128, alpha_sweep=(0.0, 0.05, 0.10, 0.20, 0.32)),
}
# BASELINE.json configs[3]/[4]: ogbn-papers100M-shaped (111M nodes, 1.6B
# edges = 3.3B CSR slots, 8 partitions). configs[4] is the VIP-analysis-only
# sweep (2/3/4 hops, fanouts 5..25): `--config c5`.
CONFIGS["c4"] = dict(workload="C4 ogbn-papers100M-shaped 111M nodes / 3.3B CSR slots, 128-d fp16, "
                              "8 partitions, fanout (15,10,5), batch 1024, VIP cache 32% (sweep 0-32%)",
                     n=111_059_956, d=15, K=8, p_in=0.8, train=0.011, dim=128, dtype=1, alpha=0.32,
                     fanouts=(15, 10, 5), b=1024, wave=128, alpha_sweep=(0.0, 0.04, 0.08, 0.16, 0.32))
CONFIGS["c5"] = dict(workload="C5 VIP analysis on ogbn-papers100M-shaped 111M nodes / 3.3B CSR slots, "
                              "8 partitions, fanout sweep", n=111_059_956, d=15, K=8, p_in=0.8, train=0.011,
                     b=1024, fanouts=(15, 10, 5),
                     sweep=[(15, 10, 5), (5, 5), (25, 15), (20, 20, 20), (25, 25, 25, 25)])
RANDOM_READ_GBS = 1400.0  # measured random-record HBM reads, profiles/r01_random_read_bw.txt
PAPER_VIP_SECONDS = 11.8  # PAPER.md:1760-1763 (papers100M, fanouts 15,10,5, 8x A10G)
GRAPH_SEED, ROLES_SEED, SAMPLE_SEED, FEATURE_SEED = 7, 3, 42, 1234


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """NVML sampler (5 ms period) running during the timed region: median SM
    clock under load, max SM clock, and any throttle reasons seen."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device):
        self.ok = False
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(device)
            self.max_sm = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
        self.samples, self.mask = [], 0
        self._stop = threading.Event()

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                self.mask |= N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def stop(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [f"nvml unavailable: {self.err}"]}
        self._stop.set()
        self.t.join()
        reasons = sorted(v for k, v in self.REASONS.items() if self.mask & k)
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_sm, "reasons": reasons, "samples": len(self.samples)}


def nvlink_counters(device):
    """NVLink data bytes (tx, rx) this GPU has moved, from the NVML
    throughput counters (KiB, all links), or None where unavailable."""
    try:
        import pynvml as N
        N.nvmlInit()
        h = N.nvmlDeviceGetHandleByIndex(device)
        vals = N.nvmlDeviceGetFieldValues(h, [N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
                                              N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX])
        out = []
        for v in vals:
            if v.nvmlReturn != 0:
                return None
            out.append(int(v.value.ullVal) * 1024)
        return tuple(out)
    except Exception:  # noqa: BLE001
        return None


def make_data(cfg, threads, world=1, rank=0):
    """The config's graph, labels and roles. With several ranks on one host,
    rank 0 generates the graph once (all host threads) and shares it through
    /dev/shm (the other ranks map it read-only: one copy in the page cache
    instead of one generation peak and one 14 GB copy per rank -- 8 C4 ranks
    would otherwise exhaust host memory); without room there, ranks generate
    one after another."""
    from paper_2305_03152_b200 import vipkit as vk
    t = time.time()
    n = cfg["n"]

    def generate(th):
        return vk.synth_community_powerlaw(n, cfg["d"], cfg["K"], cfg["p_in"], GRAPH_SEED, th,
                                           skew=cfg.get("skew", 2.0))

    if world == 1:
        off, tgt, labels = generate(threads)
    else:
        import torch.distributed as dist
        base = f"/dev/shm/vk_bench_{cfg['n']}_{cfg['d']}_{cfg['K']}_{os.environ.get('MASTER_PORT', '0')}"
        ok = np.zeros(1, np.int64)
        if rank == 0:
            off, tgt, labels = generate(os.cpu_count() or threads)
            try:
                for name, a in (("off", off), ("tgt", tgt), ("lab", labels)):
                    a.tofile(f"{base}.{name}.tmp")
                    os.replace(f"{base}.{name}.tmp", f"{base}.{name}")
                ok[0] = len(tgt)
            except OSError as e:
                log(f"[bench] /dev/shm share failed ({e}); ranks generate in turn")
                for name in ("off", "tgt", "lab"):
                    for suffix in ("", ".tmp"):
                        try:
                            os.remove(f"{base}.{name}{suffix}")
                        except OSError:
                            pass
        t_ok = __import__("torch").from_numpy(ok)
        dist.broadcast(t_ok, 0)
        m = int(t_ok[0])
        if rank != 0:
            if m:
                off = np.memmap(f"{base}.off", np.uint64, "r", shape=(n + 1,))
                tgt = np.memmap(f"{base}.tgt", np.uint32, "r", shape=(m,))
                labels = np.fromfile(f"{base}.lab", np.uint32)
            else:
                for r in range(1, world):  # one generation at a time
                    if r == rank:
                        off, tgt, labels = generate(threads)
                    dist.barrier()
        dist.barrier()
        if rank == 0 and m:
            for name in ("off", "tgt", "lab"):  # unlinked now, mapped pages stay valid
                os.remove(f"{base}.{name}")
    roles = vk.synth_roles(n, cfg["train"], 0.0, 0.0, ROLES_SEED)
    log(f"[bench] graph n={n} m={len(tgt)} ready in {time.time() - t:.1f}s")
    return off, tgt, labels, roles


def schedule(vk, cfg, roles, labels, parts, count):
    """(epoch, partition, batch_index, seeds), round-robin over `parts`."""
    from paper_2305_03152_b200.dist import minibatch_schedule
    return minibatch_schedule(lambda k, e: vk.epoch_permutation(roles, labels, k, cfg["b"], e, SAMPLE_SEED),
                              parts, cfg["b"], count)


# ------------------------------------------------------------------ b200 arm
def run_b200(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_2305_03152_b200 import vipkit as vk

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")  # host-side plumbing only (barriers, handle exchange, max)
    dev = local
    K, M, L = cfg["K"], args.wave, len(cfg["fanouts"])
    nthreads = max(1, (os.cpu_count() or 8) // world)
    off, tgt, labels, roles = make_data(cfg, nthreads, world, rank)
    n, m = cfg["n"], len(tgt)
    g = vk.Graph.from_csr(off, tgt, undirected=True, device=dev)
    if world > 1:  # the host CSR is only needed again by the N=1 CPU baseline
        off = tgt = None
    stream = torch.cuda.Stream(device=dev)
    sh = stream.cuda_stream

    # ---- VIP analysis for all K partitions in one multi-column pass (timed)
    p0 = np.stack([vk.initial_probs(roles, labels, k, cfg["b"]) for k in range(K)])
    p0_d = torch.from_numpy(p0).to(f"cuda:{dev}")
    del p0  # K x n f64 on every rank: keep host memory for N ranks per box
    tot_d = torch.empty((K, n), dtype=torch.float64, device=f"cuda:{dev}")
    with torch.cuda.stream(stream):
        vk.propagate_device(g, cfg["fanouts"], K, p0_d.data_ptr(), None, tot_d.data_ptr(), sh)  # warm
        torch.cuda.synchronize(dev)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        reps = 3
        ev[0].record(stream)
        for _ in range(reps):
            vk.propagate_device(g, cfg["fanouts"], K, p0_d.data_ptr(), None, tot_d.data_ptr(), sh)
        ev[1].record(stream)
        torch.cuda.synchronize(dev)
    vip_ms = ev[0].elapsed_time(ev[1]) / reps
    totals = tot_d.cpu().numpy()
    vip_bytes = L * (8 * n + 4 * m + 8 * K * m + 32 * K * n)
    vip = {"edges_per_s": L * m * K / (vip_ms / 1e3), "ms": vip_ms, "partitions": K, "hops": L,
           "m": m, "achieved_gbs": vip_bytes / (vip_ms / 1e3) / 1e9}

    # ---- ranking, cache plan, VIP-ordered feature plane
    orders = [vk.rank_by_scores(labels, k, totals[k], device=dev)[0] for k in range(K)]
    plan = vk.build_cache(orders, cfg["alpha"], n)
    oon, ranges = vk.build_reorder(labels, K, totals, device=dev)
    plane = vk.FeaturePlane(n, K, cfg["dim"], labels, oon, ranges, dtype=cfg["dtype"], device=dev)
    from paper_2305_03152_b200.dist import exchange_plane_handles, max_over_ranks, owned_partitions
    mine = owned_partitions(K, world, rank)
    for k in mine:
        plane.load_partition(k, plan.cached[k], feature_seed=FEATURE_SEED)
    if world > 1:
        exchange_plane_handles(plane, mine)

    # ---- minibatch schedule + device-resident seeds
    W, S = args.warmup, args.steps
    sched = schedule(vk, cfg, roles, labels, mine, (W + 2 * S) * M)
    waves = [sched[i * M:(i + 1) * M] for i in range(W + 2 * S)]
    # multi-GPU: two samplers alternate so wave i+1 samples while wave i's
    # NVLink miss exchange runs (vk_plane_prefetch on the plane's aux stream)
    prefetch = (world > 1) if args.prefetch == "auto" else args.prefetch == "1"
    overlap = args.sched == "overlap"
    P = 1 if (prefetch or overlap) else args.pipes
    samplers = [vk.Sampler(g, cfg["fanouts"], cfg["b"], M, SAMPLE_SEED, frontier=args.frontier)
                for _ in range(2 if (prefetch or overlap) else P)]
    # overlap schedule: samplers on a high-priority stream, gathers on the
    # main one, so wave i+1 samples (L2/latency bound) while wave i gathers
    # (HBM bound); the sampler's CTAs take SM slots as gather CTAs retire
    hi_stream = torch.cuda.Stream(device=dev, priority=-1) if overlap else None
    view = samplers[0].view()
    cap_all = view.all_stride
    rb = plane.row_bytes
    outs = [torch.empty(M * cap_all * rb, dtype=torch.uint8, device=f"cuda:{dev}") for _ in range(P)]
    streams = [stream] + [torch.cuda.Stream(device=dev) for _ in range(P - 1)]
    seeds_all = np.concatenate([w[3] for wv in waves for w in wv]).astype(np.uint32)
    seeds_d = torch.from_numpy(seeds_all.view(np.int32)).to(f"cuda:{dev}")
    wave_offsets, pos = [], 0
    for wv in waves:
        o = np.zeros(len(wv) + 1, np.uint64)
        o[1:] = np.cumsum([len(w[3]) for w in wv])
        wave_offsets.append(o + pos)
        pos += int(o[-1])
    cw = samplers[0].count_words()
    hist_counts = torch.zeros((W + 2 * S, cw), dtype=torch.int32, device=f"cuda:{dev}")
    hist_tally = torch.zeros((W + 2 * S, M, 4), dtype=torch.int64, device=f"cuda:{dev}")
    # per wave: sampler start/end, gather start/end
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(W + 2 * S)]

    # e2e: the schedule itself is produced inside the timed region
    from paper_2305_03152_b200.dist import MinibatchStream
    src = {"stream": None}

    def fetch(i, host):
        if host and src["stream"] is not None:
            waves[i] = src["stream"].take(M)
        return waves[i]

    def wave(i, host=False, pinned=None):
        # wave i runs on pipe i % P: sampler and gather of consecutive waves
        # overlap on separate streams (sampler is L2-latency bound, gather HBM bound)
        p = i % P
        st, sp = streams[p], samplers[p]
        sh_p = st.cuda_stream
        wv = fetch(i, host)
        refs = [(e, k, bi) for (e, k, bi, _) in wv]
        evs[i][0].record(st)
        if host:
            sp.run([w[3] for w in wv], refs, stream=sh_p)
        else:
            sp.run(wave_offsets[i], refs, stream=sh_p, seeds_device_ptr=seeds_d.data_ptr())
        evs[i][1].record(st)
        evs[i][2].record(st)
        plane.gather(sp, outs[p].data_ptr(), cap_all, hist_tally[i].data_ptr(), stream=sh_p)
        evs[i][3].record(st)
        sp.snapshot_counts(hist_counts[i].data_ptr(), stream=sh_p)
        if pinned is not None:
            with torch.cuda.stream(st):
                pinned[i].copy_(hist_tally[i], non_blocking=True)

    def sample(i, host):
        sp = samplers[i % 2]
        wv = fetch(i, host)
        refs = [(e, k, bi) for (e, k, bi, _) in wv]
        evs[i][0].record(stream)
        if host:
            sp.run([w[3] for w in wv], refs, stream=sh)
        else:
            sp.run(wave_offsets[i], refs, stream=sh, seeds_device_ptr=seeds_d.data_ptr())
        evs[i][1].record(stream)

    def waves_prefetch(lo, hi, host, pinned):
        # main: S(i+1) G(i) S(i+2) G(i+1) ...; aux: the NVLink exchange of
        # wave i+1, issued after S(i+1) (runs during the HBM-bound G(i)) or,
        # --prefetch-order gather, after G(i) (runs during S(i+2))
        sample(lo, host)
        plane.prefetch(samplers[lo % 2])
        for i in range(lo, hi):
            sp = samplers[i % 2]
            if i + 1 < hi:
                sample(i + 1, host)
                if args.prefetch_order == "sample":
                    plane.prefetch(samplers[(i + 1) % 2])
            evs[i][2].record(stream)
            plane.gather(sp, outs[0].data_ptr(), cap_all, hist_tally[i].data_ptr(), stream=sh)
            evs[i][3].record(stream)
            if i + 1 < hi and args.prefetch_order == "gather":
                plane.prefetch_after(samplers[(i + 1) % 2], sh)
            sp.snapshot_counts(hist_counts[i].data_ptr(), stream=sh)
            if pinned is not None:
                with torch.cuda.stream(stream):
                    pinned[i].copy_(hist_tally[i], non_blocking=True)

    def waves_overlap(lo, hi, host, pinned):
        hs = hi_stream.cuda_stream
        for i in range(lo, hi):
            sp = samplers[i % 2]
            wv = fetch(i, host)
            refs = [(e, k, bi) for (e, k, bi, _) in wv]
            if i - 2 >= lo:
                hi_stream.wait_event(evs[i - 2][3])  # same sampler: its gather has read it
            evs[i][0].record(hi_stream)
            if host:
                sp.run([w[3] for w in wv], refs, stream=hs)
            else:
                sp.run(wave_offsets[i], refs, stream=hs, seeds_device_ptr=seeds_d.data_ptr())
            evs[i][1].record(hi_stream)
            stream.wait_event(evs[i][1])
            if prefetch:
                plane.prefetch(sp)
            evs[i][2].record(stream)
            plane.gather(sp, outs[0].data_ptr(), cap_all, hist_tally[i].data_ptr(), stream=sh)
            evs[i][3].record(stream)
            sp.snapshot_counts(hist_counts[i].data_ptr(), stream=sh)
            if pinned is not None:
                with torch.cuda.stream(stream):
                    pinned[i].copy_(hist_tally[i], non_blocking=True)

    def region(lo, hi, host=False, pinned=None):
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for st in streams[1:]:
            st.wait_event(t0)
        if overlap:
            hi_stream.wait_event(t0)
            waves_overlap(lo, hi, host, pinned)
            e_hi = torch.cuda.Event()
            e_hi.record(hi_stream)
            stream.wait_event(e_hi)
        elif prefetch:
            waves_prefetch(lo, hi, host, pinned)
        else:
            for i in range(lo, hi):
                wave(i, host, pinned)
        for st in streams[1:]:
            e = torch.cuda.Event()
            e.record(st)
            stream.wait_event(e)
        t1.record(stream)
        torch.cuda.synchronize(dev)
        return t0.elapsed_time(t1)

    region(0, W)
    if world > 1:
        dist.barrier()
    clocks = Clocks(dev)
    clocks.start()
    nvl0 = nvlink_counters(dev) if world > 1 else None
    l0 = vk.launch_count()
    ms = region(W, W + S)
    launches = vk.launch_count() - l0
    nvl1 = nvlink_counters(dev) if world > 1 else None
    clk = clocks.stop()
    # e2e: host seeds (H2D inside the region) + tallies read back to the host
    pinned = torch.zeros((W + 2 * S, M, 4), dtype=torch.int64).pin_memory()
    # steady state: the schedule worker runs one epoch ahead of the waves
    src["stream"] = MinibatchStream(vk, roles, labels, mine, cfg["b"], SAMPLE_SEED).ready()
    if world > 1:
        dist.barrier()
    e2e_ms = region(W + S, W + 2 * S, host=True, pinned=pinned)
    src["stream"].close()
    ms, e2e_ms = max_over_ranks([ms, e2e_ms])

    # ---- roofline of the dominant kernel (gather) and of the sampler, from the timed waves
    tally = hist_tally.cpu().numpy()
    cnts = hist_counts.cpu().numpy().view(np.uint32)
    gather_ms = [evs[i][2].elapsed_time(evs[i][3]) for i in range(W, W + S)]
    sample_ms = [evs[i][0].elapsed_time(evs[i][1]) for i in range(W, W + S)]
    g_bytes, s_bytes, rows, misses, peer, cache_hits = 0, 0, 0, 0, 0, 0
    for i in range(W, W + S):
        nmb = len(waves[i])
        allc = tally[i, :nmb, :3].sum(axis=1)
        rows += int(allc.sum())
        misses += int(tally[i, :nmb, 2].sum())
        cache_hits += int(tally[i, :nmb, 1].sum())
        peer += int(tally[i, :nmb, 3].sum())
        fc = cnts[i, :(L + 1) * M].reshape(L + 1, M)[:, :nmb].astype(np.int64)
        ec = cnts[i, (L + 1) * M:2 * (L + 1) * M].reshape(L + 1, M)[:, :nmb].astype(np.int64)
        ac = cnts[i, 2 * (L + 1) * M:2 * (L + 1) * M + M][:nmb].astype(np.int64)
        s_bytes += int(sum(16 * fc[h - 1].sum() + 8 * ec[h].sum() for h in range(1, L + 1))
                       + 8 * (fc[1:].sum() + ac.sum()))
    # compulsory gather bytes: every output row written once, its 4-byte id
    # read once, and each DISTINCT source row of the wave read once (rows
    # shared by minibatches of a wave are L2 hits, not HBM reads). The
    # distinct count comes from the last wave still held by its sampler.
    last = W + 2 * S - 1
    distinct = distinct_rows(samplers[last % len(samplers)], len(waves[last]), dev)
    rows_last = int(tally[last, :len(waves[last]), :3].sum())
    g_bytes = int(rows / S * (rb + 4) + distinct * rb) * S
    hbm, peak_kind = peaks()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f).get(args.config)
        if t and t.get("minibatches_per_launch") == M:
            traffic = t["dram_bytes_read"] + t["dram_bytes_write"]
    except Exception:  # noqa: BLE001
        pass
    sampler_bound = {"bound": "l2"}
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            ts = json.load(f).get(args.config + "_sampler")
        if ts and ts.get("minibatches_per_launch") == M:
            sampler_bound.update({"ncu_kernel": ts["kernel"], "ncu_l2_throughput_pct": ts["lts_throughput_pct"],
                                  "ncu_dram_throughput_pct": ts["dram_throughput_pct"], "note": ts["note"]})
    except Exception:  # noqa: BLE001
        pass
    g_ach = g_bytes / S / (statistics.mean(gather_ms) / 1e3) / 1e9
    s_ach = s_bytes / S / (statistics.mean(sample_ms) / 1e3) / 1e9
    total_mb = sum(len(waves[i]) for i in range(W, W + S)) * world
    value = total_mb / (ms / 1e3)
    e2e_val = total_mb / (e2e_ms / 1e3)
    # seeds plus the per-minibatch wave descriptors (WaveDesc, 80 B) every wave
    h2d = int(sum(len(w[3]) * 4 + 80 for i in range(W + S, W + 2 * S) for w in waves[i]) / S)
    result = {
        "metric": "sample+gather minibatches/s", "value": value, "unit": "minibatches/s",
        "n_gpus": world, "steps": S, "warmup": W, "ms_per_step": ms / S, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32 ids / fp32 rows / fp64 VIP",
        "data": "synthetic (community power-law graph, counter-hashed feature rows)",
        "config": {"workload": cfg["workload"], "n": n, "m_slots": m, "partitions": K, "pipes": P,
                   "exchange_prefetch": bool(prefetch), "prefetch_order": args.prefetch_order, "frontier": args.frontier,
                   "schedule": args.sched,
                   "fanouts": list(cfg["fanouts"]), "batch": cfg["b"], "minibatches_per_step_per_gpu": M,
                   "feature_dim": cfg["dim"], "row_bytes": rb, "alpha": cfg["alpha"],
                   "partitions_per_gpu": len(mine), "l2": "inputs larger than L2 (graph "
                   f"{(8 * n + 4 * m) / 1e9:.2f} GB, features {n * rb / 1e9:.2f} GB); no flush"},
        "e2e": {"value": e2e_val, "unit": "minibatches/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": M * 4 * 8},
        "roofline": {"bound": "hbm", "kernel": "k_gather (classify+gather)", "achieved": g_ach,
                     "peak": hbm, "unit": "GB/s", "frac": g_ach / hbm, "traffic": traffic,
                     "traffic_note": "ncu dram read+write per launch (profiles/traffic.json)",
                     "algorithmic_bytes": "rows x (row_bytes + 4 B id) + distinct rows of the wave x row_bytes "
                                          f"(distinct {distinct} of {rows_last} rows in the last wave)",
                     "peak_kind": peak_kind, "bytes_per_launch": g_bytes / S,
                     "ms_per_launch": statistics.mean(gather_ms)},
        "sampler": {"ms_per_wave": statistics.mean(sample_ms), "achieved_gbs": s_ach,
                    "frac": s_ach / hbm, "bytes_per_wave": s_bytes / S, **sampler_bound},
        "vip": {**vip, "unit": "edges/s", "frac": vip["achieved_gbs"] / hbm},
        "tallies": {"rows": rows, "miss_rows": misses, "miss_rows_no_cache": misses + cache_hits,
                    "miss_reduction_by_vip_cache": 1.0 - misses / max(misses + cache_hits, 1),
                    "miss_rows_over_nvlink": peer, "miss_fraction": misses / max(rows, 1)},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if world > 1:
        # the miss exchange of the last timed wave: distinct rows pulled over NVLink
        pulled = plane.pulled_rows()
        result["nvlink"] = {"rows_pulled_last_wave": pulled, "bytes_pulled_last_wave": pulled * rb,
                            "rows_requested_last_wave": int(tally[W + 2 * S - 1, :len(waves[W + 2 * S - 1]), 3].sum())}
        if nvl0 and nvl1:
            # hardware counters over the timed region (this rank's GPU, all
            # links): rx = rows this GPU pulled, tx = rows peers pulled from it
            tx, rx = (nvl1[0] - nvl0[0]) / S, (nvl1[1] - nvl0[1]) / S
            result["nvlink"].update({"hw_rx_bytes_per_wave": rx, "hw_tx_bytes_per_wave": tx,
                                     "hw_rx_gbs": rx / (ms / S / 1e3) / 1e9,
                                     "peak_gbs_per_direction": 900.0,
                                     "source": "NVML NVLINK_THROUGHPUT_DATA_{TX,RX} around the timed region"})
    if cfg.get("alpha_sweep") and rank == 0:
        # vipkit::simulate over one full epoch of every partition on the device
        # (vk_simulate): one expansion pass scored against every
        # cache size at once (nested VIP-ranking prefixes). Untimed for the
        # headline; its own wall time is reported.
        alphas = list(cfg["alpha_sweep"])
        plans = [vk.build_cache(orders, a, n) for a in alphas]
        takes = [[len(p_.cached[k]) for k in range(K)] for p_ in plans]
        top = plans[int(np.argmax([sum(t) for t in takes]))]
        t0 = time.perf_counter()
        cells = vk.simulate(g, roles, labels, K, list(cfg["fanouts"]), cfg["b"], 1, SAMPLE_SEED, top.cached,
                            takes=takes)
        sim_s = time.perf_counter() - t0
        sweep = []
        for i, a in enumerate(alphas):
            c = cells[i].sum(axis=(0, 1))
            sweep.append({"alpha": a, "cache_rows_per_partition": int(takes[i][0]), "local": int(c[0]),
                          "cache_hits": int(c[1]), "miss_rows": int(c[2]),
                          "miss_bytes": int(c[2]) * rb})
        base = max(sweep[0]["miss_rows"], 1)
        for r_ in sweep:
            r_["miss_reduction_vs_no_cache"] = 1.0 - r_["miss_rows"] / base
        mbs = sum(int(np.ceil(np.count_nonzero((labels == k) & (roles == 0)) / cfg["b"])) for k in range(K))
        result["alpha_sweep"] = {"scope": "one epoch, all partitions (vk_simulate)", "minibatches": mbs,
                                 "seconds": sim_s, "rows": sweep}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(cfg, off, tgt, labels, roles, M)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------ VIP-only (C5)
def run_vip_sweep(args, cfg):
    """VIP analysis for every partition on the papers100M-shaped graph: one
    multi-column pass per fanout setting; GPU g computes partitions k = g mod N.
    value = edge-hops/s for (15,10,5) = K*L*m / t (max over ranks)."""
    import torch
    import torch.distributed as dist

    from paper_2305_03152_b200 import vipkit as vk
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    K = cfg["K"]
    off, tgt, labels, roles = make_data(cfg, max(1, (os.cpu_count() or 8) // world), world, rank)
    n, m = cfg["n"], len(tgt)
    g = vk.Graph.from_csr(off, tgt, undirected=True, device=local)
    off = tgt = None
    mine = [k for k in range(K) if k % world == rank]
    p0 = np.stack([vk.initial_probs(roles, labels, k, cfg["b"]) for k in mine])
    stream = torch.cuda.Stream(device=local)
    p0_d = torch.from_numpy(p0).to(f"cuda:{local}")
    tot_d = torch.empty((len(mine), n), dtype=torch.float64, device=f"cuda:{local}")
    rows = []
    for fan in cfg["sweep"]:
        with torch.cuda.stream(stream):
            vk.propagate_device(g, fan, len(mine), p0_d.data_ptr(), None, tot_d.data_ptr(), stream.cuda_stream)
            torch.cuda.synchronize(local)
            if world > 1:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = max(1, args.steps // 5)
            e0.record(stream)
            for _ in range(reps):
                vk.propagate_device(g, fan, len(mine), p0_d.data_ptr(), None, tot_d.data_ptr(),
                                    stream.cuda_stream)
            e1.record(stream)
            torch.cuda.synchronize(local)
        t = torch.tensor([e0.elapsed_time(e1) / reps / 1e3], dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec = float(t[0])
        rows.append({"fanouts": list(fan), "hops": len(fan), "seconds_all_partitions": sec,
                     "edge_hops_per_s": K * len(fan) * m / sec})
        log(f"[bench] VIP {fan}: {sec * 1e3:.1f} ms for {K} partitions")
    head = rows[0]
    # roofline: the pull kernels gather one 32 B sector of hoisted log terms
    # (float, up to 8 columns per pass) per in-edge per hop from a table far
    # larger than L2 -> bound by random-record HBM reads, measured at
    # ~1.4 TB/s on this part (profiles/r01_random_read_bw.txt)
    passes = (len(mine) + 7) // 8
    sector_bytes = 3 * m * 32 * passes
    ach = sector_bytes / head["seconds_all_partitions"] / 1e9
    formula = 3 * (12 * m + 40 * n) * len(mine)  # SURVEY §8d per hop per column (fp64 lm)
    roof = {"bound": "hbm-random", "achieved": ach, "peak": RANDOM_READ_GBS, "unit": "GB/s",
            "frac": ach / RANDOM_READ_GBS, "traffic": None,
            "peak_kind": "measured random 32-128 B record reads (profiles/r01_random_read_bw.txt)",
            "algorithmic": "3 hops x m in-edges x one 32 B sector per pass of <= 8 float columns",
            "survey_formula_gbs": formula / head["seconds_all_partitions"] / 1e9}
    # the paper's 11.8 s produced every partition's VIP on 8 machines in parallel
    paper_rate = K * 3 * 3.2e9 / PAPER_VIP_SECONDS
    if rank == 0:
        print(json.dumps({
            "metric": "VIP analysis edge-hops/s (all partitions, fanout 15,10,5)",
            "value": head["edge_hops_per_s"], "unit": "edge-hops/s", "n_gpus": world,
            "steps": max(1, args.steps // 5), "warmup": 1, "ms_per_step": head["seconds_all_partitions"] * 1e3,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": head["edge_hops_per_s"] / paper_rate,
            "vs_baseline_note": f"paper: {PAPER_VIP_SECONDS} s on 8x A10G for papers100M (PAPER.md:1760-1763), "
                                f"taken as all {K} partitions -> {paper_rate:.3g} edge-hops/s",
            "dtype": "fp64 (hoisted log terms stored fp32, accumulation fp64)", "data": "synthetic",
            "config": {"workload": cfg["workload"], "n": n, "m_slots": m, "partitions": K,
                       "partitions_per_gpu": len(mine)},
            "roofline": roof, "sweep": rows, "gpu_launches": None}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# -------------------------------------------------------------- CPU baseline
def capacity_all(cfg, max_deg):
    """The sampler's per-minibatch all_vertices capacity (vk_sampler_create)."""
    n, cap_prev, tot = cfg["n"], cfg["b"], cfg["b"]
    for f in cfg["fanouts"]:
        cap_prev = min(n, cap_prev * min(f, max(1, max_deg)))
        tot += cap_prev
    return min(n, tot)


class CpuReference:
    """The reference's own CPU path on this config (oracle/_ref = the
    unmodified vipkit library; test infrastructure, used here only as the
    measured baseline): the schedule comes from epoch_minibatches over a
    PartitionMap built once (sampling.cpp:45-70, as for_each_expansion does,
    commsim.cpp:38-52), each minibatch is expanded (sampling.cpp:94-128) and
    classified (commsim.cpp:61-73), and its all_vertices rows are gathered from
    the host feature table by a labelled restatement (the reference never
    materialises features). Workers over independent minibatches
    (expand is pure, sampling.cpp:82).

    The cache plan is build_cache (policies.cpp:149-163) over rank_by_scores of
    the out-degree: classify's cost does not depend on which rows are cached,
    and the reference's own VIP propagate over 3.3 B slots x 8 partitions
    would take ~10 min on the host."""

    def __init__(self, cfg, off, tgt, labels, roles, threads, with_table=True):
        import concurrent.futures as cf
        from oracle import oracle as O
        self.cfg, self.threads = cfg, threads
        P, R = O.port(), O.ref()
        self.R = R
        t = time.time()
        n, K = cfg["n"], cfg["K"]
        self.G = O.CSR(n, off, tgt)
        R.graph_symmetric(self.G, threads)
        self.ctx = R.context(roles, labels, K)
        deg = np.diff(off).astype(np.float64)
        with cf.ThreadPoolExecutor(max_workers=min(K, threads)) as ex:
            orders = list(ex.map(lambda k: R.rank_by_scores(labels, K, k, deg)[0], range(K)))
        _, self.bits = R.build_cache(orders, cfg["alpha"], n)
        del orders, deg
        self.labels = labels
        fp16 = cfg.get("dtype", 0) == 1
        self.table = P.feature_table(FEATURE_SEED, cfg["dim"], n, fp16=fp16, threads=threads) if with_table else None
        cap = capacity_all(cfg, int(np.diff(off).max()))
        self.work = (np.empty((threads, cap, cfg["dim"]), np.float16 if fp16 else np.float32)
                     if with_table else None)
        self._epoch, self._buf, self._pos = 0, [], 0
        log(f"[bench] reference setup (graph, plan, feature table) {time.time() - t:.1f}s")

    def take(self, count):
        """Next `count` (epoch, k, i, seeds) in minibatch_schedule order;
        epochs are scheduled by the reference's epoch_minibatches on demand."""
        cfg, out = self.cfg, []
        while len(out) < count:
            if self._pos == len(self._buf):
                b, e = cfg["b"], self._epoch
                per = {k: self.ctx.epoch(k, b, e, SAMPLE_SEED) for k in range(cfg["K"])}
                nb = {k: (len(per[k]) + b - 1) // b for k in per}
                self._buf = [(e, k, i, per[k][i * b:(i + 1) * b]) for i in range(max(nb.values()))
                             for k in per if i < nb[k]]
                self._pos, self._epoch = 0, e + 1
            t = min(count - len(out), len(self._buf) - self._pos)
            out.extend(self._buf[self._pos:self._pos + t])
            self._pos += t
        return out

    def step(self, count, gather=True, threads=None):
        """One timed step: schedule + expand + classify (+ gather) of `count` minibatches."""
        t0 = time.perf_counter()
        mbs = self.take(count)
        self.R.bench_minibatches(self.G, mbs, self.cfg["fanouts"], SAMPLE_SEED, self.labels, self.bits,
                                 self.table if gather else None, self.work if gather else None,
                                 threads or self.threads)
        return time.perf_counter() - t0


def cpu_baseline(cfg, off, tgt, labels, roles, M, budget_s=20.0):
    """cpu_baseline of the GPU arm (rank 0, N=1): the reference CPU path
    (CpuReference) on a bounded sample of the same workload."""
    from oracle import oracle as O
    if not O.ref_available():
        return {"value": None, "unit": "minibatches/s", "cores": 0, "kind": "reference",
                "sample": "oracle/_ref not built"}
    threads = os.cpu_count() or 1
    ref = CpuReference(cfg, off, tgt, labels, roles, threads)
    per = max(threads, min(M, 64))
    ref.step(per)  # warm (page-in of the feature table and graph)
    t1 = ref.step(per)
    steps = max(1, min(20, int(budget_s / 2 / max(t1, 1e-3))))
    tt = sum(ref.step(per) for _ in range(steps))
    no_gather = per / ref.step(per, gather=False)
    single = 2 / ref.step(2, threads=1)
    return {"value": steps * per / tt, "unit": "minibatches/s", "cores": threads, "kind": "reference",
            "expand_classify_only": no_gather, "single_thread_value": single,
            "sample": f"{steps} steps x {per} minibatches of the bench schedule: reference epoch_minibatches + "
                      f"expand + classify (unmodified vipkit, oracle/_ref) + row gather restatement "
                      f"(oracle/workload.c) on {threads} threads; cache plan = build_cache over a degree "
                      f"ranking (classify cost is plan-independent)"}


class _DevArray:
    """Minimal __cuda_array_interface__ view of a device pointer (for torch)."""

    def __init__(self, ptr, count, typestr="<u4"):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3}


def distinct_rows(sampler, nmb, dev):
    """Number of distinct vertices across the all_vertices lists of the
    sampler's current wave (torch.unique on the device, outside timed regions)."""
    import torch
    v = sampler.view()
    cnt = torch.as_tensor(_DevArray(v.all_count, nmb), device=f"cuda:{dev}").to(torch.int64).cpu().tolist()
    allv = torch.as_tensor(_DevArray(v.all, nmb * v.all_stride), device=f"cuda:{dev}").view(torch.int32)
    parts = [allv[i * v.all_stride:i * v.all_stride + c] for i, c in enumerate(cnt)]
    return int(torch.unique(torch.cat(parts)).numel())


def run_reference(args, cfg):
    """--impl reference: the unmodified reference CPU path (CpuReference) on
    the same config, steps of --wave minibatches. Never imports the product
    package: the graph comes from the oracle's restatement of the bench
    generator (oracle/workload.c, pinned to the product's by tests), roles
    from the reference's make_roles."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as O
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    threads = os.cpu_count() or 1
    t = time.time()
    off, tgt, labels = O.port().synth_community_powerlaw(cfg["n"], cfg["d"], cfg["K"], cfg["p_in"], GRAPH_SEED,
                                                         threads)
    roles = O.ref().make_roles(cfg["n"], cfg["train"], 0.0, 0.0, ROLES_SEED)
    log(f"[bench] reference arm: graph n={cfg['n']} m={len(tgt)} in {time.time() - t:.1f}s")
    ref = CpuReference(cfg, off, tgt, labels, roles, threads)
    M, W, S = args.wave, args.warmup, args.steps
    for _ in range(W):
        ref.step(M)
    tt = sum(ref.step(M) for _ in range(S))
    value = S * M / tt
    no_gather = M / ref.step(M, gather=False)
    print(json.dumps({
        "impl": "reference", "metric": "sample+gather minibatches/s", "value": value,
        "unit": "minibatches/s", "n_gpus": args.gpus, "steps": S, "warmup": W,
        "ms_per_step": tt / S * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32 ids / fp32 or fp16 rows",
        "data": "synthetic (community power-law graph, counter-hashed feature rows)",
        "config": {"workload": cfg["workload"], "n": cfg["n"], "m_slots": int(len(tgt)), "partitions": cfg["K"],
                   "fanouts": list(cfg["fanouts"]), "batch": cfg["b"], "minibatches_per_step_per_gpu": M,
                   "feature_dim": cfg["dim"], "alpha": cfg["alpha"]},
        "cpu_baseline": {"value": value, "unit": "minibatches/s", "cores": threads, "kind": "reference",
                         "expand_classify_only": no_gather,
                         "sample": f"{S} steps x {M} minibatches: reference epoch_minibatches + expand + "
                                   f"classify + row gather restatement, {threads} host threads"},
        "e2e": {"value": value, "unit": "minibatches/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--alpha-sweep", action="store_true", help="also tally misses for cache sizes 0-32%%")
    ap.add_argument("--wave", type=int, default=None,
                    help="minibatches per step per GPU (default: the config's; 128 for c1-c3, 64 for c4)")
    ap.add_argument("--pipes", type=int, default=1, help="overlapped sampler+gather pipelines (streams)")
    ap.add_argument("--prefetch", default="auto", choices=["auto", "0", "1"],
                    help="overlap the multi-GPU miss exchange with the next wave's sampling (auto: on for N>1)")
    ap.add_argument("--prefetch-order", default="sample", choices=["sample", "gather"],
                    help="issue wave i+1's exchange after its sampling (overlaps gather i) or after gather i "
                         "(overlaps the sampling of wave i+2)")
    ap.add_argument("--sched", default="serial", choices=["serial", "overlap"],
                    help="overlap: sample wave i+1 on a high-priority stream while wave i gathers")
    ap.add_argument("--frontier", default="auto", choices=["auto", "dense", "sparse"],
                    help="sampler frontier representation (default: automatic by graph size)")
    ap.add_argument("--vip-storage", type=int, default=0, choices=[0, 32, 64],
                    help="VIP hoisted-term storage width (0: automatic)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--alpha", type=float, default=None, help="override the config's VIP cache fraction")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = dict(CONFIGS[args.config])
    if args.alpha is not None:
        cfg["alpha"] = args.alpha
    if args.wave is None:
        args.wave = cfg.get("wave", 32)
    if args.alpha_sweep and "alpha_sweep" not in cfg:
        cfg["alpha_sweep"] = (0.0, 0.04, 0.08, 0.16, 0.32)
    if args.vip_storage and args.impl != "reference":
        from paper_2305_03152_b200 import vipkit as vk
        vk.vip_force_storage(args.vip_storage)
    if args.config == "c5" and args.impl != "reference":
        run_vip_sweep(args, cfg)
        return
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_b200(args, cfg)


if __name__ == "__main__":
    main()
