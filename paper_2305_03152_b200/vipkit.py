"""Python mirror of the reference ``vipkit`` hot-path API over the C ABI.

The reference (/root/reference/proj) is C++; its drop-in replacement is the
C ABI in ``include/vipkit_b200.h`` plus the C++ mirror
``include/vipkit_b200/vipkit.hpp``. This module is the same surface for Python
callers (tests, bench.py): the same function names, argument meaning and error
types as ``namespace vipkit`` (``graph.hpp``, ``vip.hpp``, ``sampling.hpp``,
``policies.hpp``, ``reorder.hpp``). Every compute call goes to
``libvipkit_b200.so``; there is no CPU fallback — without the built library or
an sm_100 GPU the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libvipkit_b200.so")
MAX_HOPS = 8
VK_MISS = 0xFFFFFFFF
F32, F16 = 0, 1


# ---------------------------------------------------------------- errors
class VipkitError(RuntimeError):
    """vipkit::error (error.hpp:8-10)."""
    code = 23


class ParseError(VipkitError): code = 1          # noqa: E701
class RangeError(VipkitError): code = 2          # noqa: E701
class ParameterError(VipkitError): code = 3      # noqa: E701
class FormatError(VipkitError): code = 4         # noqa: E701
class PartitionError(VipkitError): code = 5      # noqa: E701
class SamplingError(VipkitError): code = 6       # noqa: E701
class ConfigError(VipkitError): code = 7         # noqa: E701
class ShapeError(VipkitError): code = 8          # noqa: E701
class IOError_(VipkitError): code = 9            # noqa: E701
class CudaError(VipkitError): code = 20          # noqa: E701
class UnsupportedError(VipkitError): code = 22   # noqa: E701


_BY_CODE = {c.code: c for c in (ParseError, RangeError, ParameterError, FormatError,
                                PartitionError, SamplingError, ConfigError, ShapeError,
                                IOError_, CudaError, UnsupportedError)}

# ------------------------------------------------------------------ library
_lib = None
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
c_u64, c_u32, c_int, c_vp, c_double = C.c_uint64, C.c_uint32, C.c_int, C.c_void_p, C.c_double


class BatchRef(C.Structure):
    """vipkit::BatchRef (sampling.hpp:33-37)."""
    _fields_ = [("epoch", c_u64), ("batch_index", c_u64), ("partition", c_u32), ("reserved", c_u32)]


class SamplerConfig(C.Structure):
    _fields_ = [("num_hops", c_u32), ("fanouts", c_u32 * MAX_HOPS), ("batch_size", c_u64),
                ("max_minibatches", c_u32), ("flags", c_u32), ("global_seed", c_u64)]


class SamplerView(C.Structure):
    _fields_ = [("nmb", c_u32), ("num_hops", c_u32),
                ("all", c_vp), ("all_stride", c_u64), ("all_count", c_vp),
                ("frontier", c_vp * (MAX_HOPS + 1)), ("frontier_stride", c_u64 * (MAX_HOPS + 1)),
                ("frontier_count", c_vp * (MAX_HOPS + 1)),
                ("mfg_indptr", c_vp * (MAX_HOPS + 1)),
                ("mfg_dst", c_vp * (MAX_HOPS + 1)), ("mfg_stride", c_u64 * (MAX_HOPS + 1)),
                ("all_index", c_vp * (MAX_HOPS + 1))]


def lib():
    """Load libvipkit_b200.so (fails loudly when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (or `make -C paper_2305_03152_b200/csrc`)")
    L = C.CDLL(LIB_PATH)
    L.vk_last_error.restype = C.c_char_p
    L.vk_status_name.restype = C.c_char_p
    L.vk_status_name.argtypes = [c_int]
    L.vk_launch_count.restype = c_u64
    L.vk_device_count.argtypes = [C.POINTER(c_int)]
    L.vk_device_alloc.argtypes = [c_int, C.c_size_t, C.POINTER(c_vp)]
    L.vk_device_free.argtypes = [c_vp]
    L.vk_memcpy.argtypes = [c_vp, c_vp, C.c_size_t, c_int]
    L.vk_stream_sync.argtypes = [c_vp]
    L.vk_host_free.argtypes = [c_vp]
    L.vk_host_free.restype = None
    L.vk_graph_create.argtypes = [c_int, c_u64, c_u64, u64p, c_vp, c_vp, c_vp, c_u32, C.POINTER(c_vp)]
    L.vk_graph_load_vcsr.argtypes = [c_int, C.c_char_p, c_u32, C.POINTER(c_vp)]
    L.vk_graph_destroy.argtypes = [c_vp]
    L.vk_graph_info.argtypes = [c_vp, C.POINTER(c_u64), C.POINTER(c_u64), C.POINTER(c_int), C.POINTER(c_int)]
    L.vk_graph_copy_reverse.argtypes = [c_vp, u64p, u32p]
    L.vk_graph_copy_forward.argtypes = [c_vp, u64p, u32p]
    L.vk_graph_apply_reorder.argtypes = [c_vp, u32p, C.POINTER(c_vp)]
    L.vk_initial_probs.argtypes = [c_u64, u8p, u32p, c_u32, c_u64, f64p]
    L.vk_vip_propagate.argtypes = [c_vp, u32p, c_u32, c_u32, f64p, c_vp, f64p]
    L.vk_vip_force_storage.argtypes = [c_int]
    L.vk_vip_propagate_device.argtypes = [c_vp, u32p, c_u32, c_u32, c_vp, c_vp, c_vp, c_vp]
    L.vk_train_members.argtypes = [c_u64, u8p, u32p, c_u32, u32p, C.POINTER(c_u64)]
    L.vk_epoch_shuffle.argtypes = [u32p, c_u64, c_u32, c_u64, c_u64, u32p]
    L.vk_epoch_minibatches.argtypes = [c_u64, u8p, u32p, c_u32, c_u64, c_u64, c_u64, c_vp, u32p,
                                       C.POINTER(c_u64)]
    L.vk_sampler_create.argtypes = [c_vp, C.POINTER(SamplerConfig), C.POINTER(c_vp)]
    L.vk_sampler_destroy.argtypes = [c_vp]
    L.vk_sampler_set_seed_keys.argtypes = [c_vp, c_vp]
    L.vk_sampler_run.argtypes = [c_vp, c_u32, C.POINTER(BatchRef), c_vp, u64p, c_int, c_vp]
    L.vk_sampler_sizes.argtypes = [c_vp, c_vp, c_vp, c_vp]
    L.vk_sampler_copy_frontier.argtypes = [c_vp, c_u32, c_u32, u32p]
    L.vk_sampler_copy_all.argtypes = [c_vp, c_u32, u32p]
    L.vk_sampler_copy_mfg.argtypes = [c_vp, c_u32, c_u32, c_vp, c_vp]
    L.vk_sampler_copy_relabel.argtypes = [c_vp, c_u32, c_u32, u32p]
    L.vk_sampler_get_view.argtypes = [c_vp, C.POINTER(SamplerView)]
    L.vk_sampler_snapshot_counts.argtypes = [c_vp, c_vp, C.POINTER(c_u64), c_vp]
    L.vk_rank_by_scores.argtypes = [c_int, c_u64, u32p, c_u32, f64p, c_u64, u32p, f64p, C.POINTER(c_u64)]
    L.vk_cache_capacity.argtypes = [c_double, c_u64, c_u32, C.POINTER(c_u64)]
    L.vk_rank_degree.argtypes = [c_vp, u8p, u32p, c_u32, c_u32, c_u32, u32p, f64p, C.POINTER(c_u64)]
    L.vk_rank_halo_1hop.argtypes = [c_vp, u32p, c_u32, c_u32, u32p, f64p, C.POINTER(c_u64),
                                    C.POINTER(c_double)]
    L.vk_rank_wpr.argtypes = [c_vp, u8p, u32p, c_u32, c_u32, c_u32, c_u32, c_double, u32p, f64p,
                              C.POINTER(c_u64)]
    L.vk_rank_numpaths.argtypes = [c_vp, u8p, u32p, c_u32, c_u32, c_u32, u32p, f64p, C.POINTER(c_u64)]
    L.vk_build_reorder.argtypes = [c_int, c_u64, c_u32, u32p, f64p, u32p, u64p]
    L.vk_plane_create.argtypes = [c_int, c_u64, c_u32, c_u32, c_int, u32p, u32p, u64p, C.POINTER(c_vp)]
    L.vk_plane_destroy.argtypes = [c_vp]
    L.vk_plane_load_partition.argtypes = [c_vp, c_u32, c_vp, c_u64, c_vp, c_u64]
    L.vk_plane_is_cached.argtypes = [c_vp, c_u32, c_u32, C.POINTER(c_int)]
    L.vk_plane_export.argtypes = [c_vp, c_u32, c_vp, C.POINTER(c_u64)]
    L.vk_plane_attach.argtypes = [c_vp, c_u32, c_vp, c_u64]
    L.vk_plane_gather.argtypes = [c_vp, c_vp, c_vp, c_u64, c_vp, c_vp]
    L.vk_plane_row_bytes.argtypes = [c_vp, C.POINTER(c_u64)]
    L.vk_plane_pulled_rows.argtypes = [c_vp, C.POINTER(c_u64)]
    L.vk_plane_prefetch.argtypes = [c_vp, c_vp]
    L.vk_plane_prefetch_after.argtypes = [c_vp, c_vp, c_vp]
    L.vk_simulate.argtypes = [c_vp, u8p, u32p, c_u32, u32p, c_u32, c_u64, c_u64, c_u64, c_vp, c_vp, u64p,
                              c_vp, c_u32, c_u32, u64p]
    L.vk_empirical_vip.argtypes = [c_vp, u8p, u32p, c_u32, c_u32, c_u64, u32p, c_u32, c_u64, c_u64, f64p]
    L.vk_access_counts.argtypes = [c_vp, u8p, u32p, c_u32, u32p, c_u32, c_u64, c_u64, c_u64, f64p]
    L.vk_synth_community_powerlaw_skew.argtypes = [c_u64, c_u64, c_u32, c_double, c_double, c_u64, C.c_uint,
                                                   C.POINTER(c_vp), C.POINTER(c_vp), C.POINTER(c_u64), u32p]
    L.vk_synth_community_powerlaw.argtypes = [c_u64, c_u64, c_u32, c_double, c_u64, C.c_uint,
                                              C.POINTER(c_vp), C.POINTER(c_vp), C.POINTER(c_u64), u32p]
    L.vk_debug_stream_draws.argtypes = [c_int, c_u64, c_u64, c_u64, u64p]
    L.vk_synth_roles.argtypes = [c_u64, c_double, c_double, c_double, c_u64, u8p]
    L.vk_graph_sample_neighbors.argtypes = [c_vp, c_u32, c_u32, C.POINTER(c_u64), c_vp, u32p, C.POINTER(c_u64)]
    L.vk_simulate_batches.argtypes = [c_vp, u8p, u32p, c_u32, u32p, c_u32, c_u64, c_u64, c_u64, c_vp, c_vp, u64p,
                                      c_vp, c_vp, c_double, u64p, c_vp, c_u64, C.POINTER(c_u64)]
    L.vk_partition_from_file.argtypes = [C.c_char_p, c_u32, c_u64, u32p, C.POINTER(c_u32)]
    L.vk_write_partition_labels.argtypes = [C.c_char_p, u32p, c_u64]
    L.vk_load_roles.argtypes = [C.c_char_p, C.POINTER(c_vp), C.POINTER(c_u64)]
    L.vk_write_roles.argtypes = [C.c_char_p, u8p, c_u64]
    L.vk_write_vip_binary.argtypes = [C.c_char_p, f64p, c_u64]
    L.vk_load_vip_binary.argtypes = [C.c_char_p, C.POINTER(c_vp), C.POINTER(c_u64)]
    L.vk_write_vcsr.argtypes = [C.c_char_p, c_u64, c_u64, u64p, u32p]
    _lib = L
    return L


def check(rc: int):
    if rc != 0:
        msg = lib().vk_last_error().decode(errors="replace")
        raise _BY_CODE.get(rc, VipkitError)(f"{lib().vk_status_name(rc).decode()}: {msg}")


def device_count() -> int:
    c = c_int()
    check(lib().vk_device_count(C.byref(c)))
    return c.value


def stream_draws(key, bound, count, device=0) -> np.ndarray:
    """RngStream draws computed on the device (conformance testing)."""
    out = np.zeros(count, np.uint64)
    check(lib().vk_debug_stream_draws(device, key, bound, count, out))
    return out


def launch_count() -> int:
    return int(lib().vk_launch_count())


def _a32(x):
    return np.ascontiguousarray(x, dtype=np.uint32)


def _a64(x):
    return np.ascontiguousarray(x, dtype=np.uint64)


# ------------------------------------------------------------------- graph
class Graph:
    """Device-resident vipkit::Graph (graph.hpp:20-46)."""

    UNDIRECTED, VALIDATE = 1, 2

    def __init__(self, handle, device):
        self._h = c_vp(handle) if not isinstance(handle, c_vp) else handle
        self.device = device
        n, m, sym, dev = c_u64(), c_u64(), c_int(), c_int()
        check(lib().vk_graph_info(self._h, C.byref(n), C.byref(m), C.byref(sym), C.byref(dev)))
        self.n, self.m, self.symmetric = n.value, m.value, bool(sym.value)
        self._samplers = {}

    @classmethod
    def from_csr(cls, offsets, targets, rev_offsets=None, rev_targets=None, undirected=False,
                 validate=False, device=0):
        off = _a64(offsets)
        tgt = _a32(targets)
        n = len(off) - 1
        flags = (cls.UNDIRECTED if undirected else 0) | (cls.VALIDATE if validate else 0)
        roff = None if rev_offsets is None else _a64(rev_offsets)
        rtgt = None if rev_targets is None else _a32(rev_targets)
        h = c_vp()
        check(lib().vk_graph_create(device, n, len(tgt), off, tgt.ctypes.data,
                                    None if roff is None else roff.ctypes.data,
                                    None if rtgt is None else rtgt.ctypes.data, flags, C.byref(h)))
        return cls(h, device)

    @classmethod
    def load_vcsr(cls, path, device=0):
        """load_binary_csr (graph.hpp:117)."""
        h = c_vp()
        check(lib().vk_graph_load_vcsr(device, os.fsencode(path), 0, C.byref(h)))
        return cls(h, device)

    def forward(self):
        off = np.zeros(self.n + 1, np.uint64)
        tgt = np.zeros(self.m, np.uint32)
        check(lib().vk_graph_copy_forward(self._h, off, tgt))
        return off, tgt

    def reverse(self):
        roff = np.zeros(self.n + 1, np.uint64)
        rtgt = np.zeros(self.m, np.uint32)
        check(lib().vk_graph_copy_reverse(self._h, roff, rtgt))
        return roff, rtgt

    @property
    def handle(self):
        return self._h

    def close(self):
        for s in self._samplers.values():
            s.close()
        self._samplers.clear()
        if self._h:
            lib().vk_graph_destroy(self._h)
            self._h = c_vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --------------------------------------------------------------------- VIP
@dataclass
class VipScores:
    """vipkit::VipScores (vip.hpp:31-36)."""
    partition: int
    p0: np.ndarray
    hop: np.ndarray     # [L, n]
    total: np.ndarray   # [n]


@dataclass
class FanoutSpec:
    """vipkit::FanoutSpec (sampling.hpp:14-21)."""
    fanouts: list

    def hops(self):
        return len(self.fanouts)

    def validate(self):
        if not self.fanouts:
            raise ParameterError("fanout list must have at least one hop")
        if any(f < 1 for f in self.fanouts):
            raise ParameterError("each fanout must be >= 1")

    def label(self):
        return "-".join(str(f) for f in self.fanouts)

    @staticmethod
    def parse(s: str) -> "FanoutSpec":
        out = []
        for tok in s.replace("-", ",").split(","):
            if not tok.isdigit():
                raise ParameterError(f"bad fanout list: {s}")
            out.append(int(tok))
        spec = FanoutSpec(out)
        spec.validate()
        return spec


def initial_probs(roles, part_of, k, b) -> np.ndarray:
    """vipkit::initial_probs (vip.hpp:39-40)."""
    roles = np.ascontiguousarray(roles, np.uint8)
    out = np.zeros(len(roles), np.float64)
    check(lib().vk_initial_probs(len(roles), roles, _a32(part_of), k, b, out))
    return out


def _fan(fanouts):
    f = fanouts.fanouts if isinstance(fanouts, FanoutSpec) else list(fanouts)
    return _a32(f)


def propagate(g: Graph, fanouts, p0, partition: int = 0, with_hops: bool = True):
    """vipkit::propagate (vip.hpp:45-46). p0 may be [n] or [ncols, n] (one
    pass serves every column). Returns VipScores (or a list for 2-D p0)."""
    f = _fan(fanouts)
    p = np.ascontiguousarray(p0, np.float64)
    cols = p.reshape(-1, p.shape[-1]) if p.ndim > 1 else p.reshape(1, -1)
    if cols.shape[1] != g.n:
        raise ShapeError("p0 length does not match vertex count")
    nc = cols.shape[0]
    hop = np.zeros((nc, len(f), g.n), np.float64) if with_hops else None
    total = np.zeros((nc, g.n), np.float64)
    check(lib().vk_vip_propagate(g.handle, f, len(f), nc, np.ascontiguousarray(cols),
                                 None if hop is None else hop.ctypes.data, total))
    res = [VipScores(partition + c if p.ndim > 1 else partition, cols[c],
                     None if hop is None else hop[c], total[c]) for c in range(nc)]
    return res if p.ndim > 1 else res[0]


def vip_force_storage(bits):
    """vk_vip_force_storage: 0 automatic, 32 / 64 force the hoisted-term width."""
    check(lib().vk_vip_force_storage(bits))


def propagate_device(g: Graph, fanouts, ncols, p0_ptr, hop_ptr, total_ptr, stream=0):
    """Device-buffer propagate (pointers are device addresses, e.g. torch data_ptr())."""
    f = _fan(fanouts)
    check(lib().vk_vip_propagate_device(g.handle, f, len(f), ncols, p0_ptr, hop_ptr, total_ptr,
                                        stream or None))


# ---------------------------------------------------------------- sampling
def epoch_permutation(roles, part_of, k, b, epoch, seed, seed_keys=None) -> np.ndarray:
    roles = np.ascontiguousarray(roles, np.uint8)
    out = np.zeros(len(roles), np.uint32)
    cnt = c_u64()
    sk = None if seed_keys is None else _a32(seed_keys)
    check(lib().vk_epoch_minibatches(len(roles), roles, _a32(part_of), k, b, epoch, seed,
                                     None if sk is None else sk.ctypes.data, out, C.byref(cnt)))
    return out[:cnt.value]


def train_members(roles, part_of, k) -> np.ndarray:
    """PartitionMap::train_members (graph.hpp:68): partition k's train ids, ascending."""
    roles = np.ascontiguousarray(roles, np.uint8)
    out = np.zeros(len(roles), np.uint32)
    cnt = c_u64()
    check(lib().vk_train_members(len(roles), roles, _a32(part_of), k, out, C.byref(cnt)))
    return out[:cnt.value].copy()


def epoch_shuffle(train, k, epoch, seed) -> np.ndarray:
    """epoch_minibatches' permutation from a precomputed train list."""
    train = _a32(train)
    out = np.empty_like(train)
    check(lib().vk_epoch_shuffle(train, len(train), k, epoch, seed, out))
    return out


def epoch_minibatches(roles, part_of, k, b, epoch, seed, seed_keys=None):
    """vipkit::epoch_minibatches (sampling.hpp:43-47)."""
    perm = epoch_permutation(roles, part_of, k, b, epoch, seed, seed_keys)
    return [perm[i:i + b] for i in range(0, len(perm), b)]


@dataclass
class ExpandedNeighborhood:
    """vipkit::ExpandedNeighborhood (sampling.hpp:26-30) + the MFG."""
    batch: np.ndarray
    frontier: list = field(default_factory=list)
    all_vertices: np.ndarray = None
    mfg_indptr: list = field(default_factory=list)   # per hop, u64 [|F_{h-1}|+1]
    mfg_dst: list = field(default_factory=list)      # per hop, index into F_h
    all_index: list = field(default_factory=list)    # per h = 0..L, index into all_vertices


class Sampler:
    """Batched device sampler: one run = expand() of a wave of minibatches."""

    FRONTIERS = {"auto": 0, "dense": 1, "sparse": 2}  # VK_SAMPLER_FORCE_*

    def __init__(self, g: Graph, fanouts, batch_size, max_minibatches=1, seed=0, frontier="auto"):
        self.g = g
        f = _fan(fanouts)
        cfg = SamplerConfig()
        cfg.flags = self.FRONTIERS[frontier]
        cfg.num_hops = len(f)
        for i, x in enumerate(f[:MAX_HOPS]):
            cfg.fanouts[i] = int(x)
        cfg.batch_size = batch_size
        cfg.max_minibatches = max_minibatches
        cfg.global_seed = seed
        self.cfg = cfg
        self.L = len(f)
        h = c_vp()
        check(lib().vk_sampler_create(g.handle, C.byref(cfg), C.byref(h)))
        self._h = h
        self.nmb = 0
        self._keys = None

    def set_seed_keys(self, seed_keys):
        """seed_keys replay (vk_sampler_set_seed_keys); None turns it off."""
        if seed_keys is None:
            if self._keys is not None:
                check(lib().vk_sampler_set_seed_keys(self._h, None))
                self._keys = None
            return
        sk = _a32(seed_keys)
        if len(sk) != self.g.n:
            raise ShapeError("seed_keys length does not match vertex count")
        if self._keys is not None and np.array_equal(self._keys, sk):
            return
        check(lib().vk_sampler_set_seed_keys(self._h, sk.ctypes.data))
        self._keys = sk.copy()

    @property
    def handle(self):
        return self._h

    def run(self, batches: Sequence, refs: Sequence[tuple], stream=0, seeds_device_ptr=None):
        """batches: list of id arrays (host) -- or, with seeds_device_ptr, a
        u64 offsets array describing the device seed buffer."""
        nmb = len(refs)
        r = (BatchRef * nmb)()
        for i, (e, k, b) in enumerate(refs):
            r[i].epoch, r[i].partition, r[i].batch_index = e, k, b
        if seeds_device_ptr is None:
            offs = np.zeros(nmb + 1, np.uint64)
            offs[1:] = np.cumsum([len(b) for b in batches])
            cat = _a32(np.concatenate([np.asarray(b, np.uint32) for b in batches]))
            self._keep = cat
            check(lib().vk_sampler_run(self._h, nmb, r, cat.ctypes.data, offs, 0, stream or None))
        else:
            offs = _a64(batches)
            check(lib().vk_sampler_run(self._h, nmb, r, seeds_device_ptr, offs, 1, stream or None))
        self.nmb = nmb

    def sizes(self):
        fs = np.zeros(self.nmb * self.L, np.uint64)
        ec = np.zeros(self.nmb * self.L, np.uint64)
        al = np.zeros(self.nmb, np.uint64)
        check(lib().vk_sampler_sizes(self._h, fs.ctypes.data, ec.ctypes.data, al.ctypes.data))
        return fs.reshape(self.nmb, self.L), ec.reshape(self.nmb, self.L), al

    def result(self, mb: int) -> ExpandedNeighborhood:
        """Host copy of minibatch `mb` of the last run."""
        fs, ec, al = self.sizes()
        L = self.L
        nb = self._batch_len(mb)
        b0 = np.zeros(nb, np.uint32)
        check(lib().vk_sampler_copy_frontier(self._h, mb, 0, b0))
        out = ExpandedNeighborhood(batch=b0)
        for h in range(1, L + 1):
            fr = np.zeros(int(fs[mb, h - 1]), np.uint32)
            check(lib().vk_sampler_copy_frontier(self._h, mb, h, fr))
            out.frontier.append(fr)
        a = np.zeros(int(al[mb]), np.uint32)
        check(lib().vk_sampler_copy_all(self._h, mb, a))
        out.all_vertices = a
        for h in range(1, L + 1):
            nsrc = nb if h == 1 else int(fs[mb, h - 2])
            ip = np.zeros(nsrc + 1, np.uint64)
            dst = np.zeros(int(ec[mb, h - 1]), np.uint32)
            check(lib().vk_sampler_copy_mfg(self._h, mb, h, ip.ctypes.data, dst.ctypes.data))
            out.mfg_indptr.append(ip)
            out.mfg_dst.append(dst)
        for h in range(0, L + 1):
            cnt = nb if h == 0 else int(fs[mb, h - 1])
            ai = np.zeros(cnt, np.uint32)
            check(lib().vk_sampler_copy_relabel(self._h, mb, h, ai))
            out.all_index.append(ai)
        return out

    def _batch_len(self, mb):
        v = self.view()
        cnt = np.zeros(1, np.uint32)
        check(lib().vk_memcpy(cnt.ctypes.data, v.frontier_count[0] + 4 * mb, 4, 2))
        return int(cnt[0])

    def count_words(self) -> int:
        w = c_u64()
        check(lib().vk_sampler_snapshot_counts(self._h, None, C.byref(w), None))
        return w.value

    def snapshot_counts(self, dst_ptr, stream=0):
        check(lib().vk_sampler_snapshot_counts(self._h, dst_ptr, None, stream or None))

    def view(self) -> SamplerView:
        v = SamplerView()
        check(lib().vk_sampler_get_view(self._h, C.byref(v)))
        return v

    def close(self):
        if self._h:
            lib().vk_sampler_destroy(self._h)
            self._h = c_vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def expand(g: Graph, batch, fanouts, seeds, ref=(0, 0, 0), seed_keys=None) -> ExpandedNeighborhood:
    """vipkit::expand (sampling.hpp:62-64) for one minibatch. `seeds` is the
    SeedSpec global seed; `ref` = (epoch, partition, batch_index);
    `seed_keys` replays another labelling's streams (sampling.hpp:46-56)."""
    f = tuple(int(x) for x in _fan(fanouts))
    if len(f) == 0:
        raise ParameterError("fanout list must have at least one hop")
    if any(x < 1 for x in f):
        raise ParameterError("each fanout must be >= 1")
    b = _a32(batch)
    if len(b) == 0:
        raise SamplingError("cannot expand an empty batch")
    key = (f, int(seeds))
    s = g._samplers.get(key)
    if s is None or s.cfg.batch_size < len(b):
        if s is not None:
            s.close()
        s = Sampler(g, f, max(len(b), 1024), 1, seeds)
        g._samplers[key] = s
    s.set_seed_keys(seed_keys)
    s.run([b], [ref])
    return s.result(0)


# ---------------------------------------------------------- cache / store
def rank_by_scores(part_of, k, scores, device=0):
    """vipkit::rank_by_scores (policies.hpp:48) -> (order, score)."""
    part_of = _a32(part_of)
    scores = np.ascontiguousarray(scores, np.float64)
    n = len(part_of)
    order = np.zeros(n, np.uint32)
    sc = np.zeros(n, np.float64)
    cnt = c_u64()
    check(lib().vk_rank_by_scores(device, n, part_of, k, scores, len(scores), order, sc, C.byref(cnt)))
    return order[:cnt.value], sc[:cnt.value]


def _ranked(fn, g, *args):
    order = np.zeros(g.n, np.uint32)
    sc = np.zeros(g.n, np.float64)
    cnt = c_u64()
    fn(*args, order, sc, C.byref(cnt))
    return order[:cnt.value], sc[:cnt.value]


def rank_degree(g: Graph, roles, part_of, K, k, L):
    """vipkit::rank_degree (policies.hpp:28-29) -> (order, score)."""
    return _ranked(lambda *a: check(lib().vk_rank_degree(g.handle, np.ascontiguousarray(roles, np.uint8),
                                                         _a32(part_of), K, k, L, *a)), g)


def rank_halo_1hop(g: Graph, part_of, K, k):
    """vipkit::rank_halo_1hop (policies.hpp:32) -> (order, score, effective_alpha)."""
    ea = c_double()
    o, sc = _ranked(lambda *a: check(lib().vk_rank_halo_1hop(g.handle, _a32(part_of), K, k, *a, C.byref(ea))), g)
    return o, sc, ea.value


def rank_wpr(g: Graph, roles, part_of, K, k, hop1_fanout, iters=5, damping=0.85):
    """vipkit::rank_wpr (policies.hpp:38-40), TransitionModel of fanout
    hop1_fanout at hop 1 -> (order, score)."""
    return _ranked(lambda *a: check(lib().vk_rank_wpr(g.handle, np.ascontiguousarray(roles, np.uint8),
                                                      _a32(part_of), K, k, hop1_fanout, iters, damping, *a)), g)


def rank_numpaths(g: Graph, roles, part_of, K, k, L):
    """vipkit::rank_numpaths (policies.hpp:44-45) -> (order, score)."""
    return _ranked(lambda *a: check(lib().vk_rank_numpaths(g.handle, np.ascontiguousarray(roles, np.uint8),
                                                           _a32(part_of), K, k, L, *a)), g)


def cache_capacity(alpha, n, K) -> int:
    cap = c_u64()
    check(lib().vk_cache_capacity(alpha, n, K, C.byref(cap)))
    return cap.value


@dataclass
class CachePlan:
    """vipkit::CachePlan (policies.hpp:52-62)."""
    K: int
    alpha: float
    cached: list
    member_bits: np.ndarray

    def is_cached(self, k, v) -> bool:
        return bool((int(self.member_bits[k][v >> 6]) >> (v & 63)) & 1)


def build_cache(rankings: Sequence, alpha: float, n: int) -> CachePlan:
    """vipkit::build_cache (policies.hpp:64): prefix of each ranking's order."""
    K = len(rankings)
    if K == 0:
        raise ParameterError("need at least one ranking")
    cap = cache_capacity(alpha, n, K)
    cached = [np.asarray(r[0] if isinstance(r, tuple) else r, np.uint32)[:cap] for r in rankings]
    W = (n + 63) // 64
    bits = np.zeros((K, W), np.uint64)
    for k, c in enumerate(cached):
        c64 = c.astype(np.uint64)
        np.bitwise_or.at(bits[k], (c64 >> np.uint64(6)).astype(np.int64),
                         np.left_shift(np.uint64(1), c64 & np.uint64(63)))
    return CachePlan(K, alpha, cached, bits)


def simulate(g: Graph, roles, part_of, K, fanouts, b, epochs, seed, cached, takes=None, wave=0,
             seed_keys=None):
    """vipkit::simulate (commsim.hpp:56-59) on the device -> cells[E, K, 3]
    = (local_hits, cache_hits, remote_misses) per (epoch, partition).

    `cached` is each partition's cached id list (CachePlan::cached). With
    `takes` (shape [A, K]) it is read as ranking prefixes and A nested plans
    are scored from one expansion pass -> cells[A, E, K, 3] (the alpha axis
    of sweep, commsim.cpp:140-259)."""
    part_of = _a32(part_of)
    fan = _a32(fanouts)
    offs = np.zeros(K + 1, np.uint64)
    offs[1:] = np.cumsum([len(c) for c in cached])
    ids = _a32(np.concatenate([np.asarray(c, np.uint32) for c in cached]) if K else [])
    A = 1
    tk = None
    if takes is not None:
        tk = np.ascontiguousarray(np.asarray(takes, np.uint64).reshape(-1, K))
        A = tk.shape[0]
    cells = np.zeros(A * epochs * K * 3, np.uint64)
    sk = None if seed_keys is None else _a32(seed_keys)
    check(lib().vk_simulate(g.handle, np.ascontiguousarray(roles, np.uint8), part_of, K, fan, len(fan), b,
                            epochs, seed, None if sk is None else sk.ctypes.data,
                            ids.ctypes.data if ids.size else None, offs,
                            tk.ctypes.data if tk is not None else None, A, wave, cells))
    cells = cells.reshape(A, epochs, K, 3)
    return cells if takes is not None else cells[0]


def simulate_batches(g: Graph, roles, part_of, K, fanouts, b, epochs, seed, cached, seed_keys=None,
                     gpu_orderings=None, gamma=0.0):
    """simulate with SimulateOptions::batch_costs (commsim.cpp:104-118) ->
    (cells[E, K, 3], rows[B, 7]); row = (epoch, batch_index, partition,
    local - gpu, gpu, cache, miss) in for_each_expansion order."""
    part_of = _a32(part_of)
    roles = np.ascontiguousarray(roles, np.uint8)
    fan = _a32(fanouts)
    offs = np.zeros(K + 1, np.uint64)
    offs[1:] = np.cumsum([len(c) for c in cached])
    ids = _a32(np.concatenate([np.asarray(c, np.uint32) for c in cached]) if K else [])
    total = epochs * sum((len(train_members(roles, part_of, k)) + b - 1) // b for k in range(K))
    rows = np.zeros(max(1, total) * 7, np.uint64)
    cells = np.zeros(epochs * K * 3, np.uint64)
    sk = None if seed_keys is None else _a32(seed_keys)
    keep, ptrs, sizes = [], None, None
    if gpu_orderings is not None:
        keep = [_a32(o) for o in gpu_orderings]
        ptrs = (c_vp * K)(*[o.ctypes.data for o in keep])
        sizes = np.array([len(o) for o in keep], np.uint64)
    got = c_u64()
    check(lib().vk_simulate_batches(g.handle, roles, part_of, K, fan, len(fan), b, epochs, seed,
                                    None if sk is None else sk.ctypes.data, ids.ctypes.data if ids.size else None,
                                    offs, ptrs, None if sizes is None else sizes.ctypes.data, gamma, cells,
                                    rows.ctypes.data, total, C.byref(got)))
    return cells.reshape(epochs, K, 3), rows[:got.value * 7].reshape(-1, 7)


def sample_neighbors(g: Graph, v, fanout, stream_state, seed_keys=None, offsets=None, targets=None):
    """vipkit::sample_neighbors (sampling.hpp:54-56) on the device ->
    (ids, advanced stream state). stream_state is RngStream's counter
    (mix64(key) for a fresh stream). With seed_keys, the keys of v's
    neighbours are marshalled from the host CSR (offsets, targets)."""
    out = np.zeros(max(1, fanout), np.uint32)
    cnt, st = c_u64(), c_u64(stream_state)
    keys = None
    if seed_keys is not None:
        if offsets is None:
            offsets, targets = g.forward()
        keys = _a32(np.asarray(seed_keys, np.uint32)[targets[int(offsets[v]):int(offsets[v + 1])]])
    check(lib().vk_graph_sample_neighbors(g.handle, v, fanout, C.byref(st), None if keys is None else keys.ctypes.data,
                                          out, C.byref(cnt)))
    return out[:cnt.value].copy(), st.value


# ------------------------------------------------------------ file formats
def partition_from_file(path, K, n):
    """partition_from_file (graph.hpp:105) -> (part_of, K)."""
    out = np.zeros(n, np.uint32)
    k_out = c_u32()
    check(lib().vk_partition_from_file(os.fsencode(path), K, n, out, C.byref(k_out)))
    return out, k_out.value


def write_partition_labels(part_of, path):
    p = _a32(part_of)
    check(lib().vk_write_partition_labels(os.fsencode(path), p, len(p)))


def load_roles(path):
    """load_roles (graph.hpp:119) -> u8 codes."""
    ptr, n = c_vp(), c_u64()
    check(lib().vk_load_roles(os.fsencode(path), C.byref(ptr), C.byref(n)))
    out = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint8)), shape=(max(1, n.value),))[:n.value].copy()
    lib().vk_host_free(ptr)
    return out


def write_roles(roles, path):
    r = np.ascontiguousarray(roles, np.uint8)
    check(lib().vk_write_roles(os.fsencode(path), r, len(r)))


def write_vip_binary(total, path):
    """write_vip_binary (vip.hpp:58): n little-endian f64 totals."""
    t = np.ascontiguousarray(total, np.float64)
    check(lib().vk_write_vip_binary(os.fsencode(path), t, len(t)))


def load_vip_binary(path):
    ptr, n = c_vp(), c_u64()
    check(lib().vk_load_vip_binary(os.fsencode(path), C.byref(ptr), C.byref(n)))
    out = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_double)), shape=(max(1, n.value),))[:n.value].copy()
    lib().vk_host_free(ptr)
    return out


def write_binary_csr(offsets, targets, path):
    """write_binary_csr (graph.hpp:116): the VCSR file Graph.load_vcsr reads."""
    off, tgt = _a64(offsets), _a32(targets)
    check(lib().vk_write_vcsr(os.fsencode(path), len(off) - 1, len(tgt), off, tgt))


def access_counts(g: Graph, roles, part_of, K, fanouts, b, epochs, seed):
    """The oracle policy's access counts (commsim.cpp:155-166) -> [K, n] f64."""
    part_of = _a32(part_of)
    fan = _a32(fanouts)
    out = np.zeros(K * len(part_of), np.float64)
    check(lib().vk_access_counts(g.handle, np.ascontiguousarray(roles, np.uint8), part_of, K, fan, len(fan), b,
                                 epochs, seed, out))
    return out.reshape(K, -1)


def empirical_vip(g: Graph, roles, part_of, K, k, b, fanouts, S, seed):
    """vipkit::empirical_vip (vip.hpp:52-55) on the device -> freq[n] (f64)."""
    part_of = _a32(part_of)
    fan = _a32(fanouts)
    out = np.zeros(len(part_of), np.float64)
    check(lib().vk_empirical_vip(g.handle, np.ascontiguousarray(roles, np.uint8), part_of, K, k, b, fan,
                                 len(fan), S, seed, out))
    return out


def apply_reorder(g: Graph, roles, part_of, old_of_new):
    """vipkit::apply_reorder (reorder.hpp:34-35) -> (Graph, roles, part_of):
    the relabelled graph is built on the device; roles/labels permute."""
    oon = _a32(old_of_new)
    if len(oon) != g.n:
        raise ShapeError("reorder map size does not match vertex count")  # reorder.cpp:39
    h = c_vp()
    check(lib().vk_graph_apply_reorder(g.handle, oon, C.byref(h)))
    ng = Graph(h, g.device)
    return ng, np.ascontiguousarray(roles, np.uint8)[oon], _a32(part_of)[oon]


def build_reorder(part_of, K, scores, device=0):
    """vipkit::build_reorder (reorder.hpp:25-26) -> (old_of_new, ranges[K,2])."""
    part_of = _a32(part_of)
    n = len(part_of)
    s = np.ascontiguousarray(np.asarray(scores, np.float64).reshape(K, n))
    oon = np.zeros(n, np.uint32)
    ranges = np.zeros(2 * K, np.uint64)
    check(lib().vk_build_reorder(device, n, K, part_of, s, oon, ranges))
    return oon, ranges.reshape(K, 2)


class FeaturePlane:
    """VIP-ordered feature store (north-star (3)), one per device."""

    def __init__(self, n, K, dim, part_of, old_of_new, ranges, dtype=F32, device=0):
        h = c_vp()
        self.part_of = _a32(part_of)
        check(lib().vk_plane_create(device, n, K, dim, dtype, self.part_of, _a32(old_of_new),
                                    _a64(np.asarray(ranges).reshape(-1)), C.byref(h)))
        self._h = h
        self.n, self.K, self.dim, self.dtype, self.device = n, K, dim, dtype, device
        rb = c_u64()
        check(lib().vk_plane_row_bytes(h, C.byref(rb)))
        self.row_bytes = rb.value

    @property
    def handle(self):
        return self._h

    def load_partition(self, k, cache_ids, features=None, feature_seed=0):
        c = _a32(cache_ids)
        f = None
        if features is not None:
            f = np.ascontiguousarray(features)
        check(lib().vk_plane_load_partition(self._h, k, c.ctypes.data if len(c) else None, len(c),
                                            None if f is None else f.ctypes.data, feature_seed))

    def is_cached(self, k, v) -> bool:
        out = c_int()
        check(lib().vk_plane_is_cached(self._h, k, v, C.byref(out)))
        return bool(out.value)

    def export(self, k):
        buf = (C.c_char * 64)()
        rows = c_u64()
        check(lib().vk_plane_export(self._h, k, buf, C.byref(rows)))
        return bytes(buf), rows.value

    def attach(self, k, handle: bytes, rows: int):
        buf = (C.c_char * 64).from_buffer_copy(handle)
        check(lib().vk_plane_attach(self._h, k, buf, rows))

    def gather(self, sampler: Sampler, out_ptr, out_stride_rows, counts_ptr, stream=0):
        check(lib().vk_plane_gather(self._h, sampler.handle, out_ptr, out_stride_rows, counts_ptr,
                                    stream or None))

    def prefetch(self, sampler: Sampler):
        """Issue the multi-GPU miss exchange of the sampler's last run now
        (vk_plane_prefetch); no-op on a single GPU."""
        check(lib().vk_plane_prefetch(self._h, sampler.handle))

    def prefetch_after(self, sampler: Sampler, stream):
        """vk_plane_prefetch_after: the exchange also waits for the work
        queued so far on `stream` (a cudaStream_t)."""
        check(lib().vk_plane_prefetch_after(self._h, sampler.handle, stream))

    def pulled_rows(self) -> int:
        """Distinct remote rows pulled over NVLink by the last gather."""
        r = c_u64()
        check(lib().vk_plane_pulled_rows(self._h, C.byref(r)))
        return r.value

    def close(self):
        if self._h:
            lib().vk_plane_destroy(self._h)
            self._h = c_vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --------------------------------------------------------- synthetic data
def synth_community_powerlaw(n, d, communities, p_in=0.8, seed=7, threads=0, skew=2.0):
    """Community-structured power-law graph -> (offsets u64, targets u32, labels u32)."""
    po, pt, m = c_vp(), c_vp(), c_u64()
    labels = np.zeros(n, np.uint32)
    check(lib().vk_synth_community_powerlaw_skew(n, d, communities, p_in, skew, seed, threads, C.byref(po),
                                                 C.byref(pt), C.byref(m), labels))
    try:
        off = np.ctypeslib.as_array(C.cast(po, C.POINTER(c_u64)), shape=(n + 1,)).copy()
        tgt = (np.ctypeslib.as_array(C.cast(pt, C.POINTER(C.c_uint32)), shape=(m.value,)).copy()
               if m.value else np.zeros(0, np.uint32))
    finally:
        lib().vk_host_free(po)
        lib().vk_host_free(pt)
    return off, tgt, labels


def synth_roles(n, train, valid=0.0, test=0.0, seed=3):
    """vipkit::make_roles (graph.hpp:93-94)."""
    out = np.zeros(n, np.uint8)
    check(lib().vk_synth_roles(n, train, valid, test, seed, out))
    return out
