"""TEST INFRASTRUCTURE ONLY (see oracle/README.md).

ctypes bindings for the two CPU checkers with one Python surface:

* ``Port`` — ``_build/libvipkit_port.so``, the plain-C restatement
  (``vipkit_port.c``), always available after ``make -C oracle``.
* ``Ref``  — ``_ref/libvipkit_ref.so``, the UNMODIFIED reference library
  (``/root/reference/proj/src``) behind ``ref_shim.cpp``. Present wherever it
  was built (it travels to the GPU box as a build product).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libvipkit_port.so")
REF_SO = os.path.join(HERE, "_ref", "libvipkit_ref.so")

KINDS = {"path": 0, "star": 1, "tree": 2, "grid": 3, "pa": 4, "uniform": 5}
PARTITION_METHODS = {"random": 0, "bfs_greedy": 1}

u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
c_u64, c_u32, c_int, c_double, c_vp = C.c_uint64, C.c_uint32, C.c_int, C.c_double, C.c_void_p

ERROR_NAMES = {1: "parse_error", 2: "range_error", 3: "parameter_error", 4: "format_error",
               5: "partition_error", 6: "sampling_error", 7: "config_error", 8: "shape_error",
               9: "io_error", 23: "error"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERROR_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERROR_NAMES.get(code, "error")


def _a32(x):
    return np.ascontiguousarray(x, dtype=np.uint32)


def _a64(x):
    return np.ascontiguousarray(x, dtype=np.uint64)


@dataclass
class CSR:
    """Host CSR with the reference layout (graph.hpp:20-46)."""
    n: int
    off: np.ndarray            # u64 [n+1]
    tgt: np.ndarray            # u32 [m]
    rev_off: np.ndarray = None  # u64 [n+1]
    rev_tgt: np.ndarray = None  # u32 [m]

    @property
    def m(self) -> int:
        return int(self.tgt.shape[0])

    def ensure_reverse(self):
        if self.rev_off is None:
            self.rev_off, self.rev_tgt = transpose(self.n, self.off, self.tgt)
        return self

    def out_degree(self) -> np.ndarray:
        return np.diff(self.off)


def transpose(n, off, tgt):
    """Reverse CSR by counting transpose (same as graph.cpp:587-595)."""
    m = tgt.shape[0]
    src = np.repeat(np.arange(n, dtype=np.uint32), np.diff(off).astype(np.int64))
    order = np.lexsort((src, tgt))
    rev_tgt = src[order].astype(np.uint32)
    cnt = np.bincount(tgt, minlength=n).astype(np.uint64)
    rev_off = np.zeros(n + 1, dtype=np.uint64)
    np.cumsum(cnt, out=rev_off[1:])
    assert rev_off[-1] == m
    return rev_off, rev_tgt


@dataclass
class Expansion:
    batch: np.ndarray
    frontier: list = field(default_factory=list)
    all_vertices: np.ndarray = None
    indptr: list = field(default_factory=list)
    edges: list = field(default_factory=list)


class Port:
    """The C restatement (vipkit_port.c)."""

    name = "port"

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(path)
        L.vp_last_error.restype = C.c_char_p
        L.vp_mix64.restype = c_u64
        L.vp_mix64.argtypes = [c_u64]
        L.vp_seed_key.restype = c_u64
        L.vp_seed_key.argtypes = [c_u64, u64p, c_u32]
        L.vp_generate.argtypes = [c_int, c_u64, c_u64, c_u64, C.POINTER(c_vp), C.POINTER(c_vp),
                                  C.POINTER(c_u64)]
        L.vp_graph_from_edges.argtypes = [c_u64, u32p, u32p, c_u64, c_int, C.POINTER(c_vp),
                                          C.POINTER(c_vp), C.POINTER(c_u64)]
        L.vp_free.argtypes = [c_vp]
        L.vp_synth_community_powerlaw.argtypes = [c_u64, c_u64, c_u32, c_double, c_u64, C.c_uint,
                                                  C.POINTER(c_vp), C.POINTER(c_vp), C.POINTER(c_u64), c_vp]
        L.vp_synth_community_powerlaw_skew.argtypes = [c_u64, c_u64, c_u32, c_double, c_double, c_u64, C.c_uint,
                                                       C.POINTER(c_vp), C.POINTER(c_vp), C.POINTER(c_u64), c_vp]
        L.vp_fill_features.argtypes = [c_u64, c_u32, c_int, c_u64, c_vp, C.c_uint]
        L.vp_gather_rows.argtypes = [c_vp, c_u64, c_vp, c_u64, c_vp, C.c_uint]
        L.vp_stream_draws.argtypes = [c_u64, c_u64, c_u64, u64p]
        L.vp_make_roles.argtypes = [c_u64, c_double, c_double, c_double, c_u64, u8p]
        L.vp_epoch_minibatches.argtypes = [u8p, c_u64, u32p, c_u32, c_u64, c_u64, c_u64, u32p,
                                           C.POINTER(c_u64)]
        L.vp_expand.restype = c_vp
        L.vp_expand.argtypes = [u64p, u32p, c_u64, u32p, c_u64, u32p, c_u32, c_u64, c_u64, c_u32,
                                c_u64]
        L.vp_expansion_free.argtypes = [c_vp]
        L.vp_initial_probs.argtypes = [u8p, c_u64, u32p, c_u32, c_u64, f64p]
        L.vp_propagate.argtypes = [u64p, u64p, u32p, c_u64, u32p, c_u32, f64p, f64p, f64p]
        L.vp_rank_by_scores.argtypes = [u32p, c_u64, c_u32, f64p, u32p, f64p, C.POINTER(c_u64)]
        L.vp_cache_capacity.argtypes = [c_double, c_u64, c_u32, C.POINTER(c_u64)]
        L.vp_classify.argtypes = [u32p, c_u64, u32p, c_u32, c_vp, u64p]
        L.vp_build_reorder.argtypes = [u32p, c_u64, c_u32, f64p, u32p, u64p]
        L.vp_features.argtypes = [c_u64, c_u32, c_int, u32p, c_u64, c_vp]

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.vp_last_error().decode())

    # ---- rng ----
    def mix64(self, x):
        return self.lib.vp_mix64(x)

    def seed_key(self, seed, parts):
        p = _a64(parts)
        return self.lib.vp_seed_key(seed, p, len(p))

    def stream_draws(self, key, bound, count):
        out = np.zeros(count, np.uint64)
        self.lib.vp_stream_draws(key, bound, count, out)
        return out

    # ---- graph ----
    def _take_csr(self, n, po, pt, m):
        off = np.ctypeslib.as_array(C.cast(po, C.POINTER(c_u64)), shape=(n + 1,)).copy()
        tgt = (np.ctypeslib.as_array(C.cast(pt, C.POINTER(C.c_uint32)), shape=(m,)).copy()
               if m else np.zeros(0, np.uint32))
        self.lib.vp_free(po)
        self.lib.vp_free(pt)
        return CSR(n, off, tgt)

    def generate(self, kind, n, d=2, seed=0) -> CSR:
        po, pt, m = c_vp(), c_vp(), c_u64()
        self._check(self.lib.vp_generate(KINDS[kind], n, d, seed, C.byref(po), C.byref(pt),
                                         C.byref(m)))
        return self._take_csr(n, po, pt, m.value)

    def from_edges(self, n, edges, undirected) -> CSR:
        e = np.asarray(edges, dtype=np.uint32).reshape(-1, 2)
        po, pt, m = c_vp(), c_vp(), c_u64()
        self._check(self.lib.vp_graph_from_edges(n, _a32(e[:, 0]), _a32(e[:, 1]), len(e),
                                                 int(undirected), C.byref(po), C.byref(pt),
                                                 C.byref(m)))
        return self._take_csr(n, po, pt, m.value)

    def make_roles(self, n, train, valid=0.0, test=0.0, seed=0):
        out = np.zeros(n, np.uint8)
        self._check(self.lib.vp_make_roles(n, train, valid, test, seed, out))
        return out

    # ---- sampling ----
    def epoch_permutation(self, roles, labels, k, b, epoch, seed):
        n = len(roles)
        out = np.zeros(n, np.uint32)
        cnt = c_u64()
        self._check(self.lib.vp_epoch_minibatches(np.ascontiguousarray(roles, np.uint8), n,
                                                  _a32(labels), k, b, epoch, seed, out,
                                                  C.byref(cnt)))
        return out[:cnt.value]

    def epoch_minibatches(self, roles, labels, k, b, epoch, seed):
        perm = self.epoch_permutation(roles, labels, k, b, epoch, seed)
        return [perm[i:i + b] for i in range(0, len(perm), b)]

    def expand(self, g: CSR, batch, fanouts, seed, epoch=0, part=0, batch_index=0) -> Expansion:
        class _X(C.Structure):
            _fields_ = [("L", c_u32), ("nb", c_u64), ("batch", C.POINTER(C.c_uint32)),
                        ("fsize", C.POINTER(c_u64)), ("frontier", C.POINTER(C.POINTER(C.c_uint32))),
                        ("indptr", C.POINTER(C.POINTER(c_u64))),
                        ("edges", C.POINTER(C.POINTER(C.c_uint32))), ("nall", c_u64),
                        ("all", C.POINTER(C.c_uint32))]
        b = _a32(batch)
        f = _a32(fanouts)
        p = self.lib.vp_expand(g.off, g.tgt, g.n, b, len(b), f, len(f), seed, epoch, part,
                               batch_index)
        if not p:
            msg = self.lib.vp_last_error().decode()
            raise OracleError(6 if "empty batch" in msg else 3, msg)
        x = C.cast(p, C.POINTER(_X)).contents
        out = Expansion(batch=b.copy())
        prev = len(b)
        for h in range(x.L):
            fs = x.fsize[h]
            out.frontier.append(np.ctypeslib.as_array(x.frontier[h], shape=(fs,)).copy()
                                if fs else np.zeros(0, np.uint32))
            ip = np.ctypeslib.as_array(x.indptr[h], shape=(prev + 1,)).copy()
            out.indptr.append(ip)
            ne = int(ip[-1])
            out.edges.append(np.ctypeslib.as_array(x.edges[h], shape=(ne,)).copy()
                             if ne else np.zeros(0, np.uint32))
            prev = fs
        out.all_vertices = np.ctypeslib.as_array(x.all, shape=(x.nall,)).copy()
        self.lib.vp_expansion_free(p)
        return out

    # ---- vip ----
    def initial_probs(self, roles, labels, K, k, b):
        n = len(roles)
        out = np.zeros(n, np.float64)
        self._check(self.lib.vp_initial_probs(np.ascontiguousarray(roles, np.uint8), n,
                                              _a32(labels), k, b, out))
        return out

    def propagate(self, g: CSR, fanouts, p0):
        g.ensure_reverse()
        f = _a32(fanouts)
        hop = np.zeros((len(f), g.n), np.float64)
        total = np.zeros(g.n, np.float64)
        p0 = np.ascontiguousarray(p0, np.float64)
        if p0.shape[0] != g.n:
            raise OracleError(8, "p0 length does not match vertex count")
        self._check(self.lib.vp_propagate(g.off, g.rev_off, g.rev_tgt, g.n, f, len(f), p0, hop,
                                          total))
        return hop, total

    # ---- policies ----
    def rank_by_scores(self, labels, K, k, scores):
        labels = _a32(labels)
        scores = np.ascontiguousarray(scores, np.float64)
        if scores.shape[0] != labels.shape[0]:
            raise OracleError(8, "score vector length does not match vertex count")
        n = len(labels)
        order = np.zeros(n, np.uint32)
        sc = np.zeros(n, np.float64)
        cnt = c_u64()
        self._check(self.lib.vp_rank_by_scores(labels, n, k, scores, order, sc, C.byref(cnt)))
        return order[:cnt.value], sc[:cnt.value]

    def cache_capacity(self, alpha, n, K):
        cap = c_u64()
        self._check(self.lib.vp_cache_capacity(alpha, n, K, C.byref(cap)))
        return cap.value

    def build_cache(self, orders, alpha, n):
        cap = self.cache_capacity(alpha, n, len(orders))
        cached = [np.asarray(o[:cap], np.uint32) for o in orders]
        return cached, bitsets(cached, n)

    def classify(self, all_vertices, labels, k, bits=None):
        out = np.zeros(3, np.uint64)
        a = _a32(all_vertices)
        bp = None if bits is None else _a64(bits).ctypes.data
        keep = None if bits is None else _a64(bits)
        if keep is not None:
            bp = keep.ctypes.data
        self.lib.vp_classify(a, len(a), _a32(labels), k, bp, out)
        return tuple(int(x) for x in out)

    def build_reorder(self, labels, K, scores):
        labels = _a32(labels)
        n = len(labels)
        s = np.ascontiguousarray(np.asarray(scores, np.float64).reshape(K, n))
        oon = np.zeros(n, np.uint32)
        ranges = np.zeros(2 * K, np.uint64)
        self._check(self.lib.vp_build_reorder(labels, n, K, s, oon, ranges))
        return oon, ranges.reshape(K, 2)

    def features(self, seed, D, ids, fp16=False):
        ids = _a32(ids)
        out = np.zeros((len(ids), D), np.float16 if fp16 else np.float32)
        self.lib.vp_features(seed, D, int(fp16), ids, len(ids), out.ctypes.data)
        return out

    # ---- workload (workload.c) ----
    def synth_community_powerlaw(self, n, d, communities, p_in, seed, threads=0, skew=2.0):
        """The bench graph recipe (restated from the product generator):
        (off u64[n+1], tgt u32[m], labels u32[n])."""
        offp, tgtp, m = c_vp(), c_vp(), c_u64()
        labels = np.zeros(n, np.uint32)
        rc = self.lib.vp_synth_community_powerlaw_skew(n, d, communities, p_in, skew, seed,
                                                       threads or (os.cpu_count() or 1), C.byref(offp),
                                                       C.byref(tgtp), C.byref(m), labels.ctypes.data)
        if rc != 0:
            raise OracleError(rc, "bad generator parameters")
        off = np.ctypeslib.as_array(C.cast(offp, C.POINTER(C.c_uint64)), shape=(n + 1,)).copy()
        self.lib.vp_free(offp)
        if m.value:
            tgt = np.empty(m.value, np.uint32)
            C.memmove(tgt.ctypes.data, tgtp, m.value * 4)
        else:
            tgt = np.zeros(0, np.uint32)
        self.lib.vp_free(tgtp)
        return off, tgt, labels

    def feature_table(self, seed, D, n, fp16=False, threads=0):
        out = np.empty((n, D), np.float16 if fp16 else np.float32)
        self.lib.vp_fill_features(seed, D, int(fp16), n, out.ctypes.data, threads or (os.cpu_count() or 1))
        return out

    def gather_rows(self, table, ids, out=None, threads=0):
        ids = _a32(ids)
        rb = table.shape[1] * table.itemsize
        if out is None:
            out = np.empty((len(ids), table.shape[1]), table.dtype)
        self.lib.vp_gather_rows(table.ctypes.data, rb, ids.ctypes.data, len(ids), out.ctypes.data,
                                threads or (os.cpu_count() or 1))
        return out


def bitsets(cached, n):
    """CachePlan::member_bits layout (policies.hpp:55-60): K x ceil(n/64) u64."""
    W = (n + 63) // 64
    bits = np.zeros((len(cached), W), np.uint64)
    for k, c in enumerate(cached):
        c = np.asarray(c, np.uint64)
        np.bitwise_or.at(bits[k], (c >> np.uint64(6)).astype(np.int64),
                         np.left_shift(np.uint64(1), c & np.uint64(63)))
    return bits


class Ref:
    """The unmodified reference library behind ref_shim.cpp."""

    name = "reference"

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_threads.argtypes = [C.c_uint]
        L.ref_mix64.restype = c_u64
        L.ref_mix64.argtypes = [c_u64]
        L.ref_seed_key.restype = c_u64
        L.ref_seed_key.argtypes = [c_u64, u64p, c_u32]
        L.ref_stream_draws.argtypes = [c_u64, c_u64, c_u64, u64p]
        for fn in ("ref_graph_generate", "ref_graph_from_edges", "ref_graph_from_csr",
                   "ref_graph_load_vcsr", "ref_expand"):
            getattr(L, fn).restype = c_vp
        L.ref_graph_generate.argtypes = [c_int, c_u64, c_u64, c_u64]
        L.ref_graph_from_edges.argtypes = [c_u64, u32p, u32p, c_u64, c_int]
        L.ref_graph_from_csr.argtypes = [c_u64, c_u64, u64p, u32p]
        L.ref_graph_from_symmetric_csr.restype = c_vp
        L.ref_graph_from_symmetric_csr.argtypes = [c_u64, c_u64, u64p, u32p, C.c_uint, c_int]
        L.ref_ctx_create.restype = c_vp
        L.ref_ctx_create.argtypes = [u8p, u32p, c_u64, c_u32]
        L.ref_ctx_free.argtypes = [c_vp]
        L.ref_ctx_epoch.argtypes = [c_vp, c_u32, c_u64, c_u64, c_u64, u32p, C.POINTER(c_u64)]
        L.ref_sample_neighbors_state.argtypes = [c_vp, c_u32, c_u32, c_u64, c_vp, u32p, C.POINTER(c_u64),
                                                 C.POINTER(c_u64)]
        L.ref_write_partition_labels.argtypes = [u32p, c_u64, c_u32, C.c_char_p]
        L.ref_partition_from_file.argtypes = [C.c_char_p, c_u32, c_u64, u32p, C.POINTER(c_u32)]
        L.ref_write_roles.argtypes = [u8p, c_u64, C.c_char_p]
        L.ref_load_roles.argtypes = [C.c_char_p, u8p, c_u64, C.POINTER(c_u64)]
        L.ref_write_vip_binary.argtypes = [f64p, c_u64, C.c_char_p]
        L.ref_load_vip_binary.argtypes = [C.c_char_p, f64p, c_u64, C.POINTER(c_u64)]
        L.ref_simulate_streams.argtypes = [c_vp, u8p, u32p, c_u32, u32p, c_u32, c_u64, c_u64, c_u64, u32p, u64p,
                                           C.c_char_p, C.c_char_p, c_vp, c_vp, c_double, u64p]
        L.ref_bench_minibatches.argtypes = [c_vp, c_u32, u32p, u64p, u64p, u32p, c_u32, c_u64, u32p, c_vp,
                                            c_u64, c_vp, c_u64, c_vp, c_u64, C.c_uint, u64p]
        L.ref_graph_load_vcsr.argtypes = [C.c_char_p]
        L.ref_graph_write_vcsr.argtypes = [c_vp, C.c_char_p]
        L.ref_graph_n.restype = c_u64
        L.ref_graph_n.argtypes = [c_vp]
        L.ref_graph_m.restype = c_u64
        L.ref_graph_m.argtypes = [c_vp]
        L.ref_graph_copy.argtypes = [c_vp, c_vp, c_vp, c_vp, c_vp]
        L.ref_graph_free.argtypes = [c_vp]
        L.ref_make_roles.argtypes = [c_u64, c_double, c_double, c_double, c_u64, u8p]
        L.ref_partition_graph.argtypes = [c_vp, u8p, c_u64, c_u32, c_int, c_u64, u32p]
        L.ref_epoch_minibatches.argtypes = [u8p, c_u64, u32p, c_u32, c_u32, c_u64, c_u64, c_u64,
                                            c_vp, u32p, C.POINTER(c_u64)]
        L.ref_expand.argtypes = [c_vp, u32p, c_u64, u32p, c_u32, c_u64, c_u64, c_u32, c_u64, c_int, c_vp]
        for fn in ("ref_exp_frontier_size", "ref_exp_edges_size"):
            getattr(L, fn).restype = c_u64
            getattr(L, fn).argtypes = [c_vp, c_u32]
        L.ref_exp_all_size.restype = c_u64
        L.ref_exp_all_size.argtypes = [c_vp]
        for fn in ("ref_exp_frontier", "ref_exp_edges"):
            getattr(L, fn).restype = C.POINTER(C.c_uint32)
            getattr(L, fn).argtypes = [c_vp, c_u32]
        L.ref_exp_all.restype = C.POINTER(C.c_uint32)
        L.ref_exp_all.argtypes = [c_vp]
        L.ref_exp_indptr.restype = C.POINTER(c_u64)
        L.ref_exp_indptr.argtypes = [c_vp, c_u32]
        L.ref_exp_free.argtypes = [c_vp]
        L.ref_expand_classify_range.argtypes = [c_vp, u32p, c_u64, c_u64, u32p, c_u32, c_u64,
                                                c_u64, c_u32, c_u64, c_u64, u32p, c_vp, C.c_uint,
                                                u64p]
        L.ref_initial_probs.argtypes = [u8p, c_u64, u32p, c_u32, c_u32, c_u64, f64p]
        L.ref_propagate.argtypes = [c_vp, u32p, c_u32, f64p, c_vp, f64p]
        L.ref_empirical_vip.argtypes = [c_vp, u8p, u32p, c_u32, c_u32, c_u64, u32p, c_u32, c_u64,
                                        c_u64, f64p]
        L.ref_rank_by_scores.argtypes = [u32p, c_u64, c_u32, c_u32, f64p, c_u64, u32p, f64p,
                                         C.POINTER(c_u64)]
        L.ref_build_cache.argtypes = [u32p, u64p, c_u32, c_double, c_u64, u64p, u64p]
        L.ref_simulate.argtypes = [c_vp, u8p, u32p, c_u32, u32p, c_u32, c_u64, c_u64, c_u64, u32p,
                                   u64p, u64p, c_vp]
        L.ref_build_reorder.argtypes = [u32p, c_u64, c_u32, f64p, u32p, u64p]
        L.ref_apply_reorder.restype = c_vp
        L.ref_rank_policy.argtypes = [c_vp, c_int, u8p, u32p, c_u32, c_u32, c_u64, c_u32, c_u32, c_double,
                                      u32p, f64p, C.POINTER(c_u64), C.POINTER(c_double)]
        L.ref_apply_reorder.argtypes = [c_vp, u8p, u32p, c_u32, u32p, u8p, u32p]
        self._handles = {}

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def _ptr(self, p):
        if not p:
            msg = self.lib.ref_last_error().decode()
            code = 3
            for c, nm in ((6, "empty"), (6, "no train"), (8, "length"), (2, "out of range"),
                          (4, "offsets"), (4, "target")):
                if nm in msg:
                    code = c
                    break
            raise OracleError(code, msg)
        return p

    def set_threads(self, n):
        self.lib.ref_set_threads(n)

    # ---- rng ----
    def mix64(self, x):
        return self.lib.ref_mix64(x)

    def seed_key(self, seed, parts):
        p = _a64(parts)
        return self.lib.ref_seed_key(seed, p, len(p))

    def stream_draws(self, key, bound, count):
        out = np.zeros(count, np.uint64)
        self.lib.ref_stream_draws(key, bound, count, out)
        return out

    # ---- graph: a reference Graph lives as long as the CSR that names it ----
    def _graph(self, g: CSR):
        h = self._handles.get(id(g))
        if h is None or h[0] is not g:
            p = self._ptr(self.lib.ref_graph_from_csr(g.n, g.m, _a64(g.off), _a32(g.tgt)))
            h = (g, p)
            self._handles[id(g)] = h
        return h[1]

    def graph_symmetric(self, g: CSR, threads=0, check=False):
        """Reference Graph of an undirected canonical CSR (reverse = forward,
        copied instead of transposed); registered like _graph."""
        p = self._ptr(self.lib.ref_graph_from_symmetric_csr(g.n, g.m, _a64(g.off), _a32(g.tgt),
                                                            threads or (os.cpu_count() or 1), int(check)))
        self._handles[id(g)] = (g, p)
        return p

    def sample_neighbors(self, g: CSR, v, fanout, key, seed_keys=None):
        """(ids, next draw of the stream afterwards)."""
        out = np.zeros(max(1, fanout), np.uint32)
        cnt, nxt = c_u64(), c_u64()
        sk = None if seed_keys is None else _a32(seed_keys)
        self._check(self.lib.ref_sample_neighbors_state(self._graph(g), v, fanout, key,
                                                        None if sk is None else sk.ctypes.data, out,
                                                        C.byref(cnt), C.byref(nxt)))
        return out[:cnt.value].copy(), nxt.value

    # ---- file formats (the reference's own readers / writers) ----
    def write_partition_labels(self, labels, K, path):
        labels = _a32(labels)
        self._check(self.lib.ref_write_partition_labels(labels, len(labels), K, path.encode()))

    def partition_from_file(self, path, K, n):
        out = np.zeros(n, np.uint32)
        k_out = c_u32()
        self._check(self.lib.ref_partition_from_file(path.encode(), K, n, out, C.byref(k_out)))
        return out, k_out.value

    def write_roles(self, roles, path):
        r = np.ascontiguousarray(roles, np.uint8)
        self._check(self.lib.ref_write_roles(r, len(r), path.encode()))

    def load_roles(self, path, cap=1 << 24):
        out = np.zeros(cap, np.uint8)
        n = c_u64()
        self._check(self.lib.ref_load_roles(path.encode(), out, cap, C.byref(n)))
        return out[:n.value].copy()

    def write_vip_binary(self, total, path):
        t = np.ascontiguousarray(total, np.float64)
        self._check(self.lib.ref_write_vip_binary(t, len(t), path.encode()))

    def load_vip_binary(self, path, cap=1 << 24):
        out = np.zeros(cap, np.float64)
        n = c_u64()
        self._check(self.lib.ref_load_vip_binary(path.encode(), out, cap, C.byref(n)))
        return out[:n.value].copy()

    def simulate_streams(self, g: CSR, roles, labels, K, fanouts, b, E, seed, cached, trace_path=None,
                         costs_path=None, orderings=None, gamma=0.0):
        offs = np.zeros(K + 1, np.uint64)
        offs[1:] = np.cumsum([len(c) for c in cached])
        cat = _a32(np.concatenate([np.asarray(c, np.uint32) for c in cached]) if K else [])
        cells = np.zeros(E * K * 3, np.uint64)
        f = _a32(fanouts)
        oc = oo = None
        if orderings is not None:
            oo = np.zeros(K + 1, np.uint64)
            oo[1:] = np.cumsum([len(o) for o in orderings])
            oc = _a32(np.concatenate([np.asarray(o, np.uint32) for o in orderings]))
        self._check(self.lib.ref_simulate_streams(
            self._graph(g), np.ascontiguousarray(roles, np.uint8), _a32(labels), K, f, len(f), b, E, seed, cat, offs,
            None if trace_path is None else trace_path.encode(), None if costs_path is None else costs_path.encode(),
            None if oc is None else oc.ctypes.data, None if oo is None else oo.ctypes.data, gamma, cells))
        return cells.reshape(E, K, 3)

    def context(self, roles, labels, K):
        """(VertexRoles, PartitionMap) built once; .epoch(k, b, e, seed) ->
        the epoch_minibatches permutation (sampling.cpp:45-70)."""
        lib, chk = self.lib, self._check
        roles = np.ascontiguousarray(roles, np.uint8)
        h = self._ptr(lib.ref_ctx_create(roles, _a32(labels), len(roles), K))
        n = len(roles)

        class _Ctx:
            def epoch(self, k, b, e, seed):
                out = np.zeros(n, np.uint32)
                cnt = c_u64()
                chk(lib.ref_ctx_epoch(h, k, b, e, seed, out, C.byref(cnt)))
                return out[:cnt.value]

            def __del__(self):
                lib.ref_ctx_free(h)
        return _Ctx()

    def bench_minibatches(self, g: CSR, mbs, fanouts, seed, labels, cache_bits=None, table=None, work=None,
                          threads=0):
        """One CPU-arm step: mbs = [(epoch, k, i, seeds)]; reference expand +
        classify (+ gather of all_vertices rows from `table` into `work`).
        Returns tallies [nmb, 4] = (all, local, cache, miss)."""
        nmb = len(mbs)
        seeds = _a32(np.concatenate([np.asarray(w[3], np.uint32) for w in mbs]))
        offs = np.zeros(nmb + 1, np.uint64)
        offs[1:] = np.cumsum([len(w[3]) for w in mbs])
        refs = np.array([[w[0], w[1], w[2]] for w in mbs], np.uint64).ravel()
        f = _a32(fanouts)
        bits = None if cache_bits is None else np.ascontiguousarray(cache_bits, np.uint64)
        W = 0 if bits is None else bits.shape[-1]
        rb = 0 if table is None else table.shape[1] * table.itemsize
        cap = 0 if work is None else work.shape[1]
        t = np.zeros(nmb * 4, np.uint64)
        self._check(self.lib.ref_bench_minibatches(
            self._graph(g), nmb, seeds, offs, refs, f, len(f), seed, _a32(labels),
            None if bits is None else bits.ctypes.data, W, None if table is None else table.ctypes.data, rb,
            None if work is None else work.ctypes.data, cap, threads or (os.cpu_count() or 1), t))
        return t.reshape(nmb, 4)

    def release(self, g: CSR):
        h = self._handles.pop(id(g), None)
        if h is not None:
            self.lib.ref_graph_free(h[1])

    def _copy_graph(self, p) -> CSR:
        n, m = self.lib.ref_graph_n(p), self.lib.ref_graph_m(p)
        off = np.zeros(n + 1, np.uint64)
        tgt = np.zeros(m, np.uint32)
        roff = np.zeros(n + 1, np.uint64)
        rtgt = np.zeros(m, np.uint32)
        self.lib.ref_graph_copy(p, off.ctypes.data, tgt.ctypes.data, roff.ctypes.data,
                                rtgt.ctypes.data)
        g = CSR(n, off, tgt, roff, rtgt)
        self._handles[id(g)] = (g, p)
        return g

    def generate(self, kind, n, d=2, seed=0) -> CSR:
        return self._copy_graph(self._ptr(self.lib.ref_graph_generate(KINDS[kind], n, d, seed)))

    def from_edges(self, n, edges, undirected) -> CSR:
        e = np.asarray(edges, dtype=np.uint32).reshape(-1, 2)
        return self._copy_graph(self._ptr(self.lib.ref_graph_from_edges(
            n, _a32(e[:, 0]), _a32(e[:, 1]), len(e), int(undirected))))

    def load_vcsr(self, path) -> CSR:
        return self._copy_graph(self._ptr(self.lib.ref_graph_load_vcsr(path.encode())))

    def write_vcsr(self, g: CSR, path):
        self._check(self.lib.ref_graph_write_vcsr(self._graph(g), path.encode()))

    def make_roles(self, n, train, valid=0.0, test=0.0, seed=0):
        out = np.zeros(n, np.uint8)
        self._check(self.lib.ref_make_roles(n, train, valid, test, seed, out))
        return out

    def partition(self, g: CSR, roles, K, method="bfs_greedy", seed=1):
        out = np.zeros(g.n, np.uint32)
        self._check(self.lib.ref_partition_graph(self._graph(g), np.ascontiguousarray(roles, np.uint8),
                                                 g.n, K, PARTITION_METHODS[method], seed, out))
        return out

    # ---- sampling ----
    def epoch_permutation(self, roles, labels, k, b, epoch, seed, K=None, seed_keys=None):
        n = len(roles)
        labels = _a32(labels)
        K = int(labels.max()) + 1 if K is None else K
        out = np.zeros(n, np.uint32)
        cnt = c_u64()
        sk = None if seed_keys is None else _a32(seed_keys)
        self._check(self.lib.ref_epoch_minibatches(np.ascontiguousarray(roles, np.uint8), n,
                                                   labels, K, k, b, epoch, seed,
                                                   None if sk is None else sk.ctypes.data, out,
                                                   C.byref(cnt)))
        return out[:cnt.value]

    def epoch_minibatches(self, roles, labels, k, b, epoch, seed, K=None):
        perm = self.epoch_permutation(roles, labels, k, b, epoch, seed, K)
        return [perm[i:i + b] for i in range(0, len(perm), b)]

    def expand(self, g: CSR, batch, fanouts, seed, epoch=0, part=0, batch_index=0,
               with_mfg=True, seed_keys=None) -> Expansion:
        b = _a32(batch)
        f = _a32(fanouts)
        sk = None if seed_keys is None else _a32(seed_keys)
        p = self._ptr(self.lib.ref_expand(self._graph(g), b, len(b), f, len(f), seed, epoch, part,
                                          batch_index, int(with_mfg), None if sk is None else sk.ctypes.data))
        L = self.lib
        out = Expansion(batch=b.copy())
        for h in range(len(f)):
            fs = L.ref_exp_frontier_size(p, h)
            out.frontier.append(np.ctypeslib.as_array(L.ref_exp_frontier(p, h), shape=(fs,)).copy()
                                if fs else np.zeros(0, np.uint32))
            if with_mfg:
                prev = len(b) if h == 0 else len(out.frontier[h - 1])
                out.indptr.append(np.ctypeslib.as_array(L.ref_exp_indptr(p, h),
                                                        shape=(prev + 1,)).copy())
                ne = L.ref_exp_edges_size(p, h)
                out.edges.append(np.ctypeslib.as_array(L.ref_exp_edges(p, h), shape=(ne,)).copy()
                                 if ne else np.zeros(0, np.uint32))
        na = L.ref_exp_all_size(p)
        out.all_vertices = np.ctypeslib.as_array(L.ref_exp_all(p), shape=(na,)).copy()
        L.ref_exp_free(p)
        return out

    def expand_classify_range(self, g: CSR, perm, b, fanouts, seed, epoch, k, i0, i1, labels,
                              cache_bits=None, threads=1):
        t = np.zeros(4, np.uint64)
        bits = None if cache_bits is None else _a64(cache_bits)
        self._check(self.lib.ref_expand_classify_range(
            self._graph(g), _a32(perm), len(perm), b, _a32(fanouts), len(fanouts), seed, epoch, k,
            i0, i1, _a32(labels), None if bits is None else bits.ctypes.data, threads, t))
        return tuple(int(x) for x in t)

    # ---- vip ----
    def initial_probs(self, roles, labels, K, k, b):
        n = len(roles)
        out = np.zeros(n, np.float64)
        self._check(self.lib.ref_initial_probs(np.ascontiguousarray(roles, np.uint8), n,
                                               _a32(labels), K, k, b, out))
        return out

    def propagate(self, g: CSR, fanouts, p0):
        f = _a32(fanouts)
        p0 = np.ascontiguousarray(p0, np.float64)
        if p0.shape[0] != g.n:
            raise OracleError(8, "p0 length does not match vertex count")
        hop = np.zeros((len(f), g.n), np.float64)
        total = np.zeros(g.n, np.float64)
        self._check(self.lib.ref_propagate(self._graph(g), f, len(f), p0, hop.ctypes.data, total))
        return hop, total

    def empirical_vip(self, g: CSR, roles, labels, K, k, b, fanouts, S, seed):
        out = np.zeros(g.n, np.float64)
        f = _a32(fanouts)
        self._check(self.lib.ref_empirical_vip(self._graph(g), np.ascontiguousarray(roles, np.uint8),
                                               _a32(labels), K, k, b, f, len(f), S, seed, out))
        return out

    # ---- policies ----
    def rank_by_scores(self, labels, K, k, scores):
        labels = _a32(labels)
        n = len(labels)
        scores = np.ascontiguousarray(scores, np.float64)
        order = np.zeros(n, np.uint32)
        sc = np.zeros(n, np.float64)
        cnt = c_u64()
        self._check(self.lib.ref_rank_by_scores(labels, n, K, k, scores, len(scores), order, sc,
                                                C.byref(cnt)))
        return order[:cnt.value], sc[:cnt.value]

    def build_cache(self, orders, alpha, n):
        K = len(orders)
        offs = np.zeros(K + 1, np.uint64)
        offs[1:] = np.cumsum([len(o) for o in orders])
        cat = _a32(np.concatenate([np.asarray(o, np.uint32) for o in orders])
                   if K else np.zeros(0, np.uint32))
        take = np.zeros(max(K, 1), np.uint64)
        W = (n + 63) // 64
        bits = np.zeros(max(K, 1) * W, np.uint64)
        self._check(self.lib.ref_build_cache(cat, offs, K, alpha, n, take, bits))
        cached = [np.asarray(orders[k][:int(take[k])], np.uint32) for k in range(K)]
        return cached, bits.reshape(max(K, 1), W)[:K]

    def simulate(self, g: CSR, roles, labels, K, fanouts, b, E, seed, cached, seed_keys=None):
        offs = np.zeros(K + 1, np.uint64)
        offs[1:] = np.cumsum([len(c) for c in cached])
        cat = _a32(np.concatenate([np.asarray(c, np.uint32) for c in cached]) if K else [])
        cells = np.zeros(E * K * 3, np.uint64)
        f = _a32(fanouts)
        self._check(self.lib.ref_simulate(self._graph(g), np.ascontiguousarray(roles, np.uint8),
                                          _a32(labels), K, f, len(f), b, E, seed, cat, offs, cells,
                                          None if seed_keys is None else _a32(seed_keys).ctypes.data))
        return cells.reshape(E, K, 3)

    def build_reorder(self, labels, K, scores):
        labels = _a32(labels)
        n = len(labels)
        s = np.ascontiguousarray(np.asarray(scores, np.float64).reshape(K, n))
        oon = np.zeros(n, np.uint32)
        ranges = np.zeros(2 * K, np.uint64)
        self._check(self.lib.ref_build_reorder(labels, n, K, s, oon, ranges))
        return oon, ranges.reshape(K, 2)

    def rank_policy(self, g: CSR, which, roles, labels, K, k, L=0, f1=1, iters=5, damping=0.85):
        """rank_degree (0) / rank_halo_1hop (1) / rank_wpr (2) / rank_numpaths (3)
        (policies.cpp:57-132) -> (order, score, effective_alpha)."""
        order = np.zeros(g.n, np.uint32)
        score = np.zeros(g.n, np.float64)
        cnt, ea = c_u64(), c_double()
        self._check(self.lib.ref_rank_policy(self._graph(g), which, np.ascontiguousarray(roles, np.uint8),
                                             _a32(labels), K, k, L, f1, iters, damping, order, score,
                                             C.byref(cnt), C.byref(ea)))
        return order[:cnt.value], score[:cnt.value], ea.value

    def apply_reorder(self, g: CSR, roles, labels, K, old_of_new):
        """apply_reorder (reorder.cpp:36-70) -> (CSR incl. reverse, roles, labels)."""
        n = g.n
        r_out = np.zeros(n, np.uint8)
        l_out = np.zeros(n, np.uint32)
        p = self._ptr(self.lib.ref_apply_reorder(self._graph(g), np.ascontiguousarray(roles, np.uint8),
                                                 _a32(labels), K, _a32(old_of_new), r_out, l_out))
        try:
            out = self._copy_graph(p)
        finally:
            self.lib.ref_graph_free(p)
        return out, r_out, l_out


def port() -> Port:
    return Port()


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> Ref:
    return Ref()
