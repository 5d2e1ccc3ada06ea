"""TEST INFRASTRUCTURE ONLY -- the parity checker.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package. It wraps:

* ``build/liboracle.so`` -- the plain-C restatement of the reference listing
  path (oracle.c; each function cites the reference file:line it follows);
* ``_ref/libtrilist_ref.so`` -- the UNMODIFIED reference core compiled in place
  from /root/reference/proj/core (oracle/Makefile) plus ref_harness.cpp.

The restatement is pinned against the reference build and the golden vectors
in tests/golden/ (tests/test_oracle.py).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(_HERE, "build", "liboracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libtrilist_ref.so")

APP, APM = 0, 1
MASK64 = (1 << 64) - 1


class OrStats(C.Structure):
    _fields_ = [("triangle_count", C.c_uint64), ("inner_ops", C.c_uint64),
                ("mark_ops", C.c_uint64), ("checksum", C.c_uint64), ("wall_ms", C.c_double)]


RefStats = OrStats  # same layout (ref_harness.cpp ref_stats)

_vp, _u32, _u64 = C.c_void_p, C.c_uint32, C.c_uint64


@lru_cache(maxsize=None)
def lib() -> C.CDLL:
    L = C.CDLL(ORACLE_SO)
    L.or_mix64.argtypes = [_u64]
    L.or_mix64.restype = _u64
    L.or_triangle_hash.argtypes = [_u32, _u32, _u32]
    L.or_triangle_hash.restype = _u64
    L.or_orient.argtypes = [_u32, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
    L.or_orient.restype = C.c_int
    L.or_list.argtypes = [C.c_int, _u32, _vp, _vp, _vp, _vp, _vp, _vp, _u32, _u32, C.c_int,
                          _vp, _vp, _u64, C.POINTER(OrStats)]
    L.or_list.restype = _u64
    L.or_cost.argtypes = [_u32, _vp, _vp, _vp]
    L.or_cost.restype = None
    L.or_brute.argtypes = [_u32, _vp, _vp, _vp, _u64]
    L.or_brute.restype = _u64
    L.or_canonicalize.argtypes = [_vp, _u64]
    L.or_canonicalize.restype = None
    L.or_list_ranges.argtypes = [C.c_int, _u32, _vp, _vp, _vp, _vp, _vp, _vp, _u64, C.c_int,
                                 C.POINTER(OrStats)]
    L.or_list_ranges.restype = C.c_int
    L.or_orient_parallel.argtypes = [_u32, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, C.c_int]
    L.or_orient_parallel.restype = C.c_int
    L.or_sort_triples.argtypes = [_vp, _u64, C.c_int]
    L.or_sort_triples.restype = None
    L.or_core_decompose.argtypes = [_u32, _vp, _vp, _vp, _vp]
    L.or_core_decompose.restype = _u32
    return L


def ref_available() -> bool:
    return os.path.exists(REF_SO)


@lru_cache(maxsize=None)
def ref() -> C.CDLL:
    L = C.CDLL(REF_SO)
    L.ref_last_error.restype = C.c_char_p
    L.ref_graph_from_csr.argtypes = [_u32, _vp, _vp]
    L.ref_graph_from_csr.restype = _vp
    L.ref_graph_from_edges.argtypes = [_u32, _u64, _vp]
    L.ref_graph_from_edges.restype = _vp
    L.ref_graph_normalize.argtypes = [_u64, _vp, C.POINTER(_u64), C.POINTER(_u64)]
    L.ref_graph_normalize.restype = _vp
    L.ref_graph_labels.argtypes = [_vp, _vp]
    L.ref_graph_labels.restype = None
    L.ref_graph_gnm.argtypes = [_u32, _u64, _u64]
    L.ref_graph_gnm.restype = _vp
    L.ref_graph_random_small.argtypes = [_u64, _u32, _u64]
    L.ref_graph_random_small.restype = _vp
    L.ref_graph_free.argtypes = [_vp]
    L.ref_graph_n.argtypes = [_vp]
    L.ref_graph_n.restype = _u32
    L.ref_graph_m.argtypes = [_vp]
    L.ref_graph_m.restype = _u64
    L.ref_graph_csr.argtypes = [_vp, _vp, _vp]
    L.ref_order.argtypes = [_vp, C.c_char_p, _u64, _vp]
    L.ref_order.restype = C.c_int
    L.ref_core_decompose.argtypes = [_vp, _vp, _vp]
    L.ref_core_decompose.restype = C.c_int64
    L.ref_cost.argtypes = [_vp, _vp, _vp]
    L.ref_cost.restype = C.c_int
    L.ref_view.argtypes = [_vp, _vp, _u32]
    L.ref_view.restype = _vp
    L.ref_view_free.argtypes = [_vp]
    L.ref_view_csr.argtypes = [_vp, _vp, _vp, _vp, _vp]
    L.ref_orient_ms.argtypes = [_vp, _vp]
    L.ref_orient_ms.restype = C.c_double
    L.ref_list.argtypes = [_vp, C.c_int, C.c_int, _u32, _u32, _vp, _vp, _u64, C.POINTER(_u64),
                           C.POINTER(RefStats)]
    L.ref_list.restype = C.c_int
    L.ref_list_ranges.argtypes = [_vp, C.c_int, C.c_int, _vp, _u64, C.POINTER(RefStats)]
    L.ref_list_ranges.restype = C.c_int
    # synthetic-graph generators (trihost.cpp compiled into this library)
    L.th_last_error.restype = C.c_char_p
    L.th_gen_gnm.argtypes = [_u32, _u64, _u64, _vp]
    L.th_gen_rmat.argtypes = [_u32, _u32, _u64, _vp]
    L.th_gen_chung_lu.argtypes = [_u32, _u64, C.c_double, C.c_double, C.c_double, _u64, _vp]
    L.th_gen_ws.argtypes = [_u32, _u32, C.c_double, _u64, _vp]
    L.th_csr_free.argtypes = [_vp]
    for f in (L.th_gen_gnm, L.th_gen_rmat, L.th_gen_chung_lu, L.th_gen_ws):
        f.restype = C.c_int
    L.ref_brute.argtypes = [_vp, _u32, _vp, _u64]
    L.ref_brute.restype = C.c_int64
    return L


def mix64(z: int) -> int:
    return int(lib().or_mix64(z & MASK64))


def triangle_hash(a: int, b: int, c: int) -> int:
    return int(lib().or_triangle_hash(a, b, c))


# -- restatement ---------------------------------------------------------------

@dataclass
class OrientedCSR:
    succ_off: np.ndarray
    succ: np.ndarray
    pred_off: np.ndarray
    pred: np.ndarray
    inverse: np.ndarray
    rank: np.ndarray


def orient(offsets: np.ndarray, adj: np.ndarray, rank: np.ndarray, threads: int = 1) -> OrientedCSR:
    """or_orient <- oriented_view.cpp:7-47 (threads > 1: or_orient_parallel, same output)."""
    n = offsets.shape[0] - 1
    m = adj.shape[0] // 2
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    adj = np.ascontiguousarray(adj, dtype=np.uint32)
    rank = np.ascontiguousarray(rank, dtype=np.uint32)
    if rank.shape[0] != n:
        raise ValueError("orient: ordering does not match graph")
    so = np.zeros(n + 1, np.uint64)
    po = np.zeros(n + 1, np.uint64)
    s = np.zeros(max(m, 1), np.uint32)
    p = np.zeros(max(m, 1), np.uint32)
    inv = np.zeros(max(n, 1), np.uint32)
    if threads > 1:
        rc = lib().or_orient_parallel(n, m, offsets.ctypes.data, adj.ctypes.data, rank.ctypes.data,
                                      so.ctypes.data, s.ctypes.data, po.ctypes.data, p.ctypes.data,
                                      inv.ctypes.data, threads)
    else:
        rc = lib().or_orient(n, m, offsets.ctypes.data, adj.ctypes.data, rank.ctypes.data,
                             so.ctypes.data, s.ctypes.data, po.ctypes.data, p.ctypes.data, inv.ctypes.data)
    if rc != 0:
        raise ValueError("orient: ordering does not match graph")
    return OrientedCSR(so, s[:m], po, p[:m], inv[:n], rank)


@dataclass
class ListResult:
    triangle_count: int
    inner_ops: int
    mark_ops: int
    checksum: int
    wall_ms: float
    vcounts: np.ndarray | None = None
    triangles: np.ndarray | None = None


def list_triangles(view: OrientedCSR, algo: int, threads: int = 1, vcounts: bool = False,
                   collect: bool = False, rank_begin: int = 0, rank_end: int | None = None,
                   tri_cap: int | None = None) -> ListResult:
    """or_list <- listing.hpp:69-107 / 122-155."""
    n = view.succ_off.shape[0] - 1
    re = n if rank_end is None else rank_end
    vc = np.zeros(max(n, 1), np.uint64) if vcounts else None
    tri = None
    cap = 0
    if collect:
        cap = tri_cap if tri_cap is not None else int(view.succ.shape[0] * 4 + 16)
        tri = np.zeros((cap, 3), np.uint32)
    st = OrStats()
    succ = view.succ if view.succ.shape[0] else np.zeros(1, np.uint32)
    pred = view.pred if view.pred.shape[0] else np.zeros(1, np.uint32)
    k = lib().or_list(algo, n, view.succ_off.ctypes.data, succ.ctypes.data,
                      view.pred_off.ctypes.data, pred.ctypes.data, view.inverse.ctypes.data,
                      view.rank.ctypes.data, rank_begin, re, threads,
                      vc.ctypes.data if vc is not None else None,
                      tri.ctypes.data if tri is not None else None, cap, C.byref(st))
    if collect and st.triangle_count > cap:
        return list_triangles(view, algo, threads, vcounts, True, rank_begin, rank_end,
                              tri_cap=int(st.triangle_count))
    return ListResult(int(st.triangle_count), int(st.inner_ops), int(st.mark_ops),
                      int(st.checksum), float(st.wall_ms),
                      vc[:n] if vc is not None else None,
                      tri[:k] if tri is not None else None)


def list_ranges(view: OrientedCSR, algo: int, ranges, threads: int = 1) -> ListResult:
    """or_list_ranges: count + checksum over a sample of rank ranges, one pass."""
    n = view.succ_off.shape[0] - 1
    r = np.ascontiguousarray(np.asarray(ranges, dtype=np.uint32).reshape(-1, 2))
    st = OrStats()
    succ = view.succ if view.succ.shape[0] else np.zeros(1, np.uint32)
    pred = view.pred if view.pred.shape[0] else np.zeros(1, np.uint32)
    lib().or_list_ranges(algo, n, view.succ_off.ctypes.data, succ.ctypes.data, view.pred_off.ctypes.data,
                         pred.ctypes.data, view.inverse.ctypes.data, r.ctypes.data, r.shape[0], threads,
                         C.byref(st))
    return ListResult(int(st.triangle_count), int(st.inner_ops), int(st.mark_ops), int(st.checksum),
                      float(st.wall_ms))


def cost(view: OrientedCSR) -> tuple[int, int, int, int]:
    """or_cost <- cost.cpp:27-38: (c_pp, c_pm, c_mm, sum_deg_sq)."""
    n = view.succ_off.shape[0] - 1
    out = np.zeros(4, np.uint64)
    lib().or_cost(n, view.succ_off.ctypes.data, view.pred_off.ctypes.data, out.ctypes.data)
    return tuple(int(x) for x in out)


def core_decompose(offsets: np.ndarray, adj: np.ndarray) -> tuple[np.ndarray, np.ndarray, int]:
    """or_core_decompose <- ordering.cpp:141-188: (ranks of the removal order, coreness, degeneracy)."""
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    adj = np.ascontiguousarray(adj if adj.shape[0] else np.zeros(1, np.uint32), dtype=np.uint32)
    n = offsets.shape[0] - 1
    rank = np.zeros(max(n, 1), np.uint32)
    core = np.zeros(max(n, 1), np.uint32)
    dg = lib().or_core_decompose(n, offsets.ctypes.data, adj.ctypes.data, rank.ctypes.data, core.ctypes.data)
    return rank[:n], core[:n], int(dg)


def brute(offsets: np.ndarray, adj: np.ndarray) -> np.ndarray:
    """or_brute <- oracle.cpp:12-30 (sorted u<v<w triples)."""
    n = offsets.shape[0] - 1
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    adj = np.ascontiguousarray(adj if adj.shape[0] else np.zeros(1, np.uint32), dtype=np.uint32)
    k = lib().or_brute(n, offsets.ctypes.data, adj.ctypes.data, None, 0)
    out = np.zeros((max(k, 1), 3), np.uint32)
    lib().or_brute(n, offsets.ctypes.data, adj.ctypes.data, out.ctypes.data, k)
    return out[:k]


def sort_triples(tri: np.ndarray, threads: int = 1) -> np.ndarray:
    """CollectingSink::canonical in place on a (k, 3) uint32 array (or_sort_triples)."""
    assert tri.dtype == np.uint32 and tri.flags["C_CONTIGUOUS"] and tri.ndim == 2 and tri.shape[1] == 3
    if tri.shape[0]:
        lib().or_sort_triples(tri.ctypes.data, tri.shape[0], threads)
    return tri


def canonical(tri: np.ndarray) -> np.ndarray:
    """CollectingSink::canonical (listing.hpp:57-62)."""
    t = np.ascontiguousarray(np.asarray(tri, dtype=np.uint32).reshape(-1, 3)).copy()
    if t.shape[0]:
        lib().or_canonicalize(t.ctypes.data, t.shape[0])
    return t


# -- reference harness ---------------------------------------------------------------

class RefGraph:
    """trilist::Graph owned by the reference harness."""

    def __init__(self, handle):
        if not handle:
            raise ValueError(ref().ref_last_error().decode())
        self.h = handle

    @classmethod
    def gnm(cls, n, m, seed):
        return cls(ref().ref_graph_gnm(n, m, seed))

    @classmethod
    def random_small(cls, seed, max_n, max_m):
        """acceptance_main.cpp:89-95 / test_support.hpp:26-32."""
        return cls(ref().ref_graph_random_small(seed, max_n, max_m))

    @classmethod
    def from_csr(cls, offsets, adj):
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        adj = np.ascontiguousarray(adj if adj.shape[0] else np.zeros(1, np.uint32), dtype=np.uint32)
        return cls(ref().ref_graph_from_csr(offsets.shape[0] - 1, offsets.ctypes.data, adj.ctypes.data))

    @classmethod
    def from_edges(cls, n, edges):
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
        if e.shape[0] == 0:
            e = np.zeros((1, 2), np.uint32)
            return cls(ref().ref_graph_from_edges(n, 0, e.ctypes.data))
        return cls(ref().ref_graph_from_edges(n, e.shape[0], e.ctypes.data))

    @classmethod
    def normalize(cls, raw_pairs):
        """normalize (graph.cpp:115-151): returns (graph, loops_removed, duplicates_removed)."""
        e = np.ascontiguousarray(np.asarray(raw_pairs, dtype=np.int64).reshape(-1, 2))
        k = e.shape[0]
        if k == 0:
            e = np.zeros((1, 2), np.int64)
        lo, du = C.c_uint64(0), C.c_uint64(0)
        h = ref().ref_graph_normalize(k, e.ctypes.data, C.byref(lo), C.byref(du))
        if not h:
            raise ValueError(ref().ref_last_error().decode())
        return cls(h), int(lo.value), int(du.value)

    def labels(self) -> np.ndarray:
        out = np.zeros(max(self.n, 1), np.int64)
        ref().ref_graph_labels(self.h, out.ctypes.data)
        return out[: self.n]

    def __del__(self):
        try:
            ref().ref_graph_free(self.h)
        except Exception:
            pass

    @property
    def n(self):
        return int(ref().ref_graph_n(self.h))

    @property
    def m(self):
        return int(ref().ref_graph_m(self.h))

    def csr(self):
        off = np.zeros(self.n + 1, np.uint64)
        adj = np.zeros(max(2 * self.m, 1), np.uint32)
        ref().ref_graph_csr(self.h, off.ctypes.data, adj.ctypes.data)
        return off, adj[: 2 * self.m]

    def order(self, method: str, seed: int = 0) -> np.ndarray:
        r = np.zeros(max(self.n, 1), np.uint32)
        if ref().ref_order(self.h, method.encode(), seed, r.ctypes.data) != 0:
            raise ValueError(ref().ref_last_error().decode())
        return r[: self.n]

    def core_decompose(self) -> tuple[np.ndarray, np.ndarray, int]:
        """The reference's core_decompose(g): (ranks, coreness, degeneracy)."""
        r = np.zeros(max(self.n, 1), np.uint32)
        c = np.zeros(max(self.n, 1), np.uint32)
        dg = ref().ref_core_decompose(self.h, r.ctypes.data, c.ctypes.data)
        if dg < 0:
            raise ValueError(ref().ref_last_error().decode())
        return r[: self.n], c[: self.n], int(dg)

    def cost(self, rank) -> tuple[int, int, int, int]:
        rank = np.ascontiguousarray(rank, dtype=np.uint32)
        out = np.zeros(4, np.uint64)
        if ref().ref_cost(self.h, rank.ctypes.data, out.ctypes.data) != 0:
            raise ValueError(ref().ref_last_error().decode())
        return tuple(int(x) for x in out)

    def brute(self, guard: int = 500) -> np.ndarray:
        k = ref().ref_brute(self.h, guard, None, 0)
        if k < 0:
            raise ValueError(ref().ref_last_error().decode())
        out = np.zeros((max(k, 1), 3), np.uint32)
        ref().ref_brute(self.h, guard, out.ctypes.data, k)
        return out[:k]


class RefView:
    """trilist::OrientedView built by the reference constructor."""

    def __init__(self, g: RefGraph, rank):
        rank = np.ascontiguousarray(rank, dtype=np.uint32)
        r = rank if rank.shape[0] else np.zeros(1, np.uint32)
        self.h = ref().ref_view(g.h, r.ctypes.data, rank.shape[0])
        if not self.h:
            raise ValueError(ref().ref_last_error().decode())
        self.n, self.m = g.n, g.m

    def __del__(self):
        try:
            ref().ref_view_free(self.h)
        except Exception:
            pass

    def list_ranges(self, algo: int, ranges, threads: int = 1) -> ListResult:
        """The reference's run_*_range loops over a sample of rank ranges in one
        run_parallel-style pulling pass (ref_list_ranges)."""
        r = np.ascontiguousarray(np.asarray(ranges, dtype=np.uint32).reshape(-1, 2))
        st = RefStats()
        if ref().ref_list_ranges(self.h, algo, threads, r.ctypes.data, r.shape[0], C.byref(st)) != 0:
            raise ValueError(ref().ref_last_error().decode())
        return ListResult(int(st.triangle_count), int(st.inner_ops), int(st.mark_ops), int(st.checksum),
                          float(st.wall_ms))

    def csr(self):
        so = np.zeros(self.n + 1, np.uint64)
        po = np.zeros(self.n + 1, np.uint64)
        s = np.zeros(max(self.m, 1), np.uint32)
        p = np.zeros(max(self.m, 1), np.uint32)
        ref().ref_view_csr(self.h, so.ctypes.data, s.ctypes.data, po.ctypes.data, p.ctypes.data)
        return so, s[: self.m], po, p[: self.m]

    def list(self, algo: int, threads: int = 1, vcounts=False, collect=False, rank_begin=0,
             rank_end=None, tri_cap=None) -> ListResult:
        re = self.n if rank_end is None else rank_end
        vc = np.zeros(max(self.n, 1), np.uint64) if vcounts else None
        cap = 0
        tri = None
        if collect:
            cap = 4 * self.m + 16 if tri_cap is None else max(int(tri_cap), 1)
            tri = np.zeros((cap, 3), np.uint32)
        k = C.c_uint64(0)
        st = RefStats()
        rc = ref().ref_list(self.h, algo, threads, rank_begin, re,
                            vc.ctypes.data if vc is not None else None,
                            tri.ctypes.data if tri is not None else None, cap, C.byref(k),
                            C.byref(st))
        if rc != 0:
            raise ValueError(ref().ref_last_error().decode())
        if collect and k.value > cap:
            cap = k.value
            tri = np.zeros((cap, 3), np.uint32)
            rc = ref().ref_list(self.h, algo, threads, rank_begin, re,
                                vc.ctypes.data if vc is not None else None, tri.ctypes.data, cap,
                                C.byref(k), C.byref(st))
            if rc != 0:
                raise ValueError(ref().ref_last_error().decode())
        return ListResult(int(st.triangle_count), int(st.inner_ops), int(st.mark_ops),
                          int(st.checksum), float(st.wall_ms),
                          vc[: self.n] if vc is not None else None,
                          tri[: min(k.value, cap)] if tri is not None else None)


# -- synthetic inputs for the reference arm ------------------------------------------

class _ThCsr(C.Structure):
    _fields_ = [("n", C.c_uint32), ("m", C.c_uint64), ("offsets", C.POINTER(C.c_uint64)),
                ("adj", C.POINTER(C.c_uint32))]


class GenGraph:
    """A BASELINE config graph (offsets uint64[n+1], adjacency uint32[2m]) from
    the same counter-based generators the engine's host side uses, built into
    _ref/libtrilist_ref.so so the reference arm loads nothing outside oracle/."""

    def __init__(self, kind: str, **kw):
        csr = _ThCsr()
        L = ref()
        if kind == "gnm":
            rc = L.th_gen_gnm(kw["n"], kw["m"], kw["seed"], C.byref(csr))
        elif kind == "rmat":
            rc = L.th_gen_rmat(kw["scale"], kw["ef"], kw["seed"], C.byref(csr))
        elif kind == "chung_lu":
            rc = L.th_gen_chung_lu(kw["n"], kw["draws"], 2.1, 2.0, 50000.0, kw["seed"], C.byref(csr))
        elif kind == "ws":
            rc = L.th_gen_ws(kw["n"], kw["k"], kw["p"], kw["seed"], C.byref(csr))
        else:
            raise ValueError(kind)
        if rc != 0:
            raise RuntimeError(L.th_last_error().decode())
        self._csr = csr
        self.n, self.m = int(csr.n), int(csr.m)
        self.offsets = np.ctypeslib.as_array(csr.offsets, shape=(self.n + 1,))
        self.adjacency = np.ctypeslib.as_array(csr.adj, shape=(max(2 * self.m, 1),))[: 2 * self.m]

    def free(self):
        if self._csr is not None:
            self.offsets = self.adjacency = None
            ref().th_csr_free(C.byref(self._csr))
            self._csr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
