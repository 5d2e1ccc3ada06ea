"""Host-side inputs of the listing path: graphs, orderings, cost reports.

Mirrors the reference types the listing path consumes:

* :class:`Graph`    -- trilist::Graph (core/include/trilist/graph.hpp:20-62): CSR
  ``offsets`` uint64[n+1], ``adjacency`` uint32[2m], rows strictly increasing.
* :class:`Ordering` -- trilist::Ordering (ordering.hpp:16-38): ``ranks`` and
  ``sequence`` (inverse) as uint32[n].
* ``identity_order`` ... ``neigh_order`` -- the reference's own C++ orderings
  (ordering.cpp / neigh.cpp), called unchanged through ``libtrihost.so``.
* ``cost_report`` -- cost.cpp:7-25, also the reference's code.
* ``gen_gnm`` -- the reference's generator (graph.cpp:210-243); ``gen_rmat``,
  ``gen_chung_lu``, ``gen_ws`` -- the BASELINE.json C2-C5 generators.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native


class HostError(RuntimeError):
    pass


def _th_err() -> str:
    return _native.trihost().th_last_error().decode()


class Graph:
    """Immutable undirected simple graph in the reference's CSR layout."""

    def __init__(self, offsets: np.ndarray, adjacency: np.ndarray, _owner=None):
        self.offsets = offsets
        self.adjacency = adjacency
        self._owner = _owner  # keeps C-allocated memory alive
        self._ref = None      # lazily built trilist::Graph handle

    # -- construction -------------------------------------------------------
    @classmethod
    def _from_th(cls, csr: _native.ThCsr) -> "Graph":
        n, m = csr.n, csr.m
        off = np.ctypeslib.as_array(csr.offsets, shape=(n + 1,))
        adj = np.ctypeslib.as_array(csr.adj, shape=(max(2 * m, 1),))[: 2 * m]
        return cls(off, adj, _owner=_CsrOwner(csr))

    @classmethod
    def from_dense_edges(cls, n: int, edges) -> "Graph":
        """Graph::from_dense_edges (graph.cpp:13-56) semantics for valid input;
        loops are dropped and duplicates merged instead of raising."""
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
        csr = _native.ThCsr()
        if _native.trihost().th_csr_from_pairs(n, e.shape[0], e.ctypes.data, C.byref(csr)) != 0:
            raise HostError(_th_err())
        return cls._from_th(csr)

    @classmethod
    def load(cls, path: str) -> "Graph":
        """load_edgelist_file (graph.cpp:164-192), the reference's own text
        loader: label pairs, loops dropped, duplicates merged, labels re-indexed
        densely in ascending order. ``labels`` / ``loops_removed`` /
        ``duplicates_removed`` are set on the result."""
        lo, du = C.c_uint64(0), C.c_uint64(0)
        h = _native.trihost().th_graph_load(path.encode(), C.byref(lo), C.byref(du))
        if not h:
            raise HostError(_th_err())
        ref = _RefGraph(h)
        csr = _native.ThCsr()
        if _native.trihost().th_graph_to_csr(h, C.byref(csr)) != 0:
            raise HostError(_th_err())
        g = cls._from_th(csr)
        g._ref = ref
        g.labels = np.zeros(max(g.n, 1), np.int64)
        _native.trihost().th_graph_labels(h, g.labels.ctypes.data)
        g.labels = g.labels[: g.n]
        g.loops_removed, g.duplicates_removed = int(lo.value), int(du.value)
        return g

    def label_of(self, u: int) -> int:
        labels = getattr(self, "labels", None)
        return int(labels[u]) if labels is not None else int(u)

    # -- accessors (graph.hpp:31-43) -----------------------------------------
    def vertex_count(self) -> int:
        return int(self.offsets.shape[0] - 1)

    def edge_count(self) -> int:
        return int(self.adjacency.shape[0] // 2)

    @property
    def n(self) -> int:
        return self.vertex_count()

    @property
    def m(self) -> int:
        return self.edge_count()

    def neighbors(self, u: int) -> np.ndarray:
        return self.adjacency[self.offsets[u]:self.offsets[u + 1]]

    def degree(self, u: int) -> int:
        return int(self.offsets[u + 1] - self.offsets[u])

    def degrees(self) -> np.ndarray:
        return np.diff(self.offsets).astype(np.uint32)

    def has_edge(self, u: int, v: int) -> bool:
        row = self.neighbors(u)
        i = np.searchsorted(row, v)
        return bool(i < row.shape[0] and row[i] == v)

    def check_invariants(self) -> None:
        csr = self._as_th()
        if _native.trihost().th_csr_check(C.byref(csr)) != 0:
            raise HostError(_th_err())

    def _as_th(self) -> _native.ThCsr:
        csr = _native.ThCsr()
        csr.n = self.vertex_count()
        csr.m = self.edge_count()
        csr.offsets = self.offsets.ctypes.data_as(C.POINTER(C.c_uint64))
        csr.adj = self.adjacency.ctypes.data_as(C.POINTER(C.c_uint32))
        return csr

    def reference_handle(self):
        """trilist::Graph built by Graph::from_dense_edges over this CSR."""
        if self._ref is None:
            h = _native.trihost().th_graph_new(C.byref(self._as_th()))
            if not h:
                raise HostError(_th_err())
            self._ref = _RefGraph(h)
        return self._ref.h


class _CsrOwner:
    def __init__(self, csr):
        self.csr = csr

    def __del__(self):
        try:
            _native.trihost().th_csr_free(C.byref(self.csr))
        except Exception:
            pass


class _RefGraph:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            _native.trihost().th_graph_free(self.h)
        except Exception:
            pass


@dataclass
class Ordering:
    """trilist::Ordering: ranks[v] = 0-based position of v; sequence = inverse."""

    ranks: np.ndarray

    def __post_init__(self):
        self.ranks = np.ascontiguousarray(self.ranks, dtype=np.uint32)

    def size(self) -> int:
        return int(self.ranks.shape[0])

    def rank_of(self, v: int) -> int:
        return int(self.ranks[v])

    @property
    def sequence(self) -> np.ndarray:
        inv = np.empty_like(self.ranks)
        inv[self.ranks] = np.arange(self.ranks.shape[0], dtype=np.uint32)
        return inv

    @classmethod
    def identity(cls, n: int) -> "Ordering":
        return cls(np.arange(n, dtype=np.uint32))

    @classmethod
    def from_sequence(cls, order) -> "Ordering":
        order = np.asarray(order, dtype=np.uint32)
        r = np.empty_like(order)
        r[order] = np.arange(order.shape[0], dtype=np.uint32)
        return cls(r)


ORDERINGS = ("identity", "random", "degree", "core", "split", "check", "neigh")


def compute_order(g: Graph, method: str, seed: int = 0) -> tuple[Ordering, float]:
    """compute_order (trilist_cli.cpp:50-64) with the reference's own
    orderings; returns (ordering, order_ms) where order_ms times the ordering
    call alone (the CLI's order_ms, trilist_cli.cpp:199-201)."""
    ranks = np.empty(g.vertex_count(), dtype=np.uint32)
    ms = C.c_double(0.0)
    rc = _native.trihost().th_order(g.reference_handle(), method.encode(), seed,
                                    ranks.ctypes.data, C.byref(ms))
    if rc != 0:
        raise HostError(_th_err())
    return Ordering(ranks), ms.value


def identity_order(g: Graph) -> Ordering:
    return compute_order(g, "identity")[0]


def random_order(g: Graph, seed: int) -> Ordering:
    return compute_order(g, "random", seed)[0]


def degree_order(g: Graph) -> Ordering:
    return compute_order(g, "degree")[0]


def core_order(g: Graph) -> Ordering:
    return compute_order(g, "core")[0]


def split_order(g: Graph) -> Ordering:
    return compute_order(g, "split")[0]


def check_order(g: Graph) -> Ordering:
    return compute_order(g, "check")[0]


def neigh_order(g: Graph) -> Ordering:
    return compute_order(g, "neigh")[0]


@dataclass
class CostReport:
    c_pp: int
    c_pm: int
    c_mm: int
    sum_deg_sq: int


def cost_report(g: Graph, pi: Ordering) -> CostReport:
    out = np.zeros(4, dtype=np.uint64)
    if _native.trihost().th_cost(g.reference_handle(), pi.ranks.ctypes.data, out.ctypes.data) != 0:
        raise HostError(_th_err())
    return CostReport(*(int(x) for x in out))


# -- generators ---------------------------------------------------------------

def _gen(fn, *args) -> Graph:
    csr = _native.ThCsr()
    if fn(*args, C.byref(csr)) != 0:
        raise HostError(_th_err())
    return Graph._from_th(csr)


def gen_gnm(n: int, m: int, seed: int) -> Graph:
    """The reference's gen_gnm (graph.cpp:210-243): config C1 is
    gen_gnm(100000, 1000000, 4242) (acceptance_main.cpp:449)."""
    return _gen(_native.trihost().th_gen_gnm, n, m, seed)


def gen_rmat(scale: int, edge_factor: int = 16, seed: int = 1) -> Graph:
    """R-MAT (0.57, 0.19, 0.19, 0.05), edge_factor * 2^scale draws (C4, C5)."""
    return _gen(_native.trihost().th_gen_rmat, scale, edge_factor, seed)


def gen_rmat_raw(scale: int, edge_factor: int = 16, seed: int = 1) -> np.ndarray:
    """The raw (k, 2) int64 draws behind gen_rmat (loops and duplicates kept)."""
    out = np.empty(((edge_factor << scale), 2), np.int64)
    if _native.trihost().th_gen_rmat_raw(scale, edge_factor, seed, out.ctypes.data) != 0:
        raise HostError(_th_err())
    return out


def gen_chung_lu(n: int, draws: int, exponent: float = 2.1, wmin: float = 2.0,
                 wmax: float = 50000.0, seed: int = 1) -> Graph:
    """Chung-Lu with Pareto(exponent, wmin) weights capped at wmax (C2)."""
    return _gen(_native.trihost().th_gen_chung_lu, n, draws, exponent, wmin, wmax, seed)


def gen_ws(n: int, k: int = 32, p: float = 0.1, seed: int = 1) -> Graph:
    """Watts-Strogatz ring lattice with rewiring probability p (C3)."""
    return _gen(_native.trihost().th_gen_ws, n, k, p, seed)


def parse_edgelist(path: str) -> np.ndarray:
    """Raw (k, 2) int64 label pairs of a text edge list, in file order, loops and
    duplicates kept: the native multi-threaded reader (th_parse_edgelist) of
    load_edgelist's grammar (graph.cpp:164-186; errors "line N: ..." as its
    ParseError). The input of normalize (graph.cpp:115) -- Context.normalize
    runs that on the GPU."""
    lib = _native.trihost()
    ptr = C.POINTER(C.c_int64)()
    k = C.c_uint64(0)
    if lib.th_parse_edgelist(path.encode(), C.byref(ptr), C.byref(k)) != 0:
        raise HostError(_th_err())
    if k.value == 0:
        return np.zeros((0, 2), np.int64)
    try:
        return np.ctypeslib.as_array(ptr, shape=(k.value, 2)).copy()
    finally:
        lib.th_free(ptr)


def host_threads() -> int:
    return int(_native.trihost().th_threads())


def bench_csv_header() -> str:
    return _native.trihost().th_bench_csv_header().decode()


def bench_csv_row(dataset, algo, ordering, mode, threads, n, m, c_pp, c_pm, inner_ops,
                  triangles, load_ms, order_ms, list_ms) -> str:
    """trilist::to_csv_row (bench.cpp:7-19), the reference's own code."""
    buf = C.create_string_buffer(1024)
    rc = _native.trihost().th_bench_csv(
        dataset.encode(), algo.encode(), ordering.encode(), mode.encode(), threads, n, m,
        c_pp, c_pm, inner_ops, triangles, load_ms, order_ms, list_ms, buf, 1024)
    if rc != 0:
        raise HostError("bench csv row too long")
    return buf.value.decode()
