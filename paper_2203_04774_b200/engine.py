"""Python mirror of the reference listing API, backed by ``libtrigpu.so``.

Reference (core/include/trilist/):

=====================================  ==========================================
reference                              here
=====================================  ==========================================
``OrientedView(g, pi)``                ``OrientedView(g, pi)`` (built on the GPU)
  oriented_view.hpp:17-50                successors/predecessors fetched on demand
``ListingStats`` listing.hpp:23-34     ``ListingStats`` (+ checksum, costs, times)
``CountingSink`` listing.hpp:40-44     ``CountingSink``
``CollectingSink`` listing.hpp:46-63   ``CollectingSink`` (+ ``canonical()``)
(new)                   ``ChecksumSink``, ``VertexCountSink``
``list_app/list_apm`` :162-183         ``list_app/list_apm(view | (g, pi), sink)``
``list_*_parallel`` :187-199           ``list_*_parallel(view, sink, threads)``
=====================================  ==========================================

Errors follow the reference: an ordering whose size does not match the graph
raises ``ValueError`` (``std::invalid_argument`` in oriented_view.cpp:8-9).
The GPU run is always parallel, so emission order is unspecified (the
contract of the reference's parallel variants, listing.hpp:185-186); counts,
checksums, per-vertex counts and ``canonical()`` lists are exact.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _native
from ._native import (TL_ALGO_APM, TL_ALGO_APP, TL_ERR_CAPACITY, TL_ERR_INVALID_ARGUMENT, TL_OK,
                      TL_OUT_CHECKSUM, TL_OUT_LIST, TL_OUT_VERTEX_COUNTS, TlStats)
from .host import Graph, Ordering

APP = TL_ALGO_APP
APM = TL_ALGO_APM


class TrigpuError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[trigpu status {status}] {msg}")
        self.status = status


def _check(ctx_ptr, rc: int):
    if rc != TL_OK:
        msg = _native.trigpu().tl_last_error(ctx_ptr).decode()
        if rc == TL_ERR_INVALID_ARGUMENT:
            raise ValueError(msg)
        raise TrigpuError(rc, msg)


class Context:
    """One device + stream + device buffers (tl_ctx)."""

    def __init__(self, device: int = 0):
        lib = _native.trigpu()
        p = C.c_void_p()
        rc = lib.tl_create(C.byref(p), device)
        if rc != TL_OK:
            raise TrigpuError(rc, lib.tl_last_error(None).decode())
        self._p = p
        self.device = device

    @property
    def ptr(self):
        return self._p

    def close(self):
        if self._p:
            _native.trigpu().tl_destroy(self._p)
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- raw C-ABI passthroughs (host buffers) -------------------------------
    def orient(self, offsets: np.ndarray, adj: np.ndarray, rank: np.ndarray) -> None:
        n = offsets.shape[0] - 1
        if rank.shape[0] != n:
            raise ValueError("orient: ordering does not match graph")
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        adj = np.ascontiguousarray(adj, dtype=np.uint32)
        rank = np.ascontiguousarray(rank, dtype=np.uint32)
        _check(self._p, _native.trigpu().tl_orient(self._p, n, adj.shape[0] // 2, offsets.ctypes.data,
                                                   adj.ctypes.data, rank.ctypes.data))

    def orient_device(self, n: int, m: int, d_offsets: int, d_adj: int, d_rank: int) -> None:
        _check(self._p, _native.trigpu().tl_orient_device(self._p, n, m, d_offsets, d_adj, d_rank))

    # device orderings (degree_order / split_order, ordering.cpp:66-109)
    _ORDERS = {"degree": _native.TL_ORDER_DEGREE, "split": _native.TL_ORDER_SPLIT}
    _ORIENT_ORDERS = {**_ORDERS, "core": _native.TL_ORDER_CORE}  # core needs the adjacency

    def order(self, offsets: np.ndarray, method: str) -> np.ndarray:
        """Ordering::ranks() of degree_order / split_order, computed on the GPU."""
        if method not in self._ORDERS:
            raise ValueError(f"order: device orderings are {sorted(self._ORDERS)}")
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        n = offsets.shape[0] - 1
        rank = np.empty(max(n, 1), dtype=np.uint32)
        _check(self._p, _native.trigpu().tl_order(self._p, n, offsets.ctypes.data, self._ORDERS[method],
                                                  rank.ctypes.data))
        return rank[:n]

    def core_decompose(self, offsets: np.ndarray, adj: np.ndarray) -> tuple[np.ndarray, np.ndarray, int]:
        """core_decompose(g) (ordering.cpp:141-188) on the GPU: (ranks of a degeneracy
        ordering, coreness, degeneracy). Coreness / degeneracy equal the reference's; the
        order is (peel round, id) - see include/trigpu.h."""
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        adj = np.ascontiguousarray(adj, dtype=np.uint32)
        n = offsets.shape[0] - 1
        rank = np.empty(max(n, 1), dtype=np.uint32)
        core = np.empty(max(n, 1), dtype=np.uint32)
        dg = C.c_uint32(0)
        _check(self._p, _native.trigpu().tl_core_decompose(self._p, n, adj.shape[0] // 2, offsets.ctypes.data,
                                                           adj.ctypes.data, rank.ctypes.data, core.ctypes.data,
                                                           C.byref(dg)))
        return rank[:n], core[:n], int(dg.value)

    def order_device(self, n: int, d_offsets: int, method: str, d_rank: int) -> None:
        _check(self._p, _native.trigpu().tl_order_device(self._p, n, d_offsets, self._ORDERS[method], d_rank))

    def orient_ordered(self, offsets: np.ndarray, adj: np.ndarray, method: str) -> None:
        """tl_orient with the ordering computed on the device (no host ordering)."""
        if method not in self._ORIENT_ORDERS:
            raise ValueError(f"orient_ordered: device orderings are {sorted(self._ORIENT_ORDERS)}")
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        adj = np.ascontiguousarray(adj, dtype=np.uint32)
        _check(self._p, _native.trigpu().tl_orient_ordered(self._p, offsets.shape[0] - 1, adj.shape[0] // 2,
                                                           offsets.ctypes.data, adj.ctypes.data,
                                                           self._ORIENT_ORDERS[method]))

    def normalize(self, raw_pairs) -> tuple[int, int, int, int]:
        """Raw labeled edges -> Graph CSR on the device (normalize, graph.cpp:115-151).
        Returns (n, m, loops_removed, duplicates_removed); tl_fetch_graph reads it."""
        e = np.ascontiguousarray(np.asarray(raw_pairs, dtype=np.int64).reshape(-1, 2))
        n, m, lo, du = C.c_uint32(0), C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
        _check(self._p, _native.trigpu().tl_normalize(self._p, e.shape[0], e.ctypes.data if e.shape[0] else None,
                                                      C.byref(n), C.byref(m), C.byref(lo), C.byref(du)))
        self._norm = (int(n.value), int(m.value))
        return int(n.value), int(m.value), int(lo.value), int(du.value)

    def fetch_graph(self):
        """(offsets uint64[n+1], adjacency uint32[2m], labels int64[n]) of the last normalize."""
        n, m = self._norm
        off = np.zeros(n + 1, np.uint64)
        adj = np.zeros(max(2 * m, 1), np.uint32)
        lab = np.zeros(max(n, 1), np.int64)
        _check(self._p, _native.trigpu().tl_fetch_graph(self._p, off.ctypes.data, adj.ctypes.data, lab.ctypes.data))
        return off, adj[: 2 * m], lab[:n]

    def iter_triangles(self, chunk: int = 1 << 24, labels: np.ndarray | None = None, use_labels: bool = False):
        """Stream the last TL_OUT_LIST result in chunks: uint32 (k, 3) dense ids,
        or int64 labels (labels=table, or use_labels=True for the tl_normalize labels)."""
        first = 0
        k = C.c_uint64(0)
        lab = None if labels is None else np.ascontiguousarray(labels, dtype=np.int64)
        while True:
            if lab is None and not use_labels:
                buf = np.empty((chunk, 3), np.uint32)
                _check(self._p, _native.trigpu().tl_fetch_triangles_range(self._p, first, chunk, buf.ctypes.data,
                                                                          C.byref(k)))
            else:
                buf = np.empty((chunk, 3), np.int64)
                _check(self._p, _native.trigpu().tl_fetch_triangle_labels(
                    self._p, first, chunk, lab.ctypes.data if lab is not None else None, buf.ctypes.data, C.byref(k)))
            if k.value == 0:
                return
            yield buf[: k.value]
            first += k.value

    def orient_normalized(self, method: str) -> None:
        _check(self._p, _native.trigpu().tl_orient_normalized(self._p, self._ORIENT_ORDERS[method]))

    def fetch_ranks(self, n: int) -> np.ndarray:
        rank = np.empty(max(n, 1), dtype=np.uint32)
        _check(self._p, _native.trigpu().tl_fetch_ranks(self._p, rank.ctypes.data))
        return rank[:n]

    def list(self, algo: int, flags: int) -> TlStats:
        st = TlStats()
        _check(self._p, _native.trigpu().tl_list(self._p, algo, flags, C.byref(st)))
        return st

    def list_range(self, algo: int, flags: int, rank_begin: int, rank_end: int) -> TlStats:
        """run_*_range (listing.hpp:69-107) over the seeds ranked [rank_begin, rank_end)."""
        st = TlStats()
        _check(self._p, _native.trigpu().tl_list_range(self._p, algo, flags, rank_begin, rank_end, C.byref(st)))
        return st

    def fetch_triangles(self) -> np.ndarray:
        k = C.c_uint64(0)
        lib = _native.trigpu()
        rc = lib.tl_fetch_triangles(self._p, None, 0, C.byref(k))
        if rc not in (TL_OK, TL_ERR_CAPACITY):
            _check(self._p, rc)
        out = np.empty((k.value, 3), dtype=np.uint32)
        _check(self._p, lib.tl_fetch_triangles(self._p, out.ctypes.data, k.value, C.byref(k)))
        return out

    def fetch_vertex_counts(self, n: int) -> np.ndarray:
        out = np.zeros(n, dtype=np.uint64)
        _check(self._p, _native.trigpu().tl_fetch_vertex_counts(self._p, out.ctypes.data))
        return out

    def fetch_oriented(self, n: int, m: int):
        so = np.empty(n + 1, dtype=np.uint64)
        s = np.empty(max(m, 1), dtype=np.uint32)
        po = np.empty(n + 1, dtype=np.uint64)
        p = np.empty(max(m, 1), dtype=np.uint32)
        _check(self._p, _native.trigpu().tl_fetch_oriented(self._p, so.ctypes.data, s.ctypes.data,
                                                           po.ctypes.data, p.ctypes.data))
        return so, s[:m], po, p[:m]

    def cost_report(self) -> np.ndarray:
        out = np.zeros(4, dtype=np.uint64)
        _check(self._p, _native.trigpu().tl_cost_report(self._p, out.ctypes.data))
        return out

    def timer_start(self) -> None:
        _check(self._p, _native.trigpu().tl_timer_start(self._p))

    def timer_stop(self) -> float:
        ms = C.c_double(0.0)
        _check(self._p, _native.trigpu().tl_timer_stop(self._p, C.byref(ms)))
        return ms.value

    def debug_set(self, key: int, value: int) -> None:
        """Test-only knobs (tl_debug_set, include/trigpu.h): TL_DEBUG_BM_SHRINK, _VARIANT, _CLASS_WORK, _H_WIDE_MIN_N, _H_SPLIT."""
        _check(self._p, _native.trigpu().tl_debug_set(self._p, key, value))

    def phase_times(self) -> dict:
        lib = _native.trigpu()
        buf = (C.c_double * 32)()
        k = lib.tl_phase_times(self._p, buf, 32)
        return {lib.tl_phase_name(i).decode(): buf[i] for i in range(k)}

    def host_register(self, arr: np.ndarray) -> None:
        _check(self._p, _native.trigpu().tl_host_register(self._p, arr.ctypes.data, arr.nbytes))

    def host_unregister(self, arr: np.ndarray) -> None:
        _check(self._p, _native.trigpu().tl_host_unregister(self._p, arr.ctypes.data))


_default_ctx = None
_default_lock = threading.Lock()


def default_context() -> Context:
    global _default_ctx
    with _default_lock:
        if _default_ctx is None:
            _default_ctx = Context(0)
        return _default_ctx


# -- ListingStats and sinks ----------------------------------------------------

@dataclass
class ListingStats:
    """ListingStats (listing.hpp:23-34) plus the engine's extras."""

    triangle_count: int = 0
    inner_ops: int = 0
    mark_ops: int = 0
    wall_ms: float = 0.0  # listing kernels only (listing.hpp:113-116 analogue)
    checksum: int = 0
    orient_ms: float = 0.0
    c_pp: int = 0
    c_pm: int = 0
    kernel_launches: int = 0

    def merge(self, other: "ListingStats") -> None:
        self.triangle_count += other.triangle_count
        self.inner_ops += other.inner_ops
        self.mark_ops += other.mark_ops


class CountingSink:
    """listing.hpp:40-44."""

    flags = 0

    def __init__(self):
        self.count = 0

    def _absorb(self, ctx: Context, view: "OrientedView", st: TlStats):
        self.count += int(st.triangle_count)

    def merge(self, other: "CountingSink"):
        self.count += other.count


class ChecksumSink(CountingSink):
    """Order-independent checksum: wrapping sum over triangles of
    h(a) * h(b) * h(c) mod 2^64, h(v) = mix64(v) | 1, (a, b, c) the dense ids."""

    flags = TL_OUT_CHECKSUM

    def __init__(self):
        super().__init__()
        self.checksum = 0

    def _absorb(self, ctx, view, st):
        super()._absorb(ctx, view, st)
        self.checksum = (self.checksum + int(st.checksum)) % (1 << 64)

    def merge(self, other):
        super().merge(other)
        self.checksum = (self.checksum + other.checksum) % (1 << 64)


class VertexCountSink(CountingSink):
    """Per-vertex triangle counts t[x] (each triangle counts for its three
    vertices), uint64[n], dense ids."""

    flags = TL_OUT_VERTEX_COUNTS

    def __init__(self):
        super().__init__()
        self.counts = None

    def _absorb(self, ctx, view, st):
        super()._absorb(ctx, view, st)
        c = ctx.fetch_vertex_counts(view.vertex_count())
        self.counts = c if self.counts is None else self.counts + c

    def merge(self, other):
        super().merge(other)
        if other.counts is not None:
            self.counts = other.counts if self.counts is None else self.counts + other.counts


class CollectingSink(CountingSink):
    """listing.hpp:46-63: triangles as (u, v, w) dense ids, rank-ascending."""

    flags = TL_OUT_LIST

    def __init__(self):
        super().__init__()
        self._chunks = []

    @property
    def triangles(self) -> np.ndarray:
        if not self._chunks:
            return np.empty((0, 3), dtype=np.uint32)
        if len(self._chunks) > 1:
            self._chunks = [np.concatenate(self._chunks)]
        return self._chunks[0]

    def _absorb(self, ctx, view, st):
        super()._absorb(ctx, view, st)
        self._chunks.append(ctx.fetch_triangles())

    def merge(self, other):
        super().merge(other)
        self._chunks.extend(other._chunks)

    def canonical(self) -> np.ndarray:
        """listing.hpp:57-62: ids sorted inside each triple, list sorted."""
        t = np.sort(self.triangles, axis=1)
        if t.shape[0] == 0:
            return t
        order = np.lexsort((t[:, 2], t[:, 1], t[:, 0]))
        return t[order]


class CompositeSink(CountingSink):
    """Several sinks fed by one listing pass (flags OR-ed)."""

    def __init__(self, *sinks):
        super().__init__()
        self.sinks = sinks
        self.flags = 0
        for s in sinks:
            self.flags |= s.flags

    def _absorb(self, ctx, view, st):
        super()._absorb(ctx, view, st)
        for s in self.sinks:
            s._absorb(ctx, view, st)


# -- OrientedView + listing ------------------------------------------------------

class OrientedView:
    """GPU-resident oriented view (OrientedView, oriented_view.hpp:17-50).

    Construction runs the relabel/orient/CSR/sort kernels; the view stays on
    the device inside its context. Host accessors fetch the reference layout
    (dense ids, rank-ascending rows) lazily.
    """

    def __init__(self, g: Graph, pi: Ordering, ctx: Context | None = None):
        if pi.size() != g.vertex_count():
            raise ValueError("orient: ordering does not match graph")
        self.ctx = ctx or default_context()
        self.graph = g
        self.ordering = pi
        self._n = g.vertex_count()
        self._m = g.edge_count()
        self.ctx.orient(g.offsets, g.adjacency, pi.ranks)
        self._host = None
        self._token = object()
        self.ctx._current_view = self._token

    def _ensure_current(self):
        if getattr(self.ctx, "_current_view", None) is not self._token:
            # the context holds one view at a time; rebuild this one
            self.ctx.orient(self.graph.offsets, self.graph.adjacency, self.ordering.ranks)
            self.ctx._current_view = self._token

    def vertex_count(self) -> int:
        return self._n

    def edge_count(self) -> int:
        return self._m

    def _fetch(self):
        if self._host is None:
            self._ensure_current()
            self._host = self.ctx.fetch_oriented(self._n, self._m)
        return self._host

    def successors(self, u: int) -> np.ndarray:
        so, s, _, _ = self._fetch()
        return s[so[u]:so[u + 1]]

    def predecessors(self, u: int) -> np.ndarray:
        _, _, po, p = self._fetch()
        return p[po[u]:po[u + 1]]

    def out_degree(self, u: int) -> int:
        so = self._fetch()[0]
        return int(so[u + 1] - so[u])

    def in_degree(self, u: int) -> int:
        po = self._fetch()[2]
        return int(po[u + 1] - po[u])

    def rank_of(self, v: int) -> int:
        return int(self.ordering.ranks[v])

    def vertex_at(self, position: int) -> int:
        return int(self.ordering.sequence[position])

    def csr(self):
        """(succ_offsets, succ, pred_offsets, pred) in the reference layout."""
        return self._fetch()


def orient(g: Graph, pi: Ordering, ctx: Context | None = None) -> OrientedView:
    return OrientedView(g, pi, ctx)


def _run(algo: int, view_or_graph, pi_or_sink, sink=None) -> ListingStats:
    if isinstance(view_or_graph, Graph):
        view = OrientedView(view_or_graph, pi_or_sink)
    else:
        view = view_or_graph
        sink = pi_or_sink
    if sink is None:
        sink = CountingSink()
    view._ensure_current()
    st = view.ctx.list(algo, sink.flags)
    sink._absorb(view.ctx, view, st)
    return ListingStats(triangle_count=int(st.triangle_count), inner_ops=int(st.inner_ops),
                        mark_ops=int(st.mark_ops), wall_ms=float(st.list_ms),
                        checksum=int(st.checksum), orient_ms=float(st.orient_ms),
                        c_pp=int(st.c_pp), c_pm=int(st.c_pm),
                        kernel_launches=int(st.kernel_launches))


def list_app(view_or_graph, pi_or_sink=None, sink=None) -> ListingStats:
    """A++ (Algorithm 1; listing.hpp:69-86, 162-166, 175-178)."""
    return _run(APP, view_or_graph, pi_or_sink, sink)


def list_apm(view_or_graph, pi_or_sink=None, sink=None) -> ListingStats:
    """A+- (Algorithm 2; listing.hpp:91-107, 168-173, 180-183)."""
    return _run(APM, view_or_graph, pi_or_sink, sink)


def list_app_parallel(view: OrientedView, sink, threads: int) -> ListingStats:
    """listing.hpp:187-192; the GPU always runs all seeds in parallel, so
    ``threads`` only documents the caller's intent."""
    return _run(APP, view, sink)


def list_apm_parallel(view: OrientedView, sink, threads: int) -> ListingStats:
    """listing.hpp:194-199."""
    return _run(APM, view, sink)
