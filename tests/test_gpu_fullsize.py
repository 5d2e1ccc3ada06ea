"""Full-size parity at the BASELINE configs, through the C-ABI, bit-exact.

* C5 (R-MAT-27, 2.1 B edges, 107 G triangles): the degree order restated
  with numpy (ordering.cpp:66-96: stable sort by degree) against the device
  ordering; the oriented view against the oracle's (or_orient_parallel, 16
  threads); per-seed-range listings (tl_list_range, the reference's
  run_apm_range over a rank range, listing.hpp:91-107) against the oracle on
  sampled ranges -- count, checksum, inner_ops, mark_ops, per-vertex counts;
  a partition of the ranks sums to the full listing; A++ = A+- (count,
  checksum, per-vertex counts); sum of per-vertex counts = 3T. (The complete
  C5 listing on the CPU takes ~15 minutes on the box's 16 cores, more than
  this suite's budget: tools/c5_parity.py runs it, profiles/r02_c5_parity.json.)
* C2 (Chung-Lu 4 M) in LIST mode + per-vertex counts against the UNMODIFIED
  reference (oracle/_ref, 16 threads): count, checksum, per-vertex counts,
  and the canonical triangle list (CollectingSink::canonical, listing.hpp:57-62)
  byte-identical, with its SHA-256.
* C3-1M (Watts-Strogatz, the config's full-list instance): canonical list.
* C3 (16 M, 256 M edges) and C4 (R-MAT-24): count, checksum, per-vertex counts
  against the reference for degree A+- (C4 also degree A++).
"""
import hashlib
import os

import numpy as np
import pytest

import oracle
import paper_2203_04774_b200 as tg
from paper_2203_04774_b200 import host
from paper_2203_04774_b200._native import (TL_ALGO_APM, TL_ALGO_APP, TL_OUT_CHECKSUM, TL_OUT_LIST,
                                           TL_OUT_VERTEX_COUNTS)

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
THREADS = os.cpu_count() or 1
CV = TL_OUT_CHECKSUM | TL_OUT_VERTEX_COUNTS


@pytest.fixture(scope="module")
def ctx():
    c = tg.Context(0)
    yield c
    c.close()


def degree_ranks_numpy(offsets):
    """degree_order (ordering.cpp:66-96): counting sort by degree, ascending,
    ties by ascending id == a stable sort of the degrees."""
    deg = np.diff(offsets.astype(np.int64))
    seq = np.argsort(deg, kind="stable")
    ranks = np.empty(seq.shape[0], np.uint32)
    ranks[seq] = np.arange(seq.shape[0], dtype=np.uint32)
    return ranks


def bit_reversed(nb):
    bits = (nb - 1).bit_length()
    return [int(format(i, f"0{bits}b")[::-1], 2) for i in range(nb)]


_C5 = {}  # C5's triangle count, checked against the oracle in test_c5_full_size


def test_c5_full_size(ctx):
    g = tg.gen_rmat(27, 16, 1)
    n, m = g.n, g.m
    ranks = degree_ranks_numpy(g.offsets)
    assert np.array_equal(ctx.order(g.offsets, "degree"), ranks)
    ctx.orient(g.offsets, g.adjacency, ranks)
    full = ctx.list(TL_ALGO_APM, CV)
    vc = ctx.fetch_vertex_counts(n)
    T = full.triangle_count
    assert T > 10**11 and int(vc.sum()) == 3 * T
    _C5["triangles"] = T
    view = oracle.orient(g.offsets, g.adjacency, ranks, threads=THREADS)
    assert ctx.cost_report().tolist() == list(oracle.cost(view))
    assert full.inner_ops == oracle.cost(view)[1] and full.mark_ops == 2 * m
    so, s, po, p = ctx.fetch_oriented(n, m)
    assert np.array_equal(so, view.succ_off) and np.array_equal(s, view.succ)
    assert np.array_equal(po, view.pred_off) and np.array_equal(p, view.pred)
    del so, s, po, p
    # sampled seed-rank ranges, bit-exact against the oracle
    nb = 256
    bs = (n + nb - 1) // nb
    checked, ops = 0, 0
    for b in bit_reversed(nb):
        lo, hi = b * bs, min(n, (b + 1) * bs)
        exp = oracle.list_triangles(view, oracle.APM, threads=THREADS, vcounts=checked < 2,
                                    rank_begin=lo, rank_end=hi)
        st = ctx.list_range(TL_ALGO_APM, CV, lo, hi)
        assert (st.triangle_count, st.checksum, st.inner_ops, st.mark_ops) == \
            (exp.triangle_count, exp.checksum, exp.inner_ops, exp.mark_ops), (lo, hi)
        if exp.vcounts is not None:
            assert np.array_equal(ctx.fetch_vertex_counts(n), exp.vcounts)
        checked += 1
        ops += exp.inner_ops
        if checked >= 8 and ops > 10**10:  # (suite time: the oracle lists ~1 % of C5 per range set)
            break
    # a partition of the rank space adds up to the full listing
    cuts = np.linspace(0, n, 17).astype(np.int64)
    tot, chk = 0, 0
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        st = ctx.list_range(TL_ALGO_APM, TL_OUT_CHECKSUM, int(lo), int(hi))
        tot += st.triangle_count
        chk = (chk + st.checksum) % (1 << 64)
    assert (tot, chk) == (T, full.checksum)
    # A++ lists the same triangles
    app = ctx.list(TL_ALGO_APP, CV)
    assert (app.triangle_count, app.checksum) == (T, full.checksum)
    assert np.array_equal(ctx.fetch_vertex_counts(n), vc)
    assert app.inner_ops == oracle.cost(view)[0]


def _reference(g, meth):
    rg = oracle.RefGraph.from_csr(g.offsets, g.adjacency)
    r = rg.order(meth, 0)
    return rg, r, oracle.RefView(rg, r)


def _sha_canonical(tri):
    t = oracle.sort_triples(np.ascontiguousarray(tri, dtype=np.uint32), threads=THREADS)
    return t, hashlib.sha256(memoryview(t).cast("B")).hexdigest()


def test_c2_list_mode_vs_reference(ctx):
    g = tg.gen_chung_lu(4_000_000, 64_000_000, seed=1)
    rg, r, rv = _reference(g, "degree")
    ctx.orient(g.offsets, g.adjacency, r)
    st = ctx.list(TL_ALGO_APM, TL_OUT_CHECKSUM | TL_OUT_VERTEX_COUNTS | TL_OUT_LIST)
    vc = ctx.fetch_vertex_counts(g.n)
    tri = ctx.fetch_triangles()
    assert tri.shape[0] == st.triangle_count > 10**9
    # every emitted triple is rank-ascending (listing.hpp:36-38)
    assert (r[tri[:, 0]] < r[tri[:, 1]]).all() and (r[tri[:, 1]] < r[tri[:, 2]]).all()
    exp = rv.list(oracle.APM, threads=THREADS, vcounts=True, collect=True, tri_cap=st.triangle_count)
    assert (st.triangle_count, st.checksum, st.inner_ops, st.mark_ops) == \
        (exp.triangle_count, exp.checksum, exp.inner_ops, exp.mark_ops)
    assert np.array_equal(vc, exp.vcounts)
    got, h_got = _sha_canonical(tri)
    del tri
    want, h_want = _sha_canonical(exp.triangles)
    assert h_got == h_want and np.array_equal(got, want)
    print(f"C2 list: {st.triangle_count} triangles, canonical sha256 {h_got}")


def test_c3_1m_list_vs_reference(ctx):
    g = tg.gen_ws(1_000_000, 32, 0.1, seed=1)
    rg, r, rv = _reference(g, "degree")
    ctx.orient(g.offsets, g.adjacency, r)
    for algo, ralgo in ((TL_ALGO_APM, oracle.APM), (TL_ALGO_APP, oracle.APP)):
        st = ctx.list(algo, TL_OUT_CHECKSUM | TL_OUT_VERTEX_COUNTS | TL_OUT_LIST)
        exp = rv.list(ralgo, threads=THREADS, vcounts=True, collect=True, tri_cap=st.triangle_count)
        assert (st.triangle_count, st.checksum, st.inner_ops) == (exp.triangle_count, exp.checksum, exp.inner_ops)
        assert np.array_equal(ctx.fetch_vertex_counts(g.n), exp.vcounts)
        got, h1 = _sha_canonical(ctx.fetch_triangles())
        want, h2 = _sha_canonical(exp.triangles)
        assert h1 == h2 and np.array_equal(got, want)


@pytest.mark.parametrize("cfg", ["c3", "c4"])
def test_full_size_counts_vs_reference(ctx, cfg):
    g = tg.gen_ws(16_000_000, 32, 0.1, seed=1) if cfg == "c3" else tg.gen_rmat(24, 16, 1)
    # (split A+- at full C4 size costs a second reference view + listing, ~2 minutes of the suite's
    # budget: tools/sweep.py runs it; here split order is checked against the degree-order results
    # at full size in test_gpu_parity.py::test_full_size_c4_properties and against the oracle on
    # the scaled configs)
    runs = [("degree", TL_ALGO_APM)] + ([("degree", TL_ALGO_APP)] if cfg == "c4" else [])
    rg = oracle.RefGraph.from_csr(g.offsets, g.adjacency)
    for meth in dict.fromkeys(m for m, _ in runs):
        r = rg.order(meth, 0)
        rv = oracle.RefView(rg, r)
        ctx.orient(g.offsets, g.adjacency, r)
        assert ctx.cost_report().tolist() == list(rg.cost(r))
        for _, algo in (x for x in runs if x[0] == meth):
            st = ctx.list(algo, CV)
            exp = rv.list(oracle.APM if algo == TL_ALGO_APM else oracle.APP, threads=THREADS, vcounts=True)
            assert (st.triangle_count, st.checksum, st.inner_ops, st.mark_ops) == \
                (exp.triangle_count, exp.checksum, exp.inner_ops, exp.mark_ops), (cfg, meth, algo)
            assert np.array_equal(ctx.fetch_vertex_counts(g.n), exp.vcounts)
        del rv


def test_c5_raw_edge_list_normalize(ctx):
    """tl_normalize at C5 scale: the 2^31 raw R-MAT-27 draws (loops and
    duplicates kept, more than 2^31 endpoints) through the device normalize
    (graph.cpp:115-151 + from_dense_edges :13-56) give gen_rmat(27)'s graph
    restricted to its non-isolated vertices: labels = those vertex ids,
    degrees and rows equal after mapping dense ids back through the labels;
    the device-resident graph then orients and lists C5's triangles."""
    # the normalize scratch is 48 B per raw edge (103 GB here): release the module
    # context's C2-C5 buffers first (this is the module's last test; close() is idempotent)
    ctx.close()
    raw = host.gen_rmat_raw(27, 16, 1)
    k = raw.shape[0]
    assert 2 * k > 2**31
    loops_expected = int(np.count_nonzero(raw[:, 0] == raw[:, 1]))
    c = tg.Context(0)
    try:
        n, m, lo, du = c.normalize(raw)
        del raw
        g = tg.gen_rmat(27, 16, 1)
        deg = np.diff(g.offsets.astype(np.int64))
        assert (m, lo, du) == (g.m, loops_expected, k - loops_expected - g.m)
        off, adj, labels = c.fetch_graph()
        assert np.array_equal(labels, np.flatnonzero(deg))
        assert np.array_equal(np.diff(off.astype(np.int64)), deg[labels])
        step = 1 << 28
        for i in range(0, adj.shape[0], step):
            assert np.array_equal(labels[adj[i:i + step]], g.adjacency[i:i + step].astype(np.int64)), i
        del off, adj
        c.orient_normalized("degree")
        st = c.list(TL_ALGO_APM, TL_OUT_CHECKSUM)
    finally:
        c.close()
    # isolated vertices carry no triangles, and the checksum hashes dense ids of
    # the normalized graph: compare counts with the full C5 listing
    if "triangles" not in _C5:  # this test run on its own
        c2 = tg.Context(0)
        try:
            c2.orient(g.offsets, g.adjacency, degree_ranks_numpy(g.offsets))
            _C5["triangles"] = c2.list(TL_ALGO_APM, 0).triangle_count
        finally:
            c2.close()
    assert st.triangle_count == _C5["triangles"]
