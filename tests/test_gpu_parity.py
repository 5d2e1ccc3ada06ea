"""GPU parity: the sm_100a engine against the oracle and the reference's golden
vectors, through the C-ABI (Context -> tl_* calls). Bit-exact for every
integer output: triangle_count, inner_ops, mark_ops, checksum, per-vertex
counts, canonical triangle lists and the oriented-view rows.
"""
import os
import subprocess

import numpy as np
import pytest

import oracle
import paper_2203_04774_b200 as tg
from paper_2203_04774_b200 import host
from paper_2203_04774_b200._native import (TL_ALGO_APM, TL_ALGO_APP, TL_DEBUG_BM_SHRINK, TL_DEBUG_H_SPLIT,
                                           TL_DEBUG_H_WIDE_MIN_N, TL_OUT_CHECKSUM, TL_OUT_LIST,
                                           TL_OUT_VERTEX_COUNTS)
from golden_io import case_csr, cases, golden, sha, sweep_graphs

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ALL = TL_OUT_CHECKSUM | TL_OUT_VERTEX_COUNTS | TL_OUT_LIST


@pytest.fixture(scope="module")
def ctx():
    c = tg.Context(0)
    yield c
    c.close()


def canon(t):
    return oracle.canonical(t)


def run_all_sinks(ctx, algo, n):
    st = ctx.list(algo, ALL)
    tri = ctx.fetch_triangles()
    vc = ctx.fetch_vertex_counts(n)
    return st, tri, vc


@pytest.mark.parametrize("case", cases(), ids=lambda c: c["name"])
def test_golden_cases(ctx, case):
    off, adj = case_csr(case)
    n, m = case["n"], case["m"]
    for key, ent in case["orderings"].items():
        r = np.array(ent["ranks"], np.uint32)
        ctx.orient(off, adj, r)
        so, s, po, p = ctx.fetch_oriented(n, m)
        gv = ent["view"]
        assert so.tolist() == gv["succ_off"] and s.tolist() == gv["succ"], key
        assert po.tolist() == gv["pred_off"] and p.tolist() == gv["pred"], key
        assert ctx.cost_report().tolist() == [ent["cost"][k] for k in ("c_pp", "c_pm", "c_mm", "sum_deg_sq")]
        for algo, an in ((TL_ALGO_APP, "app"), (TL_ALGO_APM, "apm")):
            exp = ent[an]
            st, tri, vc = run_all_sinks(ctx, algo, n)
            assert st.triangle_count == exp["triangle_count"], (key, an)
            assert st.inner_ops == exp["inner_ops"] and st.mark_ops == exp["mark_ops"]
            assert str(st.checksum) == exp["checksum"]
            assert vc.tolist() == exp["vcounts"]
            assert canon(tri).tolist() == exp["canonical"]
            # every emitted triple is rank-ascending (listing.hpp:36-38)
            if tri.shape[0]:
                assert (r[tri[:, 0]] < r[tri[:, 1]]).all() and (r[tri[:, 1]] < r[tri[:, 2]]).all()
            # count-only and checksum-only passes agree with the fused pass
            assert ctx.list(algo, 0).triangle_count == exp["triangle_count"]
            assert str(ctx.list(algo, TL_OUT_CHECKSUM).checksum) == exp["checksum"]


def test_acceptance_sweep(ctx):
    """acceptance criteria 1-3 (acceptance_main.cpp:116-149) on the GPU."""
    checks = 0
    for gi, n, off, adj, rows in sweep_graphs():
        brute = oracle.brute(off, adj)
        for oi, r, row in rows:
            ctx.orient(off, adj, r)
            assert ctx.cost_report().tolist() == row[2:6]
            for algo, base in ((TL_ALGO_APP, 6), (TL_ALGO_APM, 10)):
                st = ctx.list(algo, TL_OUT_CHECKSUM | TL_OUT_LIST)
                assert [st.triangle_count, st.inner_ops, st.mark_ops, st.checksum] == row[base:base + 4]
                assert (canon(ctx.fetch_triangles()) == brute).all()
                checks += 1
    assert checks == 2800


@pytest.mark.parametrize("meth", ["identity", "random", "degree", "core", "split", "check", "neigh"])
def test_c1_config(ctx, meth):
    """BASELINE config C1: gen_gnm(100000, 1000000, 4242), both algorithms, full list."""
    g = tg.gen_gnm(100000, 1000000, 4242)
    pi, _ = host.compute_order(g, meth, 4242)
    ent = golden()["c1"]["orderings"][meth]
    assert sha(pi.ranks) == ent["rank_sha256"]
    ctx.orient(g.offsets, g.adjacency, pi.ranks)
    assert ctx.cost_report().tolist() == ent["cost"]
    for algo, an in ((TL_ALGO_APP, "app"), (TL_ALGO_APM, "apm")):
        st, tri, vc = run_all_sinks(ctx, algo, g.n)
        e = ent[an]
        assert st.triangle_count == e["triangle_count"] == 1338
        assert st.inner_ops == e["inner_ops"]
        assert str(st.checksum) == e["checksum"]
        assert sha(vc.astype("<u8")) == e["vcounts_sha256"]
        assert sha(canon(tri).astype("<u4")) == e["canonical_sha256"]


def _oracle_check(ctx, g, pi, algos=(TL_ALGO_APP, TL_ALGO_APM), lists=True, threads=8):
    view = oracle.orient(g.offsets, g.adjacency, pi.ranks)
    ctx.orient(g.offsets, g.adjacency, pi.ranks)
    assert ctx.cost_report().tolist() == list(oracle.cost(view))
    so, s, po, p = ctx.fetch_oriented(g.n, g.m)
    assert np.array_equal(so, view.succ_off) and np.array_equal(s, view.succ)
    assert np.array_equal(po, view.pred_off) and np.array_equal(p, view.pred)
    for algo in algos:
        exp = oracle.list_triangles(view, algo, threads=threads, vcounts=True, collect=lists)
        flags = TL_OUT_CHECKSUM | TL_OUT_VERTEX_COUNTS | (TL_OUT_LIST if lists else 0)
        st = ctx.list(algo, flags)
        assert st.triangle_count == exp.triangle_count
        assert st.inner_ops == exp.inner_ops and st.mark_ops == exp.mark_ops
        assert st.checksum == exp.checksum
        assert np.array_equal(ctx.fetch_vertex_counts(g.n), exp.vcounts)
        if lists:
            assert np.array_equal(canon(ctx.fetch_triangles()), canon(exp.triangles))


# scaled-down instances of C2-C5 (same generators and recipes), every ordering
# class the configs use; sizes chosen so the oracle finishes in seconds
SCALED = {
    "rmat16": lambda: tg.gen_rmat(16, 16, 1),
    "chung_lu_200k": lambda: tg.gen_chung_lu(200000, 3200000, seed=1),
    "ws_200k": lambda: tg.gen_ws(200000, 32, 0.1, seed=1),
}


@pytest.mark.parametrize("gname", list(SCALED))
@pytest.mark.parametrize("meth", ["degree", "core", "split", "check", "neigh"])
def test_scaled_configs_vs_oracle(ctx, gname, meth):
    g = SCALED[gname]()
    pi, _ = host.compute_order(g, meth)
    _oracle_check(ctx, g, pi, lists=(meth in ("degree", "core")))


def test_giant_hubs_and_long_rows(ctx):
    """Hubs with degree > 4096 exercise the big-row sort and the class-G
    (global bitmap) seeds under every ordering that puts them early."""
    rng = np.random.default_rng(3)
    n = 30000
    hub_edges = [(0, v) for v in range(1, 20001)] + [(1, v) for v in range(2, 9000)]
    extra = rng.integers(0, n, size=(60000, 2))
    g = tg.Graph.from_dense_edges(n, np.concatenate([np.array(hub_edges), extra]))
    for pi in (tg.identity_order(g), host.compute_order(g, "split")[0], tg.degree_order(g)):
        _oracle_check(ctx, g, pi)


def test_giant_rows_shared_by_the_cta(ctx):
    """Class G seeds whose sets contain rows of more than 16 K elements: those
    rows are left to the whole CTA (every warp a share of each row's chunks)
    instead of one warp; under the identity order seed 0 (|S| = 6000) scans the
    30000- and 20000-element out-rows of vertices 1 and 2, and vertex 1 is a
    class G seed itself."""
    rng = np.random.default_rng(9)
    n = 40000
    e = [(0, v) for v in range(1, 6001)] + [(1, v) for v in range(2, 30002)] + [(2, v) for v in range(3, 20003)]
    extra = rng.integers(0, n, size=(80000, 2))
    g = tg.Graph.from_dense_edges(n, np.concatenate([np.array(e), extra]))
    for pi in (tg.identity_order(g), host.compute_order(g, "split")[0], tg.degree_order(g)):
        _oracle_check(ctx, g, pi)
    # both algorithms agree with brute-force counting on the hub triangles
    ctx.orient(g.offsets, g.adjacency, tg.identity_order(g).ranks)
    assert ctx.list(TL_ALGO_APM, 0).triangle_count == ctx.list(TL_ALGO_APP, 0).triangle_count


def test_dense_clique(ctx):
    n = 300
    e = np.array([(u, v) for u in range(n) for v in range(u + 1, n)])
    g = tg.Graph.from_dense_edges(n, e)
    view_pi = tg.random_order(g, 3)
    ctx.orient(g.offsets, g.adjacency, view_pi.ranks)
    for algo in (TL_ALGO_APP, TL_ALGO_APM):
        st = ctx.list(algo, TL_OUT_VERTEX_COUNTS)
        assert st.triangle_count == n * (n - 1) * (n - 2) // 6
        assert (ctx.fetch_vertex_counts(n) == (n - 1) * (n - 2) // 2).all()


def test_edge_cases(ctx):
    # empty graph, single vertex, edgeless
    for n in (0, 1, 7):
        g = tg.Graph.from_dense_edges(n, np.zeros((0, 2), np.uint32))
        ctx.orient(g.offsets, g.adjacency, np.arange(n, dtype=np.uint32))
        for algo in (TL_ALGO_APP, TL_ALGO_APM):
            st = ctx.list(algo, ALL)
            assert (st.triangle_count, st.inner_ops, st.mark_ops, st.checksum) == (0, 0, 0, 0)
            assert ctx.fetch_triangles().shape == (0, 3)
    g = tg.gen_gnm(20, 60, 1)
    with pytest.raises(ValueError):  # not a permutation
        ctx.orient(g.offsets, g.adjacency, np.zeros(20, np.uint32))
    with pytest.raises(ValueError):  # size mismatch (oriented_view.cpp:8-9)
        ctx.orient(g.offsets, g.adjacency, np.arange(19, dtype=np.uint32))
    bad = g.adjacency.copy()
    bad[0], bad[1] = bad[1], bad[0]  # row not increasing: Graph invariant broken
    with pytest.raises(ValueError):
        ctx.orient(g.offsets, bad, np.arange(20, dtype=np.uint32))


def test_state_errors():
    c = tg.Context(0)
    with pytest.raises(tg.TrigpuError):
        c.list(TL_ALGO_APM, 0)  # no view yet
    g = tg.gen_gnm(10, 20, 2)
    c.orient(g.offsets, g.adjacency, np.arange(10, dtype=np.uint32))
    c.list(TL_ALGO_APM, 0)
    with pytest.raises(tg.TrigpuError):
        c.fetch_triangles()  # last run did not list
    c.close()


def test_python_mirror_api():
    """engine.py mirrors listing.hpp: views, sinks, overloads, stats."""
    g = tg.gen_gnm(300, 2500, 5)
    pi = tg.degree_order(g)
    view = tg.OrientedView(g, pi)
    cs, col, chk, vcs = tg.CountingSink(), tg.CollectingSink(), tg.ChecksumSink(), tg.VertexCountSink()
    st = tg.list_apm(view, cs)
    ref = oracle.list_triangles(oracle.orient(g.offsets, g.adjacency, pi.ranks), oracle.APM,
                                vcounts=True, collect=True)
    assert cs.count == st.triangle_count == ref.triangle_count
    assert st.mark_ops == 2 * g.m and st.inner_ops == tg.cost_report(g, pi).c_pm
    tg.list_app(view, col)
    assert np.array_equal(col.canonical(), oracle.canonical(ref.triangles))
    tg.list_apm_parallel(view, chk, 8)
    assert chk.checksum == ref.checksum
    tg.list_app(g, pi, vcs)  # (g, pi, sink) overload builds a temporary view
    assert np.array_equal(vcs.counts, ref.vcounts)
    assert view.successors(5).tolist() == oracle.orient(g.offsets, g.adjacency, pi.ranks).succ[
        oracle.orient(g.offsets, g.adjacency, pi.ranks).succ_off[5]:
        oracle.orient(g.offsets, g.adjacency, pi.ranks).succ_off[6]].tolist()
    with pytest.raises(ValueError):
        tg.OrientedView(g, tg.Ordering.identity(299))


def test_device_pointer_entry_point(ctx):
    """tl_orient_device: inputs already resident in HBM (torch tensors)."""
    import torch
    g = tg.gen_rmat(14, 16, 5)
    pi = tg.degree_order(g)
    d_off = torch.from_numpy(g.offsets.view(np.int64)).cuda()
    d_adj = torch.from_numpy(g.adjacency.view(np.int32)).cuda()
    d_rank = torch.from_numpy(pi.ranks.view(np.int32)).cuda()
    torch.cuda.synchronize()
    ctx.orient_device(g.n, g.m, d_off.data_ptr(), d_adj.data_ptr(), d_rank.data_ptr())
    st_dev = ctx.list(TL_ALGO_APM, TL_OUT_CHECKSUM)
    ctx.orient(g.offsets, g.adjacency, pi.ranks)
    st_host = ctx.list(TL_ALGO_APM, TL_OUT_CHECKSUM)
    assert (st_dev.triangle_count, st_dev.checksum) == (st_host.triangle_count, st_host.checksum)


def test_cpp_shim():
    """The reference's listing tests + acceptance 1-3 and 12 through include/trigpu.hpp."""
    exe = os.path.join(ROOT, "build", "shim_test")
    if not os.path.exists(exe):
        pytest.skip("build/shim_test not built (needs the reference sources at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


def test_full_size_c4_properties(ctx):
    """C4 (R-MAT-24, ef 16) at full size: size-independent properties --
    A++ and A+- agree on count, checksum and per-vertex counts; sum of
    per-vertex counts = 3T; inner_ops = cost; degree and split orderings list
    the same triangle set (same count and checksum)."""
    g = tg.gen_rmat(24, 16, 1)
    out = {}
    for meth in ("degree", "split"):
        pi, _ = host.compute_order(g, meth)
        ctx.orient(g.offsets, g.adjacency, pi.ranks)
        cost = ctx.cost_report()
        for algo in (TL_ALGO_APM, TL_ALGO_APP):
            st = ctx.list(algo, TL_OUT_CHECKSUM | TL_OUT_VERTEX_COUNTS)
            vc = ctx.fetch_vertex_counts(g.n)
            assert int(vc.sum()) == 3 * st.triangle_count
            assert st.inner_ops == (cost[1] if algo == TL_ALGO_APM else cost[0])
            out[(meth, algo)] = (st.triangle_count, st.checksum, vc)
    vals = list(out.values())
    for v in vals[1:]:
        assert v[0] == vals[0][0] and v[1] == vals[0][1] and np.array_equal(v[2], vals[0][2])


@pytest.mark.parametrize("shrink", [4, 8, 13])
def test_probe_filter_path(shrink):
    """Each seed's set is a windowed bitmap: exact when the set's rank span
    fits, otherwise a filter whose candidates are verified exactly.
    Shrinking every class's bitmap (tl_debug_set TL_DEBUG_BM_SHRINK) pushes the seeds of
    graphs small enough for the oracle through the filter + verification path
    with many false positives; results must not change."""
    c = tg.Context(0)
    c.debug_set(TL_DEBUG_BM_SHRINK, shrink)
    try:
        for g in (tg.gen_rmat(15, 16, 3), tg.gen_chung_lu(50000, 800000, seed=4)):
            for meth in ("degree", "split"):
                pi, _ = host.compute_order(g, meth)
                _oracle_check(c, g, pi, lists=False)
        case = next(x for x in cases() if x["name"] == "gnm_60_400_11")
        off, adj = case_csr(case)
        for key, ent in case["orderings"].items():
            c.orient(off, adj, np.array(ent["ranks"], np.uint32))
            for algo, an in ((TL_ALGO_APP, "app"), (TL_ALGO_APM, "apm")):
                st = c.list(algo, ALL)
                assert str(st.checksum) == ent[an]["checksum"]
                assert canon(c.fetch_triangles()).tolist() == ent[an]["canonical"]
    finally:
        c.close()


def test_wide_h_path():
    """Class H on the CTA-per-seed 2^19-window kernel and C1 on its 2^19-window
    instance (the paths graphs above 2^25 vertices take), forced on graphs the
    oracle checks in seconds, with and without shrunken windows (filter +
    verification path), and with class H split between the warp kernel (small
    sets, back of the list) and the CTA kernel (TL_DEBUG_H_SPLIT)."""
    c = tg.Context(0)
    c.debug_set(TL_DEBUG_H_WIDE_MIN_N, 0)
    try:
        for shrink, split in ((0, 0), (6, 96), (0, 256)):
            c.debug_set(TL_DEBUG_BM_SHRINK, shrink)
            c.debug_set(TL_DEBUG_H_SPLIT, split)
            for g in (tg.gen_rmat(16, 16, 5), tg.gen_chung_lu(100000, 1600000, seed=6)):
                for meth in ("degree", "split"):
                    pi, _ = host.compute_order(g, meth)
                    _oracle_check(c, g, pi, lists=(shrink == 0))
        with pytest.raises(ValueError):
            c.debug_set(TL_DEBUG_H_SPLIT, 257)
    finally:
        c.close()


@pytest.mark.parametrize("meth", ["degree", "split"])
def test_device_orderings_match_reference(meth):
    """tl_order (degree / split on the GPU) is bit-identical to the
    reference's degree_order / split_order (ordering.cpp:66-109), including
    the tie-breaks, and tl_orient_ordered lists the same triangles."""
    c = tg.Context(0)
    try:
        graphs = [tg.gen_gnm(0, 0, 1), tg.gen_gnm(1, 0, 1), tg.gen_gnm(60, 400, 11), tg.gen_rmat(14, 16, 2),
                  tg.gen_chung_lu(30000, 400000, seed=3), tg.gen_ws(20000, 16, 0.1, seed=5)]
        for case in cases():
            off, adj = case_csr(case)
            graphs.append(host.Graph(off, adj))
        for g in graphs:
            pi, _ = host.compute_order(g, meth)
            assert np.array_equal(c.order(g.offsets, meth), pi.ranks)
            if g.n == 0:
                continue
            c.orient_ordered(g.offsets, g.adjacency, meth)
            assert np.array_equal(c.fetch_ranks(g.n), pi.ranks)
            st = c.list(TL_ALGO_APM, TL_OUT_CHECKSUM)
            view = oracle.orient(g.offsets, g.adjacency, pi.ranks)
            exp = oracle.list_triangles(view, TL_ALGO_APM, threads=8)
            assert (st.triangle_count, st.checksum) == (exp.triangle_count, exp.checksum)
        with pytest.raises(ValueError):
            c.order(graphs[2].offsets, "core")
    finally:
        c.close()


def _succ_counts(g, rank):
    """d+ per vertex under pi: neighbours of larger rank."""
    src = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.offsets.astype(np.int64)))
    later = rank[g.adjacency] > rank[src]
    return np.bincount(src[later], minlength=g.n)


def test_device_core_decompose():
    """tl_core_decompose: coreness and degeneracy equal core_decompose
    (ordering.cpp:141-188; oracle.core_decompose is pinned to it swap for swap);
    the ranks are a permutation with the degeneracy-order property d+(v) <=
    coreness(v) (so max d+ = degeneracy, as under the reference's core order),
    monotone in coreness; listing under it gives the reference's results."""
    c = tg.Context(0)
    try:
        path = host.Graph(*_path_csr(30000))
        graphs = [tg.gen_gnm(1, 0, 1), tg.gen_gnm(5, 0, 1), tg.gen_gnm(60, 400, 11), path,
                  tg.gen_gnm(100000, 1000000, 4242), tg.gen_rmat(16, 16, 2), tg.gen_chung_lu(200000, 3000000, seed=3),
                  tg.gen_ws(50000, 16, 0.1, seed=5), _hub_graph()]
        for case in cases():
            off, adj = case_csr(case)
            graphs.append(host.Graph(off, adj))
        for g in graphs:
            rank, core, dg = c.core_decompose(g.offsets, g.adjacency)
            r0, c0, d0 = oracle.core_decompose(g.offsets, g.adjacency)
            assert np.array_equal(core, c0) and dg == d0
            assert np.array_equal(np.sort(rank), np.arange(g.n, dtype=np.uint32))
            dplus = _succ_counts(g, rank.astype(np.int64))
            assert np.all(dplus <= core)
            assert int(dplus.max(initial=0)) <= dg
            order = np.argsort(rank)
            assert np.all(np.diff(core[order].astype(np.int64)) >= 0)  # peeled level by level
            # same listing results as under the reference's own core order
            c.orient_ordered(g.offsets, g.adjacency, "core")
            assert np.array_equal(c.fetch_ranks(g.n), rank)
            for algo in (TL_ALGO_APM, TL_ALGO_APP):
                st = c.list(algo, TL_OUT_CHECKSUM | TL_OUT_VERTEX_COUNTS)
                vc = c.fetch_vertex_counts(g.n)
                view = oracle.orient(g.offsets, g.adjacency, r0)
                exp = oracle.list_triangles(view, algo, threads=8, vcounts=True)
                assert (st.triangle_count, st.checksum) == (exp.triangle_count, exp.checksum)
                assert np.array_equal(vc, exp.vcounts)
        with pytest.raises(ValueError):
            c.order(graphs[2].offsets, "core")  # offsets only: core needs the adjacency
    finally:
        c.close()


def _path_csr(n):
    """Path 0-1-...-(n-1): level 1 peels it from both ends, n/2 rounds."""
    deg = np.full(n, 2, np.uint64)
    deg[0] = deg[-1] = 1
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum(deg)
    adj = np.empty(2 * (n - 1), np.uint32)
    k = 0
    for v in range(n):
        if v > 0:
            adj[k] = v - 1
            k += 1
        if v < n - 1:
            adj[k] = v + 1
            k += 1
    return off, adj


def _hub_graph():
    """A 40-clique whose members also own 3000 leaves each (long rows, high levels)."""
    k, leaves = 40, 3000
    e = [(a, b) for a in range(k) for b in range(a + 1, k)]
    nxt = k
    for a in range(k):
        e += [(a, nxt + i) for i in range(leaves)]
        nxt += leaves
    return tg.Graph.from_dense_edges(nxt, np.array(e, np.uint32))


def test_device_normalize_matches_reference():
    """tl_normalize (raw labeled edges -> Graph CSR on the GPU) equals the
    reference's normalize (graph.cpp:115-151 + from_dense_edges :13-56):
    same n, m, loop / duplicate counts, offsets, sorted rows and labels; the
    device-resident graph then orients with a device ordering and lists the
    reference's triangles."""
    rng = np.random.default_rng(11)
    c = tg.Context(0)
    try:
        inputs = [np.zeros((0, 2), np.int64), np.array([[5, 5]], np.int64), np.array([[3, -7], [-7, 3]], np.int64)]
        for trial in range(12):
            k = int(rng.integers(1, 20000))
            pool = rng.integers(-2**62, 2**62, size=int(rng.integers(2, 3000)))
            raw = rng.choice(pool, size=(k, 2))
            raw[rng.integers(0, k, size=k // 8)] = raw[rng.integers(0, k, size=k // 8)]
            inputs.append(raw)
        g4 = tg.gen_rmat(14, 16, 4)  # a larger one: a real graph's edges, relabelled and shuffled
        e = np.stack([np.repeat(np.arange(g4.n), np.diff(g4.offsets.astype(np.int64))), g4.adjacency], 1)
        lab = rng.permutation(np.arange(g4.n, dtype=np.int64) * 1000003 - 5 * 10**9)
        inputs.append(rng.permutation(lab[e]))
        for raw in inputs:
            rg, loops, dups = oracle.RefGraph.normalize(raw)
            n, m, lo, du = c.normalize(raw)
            assert (n, m, lo, du) == (rg.n, rg.m, loops, dups)
            off, adj, labels = c.fetch_graph()
            o, a = rg.csr()
            assert np.array_equal(off, o) and np.array_equal(adj, a) and np.array_equal(labels, rg.labels())
            if n == 0 or m == 0:
                continue
            c.orient_normalized("degree")
            st = c.list(TL_ALGO_APM, TL_OUT_CHECKSUM)
            pi = rg.order("degree")
            exp = oracle.RefView(rg, pi).list(TL_ALGO_APM, threads=8)
            assert (st.triangle_count, st.checksum) == (exp.triangle_count, exp.checksum)
    finally:
        c.close()


def test_chunked_triangle_stream_with_labels():
    """tl_fetch_triangles_range / tl_fetch_triangle_labels stream the list in
    chunks; concatenated they equal tl_fetch_triangles, and mapped through
    the Graph's labels they equal the reference's labelled triangle set."""
    rng = np.random.default_rng(5)
    g = tg.gen_rmat(12, 16, 9)
    e = np.stack([np.repeat(np.arange(g.n), np.diff(g.offsets.astype(np.int64))), g.adjacency], 1)
    labels_of = rng.permutation(np.arange(g.n, dtype=np.int64) * 7919 - 10**6)
    raw = labels_of[e]
    c = tg.Context(0)
    try:
        n, m, _, _ = c.normalize(raw)
        off, adj, labels = c.fetch_graph()
        c.orient_normalized("degree")
        st = c.list(TL_ALGO_APM, TL_OUT_LIST)
        whole = c.fetch_triangles()
        parts = np.concatenate(list(c.iter_triangles(chunk=1000)))
        assert np.array_equal(parts, whole) and parts.shape[0] == st.triangle_count
        lab_parts = np.concatenate(list(c.iter_triangles(chunk=777, use_labels=True)))
        assert np.array_equal(lab_parts, labels[whole])
        lab2 = np.concatenate(list(c.iter_triangles(chunk=5000, labels=labels)))
        assert np.array_equal(lab2, lab_parts)
        rg, _, _ = oracle.RefGraph.normalize(raw)
        exp = oracle.RefView(rg, rg.order("degree")).list(TL_ALGO_APM, collect=True)
        exp_lab = np.sort(rg.labels()[exp.triangles], axis=1)
        got = np.sort(lab_parts, axis=1)
        assert np.array_equal(got[np.lexsort(got.T[::-1])], exp_lab[np.lexsort(exp_lab.T[::-1])])
    finally:
        c.close()


def test_cli_list_and_bench(tmp_path, capsys):
    """The reference CLI's list / bench (trilist_cli.cpp:101-256) over the GPU:
    cli_test.cpp's toy graph gives one triangle and the --out line "0 1 2";
    relabelled inputs come back as their original labels; rows follow the
    reference BenchRecord schema."""
    from paper_2203_04774_b200 import cli
    toy = tmp_path / "toy.txt"
    toy.write_text("0 1\n0 2\n1 2\n2 3\n")
    out = tmp_path / "tri.txt"
    assert cli.main(["list", str(toy), "--out", str(out)]) == 0
    text = capsys.readouterr().out.splitlines()
    assert text[0] == "# sink collect" and text[1] == host.bench_csv_header()
    row = text[2].split(",")
    assert row[0] == "toy" and row[1] == "apm" and row[10] == "1"
    assert out.read_text() == "0 1 2\n"
    # labelled input with loops / duplicates, every ordering, both algorithms
    rng = np.random.default_rng(4)
    g = tg.gen_gnm(300, 2500, 5)
    lab = rng.permutation(np.arange(300, dtype=np.int64) * 37 + 1000)
    e = np.stack([np.repeat(np.arange(g.n), np.diff(g.offsets.astype(np.int64))), g.adjacency], 1)
    lines = [f"{lab[a]} {lab[b]}" for a, b in e[::3]] + ["5000 5000"]
    src = tmp_path / "lab.txt"
    src.write_text("\n".join(lines) + "\n")
    rg, _, _ = oracle.RefGraph.normalize(np.array([[int(x) for x in l.split()] for l in lines], np.int64))
    for meth in ("degree", "core", "neigh"):
        for algo in ("app", "apm"):
            out2 = tmp_path / f"t_{meth}_{algo}.txt"
            assert cli.main(["list", str(src), "--order", meth, "--algo", algo, "--out", str(out2)]) == 0
            got = np.array([[int(x) for x in l.split()] for l in out2.read_text().splitlines()], np.int64)
            exp = rg.labels()[rg.brute()]
            assert got.shape == exp.shape
            g_sorted = np.sort(got, axis=1)
            assert np.array_equal(g_sorted[np.lexsort(g_sorted.T[::-1])],
                                  np.sort(exp, axis=1)[np.lexsort(np.sort(exp, axis=1).T[::-1])])
    capsys.readouterr()
    assert cli.main(["bench", str(src), "--orderings", "degree,split", "--algos", "app,apm"]) == 0
    rows = capsys.readouterr().out.splitlines()
    assert rows[0] == host.bench_csv_header() and len(rows) == 5
    assert len({r.split(",")[10] for r in rows[1:]}) == 1  # same triangle count every run
    # --device-order: degree / split rows are identical to the host-ordered ones (same ranks, so
    # same costs); core is a degeneracy ordering of its own but lists the same triangles
    assert cli.main(["bench", str(src), "--orderings", "degree,split,core", "--algos", "apm", "--device-order"]) == 0
    dev = capsys.readouterr().out.splitlines()
    assert len(dev) == 4 and {r.split(",")[10] for r in dev[1:]} == {rows[1].split(",")[10]}
    host_rows = {(r.split(",")[1], r.split(",")[2]): r.split(",")[6:11] for r in rows[1:]}
    for r in dev[1:3]:
        f = r.split(",")
        assert host_rows[(f[1], f[2])] == f[6:11]  # c_pp, c_pm, inner_ops, triangles (+ n/m columns before)
