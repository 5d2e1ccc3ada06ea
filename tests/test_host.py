"""Host-side input preparation (libtrihost.so): generators and the reference's
orderings / cost report reached through it. CPU only."""
import os

import numpy as np
import pytest

import paper_2203_04774_b200 as tg
from paper_2203_04774_b200 import host
from golden_io import golden, sha


def test_gen_gnm_is_the_reference_generator_c1():
    g = tg.gen_gnm(100000, 1000000, 4242)
    assert (g.n, g.m) == (100000, 1000000)
    c1 = golden()["c1"]
    for meth in ("degree", "core", "split", "check"):
        pi, ms = host.compute_order(g, meth, 4242)
        assert sha(pi.ranks) == c1["orderings"][meth]["rank_sha256"]
        assert ms >= 0
    pi = tg.degree_order(g)
    c = tg.cost_report(g, pi)
    assert [c.c_pp, c.c_pm, c.c_mm, c.sum_deg_sq] == c1["orderings"]["degree"]["cost"]


@pytest.mark.parametrize("gen", [
    lambda: tg.gen_rmat(12, 16, 7),
    lambda: tg.gen_chung_lu(20000, 100000, seed=3),
    lambda: tg.gen_ws(5000, 8, 0.1, seed=5),
])
def test_generators_valid_and_deterministic(gen):
    a, b = gen(), gen()
    a.check_invariants()
    assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.adjacency, b.adjacency)


def test_generators_thread_count_independent(monkeypatch):
    monkeypatch.setenv("TRIHOST_THREADS", "1")
    a = tg.gen_rmat(11, 8, 3)
    monkeypatch.setenv("TRIHOST_THREADS", "5")
    b = tg.gen_rmat(11, 8, 3)
    assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.adjacency, b.adjacency)


def test_rmat_shape_and_skew():
    g = tg.gen_rmat(14, 16, 1)
    assert g.n == 1 << 14
    # symmetrised, deduplicated: fewer undirected edges than draws
    assert 0.5 * 16 * (1 << 14) < g.m < 16 * (1 << 14)
    deg = g.degrees()
    assert deg.max() > 20 * deg.mean()  # heavy hubs
    assert (deg == 0).sum() > 0         # isolated vertices kept


def test_ws_ring_structure():
    g = tg.gen_ws(1000, 32, 0.0, seed=1)  # no rewiring: exact ring lattice
    assert g.m == 1000 * 16
    assert (g.degrees() == 32).all()


def test_chung_lu_weights_capped():
    g = tg.gen_chung_lu(50000, 400000, wmax=100.0, seed=2)
    g.check_invariants()
    assert g.degrees().max() < 400


def test_orderings_match_reference_harness():
    import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    g = tg.gen_rmat(10, 8, 2)
    rg = oracle.RefGraph.from_csr(g.offsets, g.adjacency)
    for meth in tg.ORDERINGS:
        pi, _ = host.compute_order(g, meth, 9)
        assert np.array_equal(pi.ranks, rg.order(meth, 9)), meth
        c = tg.cost_report(g, pi)
        assert (c.c_pp, c.c_pm, c.c_mm, c.sum_deg_sq) == rg.cost(pi.ranks)


def test_from_dense_edges_and_accessors():
    g = tg.Graph.from_dense_edges(5, [[0, 1], [1, 2], [2, 0], [3, 4], [1, 0]])
    assert g.n == 5 and g.m == 4
    assert g.neighbors(0).tolist() == [1, 2]
    assert g.has_edge(2, 1) and not g.has_edge(0, 3)
    assert g.degree(1) == 2


def test_bench_csv_is_reference_schema():
    hdr = host.bench_csv_header()
    assert hdr == ("dataset,algo,ordering,mode,threads,n,m,c_pp,c_pm,inner_ops,triangles,"
                   "load_ms,order_ms,list_ms")
    row = host.bench_csv_row("x", "apm", "degree", "mere", 1, 3, 3, 5, 1, 1, 1, 0.0, 0.5, 1.25)
    assert row == "x,apm,degree,mere,1,3,3,5,1,1,1,0.000,0.500,1.250"


def test_unknown_ordering_raises():
    g = tg.gen_gnm(10, 10, 1)
    with pytest.raises(host.HostError):
        host.compute_order(g, "bogus")


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_bytes(text.encode() if isinstance(text, str) else text)
    return str(p)


def test_parse_edgelist_matches_reference_loader(tmp_path):
    """The native reader (th_parse_edgelist) + the reference's normalize equals
    the reference's own load_edgelist_file (graph.cpp:164-192): same n, m,
    loop / duplicate counts, CSR and labels, on the grammar's corner cases
    (CRLF, tabs, blank and '#' lines, negative and extreme labels, no final
    newline) and on a large multi-slice file."""
    import oracle
    rng = np.random.default_rng(5)
    cases = {
        "toy": "0 1\n0 2\n1 2\n2 3\n",  # cli_test.cpp's toy graph
        "crlf": "# header\r\n10\t-3\r\n\r\n-3 10\r\n  7   7  \r\n7 10",
        "extreme": f"{-2**63} {2**63 - 1}\n#c\n\t\n5 {-2**63}\n",
        "empty": "",
        "comments": "# only\n#\n",
    }
    lines = [f"{a} {b}" for a, b in rng.integers(-10**12, 10**12, size=(120_000, 2))]
    lines[::7] = [f"{a}\t{a}" for a in rng.integers(0, 50, size=len(lines[::7]))]
    cases["big"] = "\n".join(lines) + "\n"
    for name, text in cases.items():
        p = _write(tmp_path, name + ".txt", text)
        raw = tg.host.parse_edgelist(p)
        ref = tg.Graph.load(p)
        if raw.shape[0] == 0:
            assert ref.n == 0 and ref.m == 0
            continue
        rg, lo, du = oracle.RefGraph.normalize(raw)
        off, adj = rg.csr()
        assert (rg.n, rg.m, lo, du) == (ref.n, ref.m, ref.loops_removed, ref.duplicates_removed), name
        assert np.array_equal(off, ref.offsets) and np.array_equal(adj, ref.adjacency), name
        assert np.array_equal(rg.labels(), ref.labels), name


def test_parse_edgelist_errors_match_reference(tmp_path):
    """Bad lines raise the reference's ParseError text ("line N: ...",
    common.hpp:16-20, graph.cpp:180-183) for the FIRST bad line, also when
    it sits deep in a multi-slice file."""
    good = "\n".join(f"{i} {i + 1}" for i in range(300_000))
    for name, text in {
        "one_token": "1 2\n3\n",
        "trailing": "1 2\n3 4 5\n",
        "plus": "1 2\n+3 4\n",
        "word": "1 2\nx 4\n",
        "overflow": f"1 {2**63}\n",
        "deep": good + "\n1 2 3\n" + good + "\nbad\n",
        "percent": "% comment\n1 2\n",
    }.items():
        p = _write(tmp_path, name + ".txt", text)
        with pytest.raises(tg.host.HostError) as ours:
            tg.host.parse_edgelist(p)
        with pytest.raises(tg.host.HostError) as theirs:
            tg.Graph.load(p)
        assert str(ours.value) == str(theirs.value), name
    with pytest.raises(tg.host.HostError, match="cannot open"):
        tg.host.parse_edgelist(str(tmp_path / "missing.txt"))
