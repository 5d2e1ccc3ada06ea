"""Generate the golden parity fixtures from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libtrilist_ref.so, i.e. the
reference sources under /root/reference):

    python tests/golden/make_golden.py

Outputs (committed):
  golden.json   named known-answer cases: the literals the reference's own
                tests assert (listing_test.cpp, cost_test.cpp, graph_test.cpp,
                cli_test.cpp, acceptance_main.cpp) are checked here against the
                reference build before being written, plus the reference's
                outputs (counts, inner_ops, checksum, per-vertex counts,
                canonical lists) on those graphs; and the C1 config
                gen_gnm(100000, 1000000, 4242) per ordering.
  sweep.npz     acceptance criteria 1-3 sweep (acceptance_main.cpp:116-149):
                200 random_small_graph(seed, 60, 400) x 7 orderings, with the
                reference's costs and listing results.

Every value comes from running the reference core (listing.hpp templates,
cost.cpp, ordering.cpp, oracle.cpp brute_triangles) through the harness.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from oracle import RefGraph, RefView  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
ORDERS7 = ["identity", "random", "degree", "core", "split", "check", "neigh"]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def edges_of(g: RefGraph):
    off, adj = g.csr()
    out = []
    for u in range(g.n):
        for v in adj[off[u]:off[u + 1]]:
            if u < v:
                out.append([int(u), int(v)])
    return out


def run_case(name, g: RefGraph, orders, seed=0, lists=True):
    case = {"name": name, "n": g.n, "m": g.m, "edges": edges_of(g), "orderings": {}}
    brute = g.brute(guard=10**6) if g.n <= 2000 else None
    if brute is not None:
        case["brute"] = brute.tolist()
    for meth, oseed in orders:
        r = g.order(meth, oseed)
        v = RefView(g, r)
        c = g.cost(r)
        ent = {"method": meth, "seed": oseed, "ranks": r.tolist(),
               "cost": {"c_pp": c[0], "c_pm": c[1], "c_mm": c[2], "sum_deg_sq": c[3]}}
        for algo, an in ((0, "app"), (1, "apm")):
            res = v.list(algo, threads=1, vcounts=True, collect=lists)
            e = {"triangle_count": res.triangle_count, "inner_ops": res.inner_ops,
                 "mark_ops": res.mark_ops, "checksum": str(res.checksum),
                 "vcounts": res.vcounts.tolist()}
            if lists:
                e["emitted"] = res.triangles.tolist()  # single-threaded emission order
                e["canonical"] = oracle.canonical(res.triangles).tolist()
            ent[an] = e
        so, s, po, p = v.csr()
        ent["view"] = {"succ_off": so.tolist(), "succ": s.tolist(), "pred_off": po.tolist(),
                       "pred": p.tolist()}
        case["orderings"][f"{meth}:{oseed}"] = ent
    return case


def main():
    if not oracle.ref_available():
        sys.exit("oracle/_ref/libtrilist_ref.so missing: run `make oracle` first")
    cases = []
    # listing_test.cpp:15-25 (K3 identity: 1 triangle, app inner 5, apm inner 1)
    k3 = RefGraph.gnm(3, 3, 0)
    c = run_case("K3", k3, [("identity", 0)])
    o = c["orderings"]["identity:0"]
    assert o["app"]["triangle_count"] == 1 and o["app"]["inner_ops"] == 5
    assert o["apm"]["triangle_count"] == 1 and o["apm"]["inner_ops"] == 1
    # cost_test.cpp:11-18
    assert o["cost"] == {"c_pp": 5, "c_pm": 1, "c_mm": 5, "sum_deg_sq": 12}
    c["asserted_by"] = "listing_test.cpp:15-25; cost_test.cpp:11-18"
    cases.append(c)
    # listing_test.cpp:26-31 / oracle_test.cpp:14 (K4: 4 triangles)
    c = run_case("K4", RefGraph.gnm(4, 6, 0), [("identity", 0)])
    assert c["orderings"]["identity:0"]["apm"]["triangle_count"] == 4
    assert c["orderings"]["identity:0"]["app"]["triangle_count"] == 4
    c["asserted_by"] = "listing_test.cpp:26-31"
    cases.append(c)
    # listing_test.cpp:32-39 (edgeless: 0 / 0 / 0)
    c = run_case("edgeless", RefGraph.gnm(10, 0, 0), [("identity", 0)])
    e = c["orderings"]["identity:0"]["apm"]
    assert e["triangle_count"] == 0 and e["inner_ops"] == 0 and e["mark_ops"] == 0
    c["asserted_by"] = "listing_test.cpp:32-39"
    cases.append(c)
    # oracle_test.cpp:16-17 (5-cycle: 0 triangles)
    c = run_case("C5cycle", RefGraph.from_edges(5, [[0, 1], [1, 2], [2, 3], [3, 4], [0, 4]]),
                 [("identity", 0), ("degree", 0)])
    assert c["orderings"]["identity:0"]["apm"]["triangle_count"] == 0
    c["asserted_by"] = "oracle_test.cpp:16-17"
    cases.append(c)
    # cost_test.cpp:19-25 (path 1-0-2, middle first: c_pp 4, c_pm 0)
    c = run_case("path_mid_first", RefGraph.from_edges(3, [[0, 1], [0, 2]]), [("identity", 0)])
    assert c["orderings"]["identity:0"]["cost"]["c_pp"] == 4
    assert c["orderings"]["identity:0"]["cost"]["c_pm"] == 0
    c["asserted_by"] = "cost_test.cpp:19-25"
    cases.append(c)
    # graph_test.cpp:146-160 (orient triangle / star degrees)
    c = run_case("orient_triangle", RefGraph.from_edges(3, [[0, 1], [0, 2], [1, 2]]), [("identity", 0)])
    so = c["orderings"]["identity:0"]["view"]["succ_off"]
    assert [so[i + 1] - so[i] for i in range(3)] == [2, 1, 0]
    c["asserted_by"] = "graph_test.cpp:146-153"
    cases.append(c)
    c = run_case("orient_star", RefGraph.from_edges(4, [[0, 1], [0, 2], [0, 3]]), [("identity", 0)])
    so = c["orderings"]["identity:0"]["view"]["succ_off"]
    assert so[1] - so[0] == 3
    c["asserted_by"] = "graph_test.cpp:154-159"
    cases.append(c)
    # cli_test.cpp:66-67, 127-137 (toy graph 0 1, 0 2, 1 2, 2 3: one triangle "0 1 2")
    c = run_case("cli_toy", RefGraph.from_edges(4, [[0, 1], [0, 2], [1, 2], [2, 3]]),
                 [("degree", 0), ("identity", 0)])
    assert c["orderings"]["degree:0"]["apm"]["canonical"] == [[0, 1, 2]]
    c["asserted_by"] = "cli_test.cpp:66-67, 127-137"
    cases.append(c)
    # listing_test.cpp:42-62 (G(25,90,3), random pi seed 17)
    c = run_case("gnm_25_90_3", RefGraph.gnm(25, 90, 3), [("random", 17)])
    c["asserted_by"] = "listing_test.cpp:42-62"
    cases.append(c)
    # listing_test.cpp:64-78 (G(60,400,11) x 6 orderings vs brute force) + neigh
    c = run_case("gnm_60_400_11", RefGraph.gnm(60, 400, 11),
                 [("identity", 0), ("random", 1), ("degree", 0), ("core", 0), ("split", 0),
                  ("check", 0), ("neigh", 0)])
    for k, o in c["orderings"].items():
        assert o["app"]["canonical"] == c["brute"] and o["apm"]["canonical"] == c["brute"], k
    c["asserted_by"] = "listing_test.cpp:64-78"
    cases.append(c)
    # listing_test.cpp:80-93 (random_graph(seed, 40, 200), random pi seed+7)
    for seed in range(20):
        g = RefGraph.random_small(seed, 40, 200)
        c = run_case(f"random_graph_{seed}", g, [("random", seed + 7)])
        o = c["orderings"][f"random:{seed + 7}"]
        assert o["app"]["inner_ops"] == o["cost"]["c_pp"] and o["apm"]["inner_ops"] == o["cost"]["c_pm"]
        assert o["app"]["mark_ops"] == 2 * g.m
        c["asserted_by"] = "listing_test.cpp:80-93"
        cases.append(c)
    # listing_test.cpp:95-118 (G(300,2500,5), degree; parallel == single)
    g = RefGraph.gnm(300, 2500, 5)
    c = run_case("gnm_300_2500_5", g, [("degree", 0)])
    r = g.order("degree")
    par = RefView(g, r).list(1, threads=4)
    assert par.triangle_count == c["orderings"]["degree:0"]["apm"]["triangle_count"]
    c["asserted_by"] = "listing_test.cpp:95-118"
    cases.append(c)
    # graph_test.cpp:161-176 (G(50,200,123), random pi seed 5)
    c = run_case("gnm_50_200_123", RefGraph.gnm(50, 200, 123), [("random", 5)])
    c["asserted_by"] = "graph_test.cpp:161-176"
    cases.append(c)

    # C1: gen_gnm(100000, 1000000, 4242) (acceptance_main.cpp:449), every ordering
    g = RefGraph.gnm(100000, 1000000, 4242)
    c1 = {"n": g.n, "m": g.m, "seed": 4242, "orderings": {}}
    for meth in ORDERS7:
        r = g.order(meth, 4242)
        v = RefView(g, r)
        cst = g.cost(r)
        ent = {"rank_sha256": sha(r), "cost": list(cst)}
        for algo, an in ((0, "app"), (1, "apm")):
            res = v.list(algo, threads=1, vcounts=True, collect=True)
            assert res.inner_ops == (cst[0] if algo == 0 else cst[1])
            ent[an] = {"triangle_count": res.triangle_count, "inner_ops": res.inner_ops,
                       "mark_ops": res.mark_ops, "checksum": str(res.checksum),
                       "vcounts_sha256": sha(res.vcounts.astype("<u8")),
                       "canonical_sha256": sha(oracle.canonical(res.triangles).astype("<u4"))}
        c1["orderings"][meth] = ent
    assert c1["orderings"]["degree"]["apm"]["triangle_count"] == 1338

    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump({"generated_by": "tests/golden/make_golden.py (reference core via oracle/_ref)",
                   "cases": cases, "c1": c1}, f, separators=(",", ":"))

    # acceptance criteria 1-3 sweep
    E, EO, N, R, RES = [], [0], [], [], []
    for seed in range(200):
        g = RefGraph.random_small(seed, 60, 400)
        off, adj = g.csr()
        ed = [(u, int(v)) for u in range(g.n) for v in adj[off[u]:off[u + 1]] if u < v]
        E.extend(ed)
        EO.append(len(E))
        N.append(g.n)
        brute = g.brute()
        for meth in ORDERS7:
            r = g.order(meth, seed)
            v = RefView(g, r)
            cst = g.cost(r)
            row = [seed, ORDERS7.index(meth)] + list(cst)
            for algo in (0, 1):
                res = v.list(algo, collect=True)
                assert (oracle.canonical(res.triangles) == brute).all()
                row += [res.triangle_count, res.inner_ops, res.mark_ops, res.checksum]
            RES.append(row)
            R.append(np.pad(r, (0, 60 - g.n)))
    np.savez_compressed(os.path.join(OUT, "sweep.npz"), edges=np.array(E, np.uint32).reshape(-1, 2),
                        edge_off=np.array(EO, np.int64), n=np.array(N, np.uint32),
                        ranks=np.array(R, np.uint32), results=np.array(RES, np.uint64))
    print("wrote", os.path.join(OUT, "golden.json"), "and sweep.npz")


if __name__ == "__main__":
    main()
