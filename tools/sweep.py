"""Config sweep over BASELINE.json's configs (SURVEY §8d runs), on one B200.

    python tools/sweep.py [--out profiles/r01b_sweep.jsonl] [--only c1,c2] [--no-ref]

For every config: the orderings and algorithms the BASELINE config names,
timed on the GPU through the C-ABI (orient ms, list ms, algorithmic GB/s vs
the measured HBM peak), with the config's sinks. Cross-checks on every row:
count and checksum identical across orderings and algorithms (both are
ordering-independent: dense ids), inner_ops = c_pm / c_pp, Σ per-vertex counts
= 3T. Parity rows (`ref`) re-run the UNMODIFIED reference listing
(oracle/_ref: the reference's own OrientedView + list_apm/list_app loops with
a count/checksum/per-vertex-count sink, all host threads) on the same graph
and ordering and compare count, checksum and the per-vertex counts bit for bit.
Synthetic inputs: the seeded generators of csrc/host/trihost.cpp (C1 is the
reference's own gen_gnm), see DESIGN.md §5.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (configs, generators, peaks)

# (config, orderings, algorithms, sinks, reference-parity runs)
PLAN = [
    ("c1", ["degree", "core"], ["apm", "app"], "list+vcounts", [("degree", "apm"), ("core", "app")]),
    ("c3_1m", ["degree"], ["apm", "app"], "list+vcounts", [("degree", "apm")]),
    ("c2", ["degree", "core", "split", "check"], ["apm", "app"], "checksum+vcounts", [("degree", "apm")]),
    ("c3", ["degree"], ["apm", "app"], "checksum", [("degree", "apm")]),
    ("c4", ["degree", "split", "check"], ["apm", "app"], "checksum", [("degree", "apm")]),
]


def vc_digest(vc: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(vc, dtype=np.uint64).tobytes()).hexdigest()[:16]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01b_sweep.jsonl"))
    ap.add_argument("--only", default="")
    ap.add_argument("--no-ref", action="store_true")
    args = ap.parse_args()
    import oracle
    import paper_2203_04774_b200 as tg
    from paper_2203_04774_b200 import host
    from paper_2203_04774_b200._native import (TL_ALGO_APM, TL_ALGO_APP, TL_OUT_CHECKSUM, TL_OUT_LIST,
                                               TL_OUT_VERTEX_COUNTS)

    peak, _ = bench.load_peaks()
    only = set(filter(None, args.only.split(",")))
    out = open(args.out, "a")
    ctx = tg.Context(0)
    threads = os.cpu_count() or 1
    for name, orders, algos, sinks, ref_runs in PLAN:
        if only and name not in only:
            continue
        cfg = bench.CONFIGS[name]
        t0 = time.perf_counter()
        g = bench.make_graph(cfg)
        gen_s = time.perf_counter() - t0
        flags = TL_OUT_CHECKSUM | (TL_OUT_VERTEX_COUNTS if "vcounts" in sinks else 0) | \
            (TL_OUT_LIST if sinks.startswith("list") else 0)
        seen = {}
        for meth in orders:
            pi, order_ms = host.compute_order(g, meth)
            for algo_name in algos:
                algo = TL_ALGO_APM if algo_name == "apm" else TL_ALGO_APP
                ctx.orient(g.offsets, g.adjacency, pi.ranks)  # warm (allocations)
                ctx.list(algo, flags)
                ctx.orient(g.offsets, g.adjacency, pi.ranks)
                ph = ctx.phase_times()
                st = ctx.list(algo, flags)
                ph2 = ctx.phase_times()
                list_ms = ph2["list"]
                cost = ctx.cost_report().tolist()
                C = cost[1] if algo == TL_ALGO_APM else cost[0]
                B = 4 * (C + 2 * g.m)
                row = {"config": name, "desc": cfg["desc"], "n": g.n, "m": g.m, "ordering": meth,
                       "algo": algo_name, "sinks": sinks, "triangles": st.triangle_count,
                       "checksum": str(st.checksum), "inner_ops": st.inner_ops,
                       "inner_ops_ok": st.inner_ops == C and st.mark_ops == 2 * g.m,
                       "order_ms": round(order_ms, 3), "orient_ms": round(ph["relabel_count"] + ph["scan"] +
                                                                       ph["scatter"] + ph["segsort"] + ph["cost"], 3),
                       "list_ms": round(list_ms, 3),
                       "triangles_per_s": st.triangle_count / (list_ms / 1e3) if list_ms > 0 else None,
                       "algorithmic_GBps": B / (list_ms / 1e3) / 1e9 if list_ms > 0 else None,
                       "frac_of_measured_peak": B / (list_ms / 1e3) / 1e9 / peak if list_ms > 0 else None,
                       "gen_s": round(gen_s, 1)}
                if flags & TL_OUT_VERTEX_COUNTS:
                    vc = ctx.fetch_vertex_counts(g.n)
                    row["vcount_sum_ok"] = int(vc.sum()) == 3 * st.triangle_count
                    row["vcounts_sha"] = vc_digest(vc)
                if flags & TL_OUT_LIST:
                    tri = ctx.fetch_triangles()
                    row["list_len_ok"] = tri.shape[0] == st.triangle_count
                    can = oracle.canonical(tri)
                    row["list_sha"] = hashlib.sha256(can.tobytes()).hexdigest()[:16]
                    row["list_unique"] = bool(can.shape[0] == 0 or (np.diff(can.view(np.uint32).reshape(-1, 3)
                                                                             .astype(np.int64), axis=0) != 0)
                                              .any(axis=1).all())
                key = (st.triangle_count, str(st.checksum), row.get("vcounts_sha"), row.get("list_sha"))
                seen[(meth, algo_name)] = key
                row["agrees_across_runs"] = len(set(seen.values())) == 1
                if (meth, algo_name) in ref_runs and not args.no_ref:
                    t1 = time.perf_counter()
                    rg = oracle.RefGraph.from_csr(g.offsets, g.adjacency)
                    rv = oracle.RefView(rg, pi.ranks)
                    r = rv.list(algo, threads=threads, vcounts=bool(flags & TL_OUT_VERTEX_COUNTS))
                    ref_s = time.perf_counter() - t1
                    ok = r.triangle_count == st.triangle_count and r.checksum == st.checksum and \
                        r.inner_ops == st.inner_ops
                    if flags & TL_OUT_VERTEX_COUNTS:
                        ok = ok and vc_digest(r.vcounts) == row["vcounts_sha"]
                    row["reference_parity"] = bool(ok)
                    row["reference_s"] = round(ref_s, 1)
                    row["reference_threads"] = threads
                    del rv, rg
                print(json.dumps(row), flush=True)
                out.write(json.dumps(row) + "\n")
                out.flush()
    ctx.close()


if __name__ == "__main__":
    main()
