"""GPU-backed callers of the listing path: the reference CLI's ``list`` and
``bench`` commands (tools/trilist_cli.cpp:101-139 ``run_listing``, :192-228
``cmd_list``, :230-256 ``cmd_bench``) over the sm_100a engine.

    python -m paper_2203_04774_b200.cli list  GRAPH [--order degree] [--algo apm]
                                              [--mode mere|full] [--sink count|collect]
                                              [--out TRIANGLES] [--device-order]
    python -m paper_2203_04774_b200.cli bench GRAPH [--orderings degree,core]
                                              [--algos app,apm] [--repeats 1]

GRAPH is a text edge list read by the reference's own loader
(load_edgelist_file, graph.cpp:164-192). Orderings are the reference's code
(ordering.cpp / neigh.cpp). Each listing is one ``BenchRecord`` row in the
reference's CSV schema (bench.hpp:28-30), formatted by the reference's
``to_csv_row`` (bench.cpp:7-19); ``list_ms`` is the wall time of the
orientation + listing, as run_listing times OrientedView + list_* (the host
to device copy of the graph is inside it). ``--out`` writes one triangle per
line as original labels, rank-ascending inside each triple, like
trilist_cli.cpp:212-220; rows come in the device's emission order (the
reference's parallel listing has no fixed order either, listing.hpp:185-186).
The threads option of the reference does not apply (the listing is always
the whole GPU); records report threads = 0.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

from . import host
from ._native import TL_ALGO_APM, TL_ALGO_APP, TL_OUT_LIST
from .engine import Context

# trilist_cli.cpp:47-48
METHODS = ("identity", "random", "degree", "core", "split", "check", "neigh")


def dataset_name(path: str) -> str:
    """trilist_cli.cpp dataset_name: file name without directory and extension."""
    base = os.path.basename(path)
    return base.rsplit(".", 1)[0] if "." in base else base


def load(path: str):
    t0 = time.perf_counter()
    g = host.Graph.load(path)
    return g, (time.perf_counter() - t0) * 1e3


DEVICE_METHODS = ("degree", "split", "core")


def compute_order(ctx: Context, g, method: str, seed: int, device_order: bool):
    """compute_order (trilist_cli.cpp:50-64): the reference's host code, or with
    --device-order the engine's degree / split ordering (bit-identical ranks) and
    k-core degeneracy ordering (tl_core_decompose). Returns (ranks, order_ms)."""
    if device_order and method in DEVICE_METHODS:
        t0 = time.perf_counter()
        ranks = ctx.core_decompose(g.offsets, g.adjacency)[0] if method == "core" else ctx.order(g.offsets, method)
        return ranks, (time.perf_counter() - t0) * 1e3
    pi, order_ms = host.compute_order(g, method, seed)
    return pi.ranks, order_ms


def run_listing(ctx: Context, g, ranks, dataset: str, algo: str, ordering: str, mode: str,
                load_ms: float, order_ms: float, collect: bool) -> tuple[str, object]:
    """run_listing (trilist_cli.cpp:101-139): one BenchRecord CSV row."""
    t0 = time.perf_counter()
    ctx.orient(g.offsets, g.adjacency, ranks)
    st = ctx.list(TL_ALGO_APP if algo == "app" else TL_ALGO_APM, TL_OUT_LIST if collect else 0)
    list_ms = (time.perf_counter() - t0) * 1e3
    row = host.bench_csv_row(dataset, algo, ordering, mode, 0, g.n, g.m, st.c_pp, st.c_pm, st.inner_ops,
                             st.triangle_count, load_ms, order_ms, list_ms)
    return row, st


def cmd_list(args) -> int:
    g, load_ms = load(args.graph)
    collect = args.sink == "collect" or bool(args.out)
    ctx = Context(args.device)
    try:
        ranks, order_ms = compute_order(ctx, g, args.order, args.seed, args.device_order)
        row, st = run_listing(ctx, g, ranks, dataset_name(args.graph), args.algo, args.order, args.mode,
                              load_ms, order_ms, collect)
        if args.out:
            with open(args.out, "w") as f:
                for chunk in ctx.iter_triangles(labels=g.labels):
                    f.write("".join(f"{a} {b} {c}\n" for a, b, c in chunk.tolist()))
    finally:
        ctx.close()
    print(f"# sink {'collect' if collect else 'count'}")
    print(host.bench_csv_header())
    print(row)
    if args.mode == "full":
        t = [float(x) for x in row.split(",")[-3:]]
        print(f"# full_time_ms {sum(t)}")
    return 0


def cmd_bench(args) -> int:
    g, load_ms = load(args.graph)
    orderings = args.orderings.split(",") if args.orderings else list(METHODS)
    algos = args.algos.split(",") if args.algos else ["app", "apm"]
    print(host.bench_csv_header())
    ctx = Context(args.device)
    try:
        for method in orderings:
            ranks, order_ms = compute_order(ctx, g, method, args.seed, args.device_order)
            for algo in algos:
                for _ in range(args.repeats):
                    row, _ = run_listing(ctx, g, ranks, dataset_name(args.graph), algo, method, "full",
                                         load_ms, order_ms, False)
                    print(row, flush=True)
    finally:
        ctx.close()
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="trigpu", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    pl = sub.add_parser("list")
    pl.add_argument("graph")
    pl.add_argument("--order", default="degree", choices=METHODS)
    pl.add_argument("--seed", type=int, default=0)
    pl.add_argument("--algo", default="apm", choices=["app", "apm"])
    pl.add_argument("--mode", default="mere", choices=["mere", "full"])
    pl.add_argument("--sink", default="count", choices=["count", "collect"])
    pl.add_argument("--out", default="")
    pl.add_argument("--device", type=int, default=0)
    pl.add_argument("--device-order", action="store_true", help="degree / split / core ordering on the GPU")
    pb = sub.add_parser("bench")
    pb.add_argument("graph")
    pb.add_argument("--orderings", default="")
    pb.add_argument("--algos", default="")
    pb.add_argument("--repeats", type=int, default=1)
    pb.add_argument("--seed", type=int, default=0)
    pb.add_argument("--device", type=int, default=0)
    pb.add_argument("--device-order", action="store_true", help="degree / split / core ordering on the GPU")
    args = ap.parse_args(argv)
    try:
        return cmd_list(args) if args.cmd == "list" else cmd_bench(args)
    except Exception as e:  # the reference CLI prints the error and exits 1 (trilist_cli.cpp:510-513)
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
