"""A/B timing of listing-kernel builds on one config (experiments, not the bench).

    python tools/ab.py [--config c4] [--libs base,_c1r4] [--flags 1] [--algo apm] [--reps 5]

Generates the graph once; for each library variant (lib/libtrigpu<suffix>.so,
"base" = lib/libtrigpu.so) orients, lists `reps` times and prints one JSON line
of mean per-phase device times. The ordering is computed on the device
(tl_order, bit-identical to the reference's degree / split order).
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_2203_04774_b200 as tg  # noqa: E402
from paper_2203_04774_b200 import _native  # noqa: E402
from paper_2203_04774_b200._native import (TL_DEBUG_CLASS_WORK, TL_DEBUG_H_SPLIT, TL_DEBUG_H_WIDE_MIN_N,
                                           TL_DEBUG_VARIANT)  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--ordering", default="degree")
ap.add_argument("--algo", default="apm")
ap.add_argument("--flags", default="1")
ap.add_argument("--libs", default="base")
ap.add_argument("--variant", type=int, default=0)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--class-work", action="store_true", help="report per-class inner_ops and GB/s")
ap.add_argument("--hsplit", default="", help="comma list of TL_DEBUG_H_SPLIT values to time (per library)")
ap.add_argument("--hwide-min-n", type=int, default=-1, help="TL_DEBUG_H_WIDE_MIN_N (0: class H always CTA-wide)")
a = ap.parse_args()
t0 = time.perf_counter()
g = bench.make_graph(bench.CONFIGS[a.config])
gen_s = time.perf_counter() - t0
ranks = None
algo = 1 if a.algo == "apm" else 0
ref = None
for lib in a.libs.split(","):
    _native.use_library_variant("" if lib == "base" else lib)
    ctx = tg.Context(0)
    if ranks is None:
        ranks = ctx.order(g.offsets, a.ordering)
    ctx.orient(g.offsets, g.adjacency, ranks)
    ctx.orient(g.offsets, g.adjacency, ranks)  # second call: buffers allocated, orient_ms is warm
    if a.variant:
        ctx.debug_set(TL_DEBUG_VARIANT, a.variant)
    if a.class_work:
        ctx.debug_set(TL_DEBUG_CLASS_WORK, 1)
    if a.hwide_min_n >= 0:
        ctx.debug_set(TL_DEBUG_H_WIDE_MIN_N, a.hwide_min_n)
    splits = [int(x) for x in a.hsplit.split(",")] if a.hsplit else [None]
    for flags, hsplit in ((int(f), sp) for f in a.flags.split(",") for sp in splits):
        if hsplit is not None:
            ctx.debug_set(TL_DEBUG_H_SPLIT, hsplit)
        st = ctx.list(algo, flags)
        if ref is None:
            ref = st.triangle_count
        assert st.triangle_count == ref or a.variant, (lib, st.triangle_count, ref)
        ph = []
        for _ in range(a.reps):
            st2 = ctx.list(algo, flags)
            assert st2.triangle_count == st.triangle_count and st2.checksum == st.checksum
            ph.append(ctx.phase_times())
        mean = {k: round(statistics.mean(p[k] for p in ph), 3) for k in ph[0]
                if k.startswith("list") or k.startswith("sort_") or k in ("classify", "in_csr")}
        if a.class_work:
            for c in ("R", "H", "C1", "C2", "G"):
                w = ph[-1]["work_" + c]
                mean["work_" + c] = int(w)
                if mean["list_" + c] > 0:
                    mean["gbs_" + c] = round(4 * w / (mean["list_" + c] / 1e3) / 1e9, 1)
        B = 4 * (st.inner_ops + 2 * g.m)
        print(json.dumps({"config": a.config, "ordering": a.ordering, "algo": a.algo, "flags": flags,
                          "variant": a.variant, "lib": lib, "hwide_min_n": a.hwide_min_n, "hsplit": hsplit, "T": st.triangle_count, "checksum": st.checksum,
                          "C": st.inner_ops, "m": g.m, "frac": round(B / (mean["list"] / 1e3) / 6550.1e9, 4),
                          "orient_ms": round(st.orient_ms, 2), "gen_s": round(gen_s, 1), **mean}), flush=True)
    ctx.close()
