"""A/B timing of the listing kernels on one config (experiments, not the bench).

    python tools/ab.py [--config c4] [--algo apm] [--flags 1] [--variant 0] [--reps 5]

Select an experimental build with TRIGPU_LIB_SUFFIX. The ordering is computed
on the device (tl_order, bit-identical to the reference's degree / split
order). Prints one JSON line: mean per-phase device times over the reps.
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2203_04774_b200 as tg  # noqa: E402
from paper_2203_04774_b200._native import TL_DEBUG_VARIANT  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--ordering", default="degree")
ap.add_argument("--algo", default="apm")
ap.add_argument("--flags", type=int, default=1)
ap.add_argument("--variant", type=int, default=0)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
t0 = time.perf_counter()
g = bench.make_graph(bench.CONFIGS[a.config])
ctx = tg.Context(0)
rank = ctx.order(g.offsets, a.ordering)
gen_s = time.perf_counter() - t0
ctx.orient(g.offsets, g.adjacency, rank)
if a.variant:
    ctx.debug_set(TL_DEBUG_VARIANT, a.variant)
algo = 1 if a.algo == "apm" else 0
st = ctx.list(algo, a.flags)
ph = []
for _ in range(a.reps):
    st2 = ctx.list(algo, a.flags)
    assert st2.triangle_count == st.triangle_count or a.variant
    ph.append(ctx.phase_times())
mean = {k: round(statistics.mean(p[k] for p in ph), 3) for k in ph[0] if k.startswith("list") or k == "classify"}
C = st.inner_ops
B = 4 * (C + 2 * g.m)
print(json.dumps({"config": a.config, "ordering": a.ordering, "algo": a.algo, "flags": a.flags,
                  "variant": a.variant, "lib": os.environ.get("TRIGPU_LIB_SUFFIX", ""),
                  "T": st.triangle_count, "checksum": st.checksum, "C": C, "m": g.m,
                  "frac": B / (mean["list"] / 1e3) / 6550.1e9, "gen_s": round(gen_s, 1), **mean}), flush=True)
