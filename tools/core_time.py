"""Time tl_core_decompose on the BASELINE configs and check it at full size.

    python tools/core_time.py c2 c4 [c5]
For each config: device k-core decomposition (H2D inside), coreness / degeneracy against
the oracle's bucket-queue restatement of core_decompose (ordering.cpp:141-188), the
degeneracy-order property d+(v) <= coreness(v), and the A+- listing under the device core
order against the degree-order listing (count, checksum). One JSON line per config.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
import oracle
import paper_2203_04774_b200 as tg

for cfg in sys.argv[1:]:
    g = bench.make_graph(bench.CONFIGS[cfg])
    ctx = tg.Context(0)
    ctx.core_decompose(g.offsets[:2].copy() * 0, np.zeros(0, np.uint32))  # warm the context
    t0 = time.perf_counter()
    rank, core, dg = ctx.core_decompose(g.offsets, g.adjacency)
    dev_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, c0, d0 = oracle.core_decompose(g.offsets, g.adjacency)
    cpu_s = time.perf_counter() - t0
    ok_core = bool(np.array_equal(core, c0)) and dg == d0
    src = np.repeat(np.arange(g.n, dtype=np.uint32), np.diff(g.offsets.astype(np.int64)))
    later = rank[g.adjacency] > rank[src]
    dplus = np.bincount(src[later], minlength=g.n)
    ok_order = bool(np.all(dplus <= core)) and bool(np.array_equal(np.sort(rank), np.arange(g.n, dtype=np.uint32)))
    del src, later
    ctx.orient(g.offsets, g.adjacency, rank)
    a = ctx.list(1, 1)
    ctx.orient(g.offsets, g.adjacency, ctx.order(g.offsets, "degree"))
    b = ctx.list(1, 1)
    print(json.dumps({"config": cfg, "n": g.n, "m": g.m, "degeneracy": dg, "device_core_s": round(dev_s, 3),
                      "cpu_bucket_queue_s": round(cpu_s, 3), "coreness_equal": ok_core, "order_valid": ok_order,
                      "max_dplus": int(dplus.max()), "list_core_ms": round(a.list_ms, 2), "c_pm_core": a.inner_ops,
                      "list_degree_ms": round(b.list_ms, 2), "c_pm_degree": b.inner_ops,
                      "same_triangles": (a.triangle_count, a.checksum) == (b.triangle_count, b.checksum)}), flush=True)
    ctx.close()
