"""Full C5 parity record (profiles/r02_c5_parity.json): the complete R-MAT-27
listing on the GPU against the oracle restatement (oracle.c, listing.hpp:91-107
via run_parallel's block pulling, all host cores) on the same graph and the
same pi -- triangle count, checksum, inner_ops, mark_ops and every per-vertex
count. The degree order is restated with numpy (stable sort by degree,
ordering.cpp:66-96) and compared with the device ordering. Run on the GPU box:

    python tools/c5_parity.py > gpurun_out/c5_parity.json
"""
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2203_04774_b200 as tg  # noqa: E402
from paper_2203_04774_b200._native import TL_ALGO_APM, TL_OUT_CHECKSUM, TL_OUT_VERTEX_COUNTS  # noqa: E402

T0 = time.perf_counter()
log = lambda *a: print(f"[{time.perf_counter() - T0:7.1f}s]", *a, file=sys.stderr, flush=True)  # noqa: E731
threads = os.cpu_count() or 1
g = tg.gen_rmat(27, 16, 1)
log("generated", g.n, g.m)
deg = np.diff(g.offsets.astype(np.int64))
seq = np.argsort(deg, kind="stable")
ranks = np.empty(g.n, np.uint32)
ranks[seq] = np.arange(g.n, dtype=np.uint32)
del seq, deg
ctx = tg.Context(0)
dev_ranks_equal = bool(np.array_equal(ctx.order(g.offsets, "degree"), ranks))
ctx.orient(g.offsets, g.adjacency, ranks)
st = ctx.list(TL_ALGO_APM, TL_OUT_CHECKSUM | TL_OUT_VERTEX_COUNTS)
vc = ctx.fetch_vertex_counts(g.n)
gpu = {"triangle_count": st.triangle_count, "checksum": str(st.checksum), "inner_ops": st.inner_ops,
       "mark_ops": st.mark_ops, "vcounts_sha256": hashlib.sha256(vc.astype("<u8").tobytes()).hexdigest(),
       "list_ms": st.list_ms, "orient_ms": st.orient_ms}
log("gpu", gpu)
ctx.close()
view = oracle.orient(g.offsets, g.adjacency, ranks, threads=threads)
log("oracle view")
cost = oracle.cost(view)
t = time.perf_counter()
exp = oracle.list_triangles(view, oracle.APM, threads=threads, vcounts=True)
cpu_s = time.perf_counter() - t
ref = {"triangle_count": exp.triangle_count, "checksum": str(exp.checksum), "inner_ops": exp.inner_ops,
       "mark_ops": exp.mark_ops, "vcounts_sha256": hashlib.sha256(exp.vcounts.astype("<u8").tobytes()).hexdigest(),
       "wall_s": cpu_s, "threads": threads}
log("oracle", ref)
same = {k: gpu[k] == ref[k] for k in ("triangle_count", "checksum", "inner_ops", "mark_ops", "vcounts_sha256")}
print(json.dumps({"config": "c5 R-MAT scale 27, edge factor 16, seed 1", "n": g.n, "m": g.m,
                  "ordering": "degree (numpy restatement of ordering.cpp:66-96)",
                  "device_ordering_identical": dev_ranks_equal, "algo": "apm",
                  "c_pm": cost[1], "gpu": gpu, "oracle": ref, "match": same,
                  "vcounts_identical": bool(np.array_equal(vc, exp.vcounts)),
                  "bit_exact": all(same.values()) and dev_ranks_equal}))
