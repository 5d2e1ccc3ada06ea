"""Probe: box resources and the setup cost of C5 (R-MAT-27) on the host."""
import os, sys, time, resource, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

def rss():
    return resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6

def T(label, t0):
    print(f"{label}: {time.perf_counter()-t0:.1f} s  (maxrss {rss():.1f} GB)", flush=True)

print(subprocess.run("nproc; free -g; lscpu | head -20", shell=True, capture_output=True, text=True).stdout, flush=True)
import paper_2203_04774_b200 as tg
import oracle
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
t0 = time.perf_counter(); g = tg.gen_rmat(scale, 16, 1); T(f"gen_rmat({scale}) n={g.n} m={g.m}", t0)
t0 = time.perf_counter(); pi, oms = tg.compute_order(g, "degree"); T(f"reference degree order (incl. Graph build; order {oms:.0f} ms)", t0)
ctx = tg.Context(0)
t0 = time.perf_counter(); r = ctx.order(g.offsets, "degree"); T("gpu degree order", t0)
assert np.array_equal(r, pi.ranks)
t0 = time.perf_counter(); ctx.orient(g.offsets, g.adjacency, pi.ranks); st = ctx.list(1, 1); T(f"gpu orient+list T={st.triangle_count} list_ms={st.list_ms:.0f}", t0)
t0 = time.perf_counter(); so, s_, po, p_ = ctx.fetch_oriented(g.n, g.m); T("fetch_oriented", t0)
ctx.close()
t0 = time.perf_counter(); view = oracle.orient(g.offsets, g.adjacency, pi.ranks); T("oracle.orient (port, 1 thread)", t0)
assert np.array_equal(view.succ, s_); del so, s_, po, p_
t0 = time.perf_counter(); rg = oracle.RefGraph.from_csr(g.offsets, g.adjacency); T("oracle RefGraph.from_csr", t0)
t0 = time.perf_counter(); rv = oracle.RefView(rg, pi.ranks); T("oracle RefView (reference OrientedView ctor)", t0)
nb = 256; bs = (g.n + nb - 1) // nb
for b in (0, 3, 100, 200):
    t0 = time.perf_counter(); x = rv.list(1, threads=os.cpu_count(), rank_begin=b*bs, rank_end=(b+1)*bs); T(f"ref block {b}: ops={x.inner_ops} tri={x.triangle_count} wall_ms={x.wall_ms:.0f}", t0)
    t0 = time.perf_counter(); y = oracle.list_triangles(view, 1, threads=os.cpu_count(), rank_begin=b*bs, rank_end=(b+1)*bs); T(f"port block {b}: ops={y.inner_ops} tri={y.triangle_count}", t0)
    assert x.triangle_count == y.triangle_count and x.checksum == y.checksum
