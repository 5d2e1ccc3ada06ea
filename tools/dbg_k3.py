import sys, numpy as np
sys.path.insert(0, '.')
import paper_2203_04774_b200 as tg
from paper_2203_04774_b200 import host
g = tg.Graph.from_dense_edges(3, [(0, 1), (0, 2), (1, 2)]) if hasattr(tg, 'Graph') else host.Graph.from_dense_edges(3, [(0, 1), (0, 2), (1, 2)])
c = tg.Context(0)
c.orient(g.offsets, g.adjacency, np.arange(3, dtype=np.uint32))
print(c.fetch_oriented(g.n, g.m))
g = tg.gen_gnm(60, 400, 11)
pi = tg.degree_order(g)
c.orient(g.offsets, g.adjacency, pi.ranks)
so, s, po, p = c.fetch_oriented(g.n, g.m)
import oracle
v = oracle.orient(g.offsets, g.adjacency, pi.ranks)
print(np.array_equal(so, v.succ_off), np.array_equal(s, v.succ), np.array_equal(po, v.pred_off), np.array_equal(p, v.pred))
bad = np.nonzero(s != v.succ)[0][:10]; print(bad, s[bad], v.succ[bad])
