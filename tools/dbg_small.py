import numpy as np, sys
sys.path.insert(0, '.')
import paper_2203_04774_b200 as tg
g = tg.gen_gnm(4, 6, 0)
for rep in range(2):
    c = tg.Context(0)
    c.orient(g.offsets, g.adjacency, np.arange(4, dtype=np.uint32))
    for f in ([4, 4, 5, 6, 0, 4] if rep == 0 else [0, 1, 2, 4]):
        st = c.list(1, f)
        print(rep, 'apm', f, st.triangle_count, st.kernel_launches, flush=True)
    c.close()
g = tg.gen_gnm(60, 400, 11)
c = tg.Context(0)
pi = tg.degree_order(g)
c.orient(g.offsets, g.adjacency, pi.ranks)
for f in (0, 4, 0, 4):
    print('g60', f, c.list(1, f).triangle_count, c.list(0, f).triangle_count)
