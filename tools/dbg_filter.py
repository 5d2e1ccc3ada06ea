"""Debug: filter-path parity per algo / flags / class (GPU box)."""
import os, sys
import numpy as np
sys.path.insert(0, '.')
import paper_2203_04774_b200 as tg
from paper_2203_04774_b200 import host
import oracle

shr = sys.argv[1] if len(sys.argv) > 1 else "4"
small = len(sys.argv) > 2
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
os.environ["TRIGPU_BM_SHRINK"] = shr
c = tg.Context(0)
graphs = ((("rmat11", tg.gen_rmat(11, 16, 3)),) if small else
          (("rmat15", tg.gen_rmat(15, 16, 3)), ("cl50k", tg.gen_chung_lu(50000, 800000, seed=4))))
for name, g in graphs * reps:
    for meth in ("degree", "split"):
        pi, _ = host.compute_order(g, meth)
        view = oracle.orient(g.offsets, g.adjacency, pi.ranks)
        c.orient(g.offsets, g.adjacency, pi.ranks)
        dout = np.diff(view.succ_off.astype(np.int64)); din = np.diff(view.pred_off.astype(np.int64))
        for algo in (0, 1):
            exp = oracle.list_triangles(view, algo, threads=8, vcounts=True)
            for flags in (0, 1, 2, 3):
                st = c.list(algo, flags)
                line = f"{name} {meth} algo{algo} F{flags}: cnt {st.triangle_count == exp.triangle_count}"
                if flags & 1: line += f" sum {st.checksum == exp.checksum}"
                if flags & 2:
                    vc = c.fetch_vertex_counts(g.n)
                    bad = np.nonzero(vc != exp.vcounts)[0]
                    line += f" vc_bad {len(bad)}"
                    if len(bad):
                        r = pi.ranks[bad].astype(np.int64)
                        dset = (dout if algo == 1 else din)[r]
                        line += f" set-deg of bad (rank space) {np.unique(dset)[:10]} diff {(vc[bad].astype(np.int64) - exp.vcounts[bad].astype(np.int64))[:8]}"
                print(line, flush=True)
c.close()
