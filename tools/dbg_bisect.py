"""Find seed-rank ranges where a library variant disagrees with the base build (debugging aid).

    python tools/dbg_bisect.py <suffix> [scale]
One context at a time (engine calls go to the currently selected library).
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2203_04774_b200 as tg
from paper_2203_04774_b200 import _native

suffix = sys.argv[1]
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 22
g = tg.gen_rmat(scale, 16, 1)
n = g.n
ranks = None


def counts(lib, ranges, reps=1):
    global ranks
    _native.use_library_variant(lib)
    c = tg.Context(0)
    if ranks is None:
        ranks = c.order(g.offsets, "degree")
    c.orient(g.offsets, g.adjacency, ranks)
    out = [[c.list_range(1, 1, lo, hi).triangle_count for lo, hi in ranges] for _ in range(reps)]
    c.close()
    return out


full = [(0, n)]
print("base full", counts("", full, 2), "variant full", counts(suffix, full, 3), flush=True)
src = np.repeat(np.arange(n, dtype=np.int64), np.diff(g.offsets.astype(np.int64)))
outdeg = np.bincount(ranks[src][ranks[g.adjacency] > ranks[src]], minlength=n)
print("n", n, "max d+", outdeg.max(), "C1 seeds", int(((outdeg > 256) & (outdeg <= 1024)).sum()), flush=True)
ranges = [(0, n)]
for rnd in range(8):
    sub = []
    for lo, hi in ranges:
        k = min(16, hi - lo)
        edges = [lo + (hi - lo) * i // k for i in range(k + 1)]
        sub += [(edges[i], edges[i + 1]) for i in range(k) if edges[i + 1] > edges[i]]
    a = counts("", sub)[0]
    b = counts(suffix, sub)[0]
    bad = [r for r, x, y in zip(sub, a, b) if x != y]
    print("round", rnd, "ranges", len(sub), "bad", len(bad), bad[:4], flush=True)
    if not bad:
        break
    ranges = bad[:4]
    if all(hi - lo == 1 for lo, hi in ranges):
        for lo, hi in ranges:
            print("seed rank", lo, "d+", int(outdeg[lo]), flush=True)
        print("repeat variant on these seeds", counts(suffix, ranges, 4), "base", counts("", ranges, 1))
        break
