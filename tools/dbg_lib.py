"""Compare a library variant with the base build on a small graph (debugging aid).

    python tools/dbg_lib.py <suffix> [scale]
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_04774_b200 as tg
from paper_2203_04774_b200 import _native
from paper_2203_04774_b200._native import TL_DEBUG_H_WIDE_MIN_N

suffix = sys.argv[1]
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 18
g = tg.gen_rmat(scale, 16, 1)
res = {}
for lib in ("", suffix):
    _native.use_library_variant(lib)
    ctx = tg.Context(0)
    ranks = ctx.order(g.offsets, "degree")
    ctx.orient(g.offsets, g.adjacency, ranks)
    ctx.debug_set(TL_DEBUG_H_WIDE_MIN_N, 0)
    for flags in (1, 3):
        st = ctx.list(1, flags)
        res[(lib, flags)] = (st.triangle_count, st.checksum)
        print(lib or "base", flags, st.triangle_count, st.checksum, ctx.phase_times()["list"], flush=True)
    ctx.close()
ok = all(res[("", f)] == res[(suffix, f)] for f in (1, 3))
print("MATCH" if ok else "MISMATCH")
