"""Diagnostic: C4 k_g2p time with the fused constitutive update (advance) vs without (phase g2p)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_04192_b200 import init_scene  # noqa: E402
from paper_2507_04192_b200.presets import c4_column3d  # noqa: E402
from paper_2507_04192_b200.solver import Context  # noqa: E402

s = c4_column3d(sys.argv[1] if len(sys.argv) > 1 else "f64")
st = init_scene(s)
ctx = Context(s, st.particles.size())
ctx.upload(st)
ctx.advance(5)
ctx.profile(True)
for name, fn in (("advance", lambda: ctx.advance(1)),
                 ("phases", lambda: (ctx.p2g(), ctx.grid_momentum_update(), ctx.grid_corrections(), ctx.g2p(),
                                     ctx.constitutive()))):
    ctx.profile_reset()
    for _ in range(5):
        fn()
    out = {}
    for k in ("k_p2g", "k_grid", "k_g2p", "k_constitutive"):
        t, c = ctx.profile_query(k)
        if c:
            out[k] = round(t / c, 4)
    print(name, out)
