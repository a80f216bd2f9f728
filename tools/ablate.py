"""time C4 f64/f32 with an alternative library build (argv[1] = path to .so)"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_04192_b200 import capi
if len(sys.argv) > 1:
    capi._lib = capi.load_library(sys.argv[1])
from paper_2507_04192_b200 import init_scene
from paper_2507_04192_b200.presets import c4_column3d
from paper_2507_04192_b200.solver import Context
for dt in ("f64", "f32"):
    s = c4_column3d(dt); st = init_scene(s); ctx = Context(s, st.particles.size()); ctx.upload(st)
    ctx.advance(3); ms = ctx.advance_timed(20)
    ctx.profile(True); ctx.advance(2)
    print(sys.argv[1:] , dt, "%.3f ms/step" % (ms / 20), {k: round(ctx.profile_query(k)[0] / 2, 3) for k in ("k_p2g", "k_g2p", "k_grid")}, flush=True)
    ctx.close()
