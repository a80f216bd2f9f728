"""P2G phase breakdown at C4, steady state. argv = dtype, then library builds compiled with
-DP2G_ABL=bits: they launch an ablated copy of k_p2g_pipe3 ("k_p2g_abl"; 1 skip reduce, 2 skip
convert, 4 skip march, 8 none) in front of the real one, whose output overwrites it, so the
simulation stays valid and the ablated copy sees the same sorted inputs as the real kernel."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_04192_b200 import capi, init_scene
from paper_2507_04192_b200.presets import c4_column3d
from paper_2507_04192_b200.solver import Context

dt = sys.argv[1]
s = c4_column3d(dt)
st = init_scene(s)
for so in sys.argv[2:]:
    capi._lib = capi.load_library(str(Path(so).resolve()))
    ctx = Context(s, st.particles.size())
    ctx.upload(st)
    ctx.advance(5)
    ctx.profile(True)
    ctx.profile_reset()
    ctx.advance(10)
    r = {k: ctx.profile_query(k) for k in ("k_p2g_abl", "k_p2g", "k_g2p_abl", "k_g2p")}
    print(Path(so).name, dt, {k: round(v[0] / max(v[1], 1), 4) for k, v in r.items()}, flush=True)
    ctx.close()
