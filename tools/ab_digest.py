"""A/B library builds at C4 steady state (k_p2g / k_g2p / step ms) and the state digest after 10
steps from the same upload (equal digests = bit-identical). argv: dtype, .so paths"""
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
    ctx.advance(10)
    dig = ctx.digest()
    ms = ctx.advance_timed(50) / 50
    ctx.profile(True)
    ctx.profile_reset()
    ctx.advance(10)
    r = {k: round(ctx.profile_query(k)[0] / max(ctx.profile_query(k)[1], 1), 4) for k in ("k_p2g", "k_g2p")}
    print(Path(so).name, dt, "step %.4f ms" % ms, r, "digest %x" % dig, flush=True)
    ctx.close()
