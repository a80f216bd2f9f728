"""Run a few forward steps (and optionally one backprop) of a config, for ncu launch lists.
usage: python tools/launch_list.py C3 [steps] [adj_steps]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_04192_b200 import init_scene
from paper_2507_04192_b200.presets import CONFIGS
from paper_2507_04192_b200.seeders import LagrangianLeastSquares
from paper_2507_04192_b200.solver import Context

cfg = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
adj = int(sys.argv[3]) if len(sys.argv) > 3 else 0
s = CONFIGS[cfg](dtype="f64")
st = init_scene(s)
ctx = Context(s, st.particles.size())
ctx.upload(st)
ctx.advance(3)
ms = ctx.advance_timed(steps)
print(cfg, "%.4f ms/step" % (ms / steps))
if adj:
    st0 = ctx.download(st)
    sd = LagrangianLeastSquares([adj], st0.particles.x[None] + 1e-3, "x")
    c0, pg, res = ctx.backprop(st0, adj, 1, sd.desc())
    print(cfg, "backprop %.4f ms/step" % (res.device_ms / adj))
