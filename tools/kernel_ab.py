"""Per-kernel A/B of library builds at C4 (steady state, profile mode: CUDA events around each launch).
usage: python tools/kernel_ab.py <f64|f32> <kernel[,kernel...]> <lib.so> [<lib.so> ...]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_04192_b200 import capi, init_scene
from paper_2507_04192_b200.presets import c4_column3d
from paper_2507_04192_b200.solver import Context

dt, names = sys.argv[1], sys.argv[2].split(",")
s = c4_column3d(dt)
st = init_scene(s)
for so in sys.argv[3:]:
    capi._lib = capi.load_library(str(Path(so).resolve()))
    ctx = Context(s, st.particles.size())
    ctx.upload(st)
    ctx.advance(5)
    ctx.profile(True)
    ctx.profile_reset()
    ctx.advance(20)
    r = {k: ctx.profile_query(k) for k in names}
    print(Path(so).name, dt, {k: round(v[0] / max(v[1], 1), 4) for k, v in r.items()}, flush=True)
    ctx.close()
