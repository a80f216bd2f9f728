"""A/B library builds on the C4 fwd+adjoint: one 10-step single-segment backprop per build, per
kernel ms and the initial cotangent's checksum (equal = bit-identical). argv: .so paths"""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_04192_b200 import capi, init_scene
from paper_2507_04192_b200.presets import c4_column3d
from paper_2507_04192_b200.seeders import LagrangianLeastSquares
from paper_2507_04192_b200.solver import Context

s = c4_column3d("f64")
st = init_scene(s)
for so in sys.argv[1:]:
    capi._lib = capi.load_library(str(Path(so).resolve()))
    ctx = Context(s, st.particles.size())
    ctx.upload(st)
    ctx.advance(3)
    st0 = ctx.download(st)
    sd = LagrangianLeastSquares([10], st0.particles.x[None] + 1e-3, "x")
    ctx.backprop(st0, 10, 1, sd.desc())
    c0, pg, res = ctx.backprop(st0, 10, 1, sd.desc())
    ctx.profile(True)
    ctx.profile_reset()
    ctx.backprop(st0, 10, 1, sd.desc())
    r = {k: round(ctx.profile_query(k)[0] / max(ctx.profile_query(k)[1], 1), 4)
         for k in ("k_adj_g2pT_gather", "k_adj_scatter", "k_adj_grid", "k_adj_p2gT")}
    chk = float(np.sum(np.abs(c0.x)) + np.sum(np.abs(c0.v)) + np.sum(np.abs(c0.sigma)))
    print(Path(so).name, "%.4f ms/step" % (res.device_ms / 10), r, "checksum %.17g" % chk, flush=True)
    ctx.close()
