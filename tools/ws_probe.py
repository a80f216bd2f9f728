"""k_p2g_ws probe: one dense 3-D case per dtype under a hard timeout, against pipe3 (bitwise).
argv: library path (optional)"""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
from paper_2507_04192_b200 import capi
if len(sys.argv) > 1 and sys.argv[1]:
    capi._lib = capi.load_library(str(Path(sys.argv[1]).resolve()))
from paper_2507_04192_b200.solver import Context
from test_gpu_p2g_impl import dense_fluid

for dt in (sys.argv[2:] or ["f32", "f64"]):
    s, st = dense_fluid(dt)
    outs = []
    for impl in ("pipe3", "ws"):
        os.environ["MPM_P2G_IMPL"] = impl
        ctx = Context(s, st.particles.size())
        ctx.upload(st)
        ctx.advance(3)
        outs.append(ctx.download(st.copy()))
        ctx.close()
        print(dt, impl, "ok", flush=True)
    print(dt, "bitwise", all(np.array_equal(getattr(outs[0].particles, f), getattr(outs[1].particles, f))
                             for f in ("x", "v", "sigma")), flush=True)
