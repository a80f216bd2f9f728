"""Small 3-D workload for compute-sanitizer (racecheck / synccheck / memcheck): forward steps through
the pipelined P2G (k_p2g_pipe3), the incremental sort kernels, G2P, one step_vjp (K5a / K5b
k_adj_scatter_pipe3 / K6 / K7) and a short backprop with the replay tape; plus 2 same-process
slab ranks (mpm_dist_*)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from helpers import dp_block_scene  # noqa: E402
from paper_2507_04192_b200 import ParamGrads, StateCotangent, init_scene  # noqa: E402
from paper_2507_04192_b200.distributed import LocalSlabGroup, SlabPlan  # noqa: E402
from paper_2507_04192_b200.solver import Context  # noqa: E402

s = dp_block_scene(3, coulomb=True, cells=[16, 12, 12])
st = init_scene(s)
rng = np.random.default_rng(3)
st.particles.v[...] = rng.uniform(-0.5, 0.5, st.particles.v.shape)
ctx = Context(s, st.particles.size())
ctx.upload(st)
ctx.advance(1)
ctx.advance(3)
cur = ctx.download(st.copy())
cot = StateCotangent.zeros_like(cur.particles)
cot.x[...] = rng.standard_normal(cot.x.shape)
cot.v[...] = rng.standard_normal(cot.v.shape)
ctx.step_vjp(cur, cot, ParamGrads(s.boundary))
ctx.backprop(st, 4, 2, {"field": "x", "obs_steps": [4], "sel": None, "target": cur.particles.x[None] + 0.01})
ctx.close()
g = LocalSlabGroup(s, SlabPlan([0, 8, 16], 8), st)
g.advance(3)
g.close()
print("sanitize driver ok")
