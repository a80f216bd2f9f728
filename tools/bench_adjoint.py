"""Adjoint throughput (SURVEY §8d B_fwd+adj): device time of step_vjp and of a checkpointed
backprop_trajectory (forward sweep + segment replays + VJPs) per kernel, for a config.

usage: python tools/bench_adjoint.py [C3|C4|C5] [steps] [n_segments]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_04192_b200 import StateCotangent, init_scene  # noqa: E402
from paper_2507_04192_b200.presets import CONFIGS  # noqa: E402
from paper_2507_04192_b200.seeders import LagrangianLeastSquares  # noqa: E402
from paper_2507_04192_b200.solver import Context  # noqa: E402
from paper_2507_04192_b200.state import ParamGrads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 20
nseg = int(sys.argv[3]) if len(sys.argv) > 3 else 4
s = CONFIGS[cfg](dtype="f64")
st = init_scene(s)
n = st.particles.size()
ctx = Context(s, n)
ctx.upload(st)
ctx.advance(2)
st = ctx.download(st)
rng = np.random.default_rng(0)
cot = StateCotangent.zeros_like(st.particles)
cot.x[...] = rng.standard_normal(cot.x.shape)
cot.v[...] = rng.standard_normal(cot.v.shape)
ctx.step_vjp(st, cot, ParamGrads(s.boundary))  # warm
ctx.profile(True)
ctx.profile_reset()
t0 = time.perf_counter()
for _ in range(3):
    ctx.step_vjp(st, cot, ParamGrads(s.boundary))
wall = (time.perf_counter() - t0) / 3
tot, _ = ctx.profile_query("")
ks = {}
for k in ("k_p2g", "k_grid", "k_adj_g2pT_gather", "k_adj_scatter", "k_adj_grid", "k_adj_p2gT", "k_pg_reduce"):
    t, c = ctx.profile_query(k)
    if c:
        ks[k] = round(t / 3, 4)
print(f"{cfg} n={n} step_vjp: device {tot / 3:.3f} ms (wall incl. host transfers {wall * 1e3:.1f} ms) {ks}")
ctx.profile(False)
sd = LagrangianLeastSquares([N], st.particles.x[None] + 0.001, "x")
ctx.backprop(st, N, nseg, sd.desc())  # first call allocates the checkpoint / replay pool
t0 = time.perf_counter()
c0, pg, res = ctx.backprop(st, N, nseg, sd.desc())
wall = time.perf_counter() - t0
print(f"{cfg} backprop N={N} nseg={nseg}: device {res.device_ms:.2f} ms = {n * N / res.device_ms / 1e6:.3f} "
      f"G particle-steps/s (fwd sweep + replay + VJP per step); wall incl. host transfers {wall * 1e3:.1f} ms")
ctx.profile(True)
ctx.profile_reset()
ctx.backprop(st, N, nseg, sd.desc())
tot, _ = ctx.profile_query("")
ks = {}
for k in ("k_p2g", "k_grid", "k_g2p", "k_adj_g2pT_gather", "k_adj_scatter", "k_adj_grid", "k_adj_p2gT", "k_seed"):
    t, c = ctx.profile_query(k)
    if c:
        ks[k] = (round(t / c, 4), c)
print(f"  device total {tot:.2f} ms over {N} steps; per launch (ms, count): {ks}")
