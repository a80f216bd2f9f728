"""dev quick check: GPU forward vs oracle on several scenes (temporary)."""
import sys, time, numpy as np
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
from oracle import CpuOracle
from paper_2507_04192_b200 import *
from paper_2507_04192_b200.presets import *
from paper_2507_04192_b200.solver import Context
orc = CpuOracle("orc")
def rel(a, b):
    return float(np.abs(a - b).max()) / max(float(np.abs(b).max()), 1e-30)
def check(name, s, steps):
    st = init_scene(s)
    ctx = Context(s, st.particles.size())
    ctx.upload(st)
    t0 = time.time(); ctx.advance(steps, nan_guard=True); t1 = time.time()
    got = ctx.download(st.copy())
    ref = st.copy(); orc.advance(s, ref, steps)
    errs = {f: rel(getattr(got.particles, f), getattr(ref.particles, f)) for f in ("x", "v", "sigma", "rho", "volume", "grad_v", "eps_eq")}
    print(f"{name:14s} n={st.particles.size():7d} steps={steps} gpu {t1-t0:.3f}s  " + " ".join(f"{k}:{v:.1e}" for k, v in errs.items()), flush=True)
    ctx.close()
s = small_fluid_scene("pic"); check("fluid pic", s, 20)
s = small_fluid_scene("flip"); s.config.gravity=[0,-9.8]; check("fluid flip g", s, 50)
s = small_fluid_scene("apic"); check("fluid apic", s, 20)
s = small_fluid_scene("tpic"); check("fluid tpic", s, 20)
s = small_fluid_scene("blend", 0.3); check("fluid blend", s, 20)
s = c1_column(); check("C1 dp 2d", s, 20)
s = c1_column("f32"); check("C1 dp 2d f32", s, 20)
s = small_fluid_scene("flip"); s.material = bui_sand(); s.config.dt=1e-5; s.config.gravity=[0,-9.8]; s.boundary.walls[2] = Wall("coulomb", [0.1, 0.4, 0.2]); check("dp coulomb", s, 30)
s3 = Scene(3, "f64"); c = s3.config; c.dh=0.05; c.cells=[16,16,16]; c.dt=1e-5; c.gravity=[0,-9.8,0]; c.scheme.kind="flip"; s3.material=bui_sand(); s3.boundary.walls[2]=Wall("no_slip")
s3.geometry.append(GeometryRegion(lo=[0.1,0.1,0.1], hi=[0.5,0.4,0.45])); check("dp 3d", s3, 20)
s3.obstacles.append(Obstacle([0.3,0.0,0.0],[0.6,0.25,0.8])); s3.config.scheme.kind="apic"; check("3d apic obst", s3, 10)
# C4 perf probe
s = c4_column3d(); st = init_scene(s); ctx = Context(s, st.particles.size()); ctx.upload(st)
ctx.advance(3); import ctypes
t0 = time.time(); ctx.advance(20); t1 = time.time()
print("C4 f64 n=%d  %.3f ms/step  %.3g p-s/s" % (st.particles.size(), (t1-t0)/20*1e3, st.particles.size()*20/(t1-t0)), ctx.grid_stats(), flush=True)
ctx.profile(True); ctx.advance(3)
for k in ["k_p2g","k_grid","k_g2p","k_seg","k_compact","k_mark","k_step"]:
    print(k, ctx.profile_query(k))
print("all", ctx.profile_query(""))
ctx.close()
s = c4_column3d("f32"); st = init_scene(s); ctx = Context(s, st.particles.size()); ctx.upload(st)
ctx.advance(3); t0 = time.time(); ctx.advance(20); t1 = time.time()
print("C4 f32  %.3f ms/step" % ((t1-t0)/20*1e3), flush=True)
s = c2_dam_break(); st = init_scene(s); ctx = Context(s, st.particles.size()); ctx.upload(st)
ctx.advance(3); t0 = time.time(); ctx.advance(100); t1 = time.time()
print("C2 f64  %.3f ms/step  %.3g p-s/s" % ((t1-t0)/100*1e3, st.particles.size()*100/(t1-t0)), flush=True)
