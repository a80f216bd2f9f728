"""profiling driver: C4 (3-D column, 4.19M particles) forward steps; argv[1] = dtype, argv[2] = steps."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_04192_b200 import init_scene
from paper_2507_04192_b200.presets import c4_column3d
from paper_2507_04192_b200.solver import Context
dtype = sys.argv[1] if len(sys.argv) > 1 else "f64"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
s = c4_column3d(dtype); st = init_scene(s)
ctx = Context(s, st.particles.size()); ctx.upload(st)
t0 = time.time(); ctx.advance(steps); t1 = time.time()
print(f"{dtype} {steps} steps {1e3*(t1-t0)/steps:.3f} ms/step")
