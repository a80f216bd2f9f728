"""Sample SM clock, power and throttle reasons at 20 ms while C4 f64 steps run back to back
(evidence for the power / clock state of the FP64-dense step). Writes gpurun_out/power_probe.csv."""
import subprocess
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_04192_b200 import init_scene
from paper_2507_04192_b200.presets import c4_column3d
from paper_2507_04192_b200.solver import Context

dt = sys.argv[1] if len(sys.argv) > 1 else "f64"
s = c4_column3d(dt)
st = init_scene(s)
ctx = Context(s, st.particles.size())
ctx.upload(st)
ctx.advance(5)
out = Path("gpurun_out") / f"power_probe_{dt}.csv"
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,clocks.sm,power.draw,power.limit,temperature.gpu,"
                        "clocks_event_reasons.active", "--format=csv", "-lms", "20"],
                       stdout=open(out, "w"), stderr=subprocess.DEVNULL)
time.sleep(1.0)
t0 = time.time()
ms = ctx.advance_timed(2000)
print(dt, "2000 steps %.3f ms/step, wall %.2f s" % (ms / 2000, time.time() - t0))
time.sleep(0.5)
smi.terminate()
