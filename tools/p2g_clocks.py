"""P2G phase clocks at C4 (f64), steady state: argv[1] = a library built with -DP2G_ABL=32, whose
ablated copy of k_p2g_pipe3 prints, for CTAs 0..3, the cycles thread 0 spent per phase (the real
kernel runs after it, so the simulation stays valid). Summarises the last step's lines."""
import os
import re
import subprocess
import sys
from pathlib import Path

if len(sys.argv) > 2:  # child: run, device printf goes to stdout
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from paper_2507_04192_b200 import capi, init_scene
    from paper_2507_04192_b200.presets import c4_column3d
    from paper_2507_04192_b200.solver import Context

    capi._lib = capi.load_library(str(Path(sys.argv[1]).resolve()))
    s = c4_column3d(sys.argv[2])
    st = init_scene(s)
    ctx = Context(s, st.particles.size())
    ctx.upload(st)
    ctx.advance(6)
    ctx.download()
    ctx.close()
    sys.exit(0)

out = subprocess.run([sys.executable, __file__, sys.argv[1], os.environ.get("DT", "f64")], capture_output=True,
                     text=True).stdout
lines = [l for l in out.splitlines() if l.startswith("p2g-clk ")][-4:]
for l in [l for l in out.splitlines() if l.startswith("p2g-clk2")][-4:]:
    print(l)
for pre in ("ws-prod", "ws-cons", "ws-red"):  # -DP2G_ABL=64 builds with MPM_P2G_IMPL=ws
    for l in [l for l in out.splitlines() if l.startswith(pre)][-4:]:
        print(l)
names = ["setup+tail", "wait", "convert", "march0", "march-imbalance", "emit"]
for l in lines:
    nums = dict(re.findall(r"([a-z+-]+\d?) (\d+)", l))
    tot = sum(int(nums[k]) for k in names)
    print(l)
    print("   fractions:", {k: round(int(nums[k]) / tot, 3) for k in names}, "total cycles", tot)
