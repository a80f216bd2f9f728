"""Host cost of the slab P2G phase when the particle count changes (diagnostic, one GPU).

C4 split into 4 slabs held by one process (LocalTransport): particles cross slab boundaries, so
a domain's count changes between steps and its P2G-phase graph must follow it (import steps run
eagerly; the steps after an export change n and recapture). Prints the host time of
`p2g()` per step, the migrations and the wall time per step.
usage: python tools/slab_recapture.py [steps]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_04192_b200 import init_scene  # noqa: E402
from paper_2507_04192_b200.distributed import GpuSlabDomain, LocalTransport, SlabPlan, SlabStepper  # noqa: E402
from paper_2507_04192_b200.presets import c4_column3d  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 60
s = c4_column3d("f64")
st = init_scene(s)
R = 4
plan = SlabPlan.make(s, R, st.particles.x)
ids = plan.partition(s, st)
doms = [GpuSlabDomain(s, plan, r, st, ids[r]) for r in range(R)]
stp = SlabStepper(doms, LocalTransport())
stp.advance(5)
T = {"p2g": 0.0}
orig = [d.p2g for d in doms]
for d, f in zip(doms, orig):
    def g(f=f):
        t0 = time.perf_counter()
        f()
        T["p2g"] += time.perf_counter() - t0
    d.p2g = g
m0 = stp.migrated
torch.cuda.synchronize()
t0 = time.perf_counter()
stp.advance(K)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / K
print(f"slabs {R} steps {K}: wall/step {wall * 1e3:.3f} ms, p2g host/step (all slabs) {T['p2g'] / K * 1e3:.3f} ms, "
      f"migrated {stp.migrated - m0}")
