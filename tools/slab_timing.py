"""Per-phase timing of the slab step at N=1 (diagnostic): host wall per phase + device time."""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_04192_b200 import init_scene  # noqa: E402
from paper_2507_04192_b200.distributed import GpuSlabDomain, SlabPlan, SlabStepper, TorchTransport, LocalTransport  # noqa
from paper_2507_04192_b200.presets import c4_column3d  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29555")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
s = c4_column3d("f64")
st = init_scene(s)
plan = SlabPlan([0, 256], 8)
dom = GpuSlabDomain(s, plan, 0, st, np.arange(st.particles.size()), local=True)
for tr in (TorchTransport(), LocalTransport()):
    stp = SlabStepper([dom], tr)
    stp.advance(5)
    T = {}
    orig = {k: getattr(dom, k) for k in ("p2g", "grid_interior", "finish_async", "commit", "migrate_export", "migrate_import")}
    def wrap(k):
        f = orig[k]
        def g(*a, **kw):
            t0 = time.perf_counter()
            r = f(*a, **kw)
            T[k] = T.get(k, 0) + time.perf_counter() - t0
            return r
        return g
    for k in orig:
        setattr(dom, k, wrap(k))
    rep = tr.report
    def rep2(*a):
        t0 = time.perf_counter()
        r = rep(*a)
        T["report"] = T.get("report", 0) + time.perf_counter() - t0
        return r
    tr.report = rep2
    K = 50
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    stp.advance(K)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / K
    print(type(tr).__name__, f"wall/step {wall*1e3:.3f} ms", {k: round(v / K * 1e3, 3) for k, v in T.items()})
    for k in orig:
        setattr(dom, k, orig[k])
    tr.report = rep
# device-only timing of the phases via the library profiler
dom.ctx.profile(True)
dom.ctx.profile_reset()
stp = SlabStepper([dom], LocalTransport())
stp.advance(5)
tot, _ = dom.ctx.profile_query("")
print("profiled device ms/step", tot / 5)
for k in ("k_reset", "k_keys", "k_seg", "k_compact", "k_mark_nodes", "k_p2g", "k_grid", "k_g2p", "k_step_end"):
    t, c = dom.ctx.profile_query(k)
    if c:
        print(k, round(t / 5, 4), c)
dist.destroy_process_group()
