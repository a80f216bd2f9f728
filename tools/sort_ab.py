"""A/B of the K1 incremental sort against the full radix sort (MPM_SORT=cub), device-timed.
usage: python tools/sort_ab.py [C4 C3 C2 ...]"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_04192_b200 import init_scene  # noqa: E402
from paper_2507_04192_b200.presets import CONFIGS  # noqa: E402
from paper_2507_04192_b200.solver import Context  # noqa: E402

for cfg in sys.argv[1:] or ["C4", "C3", "C2"]:
    s = CONFIGS[cfg](dtype="f64")
    st = init_scene(s)
    for mode in ("inc", "cub"):
        os.environ["MPM_SORT"] = mode
        ctx = Context(s, st.particles.size())
        ctx.upload(st)
        ctx.advance(3)
        k = 50 if cfg in ("C4",) else 200
        ms = min(ctx.advance_timed(k) / k for _ in range(3))
        ctx.profile(True)
        ctx.profile_reset()
        ctx.advance(10)
        parts = {}
        for name in ("k_keys", "k_sort_classify", "k_sort_count", "k_sort_offsets", "k_sort_place", "k_sort_block", "k_seg", "k_occ", "k_compact", "k_mark_nodes", "k_p2g", "k_grid", "k_g2p"):
            t, nl = ctx.profile_query(name)
            if nl:
                parts[name] = round(t / 10 * 1e3, 1)
        ctx.profile(False)
        print(f"{cfg} {mode}: {ms * 1e3:.1f} us/step (graph); eager per-kernel us/step: {parts}", flush=True)
        ctx.close()
