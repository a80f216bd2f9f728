"""Generates tests/golden/c3_gradient.npz: the C3 inverse gradient computed by the
REFERENCE itself (oracle/_ref/libmpm_ref.so = /root/reference/proj compiled unmodified against the
Eigen/doctest shims, oracle/Makefile).

C3 (§5.1, BASELINE.json configs[2]): 102,400 fluid particles, 480 x 192 cells, dt 3e-5.
  * target: the final deposit x*(N) of a twin run at the true alpha* = 2.0;
  * loss  : L = sum_p |x_p(N) - x*_p(N)|^2 at N = 1000, from the run at alpha0 = 0.1 (:908);
  * plan  : CheckpointPlan::make(1000, 10) (checkpoint.hpp:15-34), backprop_trajectory (:72-143);
  * dL/dalpha = sum_p vbar_x,p(0) (H0 - y_p) = sum_p vbar_x,p(0) v_x,p(0) / alpha.

Stored: loss, dL/dalpha, |vbar(0)| norms, and vbar(0) / xbar(0) of every 16th particle (id order).
Run here (needs /root/reference, about 6 minutes):  python tests/golden/make_c3_gradient.py
"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import CpuOracle  # noqa: E402
from paper_2507_04192_b200.presets import c3_inverse  # noqa: E402

N_STEPS, N_SEG, STRIDE = 1000, 10, 16


def main():
    ref = CpuOracle("ref")
    t0 = time.time()
    twin = c3_inverse(alpha=2.0)
    st_t = ref.init_scene(twin)
    ref.advance(twin, st_t, N_STEPS)
    target = st_t.particles.x[None].copy()
    s = c3_inverse(alpha=0.1)
    st0 = ref.init_scene(s)
    c0, pg, res = ref.backprop(s, st0.copy(), N_STEPS, N_SEG,
                               {"field": "x", "obs_steps": [N_STEPS], "sel": None, "target": target})
    alpha = s.geometry[0].velocity.alpha
    dl_dalpha = float(np.sum(c0.v[:, 0] * st0.particles.v[:, 0]) / alpha)
    out = ROOT / "tests" / "golden" / "c3_gradient.npz"
    np.savez_compressed(out, loss=res.loss, dL_dalpha=dl_dalpha, n_steps=N_STEPS, n_segments=N_SEG,
                        stride=STRIDE, n_particles=st0.particles.size(),
                        vbar0_norm=np.linalg.norm(c0.v), xbar0_norm=np.linalg.norm(c0.x),
                        vbar0_sub=c0.v[::STRIDE].copy(), xbar0_sub=c0.x[::STRIDE].copy(),
                        target_sub=target[0, ::STRIDE].copy(),
                        generator="oracle/_ref (reference compiled unmodified), backprop_trajectory")
    print(f"wrote {out}: loss {res.loss!r} dL/dalpha {dl_dalpha!r} ({time.time() - t0:.0f} s)")


if __name__ == "__main__":
    main()
