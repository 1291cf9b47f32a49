"""Stiff paper-scale configs on the GPU (Newton-Krylov policy) vs the reference CPU
path: the 70x70 lx=2pi baseline (configs/baseline.cfg) and the 100x100 delta
potential.  usage: python tools/paper_scale_timing.py"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from paper_2003_04345_b200 import nls2d  # noqa: E402

TWO_PI = 2 * np.pi
for n, gamma, v0, h, steps in ((70, -0.1, 0.0, 0.01, 20), (100, 0.1, -50.0, 0.002, 10)):
    g = nls2d.GridSpec(n, n, TWO_PI, TWO_PI)
    V = nls2d.build_delta_potential(g, v0) if v0 else np.zeros(n * n)
    model = nls2d.GridModel(g, gamma, V)
    u0 = nls2d.initial_condition(g) if not v0 else np.full(n * n, 1.0 / n, dtype=np.complex128)
    with nls2d.Session(model, nls2d.Mb4Scheme(), nls2d.NewtonConfig(1e-13, 50, 4)) as s:
        s.set_state(u0)
        s.run(h, 2, record=False)
        s.set_state(u0)
        s.profile_enable(True)
        s.profile_reset()
        t0 = time.perf_counter()
        obs, iters = s.run(h, steps)
        gpu = (time.perf_counter() - t0) / steps
        kit = s.profile()["krylov_iters"] / max(1, int(np.sum(iters))) / 3
    t0 = time.perf_counter()
    _, robs, riters, secs = O.ref_run(n, n, TWO_PI, TWO_PI, gamma, V, u0, h, steps, eps=1e-13, solver="direct",
                                      workers=3)
    print(f"{n}x{n} v0={v0}: GPU {gpu * 1e3:.2f} ms/step (iters {list(iters[:3])}, "
          f"{kit:.1f} GMRES iterations per stage solve), "
          f"reference direct/3 workers {secs / steps * 1e3:.2f} ms/step (iters {list(riters[:3])})")
