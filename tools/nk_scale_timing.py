"""Newton-Krylov stage solver (kernel 3) step time vs lattice size, with the three stage
solves batched (in flight together) when they fit the device.  The Arnoldi kernel's dot
products run in chunks of 8 (64 registers, 4 CTAs per SM), so the three concurrent
cooperative Arnoldi launches fit up to ~4x the sites of the 32-accumulator version.
usage: python tools/nk_scale_timing.py"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2003_04345_b200 import _lib, nls2d  # noqa: E402

TWO_PI = 2 * np.pi
L = _lib.lib()
for n in (70, 200, 300, 400):
    g = nls2d.GridSpec(n, n, TWO_PI, TWO_PI)
    model = nls2d.GridModel(g, 0.1)
    u0 = nls2d.initial_condition(g)
    with nls2d.Session(model, nls2d.Mb4Scheme(), nls2d.NewtonConfig(1e-13, 50, 4), kernel=3) as s:
        s.set_state(u0)
        s.run(0.01, 2, record=False)
        s.set_state(u0)
        t0 = time.perf_counter()
        _, iters = s.run(0.01, 5, record=False)
        ms = (time.perf_counter() - t0) / 5 * 1e3
    print(f"{n}x{n}: {ms:.2f} ms/step, Newton iterations {list(iters)}")
