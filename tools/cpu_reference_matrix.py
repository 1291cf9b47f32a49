#!/usr/bin/env python3
"""The reference CPU path timed on this host's cores (SURVEY.md 8(d) "CPU timing beside
it"): StepDriver(MB4) -> mb4_step of the reference library compiled from its sources
(oracle/_ref), solver Direct (sparse LU, its default) and Gmres (ILU(0)+GMRES(50)),
WorkerPool workers 1 and 3 (its maximum), on the BASELINE inputs of cfg1-cfg3.
Bounded samples (a few steps each, stated per row); cfg4 / cfg5 are not timed
(cfg4 ~4.6 min/step, cfg5 needs ~55 GB of GMRES storage).  Prints one row per run and
the same rows as JSON on the last line.  TEST / MEASUREMENT infrastructure only."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2003_04345_b200 import configs  # noqa: E402

PLAN = [  # (config, solver, workers, steps)
    ("cfg1", "direct", 1, 4), ("cfg1", "direct", 3, 4), ("cfg1", "gmres", 1, 40), ("cfg1", "gmres", 3, 40),
    ("cfg2", "direct", 3, 1), ("cfg2", "gmres", 1, 10), ("cfg2", "gmres", 3, 10),
    ("cfg3", "gmres", 3, 2),
]


def main():
    rows = []
    for name, solver, workers, steps in PLAN:
        cfg = configs.CONFIGS[name]
        V, psi = configs.make_inputs(cfg)
        u, obs, iters, secs = O.ref_run(cfg.nx, cfg.ny, float(cfg.nx), float(cfg.ny), cfg.gamma, V, psi, cfg.dt,
                                        steps, eps=cfg.epsilon, solver=solver, workers=workers)
        H = obs[:, 3]
        row = {"config": name, "sites": cfg.sites, "solver": solver, "workers": workers, "steps": steps,
               "s_per_step": secs / steps, "site_steps_per_s": cfg.sites * steps / secs,
               "newton_iters_per_step": float(np.mean(iters)),
               "energy_drift": float(np.abs(H - H[0]).max() / abs(H[0])), "nproc": os.cpu_count()}
        rows.append(row)
        print(f"{name} {solver:6s} workers={workers} steps={steps:3d}: {row['s_per_step']:.4f} s/step, "
              f"{row['site_steps_per_s']:.3e} site*steps/s, {row['newton_iters_per_step']:.1f} Newton it/step, "
              f"drift {row['energy_drift']:.2e}", flush=True)
    print(json.dumps(rows))


if __name__ == "__main__":
    main()
