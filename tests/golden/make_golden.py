#!/usr/bin/env python3
"""Regenerate the golden fixtures in tests/golden/ (run in the build container).

Sources (nothing here is hand-written data):
  scheme_exact.json  -- the reference's own exact-rational generator
                        (/root/reference/proj/tools/exact_scheme_tables.py, sympy),
                        parsed from its stdout.
  ref_*.npz          -- the reference library itself (oracle/_ref/libnls2d_ref.so,
                        StepDriver(MB4) -> mb4_step, eps = 1e-14) on the BASELINE
                        inputs produced by paper_2003_04345_b200.configs.
  ref_methods_cfg1_5.npz -- the same library's StepDriver(RK4 / GAUSS2 / GAUSS4 /
                        AVF2 / AVF4), direct solver, 5 cfg1 steps.
  ref_cfg4_sub.npz   -- the reference library on the full cfg4 lattice (4096^2, V_d ~
                        U[5,50), 4 packets; GMRES, 1 worker: 3 workers' GMRES storage exceeds
                        this container's 62 GB), 10 steps:
                        the full energy record and a deterministic subsample of the
                        state after steps 1 and 10 (every CFG4_STRIDE-th site) plus
                        whole-state checksums (sum |u|^2, sum u).

usage: python tests/golden/make_golden.py [--methods-only | --cfg4-only]
"""
import hashlib
import json
import os
import re
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2003_04345_b200 import configs  # noqa: E402

REF_TOOL = "/root/reference/proj/tools/exact_scheme_tables.py"


def input_digest(V, psi):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(V).tobytes())
    h.update(np.ascontiguousarray(psi).tobytes())
    return h.hexdigest()


def scheme_exact():
    out = subprocess.run([sys.executable, REF_TOOL], capture_output=True, text=True, check=True).stdout

    def nums(block):
        return [float(x) for x in re.findall(r"-?\d+(?:\.\d+)?(?:e-?\d+)?", block)]

    alpha = float(re.search(r"kAlpha1 = ([^;]+);", out).group(1))
    e = nums(re.search(r"kE\[3\]\[4\] = \{(.*?)\};", out, re.S).group(1))
    lam = nums(re.search(r"kEigenvalues\[3\] = \{(.*?)\};", out, re.S).group(1))
    w_block = re.search(r"kW\[3\]\[4\]\[4\]\[4\] = \{(.*?)\n\};", out, re.S).group(1)
    w = nums(w_block)
    # strip the array-dimension digits picked up from the declaration (none inside block)
    a_half = float(re.search(r"kAHalfHalf = ([^;]+);", out).group(1))
    l3_half = float(re.search(r"kL3Half = ([^;]+);", out).group(1))
    assert len(e) == 12 and len(lam) == 3 and len(w) == 192, (len(e), len(lam), len(w))
    return {"source": "reference tools/exact_scheme_tables.py (sympy, exact rationals)",
            "alpha1": alpha, "E": e, "eigenvalues": lam, "W": w, "A_half_half": a_half,
            "l3_half": l3_half}


def ref_case(name, nsteps, solver, keep_steps=(1, 10)):
    cfg = configs.CONFIGS[name]
    V, psi = configs.make_inputs(cfg)
    u = psi.copy()
    states = {}
    obs_all = [None]
    iters_all = []
    done = 0
    # step in chunks so intermediate states can be kept
    marks = sorted(set(keep_steps) | {nsteps})
    obs_series = []
    for m in marks:
        k = m - done
        u, obs, iters, secs = O.ref_run(cfg.nx, cfg.ny, float(cfg.nx), float(cfg.ny), cfg.gamma, V, u,
                                        cfg.dt, k, eps=cfg.epsilon, solver=solver)
        obs_series.append(obs if done == 0 else obs[1:])
        iters_all.extend(iters.tolist())
        done = m
        if m in keep_steps:
            states[m] = u.copy()
    obs = np.concatenate(obs_series, axis=0)
    out = {f"state_{k}": v for k, v in states.items()}
    out.update(obs=obs, iters=np.array(iters_all, dtype=np.int32), input_sha256=input_digest(V, psi),
               solver=solver, nsteps=nsteps)
    return out


def methods_case():
    cfg = configs.CONFIGS["cfg1"]
    V, psi = configs.make_inputs(cfg)
    out = {"input_sha256": input_digest(V, psi), "nsteps": 5, "solver": "direct"}
    for m in ("rk4", "gauss2", "gauss4", "avf2", "avf4"):
        u, obs, iters, _ = O.ref_run(cfg.nx, cfg.ny, float(cfg.nx), float(cfg.ny), cfg.gamma, V, psi, cfg.dt, 5,
                                     eps=cfg.epsilon, solver="direct", method=m)
        out[f"{m}_state"] = u
        out[f"{m}_obs"] = obs
        out[f"{m}_iters"] = iters
    return out


CFG4_STRIDE = 257  # sites k = 0, 257, 514, ... (65 281 of 4096^2; hits every column)


def cfg4_case(nsteps=10):
    cfg = configs.CONFIGS["cfg4"]
    V, psi = configs.make_inputs(cfg)
    idx = np.arange(0, cfg.sites, CFG4_STRIDE, dtype=np.int64)
    out = {"input_sha256": input_digest(V, psi), "solver": "gmres", "workers": 1, "nsteps": nsteps,
           "stride": CFG4_STRIDE, "idx": idx}
    u = psi
    obs_series, iters_all, done = [], [], 0
    for m in (1, nsteps):
        u, obs, iters, secs = O.ref_run(cfg.nx, cfg.ny, float(cfg.nx), float(cfg.ny), cfg.gamma, V, u, cfg.dt,
                                        m - done, eps=cfg.epsilon, solver="gmres", workers=1)
        print(f"cfg4: steps {done}..{m} in {secs:.1f} s, Newton iterations {iters.tolist()}", flush=True)
        obs_series.append(obs if done == 0 else obs[1:])
        iters_all.extend(iters.tolist())
        done = m
        out[f"sub_{m}"] = u[idx].copy()
        out[f"norm2_{m}"] = float(np.vdot(u, u).real)
        out[f"sum_{m}"] = complex(u.sum())
    out["obs"] = np.concatenate(obs_series, axis=0)
    out["iters"] = np.array(iters_all, dtype=np.int32)
    return out


def main():
    os.makedirs(HERE, exist_ok=True)
    if "--cfg4-only" in sys.argv:
        np.savez_compressed(os.path.join(HERE, "ref_cfg4_sub.npz"), **cfg4_case())
        return
    np.savez_compressed(os.path.join(HERE, "ref_methods_cfg1_5.npz"), **methods_case())
    if "--methods-only" in sys.argv:
        return
    with open(os.path.join(HERE, "scheme_exact.json"), "w") as f:
        json.dump(scheme_exact(), f, indent=1)
    # cfg1: direct solver (reference default), states after 1 and 10 steps, 10-step H series
    np.savez_compressed(os.path.join(HERE, "ref_cfg1_10.npz"), **ref_case("cfg1", 10, "direct"))
    # cfg1: full 1000-step energy record (GMRES path: equivalent to direct to ~1e-17)
    full = ref_case("cfg1", 1000, "gmres", keep_steps=())
    np.savez_compressed(os.path.join(HERE, "ref_cfg1_full.npz"), obs=full["obs"], iters=full["iters"],
                        input_sha256=full["input_sha256"], solver="gmres", nsteps=1000)
    # cfg2: 10 steps (GMRES path), state after 10 steps
    np.savez_compressed(os.path.join(HERE, "ref_cfg2_10.npz"), **ref_case("cfg2", 10, "gmres", keep_steps=(10,)))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
