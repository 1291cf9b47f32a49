"""Accuracy of the GPU energy monitor against an extended-precision host evaluation.

H(u) = Re u^H K u + sum V|u|^2 - (gamma/2) sum |u|^4 (lattice.cpp:106-137) of the same
double-precision state, evaluated on the host with every per-site term and every sum in
numpy longdouble (80-bit), row-chunked.  Compared: the fused first-sweep monitor (the
entry-state record of a step) and the observables pass (the final state).

usage: python tools/monitor_accuracy.py [cfg] [nx ny]      (default cfg5 at 8192^2;
       `cfg5 16384 32768` is the 8-GPU weak-scaling lattice on one GPU, 64 GB)
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2003_04345_b200 import configs, nls2d  # noqa: E402

LD = np.longdouble


def energy_ld(U, Vg, gamma, chunk=128):
    ny, nx = U.shape
    acc = {k: LD(0) for k in ("kin", "prob", "quart", "ext")}
    for j0 in range(0, ny, chunk):
        j1 = min(ny, j0 + chunk)
        rows = np.arange(j0 - 1, j1 + 1) % ny
        blk = U[rows]
        re, im = blk.real.astype(LD), blk.imag.astype(LD)

        def k_apply(x):  # 5-point periodic K (hx = hy = 1), rows j0..j1-1
            c = x[1:-1]
            return LD(4) * c - (np.roll(c, 1, 1) + np.roll(c, -1, 1)) - (x[:-2] + x[2:])

        kr, ki = k_apply(re), k_apply(im)
        r, i = re[1:-1], im[1:-1]
        n2 = r * r + i * i
        acc["kin"] += np.sum(r * kr + i * ki)
        acc["prob"] += np.sum(n2)
        acc["quart"] += np.sum(n2 * n2)
        acc["ext"] += np.sum(Vg[j0:j1].astype(LD) * n2)
    H = acc["kin"] - LD(0.5) * LD(gamma) * acc["quart"] + acc["ext"]
    return H, acc


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
    cfg = configs.CONFIGS[name]
    if len(sys.argv) > 3:
        cfg = cfg.with_lattice(int(sys.argv[2]), int(sys.argv[3]))
    t0 = time.time()
    V, psi = configs.make_inputs(cfg)
    model = configs.model_for(cfg, V)
    with nls2d.Session(model, nls2d.Mb4Scheme(), configs.newton_for(cfg)) as s:
        s.set_state(psi)
        obs, _ = s.run(cfg.dt, 1)  # row 0: fused monitor of psi; row 1: observables pass of u1
        u1 = s.get_state()
    t_gpu = time.time() - t0
    shape = (cfg.ny, cfg.nx)
    Vg = V.reshape(shape)
    H0, a0 = energy_ld(psi.reshape(shape), Vg, model.gamma())
    H1, a1 = energy_ld(u1.reshape(shape), Vg, model.gamma())
    rel = lambda x, ref: abs(x - float(ref)) / abs(float(ref))  # noqa: E731
    print(f"{cfg.name} {cfg.nx}x{cfg.ny} ({cfg.sites:.3e} sites), GPU part {t_gpu:.1f} s, host longdouble "
          f"{time.time() - t0 - t_gpu:.1f} s")
    print(f"  fused first-sweep monitor (entry state):  H rel err {rel(obs[0, 3], H0):.3e}   "
          f"sum|u|^2 rel err {rel(obs[0, 4], a0['prob']):.3e}")
    print(f"  observables pass (state after one step):  H rel err {rel(obs[1, 3], H1):.3e}   "
          f"sum|u|^2 rel err {rel(obs[1, 4], a1['prob']):.3e}")
    print(f"  H0 (longdouble) = {float(H0):.17g}, H1 = {float(H1):.17g}")


if __name__ == "__main__":
    main()
