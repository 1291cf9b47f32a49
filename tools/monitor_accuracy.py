"""Accuracy of the GPU energy monitor: H(u) from the fused first-sweep monitor and
from the observables pass vs an extended-precision host evaluation (numpy
longdouble, chunked).  usage: python tools/monitor_accuracy.py [cfg]"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2003_04345_b200 import configs, nls2d  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
V, psi = configs.make_inputs(cfg)
model = configs.model_for(cfg, V)
with nls2d.Session(model, nls2d.Mb4Scheme(), configs.newton_for(cfg)) as s:
    s.set_state(psi)
    obs, _ = s.run(cfg.dt, 3)
    u = s.get_state()
    o = s.observables()
nx, ny = cfg.nx, cfg.ny
U = u.reshape(ny, nx)
Vg = V.reshape(ny, nx)
acc = {k: np.longdouble(0) for k in ("uk", "p", "q", "ue")}
for j0 in range(0, ny, 256):
    rows = U[j0:j0 + 256]
    up = np.roll(U, -1, axis=0)[j0:j0 + 256]
    dn = np.roll(U, 1, axis=0)[j0:j0 + 256]
    ku = 4 * rows - (np.roll(rows, 1, 1) + np.roll(rows, -1, 1)) - (up + dn)
    re = rows.real.astype(np.longdouble)
    im = rows.imag.astype(np.longdouble)
    kr = ku.real.astype(np.longdouble)
    ki = ku.imag.astype(np.longdouble)
    n2 = re * re + im * im
    acc["uk"] += np.sum(re * kr + im * ki)
    acc["p"] += np.sum(n2)
    acc["q"] += np.sum(n2 * n2)
    acc["ue"] += np.sum(Vg[j0:j0 + 256].astype(np.longdouble) * n2)
H = acc["uk"] - np.longdouble(0.5) * np.longdouble(model.gamma()) * acc["q"] + acc["ue"]
print(f"{cfg.name}: H (longdouble) = {float(H):.17g}")
print(f"  observables pass: rel err {abs(o.total_energy - float(H)) / abs(float(H)):.3e}")
print(f"  run record last row: rel err {abs(obs[-1, 3] - float(H)) / abs(float(H)):.3e}")
print(f"  prob rel err {abs(o.probability - float(acc['p'])) / float(acc['p']):.3e}")
