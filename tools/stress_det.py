"""Determinism stress: repeat one cfg1 step (fresh session each time) and compare
with the first result and the oracle.  usage: python tools/stress_det.py [reps] [m]"""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from paper_2003_04345_b200 import configs, nls2d  # noqa: E402

pos = [a for a in sys.argv[1:] if not a.startswith("--")]
reps = int(pos[0]) if len(pos) > 0 else 100
m = int(pos[1]) if len(pos) > 1 else 1
name = pos[2] if len(pos) > 2 else "cfg1"
cfg = configs.CONFIGS[name]
V, psi = configs.make_inputs(cfg)
o = O.Oracle(cfg.nx, cfg.ny, cfg.gamma, V)
rc, ref, _, _, _ = o.step(psi, cfg.dt, eps=cfg.epsilon)
model = configs.model_for(cfg, V)
busy = "--busy" in sys.argv  # queue work on the legacy stream before each create
if busy:
    import torch
    A = torch.randn(4096, 4096, device="cuda", dtype=torch.float64)
poison = "--poison" in sys.argv  # leave stale device memory for the next cudaMalloc
if poison:
    import torch
first = None
bad = 0
hist = {}
for r in range(reps):
    st = nls2d.StepStats()
    if busy:
        B = A @ A  # noqa: F841  (async on the legacy default stream)
    if poison:
        g = torch.randn(64 << 20, device="cuda", dtype=torch.float64) * 1e3
        if r % 2:
            g.fill_(float("nan"))
        torch.cuda.synchronize()
        del g
        torch.cuda.empty_cache()
    with nls2d.Session(model, nls2d.Mb4Scheme(), configs.newton_for(cfg), neumann_terms=m) as s:
        s.set_state(psi)
        s.step(cfg.dt, st)
        u = s.get_state()
    e = np.linalg.norm(u - ref) / np.linalg.norm(ref)
    key = (st.newton_iters, st.halvings)
    hist[key] = hist.get(key, 0) + 1
    if first is None:
        first = u
    if not np.array_equal(u, first) or e > 1e-10:
        bad += 1
        d = np.abs(u - first)
        print(f"rep {r}: rel_vs_oracle={e:.3e} iters={st.newton_iters} halv={st.halvings} "
              f"ndiff={int((d > 0).sum())} maxdiff_at={int(d.argmax())} last_res={st.last_residual:.3e}")
print(f"{name} m={m}: {bad}/{reps} bad, (iters, halvings) histogram {hist}")
