"""Small cases through every kernel family, for compute-sanitizer runs:
production persistent kernel (default schedule, (2,1), (6,2), speculative miss),
tiled kernel, Newton-Krylov with the Fourier preconditioner, the other methods,
sub-domain sweeps, observables."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2003_04345_b200 import configs, dist as D, nls2d  # noqa: E402

cfg = configs.CONFIGS["cfg1"]
V, psi = configs.make_inputs(cfg)
model = configs.model_for(cfg, V)
newton = configs.newton_for(cfg)
for kw in ({}, {"neumann_terms": 1, "neumann_first": 2}, {"neumann_terms": 2, "neumann_first": 6},
           {"neumann_terms": 1, "neumann_first": 5, "first_poly": 1}, {"kernel": 1}, {"kernel": 3}):
    with nls2d.Session(model, nls2d.Mb4Scheme(), newton, **kw) as s:
        s.set_state(psi)
        for h in (cfg.dt, 2 * cfg.dt, cfg.dt):
            s.step(h)
        s.observables()
for m in ("rk4", "gauss2", "gauss4", "avf2", "avf4"):
    with nls2d.Session(model, nls2d.Mb4Scheme(), newton, method=m) as s:
        s.set_state(psi)
        s.run(cfg.dt, 2)
dec = D.Decomposition(cfg.nx, cfg.ny, 1, 1, 0)
be = D.CudaBackend(dec, V, nls2d.Mb4Scheme(), cfg.gamma, 1.0, 1.0, cfg.epsilon, cfg.max_iters, 1, 0)
be.set_state(psi)


class One:
    def allreduce_max(self, x):
        return x

    def allreduce_sum(self, x):
        return np.asarray(x)

    def allreduce_max_(self, t):
        pass

    def allreduce_sum_(self, t):
        pass


sess = D.DistributedSession(dec, be, One(), cfg.gamma, 1.0, 1.0, cfg.epsilon)
sess.run(cfg.dt, 3)
be.close()
print("sanitize case done")
