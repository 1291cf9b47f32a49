"""Profiling helper: one production-kernel launch on cfg5 inputs (with a
libmb4cu built -DMB4_DEBUG_FIRST_ONLY the launch runs the first sweep alone)."""
import sys

sys.path.insert(0, ".")
from paper_2003_04345_b200 import configs, nls2d  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg5"]
V, psi = configs.make_inputs(cfg)
model = configs.model_for(cfg, V)
with nls2d.Session(model, nls2d.Mb4Scheme(), nls2d.NewtonConfig(cfg.epsilon, 50, 0), neumann_terms=1) as s:
    for _ in range(3):
        s.set_state(psi)
        try:
            s.step(cfg.dt)
        except nls2d.NonConvergenceError:
            pass
print("done")
