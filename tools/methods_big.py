"""Every method for a few steps on a BASELINE-size lattice (memory / time check).
usage: python tools/methods_big.py [cfg] [steps]"""
import sys
import time

sys.path.insert(0, ".")
from paper_2003_04345_b200 import configs, nls2d  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
V, psi = configs.make_inputs(cfg)
model = configs.model_for(cfg, V)
for m in nls2d.METHODS:
    with nls2d.Session(model, nls2d.Mb4Scheme(), configs.newton_for(cfg), method=m) as s:
        s.set_state(psi)
        s.run(cfg.dt, 1, record=False)
        t0 = time.perf_counter()
        obs, iters = s.run(cfg.dt, steps)
        dt = (time.perf_counter() - t0) / steps
    H = obs[:, 3]
    print(f"{cfg.name} {m:7s} {dt * 1e3:9.2f} ms/step  {cfg.sites / dt:.3e} site*steps/s  iters {list(iters)}  "
          f"drift {abs(H - H[0]).max() / abs(H[0]):.2e}")
