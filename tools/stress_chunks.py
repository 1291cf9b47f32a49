"""Determinism stress of the chunked later sweeps at a BASELINE size: fresh sessions, a few
steps each, the state and the energy record hashed -- which CTA takes which chunk differs from
run to run, the bits must not.  usage (GPU box): python tools/stress_chunks.py [reps] [cfg] [steps]"""
import hashlib
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2003_04345_b200 import configs, nls2d  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 12
name = sys.argv[2] if len(sys.argv) > 2 else "cfg5"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = configs.CONFIGS[name]
V, psi = configs.make_inputs(cfg)
model = configs.model_for(cfg, V)
seen = {}
for r in range(reps):
    with nls2d.Session(model, nls2d.Mb4Scheme(), configs.newton_for(cfg), device=0) as s:
        s.set_state(psi)
        obs, it = s.run(cfg.dt, steps)
        u = s.get_state()
    h = hashlib.sha256(u.tobytes() + np.asarray(obs).tobytes() + np.asarray(it).tobytes()).hexdigest()[:16]
    seen[h] = seen.get(h, 0) + 1
print(f"{name}: {reps} runs of {steps} steps, sweeps/step {list(it)}, distinct results: {len(seen)} {seen}")
sys.exit(0 if len(seen) == 1 else 1)
