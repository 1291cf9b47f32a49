"""Per-CTA finish times of the two step launches (library built with -DMB4_CTA_TIMES,
selected by MB4CU_LIB): how evenly the persistent grids finish.
usage (GPU box): MB4CU_LIB=$PWD/paper_2003_04345_b200/lib_ct.so python tools/cta_times.py [cfg5]"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_04345_b200 import _lib, configs, nls2d  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg5"]
V, psi = configs.make_inputs(cfg)
model = configs.model_for(cfg, V)
with nls2d.Session(model, nls2d.Mb4Scheme(), configs.newton_for(cfg), device=0) as s:
    s.set_state(psi)
    s.run(cfg.dt, 8)
    buf = np.zeros((4, 2048, 4), dtype=np.uint64)
    L = ctypes.CDLL(os.environ["MB4CU_LIB"])
    rc = L.mb4cu_debug_cta_times(buf.ctypes.data_as(ctypes.c_void_p))
    assert rc == 0, rc
n1 = int((buf[1][:, 1] > 0).sum())
t_first = int(buf[1][:n1, 0].min())
starts = sorted(int(x) for x in buf[0][1][:2])
print("timeline of the last step (us after its first-sweep launch's first CTA start): "
      f"first-sweep CTAs left {(int(buf[1][:n1, 3].max()) - t_first) / 1e3:.1f}; "
      f"later-sweep CTAs start {(int(buf[2][buf[2][:, 0] > 0, 0].min()) - t_first) / 1e3:.1f}, "
      f"last sweep row done {(int(buf[2][:, 1].max()) - t_first) / 1e3:.1f}, "
      f"last CTA leaves {(int(buf[2][:, 3].max()) - t_first) / 1e3:.1f}; "
      f"period between the last two steps' first-sweep starts {(starts[1] - starts[0]) / 1e3:.1f}")
for ph in (1, 2):
    b = buf[ph]
    n = int((b[:, 1] > 0).sum())
    if n == 0:
        continue
    t0 = b[:n, 0].astype(np.int64)
    t1 = b[:n, 1].astype(np.int64)
    sm = b[:n, 2].astype(np.int64)
    base = t0.min()
    end = (t1 - base) / 1e3
    start = (t0 - base) / 1e3
    print(f"phase {ph}: {n} CTAs on {len(set(sm.tolist()))} SMs; start us min/mean/max {start.min():.1f}/{start.mean():.1f}/{start.max():.1f}; "
          f"end us min/p10/mean/p90/max {end.min():.1f}/{np.percentile(end,10):.1f}/{end.mean():.1f}/{np.percentile(end,90):.1f}/{end.max():.1f}")
    per_sm = {}
    for e, m in zip(end, sm):
        per_sm.setdefault(int(m), []).append(e)
    sm_end = np.array([max(v) for v in per_sm.values()])
    sm_cnt = np.array([len(v) for v in per_sm.values()])
    print(f"   CTAs per SM min/max {sm_cnt.min()}/{sm_cnt.max()}; SM finish us min/mean/max {sm_end.min():.1f}/{sm_end.mean():.1f}/{sm_end.max():.1f}")
    order = np.argsort(end)
    print("   slowest CTAs (block, sm, end us):", [(int(i), int(sm[i]), round(float(end[i]), 1)) for i in order[-8:]])
    print("   fastest CTAs (block, sm, end us):", [(int(i), int(sm[i]), round(float(end[i]), 1)) for i in order[:8]])
    # by SM id ranges (dies / GPCs)
    for lo in range(0, 160, 20):
        sel = (sm >= lo) & (sm < lo + 20)
        if sel.any():
            print(f"   SM {lo:3d}-{lo+19:3d}: mean end {end[sel].mean():.1f} us ({int(sel.sum())} CTAs)")
