#!/usr/bin/env python3
"""The paper's stage partition on GPUs (dist.StageSplitSession): the stiff 70x70 lx = 2*pi
baseline of the paper (configs/baseline.cfg; Newton-Krylov), the three stage systems of
each Newton iteration solved on `world` GPUs.  Run with
  python -m torch.distributed.run --nproc-per-node 3 --master-addr 127.0.0.1 tools/stage_split_bench.py
(or plainly for world 1).  Prints ms/step (max over ranks) beside the single-context
Newton-Krylov path (all three solves in flight on one GPU)."""
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2003_04345_b200 import dist as D, nls2d  # noqa: E402


def main(steps=20, n=70, h=0.01):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl")
    g = nls2d.GridSpec(n, n, 2 * np.pi, 2 * np.pi)
    model = nls2d.GridModel(g, -0.1)
    u0 = nls2d.initial_condition(g)
    cfg = nls2d.NewtonConfig()
    comm = D.Comm("cuda") if world > 1 else type("One", (), {"broadcast_": lambda self, t, src: None})()
    with nls2d.Session(model, nls2d.Mb4Scheme(), cfg, kernel=3, device=local) as s:
        s.set_state(u0)
        sess = D.StageSplitSession(s, comm, rank, world, cfg.epsilon, cfg.max_iters)
        sess.step(h)  # warm-up (plans, Krylov storage)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        its = [sess.step(h) for _ in range(steps)]
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3 / steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    single = None
    if rank == 0:
        with nls2d.Session(model, nls2d.Mb4Scheme(), cfg, kernel=3, device=local) as s:
            s.set_state(u0)
            s.step(h)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(steps):
                s.step(h)
            torch.cuda.synchronize()
            single = (time.perf_counter() - t0) * 1e3 / steps
        print(json.dumps({"lattice": [n, n], "world": world, "ms_per_step_stage_split": ms,
                          "ms_per_step_single_gpu_batched": single, "newton_iters": its[:3]}))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
