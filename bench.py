#!/usr/bin/env python3
"""MB4 FP64 lattice-site*steps/s on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5] [--impl ours|reference]

Workload (default): BASELINE configs[4] ("cfg5"), the weak-scaling lattice of
8192^2 sites per GPU (the metric's 1/2/4/8-GPU, % HBM roofline configuration
and the largest single-GPU config); --config cfg1..cfg4 selects the others.
One "step" = one MB4 time step (all stage sweeps to ||r||_inf <= 1e-14) over the
whole lattice.  Inputs are synthetic and seeded (configs.py); the state and the
stage buffers (>= 3 GiB at 8192^2) are far larger than the 126 MB L2.  For
lattices whose working set fits in L2 the bench times every step separately
and flushes L2 between steps.

Rank 0 prints ONE JSON line.  Under torchrun (N > 1) every rank steps its own
8192^2 block; `value` is the whole-job total, timed as the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "MB4 FP64 lattice-site*steps/s"
UNIT = "site*steps/s"
L2_BYTES = 126 * 1024 * 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--neumann", type=int, default=-1)
    ap.add_argument("--neumann-first", type=int, default=-1)
    ap.add_argument("--kernel", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-overlap", action="store_true",
                    help="multi-GPU: exchange halos between sweeps instead of overlapping the interior")
    ap.add_argument("--force-dist", action="store_true",
                    help="use the sub-domain (multi-GPU) path even on one GPU")
    ap.add_argument("--python-dist", action="store_true",
                    help="multi-GPU: the Python-driven sweep loop (dist.DistributedSession) instead of the "
                         "library's native NCCL stepper")
    ap.add_argument("--profile-only", action="store_true",
                    help="warm-up + a few steps, no JSON extras (for ncu captures)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- distributed


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class _StdoutToStderr:
    """fd-level redirect of stdout to stderr while NCCL initialises: its version banner is a
    plain printf to stdout, and stdout must carry only the JSON line."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


class Dist:
    def __init__(self, world: int, rank: int, local: int):
        self.world, self.rank, self.local = world, rank, local
        self.pg = None
        if world > 1:
            import torch
            import torch.distributed as dist

            torch.cuda.set_device(local)
            with _StdoutToStderr():
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
                dist.barrier()  # (the communicator is created lazily: once here, banner included)
            self.dist = dist
            self.torch = torch

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


# ----------------------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax),
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- helpers


def schedule_key(args) -> str:
    """Stage-iteration schedule of the run: 'default' (deep first sweep, adaptive m)
    or mf<first>_m<terms> when set explicitly."""
    if args.neumann < 0 and args.neumann_first < 0:
        return "default"
    return f"mf{args.neumann_first}_m{args.neumann}"


def _kernel_source_hash() -> str:
    """sha256[:16] of the sweep-kernel sources (the same as tools/update_traffic.py stamps)."""
    import hashlib

    h = hashlib.sha256()
    for f in ("sweep_march2.cu", "site_math.cuh", "async_copy.cuh", "mb4cu_internal.hpp"):
        with open(os.path.join(ROOT, "paper_2003_04345_b200", "csrc", f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def _traffic_entry(cfg_name: str, schedule: str):
    """The committed ncu capture of this workload, only if it was taken of the kernel
    sources in the tree (stamped kernel_src_sha16): a stale capture is not reported."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            e = json.load(f).get(f"{cfg_name}_{schedule}")
        if e is None or e.get("kernel_src_sha16") != _kernel_source_hash():
            return None
        return e
    except Exception:
        return None


def measured_traffic(cfg_name: str, schedule: str):
    """DRAM bytes of one step's kernel launches from the committed ncu capture (profiles/traffic.json)."""
    t = _traffic_entry(cfg_name, schedule)
    return None if t is None else float(t["dram_bytes_per_launch"])


def measured_limiters(cfg_name: str, schedule: str):
    """Pipe utilisations of the same ncu capture: with a depth-6 first sweep the
    step kernel is bounded on-chip (FP64 pipe, shared memory) rather than by HBM."""
    t = _traffic_entry(cfg_name, schedule)
    return None if t is None else t.get("limiters")


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# CPU sample window: 1024^2 sites of the workload's own inputs (cfg3's lattice size;
# the reference's GMRES at 1024^2 takes ~3 s per MB4 step on 3 workers)
REF_WINDOW = 1024


def ref_sample(cfg, V, psi):
    """Bounded CPU sample of the workload: the REF_WINDOW^2 window at the lattice
    origin of the SAME V / psi arrays (same dt, g, eps; periodic on the window)."""
    win = min(REF_WINDOW, cfg.nx, cfg.ny)
    Vs = np.ascontiguousarray(V.reshape(cfg.ny, cfg.nx)[:win, :win]).reshape(-1)
    ps = np.ascontiguousarray(psi.reshape(cfg.ny, cfg.nx)[:win, :win]).reshape(-1)
    return win, Vs, ps


def ref_time(cfg, win, Vs, ps, steps, warmup=1):
    """Time the reference stepping loop (oracle/_ref: StepDriver(MB4) -> mb4_step,
    solver=gmres, workers=3) -- or the C port when the reference library is absent.
    Returns (site*steps/s, kind, cores, seconds)."""
    import time as _t

    from oracle import oracle as O

    kind = "reference" if O.ref_available() else "port"
    if kind == "reference":
        u = ps
        if warmup:
            u, _, _, _ = O.ref_run(win, win, float(win), float(win), cfg.gamma, Vs, u, cfg.dt, warmup,
                                   eps=cfg.epsilon, solver="gmres", workers=3, record=False)
        _, _, _, secs = O.ref_run(win, win, float(win), float(win), cfg.gamma, Vs, u, cfg.dt, steps,
                                  eps=cfg.epsilon, solver="gmres", workers=3, record=False)
        cores = 3
    else:
        o = O.Oracle(win, win, cfg.gamma, Vs)
        u, _, _ = o.run(ps, cfg.dt, warmup, eps=cfg.epsilon) if warmup else (ps, None, None)
        t0 = _t.perf_counter()
        o.run(u, cfg.dt, steps, eps=cfg.epsilon)
        secs = _t.perf_counter() - t0
        cores = 1
    return win * win * steps / secs, kind, cores, secs


def cpu_baseline(cfg, V, psi, steps=3):
    win, Vs, ps = ref_sample(cfg, V, psi)
    value, kind, cores, secs = ref_time(cfg, win, Vs, ps, steps)
    return {
        "value": value,
        "unit": UNIT,
        "cores": cores,
        "nproc": os.cpu_count(),
        "kind": kind,
        "sample": (f"{win}x{win} window of the {cfg.name} inputs, {steps} MB4 steps "
                   f"(dt={cfg.dt}, eps={cfg.epsilon}), reference StepDriver(MB4) solver=gmres "
                   f"(ILU0+GMRES(50), its fastest path), workers=3 (its maximum), {secs:.1f} s"),
    }


# ----------------------------------------------------------------------------- our arm


def run_ours(args, d: Dist):
    import torch

    from paper_2003_04345_b200 import configs, nls2d

    torch.cuda.set_device(d.local)
    base = configs.CONFIGS[args.config]
    cfg = base
    if args.config == "cfg5":
        cfg = base.with_lattice(8192, 8192)
    # each rank steps its own lattice block of the configured size (weak scaling)
    t_gen = time.perf_counter()
    V, psi = configs.make_inputs(cfg)
    t_gen = time.perf_counter() - t_gen
    model = configs.model_for(cfg, V)
    sess = nls2d.Session(model, nls2d.Mb4Scheme(), configs.newton_for(cfg),
                         neumann_terms=None if args.neumann < 0 else args.neumann,
                         neumann_first=None if args.neumann_first < 0 else args.neumann_first,
                         device=d.local, kernel=args.kernel)
    sess.set_state(psi)
    obs0 = sess.observables()
    n = cfg.sites
    working_set = n * (16 + 8 + 96)
    flush = working_set < 2 * L2_BYTES
    flush_buf = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda") if flush else None

    # warm-up (device-resident run with the per-step energy record)
    obs_w, _ = sess.run(cfg.dt, args.warmup) if args.warmup > 0 else (np.zeros((1, 7)), None)
    torch.cuda.synchronize()

    sess.profile_reset()
    sess.profile_enable(True)
    stats = nls2d.StepStats()
    clocks = ClockSampler(d.local)
    d.barrier()
    torch.cuda.synchronize()
    clocks.start()
    if not flush:
        # the timed region is the user-facing device-resident run(): every step's
        # stage solve in one persistent launch + the fused per-step energy record
        # (56 B D2H per step)
        t0 = time.perf_counter()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        obs_t, iters_t = sess.run(cfg.dt, args.steps, stats=stats)
        ev1.record()
        torch.cuda.synchronize()
        step_ms_total = ev0.elapsed_time(ev1)
        wall = time.perf_counter() - t0
    else:
        step_ms_total = 0.0
        rows = []
        t0 = time.perf_counter()
        for _ in range(args.steps):
            flush_buf.zero_()
            torch.cuda.synchronize()
            st = nls2d.StepStats()
            sess.step(cfg.dt, st)
            stats.newton_iters += st.newton_iters
            stats.halvings += st.halvings
            step_ms_total += 1e3 * st.solve_seconds
        wall = time.perf_counter() - t0
        obs_t = np.array([[getattr(sess.observables(), f) for f in nls2d.OBS_FIELDS]])
    clk = clocks.stop()
    d.barrier()
    prof = sess.profile()
    sess.profile_enable(False)
    ms = d.max(step_ms_total)
    total_sites = d.sum(float(n))
    value = total_sites * args.steps / (ms * 1e-3)
    # relative energy drift over the whole run (warm-up + timed steps), every step
    H = np.concatenate([[obs0.total_energy], obs_w[:, 3], obs_t[:, 3]])
    drift = float(np.abs(H - obs0.total_energy).max() / abs(obs0.total_energy))
    drift = d.max(drift)

    peak, peak_kind = measured_peaks()
    kern_ms = prof["kernel_ms"]
    launches = max(1, prof["launches"])
    achieved = prof["alg_bytes"] / (kern_ms * 1e-3) / 1e9 if kern_ms > 0 else 0.0
    sweeps_per_step = prof["sweeps"] / max(1, args.steps)
    step_alg_bytes = prof["alg_bytes"] / max(1, args.steps)

    result = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": d.world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded defects + Gaussian packets, configs.py)",
        "config": {
            "workload": f"{cfg.name}: {cfg.nx}x{cfg.ny} sites per GPU, dt={cfg.dt}, g={cfg.g}, "
                        f"{cfg.defect_frac:.0%} defects, {cfg.npackets} packet(s) sigma={cfg.sigma}, eps={cfg.epsilon}",
            "lattice": [cfg.nx, cfg.ny],
            "sites_per_gpu": n,
            "neumann_terms": args.neumann if args.neumann >= 0 else "adaptive 1..2",
            "neumann_first": args.neumann_first if args.neumann_first >= 0 else 6,
            "schedule": schedule_key(args),
            "kernel": "tiled" if args.kernel == 1 else "default",
            "l2": "flushed between steps" if flush else "inputs larger than L2 (state+stages >= 3 GiB)",
            "parallelism": "replicas" if d.world > 1 else "single",
        },
        "sweeps_per_step": sweeps_per_step,
        "final_sweep_misses": int(prof.get("redone", 0)),
        "energy_drift": drift,
        "roofline": {
            "bound": "hbm",
            "achieved": achieved,
            "peak": peak,
            "unit": "GB/s",
            "frac": achieved / peak,
            "traffic": measured_traffic(cfg.name, schedule_key(args)),
            "traffic_source": "ncu --set full, dram__bytes_read+write of one step's launches (profiles/traffic.json)",
            "limiters": measured_limiters(cfg.name, schedule_key(args)),
            # the same metric against the HBM bound of the stage iteration SURVEY.md 8(d)
            # projected (5 sweeps at cfg5: 72 + 4 x 120 = 552 B/site-step): the deep first
            # sweep and the U3-only final sweep remove bytes, so frac above understates it
            "vs_hbm_bound_of_5_sweep_schedule": (value / d.world / (peak * 1e9 / 552.0)) if cfg.name == "cfg5" else None,
            # SURVEY.md 8(d)'s formula bytes(step) = N (72 + 120 (S - 1)) counts the U3-only final
            # sweep at 120 B/site; `frac` above uses the 88 B it moves
            "frac_survey_8d": (n * (72.0 * args.steps + 120.0 * (prof["sweeps"] - args.steps))
                               / (kern_ms * 1e-3) / 1e9 / peak) if kern_ms > 0 else None,
            "peak_kind": peak_kind,
            "kernel": "stage sweep",
            "alg_bytes_per_step": step_alg_bytes,
            "kernel_ms_per_launch": kern_ms / launches,
            "launches_per_step": launches / max(1, args.steps),
            "kernel_ms_per_step": kern_ms / max(1, args.steps),
            "sweep_ms_by_index": [round(t / n, 4) for t, n in zip(prof.get("sweep_ms", []), prof.get("sweep_n", []))
                                  if n > 0],
            "step_share": kern_ms / max(1e-9, step_ms_total),
        },
        "gpu_launches": int(prof["launches"] + prof["other_launches"]),
        "clocks": clk,
        "wall_s_timed": wall,
        "input_gen_s": t_gen,
    }

    # end-to-end through the public API with host buffers (mb4_step contract)
    if not args.no_e2e:
        host = torch.empty(2 * n, dtype=torch.float64, pin_memory=True)
        host.numpy()[:] = psi.view(np.float64)
        hv = host.numpy().view(np.complex128)
        import ctypes as C

        from paper_2003_04345_b200 import _lib

        L = _lib.lib()
        ptr = C.cast(host.data_ptr(), C.POINTER(C.c_double))
        k_e2e = max(1, min(args.steps, 10))
        d.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            L.mb4cu_set_state(sess._ctx, ptr)   # H2D of the step's input state
            sess.step(cfg.dt)
            L.mb4cu_get_state(sess._ctx, ptr)   # D2H of the step's result
        e2e_s = d.max(time.perf_counter() - t0)
        result["e2e"] = {
            "value": total_sites * k_e2e / e2e_s,
            "unit": UNIT,
            "h2d_bytes_per_step": 16 * n,
            "d2h_bytes_per_step": 16 * n,
            "steps": k_e2e,
            "api": "mb4cu_set_state -> mb4cu_step -> mb4cu_get_state (host pinned buffers)",
        }
        # the reference harness's run() (harness.cpp:64-133) through the same API: the
        # initial state up, K steps with the per-step energy record read back (its CSV
        # rows), the final state down -- host copies inside the timed region
        host.numpy()[:] = psi.view(np.float64)
        k_run = max(1, args.steps)
        d.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        L.mb4cu_set_state(sess._ctx, ptr)
        rows, _ = sess.run(cfg.dt, k_run)
        L.mb4cu_get_state(sess._ctx, ptr)
        run_s = d.max(time.perf_counter() - t0)
        result["e2e_harness"] = {
            "value": total_sites * k_run / run_s,
            "unit": UNIT,
            "h2d_bytes_per_step": 16 * n / k_run,
            "d2h_bytes_per_step": 16 * n / k_run + rows.shape[1] * 8,
            "steps": k_run,
            "api": "mb4cu_set_state -> mb4cu_run (per-step energy rows to the host) -> mb4cu_get_state",
        }
        del hv

    if d.rank == 0 and d.world == 1 and not args.no_cpu_baseline:
        try:
            result["cpu_baseline"] = cpu_baseline(cfg, V, psi)
        except Exception as exc:  # keep the GPU line even if the CPU leg fails
            result["cpu_baseline"] = {"value": None, "error": str(exc)}
    sess.close()
    return result


# ----------------------------------------------------------------------------- multi-GPU arm


def run_dist(args, d: Dist, make_backend=None, comm=None, lattice=None):
    """N GPUs: the cfg5 weak-scaling lattice (8192^2 per GPU) split over a px x py
    torus (dist.choose_grid), halo exchange + scalar all-reduces over NCCL each sweep.

    make_backend / comm / lattice: injection points for the CPU test of this control flow
    (tests/test_dist_gloo.py: gloo ranks, the numpy sub-domain backend, a small lattice)."""
    import torch

    from paper_2003_04345_b200 import configs, dist as D, nls2d

    if args.config not in ("cfg3", "cfg4", "cfg5"):
        raise SystemExit("multi-GPU runs: cfg5 (weak scaling) or cfg3 / cfg4 (strong scaling)")
    on_gpu = make_backend is None
    if on_gpu:
        torch.cuda.set_device(d.local)
    weak = args.config == "cfg5"
    if weak:  # BASELINE configs[4]: 8192^2 sites per GPU
        gnx, gny = lattice or configs.cfg5_lattice(d.world)
        cfg = configs.CONFIGS["cfg5"].with_lattice(gnx, gny)
    else:  # BASELINE configs[2] / [3]: the fixed lattice split over the GPUs
        cfg = configs.CONFIGS[args.config]
        if lattice:
            cfg = cfg.with_lattice(*lattice)
        gnx, gny = cfg.nx, cfg.ny
    px, py = D.choose_grid(d.world, gnx, gny)
    dec = D.Decomposition(gnx, gny, px, py, d.rank)
    # first-contact evidence for multi-GPU runs: the world, the process grid and NCCL's own
    # communicator lines (NCCL_DEBUG=INFO, set in main) on stderr
    print(f"[bench] rank {d.rank}/{d.world} local {d.local}: {args.config} {gnx}x{gny} on a {px}x{py} process grid, "
          f"block {dec.lnx}x{dec.lny} at ({dec.x0},{dec.y0}), transport "
          f"{'nccl' if d.world > 1 and on_gpu else 'local' if on_gpu else 'injected'}", file=sys.stderr, flush=True)
    Vb, pb, psum = configs.make_block(cfg, dec.x0, dec.y0, dec.lnx, dec.lny)
    if comm is None:
        comm = D.Comm("cuda") if d.world > 1 else _LocalComm()
    total_p = comm.allreduce_sum([psum])[0]
    pb *= 1.0 / math.sqrt(total_p)
    m = args.neumann if args.neumann >= 0 else 1
    # halo exchange overlapped with the interior sweep; the interior leaves 2 SMs to
    # NCCL's kernels when there are peers
    if on_gpu and not getattr(args, "python_dist", False):
        be = D.CudaBackend(dec, Vb, nls2d.Mb4Scheme(), cfg.gamma, 1.0, 1.0, cfg.epsilon, cfg.max_iters, m, d.local,
                           max_step_halvings=cfg.max_step_halvings)
    elif on_gpu:
        be = D.CudaBackend(dec, Vb, nls2d.Mb4Scheme(), cfg.gamma, 1.0, 1.0, cfg.epsilon, cfg.max_iters, m, d.local,
                           overlap=not args.no_overlap, reserve_sms=2 if d.world > 1 else 0)
    else:
        be = make_backend(dec, Vb, cfg)
    be.set_state(pb)
    native = on_gpu and not getattr(args, "python_dist", False)
    if native:
        # the step inside the library over NCCL (one host read per step); the communicator id
        # from rank 0 to every rank through torch.distributed
        nid = [D.nccl_unique_id() if d.rank == 0 else None]
        if d.world > 1:
            d.dist.broadcast_object_list(nid, src=0)
        with _StdoutToStderr():
            sess = D.NativeSession(dec, be, nid[0], cfg.gamma, 1.0, 1.0, adaptive_m=args.neumann < 0,
                                   grid_cap=-2 if d.world > 1 else 0)
    else:
        sess = D.DistributedSession(dec, be, comm, cfg.gamma, 1.0, 1.0, cfg.epsilon, adaptive_m=args.neumann < 0)
    obs_w, _ = sess.run(cfg.dt, args.warmup) if args.warmup > 0 else (None, None)
    H0 = obs_w[0, 3] if obs_w is not None else sess.observables()[3]
    if hasattr(be, "profile"):
        be.profile(True)
    clocks = ClockSampler(d.local)
    d.barrier()
    if on_gpu:
        torch.cuda.synchronize()
    clocks.start()
    if on_gpu:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
    t0 = time.perf_counter()
    obs_t, sweeps = sess.run(cfg.dt, args.steps)
    if on_gpu:
        ev1.record()
        torch.cuda.synchronize()
    clk = clocks.stop()
    ms = d.max(ev0.elapsed_time(ev1) if on_gpu else 1e3 * (time.perf_counter() - t0))
    d.barrier()
    p = _lib_profile(be) if on_gpu else {"alg_bytes": 0.0, "launches": 0, "other_launches": 0}
    H = np.concatenate([obs_w[:, 3] if obs_w is not None else [], obs_t[:, 3]])
    drift = float(np.abs(H - H0).max() / abs(H0))
    n_local = dec.lnx * dec.lny
    value = float(gnx) * gny * args.steps / (ms * 1e-3)
    peak, peak_kind = measured_peaks()
    # sweeps run asynchronously between device-side reductions: the time base is the
    # whole step of this rank (sweeps + halo exchanges + reductions)
    achieved = p["alg_bytes"] / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
    res = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": d.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded defects + Gaussian packets, configs.py)",
        "config": {"workload": f"{args.config} {'weak' if weak else 'strong'} scaling: {gnx}x{gny} lattice, "
                               f"{dec.lnx}x{dec.lny} sites per GPU, dt={cfg.dt}, g={cfg.g}, eps={cfg.epsilon}",
                   "lattice": [gnx, gny], "sites_per_gpu": n_local,
                   "neumann_terms": m if args.neumann >= 0 else "adaptive 1..2",
                   "process_grid": [px, py], "parallelism": f"2-D domain decomposition {px}x{py}",
                   "halo_exchange": ("in the library (mb4cu_dist_step): boundary frame first, its NCCL "
                                     "send/recv on a communication stream while the interior is swept; residual "
                                     "all-reduce and stopping test on the device, one host read per step"
                                     if native else "between sweeps" if args.no_overlap else
                                     "overlapped: boundary frame swept first, its NCCL exchange on a side "
                                     "stream while the interior is swept"),
                   "l2": (f"working set {dec.lnx * dec.lny * 120 / 2**20:.0f} MiB per GPU "
                          + ("> L2 (126 MB)" if dec.lnx * dec.lny * 120 > 126e6 else
                             "<= L2 (126 MB): not flushed between steps, strong-scaling reference only"))},
        "sweeps_per_step": float(np.mean(sweeps)),
        "energy_drift": d.max(drift),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None, "peak_kind": peak_kind,
                     "kernel": "stage sweeps, sub-domain mode, rank 0; time base = whole step incl. "
                               "halo exchange and reductions"},
        "gpu_launches": int(p["launches"] + p["other_launches"]),
        "clocks": clk,
    }
    if not args.no_e2e and on_gpu:
        # end to end per step through the public API: this rank's block host -> device,
        # one distributed step, device -> host (pinned host buffer)
        host = torch.empty(2 * n_local, dtype=torch.float64, pin_memory=True)
        host.numpy()[:] = pb.view(np.float64)
        hv = host.numpy().view(np.complex128)
        k_e2e = max(1, min(args.steps, 10))
        d.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            be.set_state(hv)
            sess.step(cfg.dt)
            hv[:] = be.get_state()
        e2e_s = d.max(time.perf_counter() - t0)
        res["e2e"] = {"value": float(gnx) * gny * k_e2e / e2e_s, "unit": UNIT,
                      "h2d_bytes_per_step": 16 * n_local * d.world, "d2h_bytes_per_step": 16 * n_local * d.world,
                      "steps": k_e2e, "api": "per rank: mb4cu_set_state -> DistributedSession.step -> mb4cu_get_state"}
    if hasattr(sess, "close"):
        sess.close()
    if hasattr(be, "close"):
        be.close()
    return res


class _LocalComm:
    """Single-rank stand-in for dist.Comm (used by --force-dist on one GPU)."""

    def allreduce_max(self, x):
        return float(x)

    def allreduce_sum(self, xs):
        return np.asarray(xs, dtype=np.float64)

    def allreduce_max_(self, t):
        pass

    def allreduce_sum_(self, t):
        pass

    def exchange(self, pairs):
        raise RuntimeError("no peers")


def _lib_profile(be):
    import ctypes as C

    from paper_2003_04345_b200 import _lib

    p = _lib.Profile()
    be.L.mb4cu_profile_get(be.ctx, C.byref(p))
    return {f: getattr(p, f) for f, _ in _lib.Profile._fields_}


# ----------------------------------------------------------------------------- reference arm


def run_reference(args, d: Dist):
    """The reference CPU path (oracle/_ref) on the host cores, same metric/config:
    one MB4 step of the bounded sample (REF_WINDOW^2 window of the workload's own
    inputs) per bench step, W warm-up steps, then K timed steps in one stepping loop."""
    from oracle import oracle as O
    from paper_2003_04345_b200 import configs  # input specs only; libmb4cu.so is never loaded here

    base = configs.CONFIGS[args.config]
    cfg = base.with_lattice(8192, 8192) if args.config == "cfg5" else base
    # the same seeded inputs from the host-only generator (oracle/libinputs.so, g++)
    V, psi = configs.make_inputs(cfg, gen=O.inputs_generator())
    win, Vs, ps = ref_sample(cfg, V, psi)
    value, kind, cores, secs = ref_time(cfg, win, Vs, ps, args.steps, warmup=args.warmup)
    return {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "impl": "reference",
        "n_gpus": d.world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded defects + Gaussian packets, configs.py)",
        "config": {"workload": f"{cfg.name} CPU sample: the {win}x{win} window at the origin of its "
                               f"{cfg.nx}x{cfg.ny} inputs (periodic on the window), one MB4 step per "
                               f"bench step; the full lattice is impractical on the CPU",
                   "lattice": [cfg.nx, cfg.ny], "window": [win, win]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "nproc": os.cpu_count(), "kind": kind,
                         "sample": f"{win}x{win} window of the {cfg.name} inputs, one MB4 step per "
                                   f"bench step, reference StepDriver(MB4) solver=gmres workers=3"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "repo_libs_mapped": repo_libs_mapped(),
    }


def repo_libs_mapped():
    """In-tree shared libraries this process has mapped (/proc/self/maps)."""
    here = os.path.dirname(os.path.abspath(__file__))
    libs = set()
    try:
        with open("/proc/self/maps") as f:
            for line in f:
                path = line.split()[-1] if len(line.split()) >= 6 else ""
                if path.startswith(here) and ".so" in path:
                    libs.add(os.path.relpath(path, here))
    except OSError:
        return None
    return sorted(libs)


def main():
    # NCCL's banner / INFO lines go to stderr: stdout carries only the JSON line
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        if rank != 0:
            return 0
        res = run_reference(args, Dist(1, 0, 0))
        res["n_gpus"] = world  # the launch's N (the CPU path itself runs on rank 0's host cores)
        print(json.dumps(res))
        return 0
    if world > 1:
        # NCCL's communicator lines (ranks, rings, NVLS) on stderr: evidence of the N-rank run
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    d = Dist(world, rank, local)
    res = run_dist(args, d) if (world > 1 or args.force_dist) else run_ours(args, d)
    if rank == 0:
        print(json.dumps(res))
    d.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
