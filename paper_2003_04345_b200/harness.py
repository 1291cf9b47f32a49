"""Run harness on the GPU path: RunConfig / run() / trajectory CSV / snapshots.

Mirrors the reference harness (run_config.hpp:19-46, run_config.cpp:9-130,
harness.hpp:18-89, harness.cpp:16-300) -- run(), compare_methods(),
parallel_bench(), convergence_study() -- backed by a device-resident Session:
the state stays in HBM, the per-step energy record comes from the energy monitor
(fused into each MB4 step's first sweep), and host copies happen only for
snapshots and the final state.  Every method of the reference runs on the GPU
(MB4: the production stage solver; RK4 / GAUSS2 / GAUSS4 / AVF2 / AVF4:
methods.cu).

Extension keys (not in the reference): the BASELINE inputs
(`baseline = cfg1..cfg5`, or `defect_frac/defect_seed/vd_min/vd_max/packets/
sigma/x0/y0/kx/ky/random_packets/packet_seed/k_max`) and `neumann_terms`.

Differences: `workers` and `solver` are accepted and ignored (no worker pool, no
sparse factorization); for MB4 `newton_iters` in the CSV counts stage sweeps;
`wall_s` is the device time of the step's chunk divided evenly over its steps
(the run is stepped in chunks between snapshot times).
"""
from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass, field, replace
from typing import List, Optional

import numpy as np

from . import configs, nls2d


class ConfigError(ValueError):
    """run_config.hpp:11-14."""


@dataclass
class RunConfig:
    lx: float = 2.0 * math.pi
    ly: float = 2.0 * math.pi
    nx: int = 70
    ny: int = 70
    t_end: float = 1.0
    dt: float = 0.01
    gamma: float = 0.1
    v0: float = 0.0
    method: str = "mb4"
    epsilon: float = 1e-13
    max_iters: int = 50
    max_halvings: int = 4
    workers: int = 1
    initial: str = "cosine"
    raw_participation: bool = False
    solver: str = "direct"
    snapshot_times: List[float] = field(default_factory=list)
    out_dir: str = ""
    # extensions
    baseline: str = ""
    defect_frac: float = 0.0
    defect_seed: int = 0
    vd_min: float = 0.0
    vd_max: float = 0.0
    packets: int = 0
    sigma: float = 1.0
    x0: float = 0.0
    y0: float = 0.0
    kx: float = 0.0
    ky: float = 0.0
    random_packets: bool = False
    packet_seed: int = 0
    k_max: float = 0.0
    neumann_terms: int = -1

    def validate(self):
        """run_config.cpp:9-20."""
        if self.nx < 2 or self.ny < 2:
            raise ConfigError("nx and ny must be >= 2")
        if not (self.lx > 0.0) or not (self.ly > 0.0):
            raise ConfigError("lx and ly must be positive")
        if not (self.dt > 0.0):
            raise ConfigError("dt must be positive")
        if not (self.t_end >= self.dt):
            raise ConfigError("t_end must be >= dt")
        if not (self.epsilon > 0.0):
            raise ConfigError("epsilon must be positive")
        if self.max_iters < 1:
            raise ConfigError("max_iters must be >= 1")
        if self.max_halvings < 0:
            raise ConfigError("max_halvings must be >= 0")
        if self.workers < 1 or self.workers > 3:
            raise ConfigError("workers must be in 1..3")
        for t in self.snapshot_times:
            if t < 0.0 or t > self.t_end + 1e-12:
                raise ConfigError("snapshot time outside [0, t_end]")
        if nls2d.parse_method(self.method) is None:
            raise ConfigError(f"unknown method '{self.method}'")

    def _lattice_cfg(self) -> Optional[configs.LatticeConfig]:
        if self.baseline:
            return configs.CONFIGS[self.baseline]
        if self.defect_frac > 0.0 or self.packets > 0:
            return configs.LatticeConfig(
                "custom", self.nx, self.ny, self.dt, 1, -self.gamma, self.defect_frac, self.defect_seed,
                self.vd_min, self.vd_max, self.packets, self.sigma, x0=self.x0, y0=self.y0, kx=self.kx,
                ky=self.ky, random_packets=self.random_packets, packet_seed=self.packet_seed,
                k_max=self.k_max, epsilon=self.epsilon)
        return None

    def make_model(self) -> nls2d.GridModel:
        """run_config.cpp:22-26 (+ the BASELINE defect potential)."""
        grid = nls2d.GridSpec(self.nx, self.ny, self.lx, self.ly)
        lc = self._lattice_cfg()
        if lc is not None and (lc.defect_frac > 0.0):
            V, _, _ = configs.make_block(lc.with_lattice(self.nx, self.ny))
            if self.v0 != 0.0:
                V[0] += self.v0
            return nls2d.GridModel(grid, self.gamma, V)
        if self.v0 != 0.0:
            return nls2d.GridModel(grid, self.gamma, nls2d.build_delta_potential(grid, self.v0))
        return nls2d.GridModel(grid, self.gamma)

    def make_initial(self, model: nls2d.GridModel) -> np.ndarray:
        """run_config.cpp:28-32 (+ the BASELINE Gaussian packets)."""
        lc = self._lattice_cfg()
        if lc is not None and lc.npackets > 0:
            _, psi = configs.make_inputs(lc.with_lattice(self.nx, self.ny))
            return psi
        if self.initial == "cosine":
            return nls2d.initial_condition(model.grid())
        n = model.points()
        return np.full(n, 1.0 / math.sqrt(n), dtype=np.complex128)


def _parse_double(key, v):
    try:
        return float(v)
    except ValueError:
        raise ConfigError(f"bad number for '{key}': {v}") from None


def _parse_int(key, v):
    try:
        return int(v)
    except ValueError:
        raise ConfigError(f"bad integer for '{key}': {v}") from None


def apply_key_value(cfg: RunConfig, key: str, value: str) -> None:
    """run_config.cpp:67-109 (+ extension keys).  Unknown keys are errors."""
    value = value.strip()
    doubles = {"lx", "ly", "t_end", "dt", "gamma", "v0", "epsilon", "defect_frac", "vd_min", "vd_max",
               "sigma", "x0", "y0", "kx", "ky", "k_max"}
    ints = {"nx", "ny", "max_iters", "max_halvings", "workers", "defect_seed", "packet_seed", "neumann_terms"}
    if key in doubles:
        setattr(cfg, key, _parse_double(key, value))
    elif key in ints:
        setattr(cfg, key, _parse_int(key, value))
    elif key == "packets":
        cfg.packets = _parse_int(key, value)
    elif key == "method":
        cfg.method = value.lower()
    elif key == "initial":
        if value not in ("cosine", "uniform"):
            raise ConfigError("initial must be 'cosine' or 'uniform'")
        cfg.initial = value
    elif key in ("raw_participation", "random_packets"):
        if value not in ("true", "false", "1", "0"):
            raise ConfigError(f"{key} must be true/false")
        setattr(cfg, key, value in ("true", "1"))
    elif key == "solver":
        if value not in ("direct", "gmres"):
            raise ConfigError("solver must be 'direct' or 'gmres'")
        cfg.solver = value
    elif key == "snapshot_times":
        cfg.snapshot_times = [_parse_double(key, x) for x in value.replace(",", " ").split()] if value else []
    elif key == "out_dir":
        cfg.out_dir = value
    elif key == "baseline":
        if value not in configs.CONFIGS:
            raise ConfigError(f"baseline must be one of {sorted(configs.CONFIGS)}")
        b = configs.CONFIGS[value]
        cfg.baseline = value
        cfg.nx, cfg.ny, cfg.lx, cfg.ly = b.nx, b.ny, float(b.nx), float(b.ny)
        cfg.dt, cfg.t_end, cfg.gamma, cfg.epsilon = b.dt, b.dt * b.steps, b.gamma, b.epsilon
    else:
        raise ConfigError(f"unknown config key '{key}'")


def parse_config_file(path: str, base: Optional[RunConfig] = None) -> RunConfig:
    """Flat `key = value` file, '#' comments (run_config.cpp:111-130)."""
    cfg = replace(base) if base is not None else RunConfig()
    with open(path) as f:
        for lineno, raw in enumerate(f, 1):
            line = raw.split("#", 1)[0].strip()
            if not line:
                continue
            if "=" not in line:
                raise ConfigError(f"{path}:{lineno}: expected key = value")
            k, v = line.split("=", 1)
            apply_key_value(cfg, k.strip(), v)
    return cfg


@dataclass
class TrajectoryRow:
    t: float
    u_kinetic: float
    u_nonlinear: float
    u_external: float
    total_energy: float
    probability: float
    participation: float
    newton_iters: int
    wall_seconds: float


@dataclass
class TrajectoryRecord:
    rows: List[TrajectoryRow]
    final_state: np.ndarray
    solve_seconds: float = 0.0
    wall_seconds: float = 0.0

    @staticmethod
    def _drift(v, base):  # harness.cpp:16-19
        return math.inf if not math.isfinite(v) else abs(v - base) / max(1.0, abs(base))

    def max_energy_drift(self) -> float:
        h0 = self.rows[0].total_energy if self.rows else 0.0
        return max((self._drift(r.total_energy, h0) for r in self.rows), default=0.0)

    def max_probability_drift(self) -> float:
        p0 = self.rows[0].probability if self.rows else 0.0
        return max((self._drift(r.probability, p0) for r in self.rows), default=0.0)


def step_count(t_end: float, dt: float) -> int:
    return int(math.ceil(t_end / dt - 1e-9))


def write_snapshot(path: str, t: float, grid: nls2d.GridSpec, u: np.ndarray) -> None:
    """harness.cpp:27-40: |u|^2 per site, one grid row per line, 17 digits."""
    with open(path, "w") as f:
        f.write(f"# {t:.17g} {grid.nx} {grid.ny}\n")
        d = (np.abs(u) ** 2).reshape(grid.ny, grid.nx)
        for j in range(grid.ny):
            f.write(" ".join(f"{x:.17g}" for x in d[j]) + "\n")


def write_trajectory_csv(f, rec: TrajectoryRecord) -> None:
    """harness.cpp:135-145."""
    f.write("t,UK,UI,UE,H,prob,participation,newton_iters,wall_s\n")
    for r in rec.rows:
        f.write(f"{r.t:.17g},{r.u_kinetic:.17g},{r.u_nonlinear:.17g},{r.u_external:.17g},"
                f"{r.total_energy:.17g},{r.probability:.17g},{r.participation:.17g},"
                f"{r.newton_iters},{r.wall_seconds:.6g}\n")


def run(cfg: RunConfig, device: int = 0) -> TrajectoryRecord:
    """harness.cpp:64-133 on the GPU path."""
    cfg.validate()
    model = cfg.make_model()
    u = cfg.make_initial(model)
    ncfg = nls2d.NewtonConfig(cfg.epsilon, cfg.max_iters, cfg.max_halvings)
    want_files = bool(cfg.out_dir)
    if want_files:
        os.makedirs(cfg.out_dir, exist_ok=True)
    snaps = sorted(cfg.snapshot_times)
    nsteps = step_count(cfg.t_end, cfg.dt)
    rows: List[TrajectoryRow] = []
    t_start = time.perf_counter()
    solve = 0.0
    with nls2d.Session(model, nls2d.Mb4Scheme(), ncfg,
                       neumann_terms=None if cfg.neumann_terms < 0 else cfg.neumann_terms,
                       device=device, method=nls2d.parse_method(cfg.method)) as s:
        s.set_state(u)

        def emit(t, obs_row, iters, wall):
            rows.append(TrajectoryRow(t, obs_row[0], obs_row[1], obs_row[2], obs_row[3], obs_row[4],
                                      obs_row[6] if cfg.raw_participation else obs_row[5], int(iters), wall))

        def maybe_snap(t):
            nonlocal snap_next
            while snap_next < len(snaps) and t + 1e-12 >= snaps[snap_next]:
                if want_files:
                    write_snapshot(os.path.join(cfg.out_dir, f"snapshot_{snaps[snap_next]:g}.txt"), t,
                                   model.grid(), s.get_state())
                snap_next += 1

        snap_next = 0
        o = s.observables()
        emit(0.0, [getattr(o, k) for k in nls2d.OBS_FIELDS], 0, 0.0)
        maybe_snap(0.0)
        done = 0
        while done < nsteps:
            # chunk up to the next snapshot (or the last, possibly shorter, step)
            chunk_end = nsteps
            if snap_next < len(snaps):
                chunk_end = min(nsteps, max(done + 1, step_count(snaps[snap_next], cfg.dt)))
            last_h = min(nsteps * cfg.dt, cfg.t_end) - (nsteps - 1) * cfg.dt
            uniform = chunk_end - done if (chunk_end < nsteps or abs(last_h - cfg.dt) < 1e-15) else chunk_end - done - 1
            for k, h in ((uniform, cfg.dt), (chunk_end - done - uniform, last_h)):
                if k <= 0:
                    continue
                st = nls2d.StepStats()
                t0 = time.perf_counter()
                try:
                    obs, iters = s.run(h, k, stats=st)
                except nls2d.NonConvergenceError as e:
                    e.at_time = done * cfg.dt
                    raise
                wall = (time.perf_counter() - t0) / k
                solve += st.solve_seconds
                for q in range(k):
                    done += 1
                    emit(min(done * cfg.dt, cfg.t_end), obs[q + 1], iters[q], wall)
            maybe_snap(min(done * cfg.dt, cfg.t_end))
        final = s.get_state()
    rec = TrajectoryRecord(rows, final, solve, time.perf_counter() - t_start)
    if want_files:
        with open(os.path.join(cfg.out_dir, "trajectory.csv"), "w") as f:
            write_trajectory_csv(f, rec)
    return rec


# ---------------------------------------------------------------------------- studies


@dataclass
class MethodReport:
    """harness.hpp:40-46."""
    method: str
    energy_drift: float
    probability_drift: float
    mean_step_seconds: float
    total_newton_iters: int


@dataclass
class CompareReport:
    """harness.hpp:48-57, harness.cpp:147-196."""
    methods: List[MethodReport]
    mb4_over_gauss2: float = 0.0
    avf4_over_gauss2: float = 0.0

    def write(self, f) -> None:
        f.write("method  energy_drift  probability_drift  mean_step_seconds  newton_iters\n")
        for m in self.methods:
            f.write(f"{nls2d.method_name(m.method):<7} {m.energy_drift:.3e}     {m.probability_drift:.3e}"
                    f"          {m.mean_step_seconds:.6f}           {m.total_newton_iters}\n")
        f.write(f"time ratio MB4/GAUSS2  = {self.mb4_over_gauss2:.3f}\n")
        f.write(f"time ratio AVF4/GAUSS2 = {self.avf4_over_gauss2:.3f}\n")


def compare_methods(cfg: RunConfig, methods, device: int = 0) -> CompareReport:
    """harness.cpp:147-178: one run per method, drifts, mean step time, iterations."""
    rep = CompareReport([])
    times = {}
    for m in methods:
        c = replace(cfg, method=m, out_dir="")
        rec = run(c, device)
        nsteps = max(1, len(rec.rows) - 1)
        mr = MethodReport(m, rec.max_energy_drift(), rec.max_probability_drift(),
                          sum(r.wall_seconds for r in rec.rows) / nsteps, sum(r.newton_iters for r in rec.rows))
        rep.methods.append(mr)
        times[m] = mr.mean_step_seconds
    if times.get("gauss2", 0.0) > 0.0:
        rep.mb4_over_gauss2 = times.get("mb4", 0.0) / times["gauss2"]
        rep.avf4_over_gauss2 = times.get("avf4", 0.0) / times["gauss2"]
    return rep


@dataclass
class BenchReport:
    """harness.hpp:59-71, harness.cpp:219-257 (workers 1 vs 3 of the reference's
    pool; the GPU path has no worker pool, so both runs take the same path and the
    trajectories must be bit-identical)."""
    serial_step_seconds: float
    parallel_step_seconds: float
    speedup: float
    solve_fraction: float
    trajectories_identical: bool

    def write(self, f) -> None:
        f.write(f"per-step seconds, 1 worker  = {self.serial_step_seconds:.6f}\n")
        f.write(f"per-step seconds, 3 workers = {self.parallel_step_seconds:.6f}\n")
        f.write(f"speedup                     = {self.speedup:.3f}\n")
        f.write(f"solve-phase fraction        = {self.solve_fraction:.3f}\n")
        f.write(f"trajectories bit-identical  = {'yes' if self.trajectories_identical else 'no'}\n")


def _rows_identical(a: TrajectoryRecord, b: TrajectoryRecord) -> bool:
    if len(a.rows) != len(b.rows):
        return False
    for x, y in zip(a.rows, b.rows):
        if (x.t, x.u_kinetic, x.u_nonlinear, x.u_external, x.total_energy, x.probability, x.participation,
                x.newton_iters) != (y.t, y.u_kinetic, y.u_nonlinear, y.u_external, y.total_energy,
                                    y.probability, y.participation, y.newton_iters):
            return False
    return bool(np.array_equal(a.final_state, b.final_state))


def parallel_bench(cfg: RunConfig, device: int = 0) -> BenchReport:
    base = replace(cfg, method="mb4", out_dir="")
    rec1 = run(replace(base, workers=1), device)
    rec3 = run(replace(base, workers=3), device)
    nsteps = max(1, len(rec1.rows) - 1)
    s1, s3 = rec1.wall_seconds / nsteps, rec3.wall_seconds / nsteps
    return BenchReport(s1, s3, s1 / s3, rec1.solve_seconds / rec1.wall_seconds, _rows_identical(rec1, rec3))


@dataclass
class ConvergenceEntry:
    method: str
    h_values: List[float]
    errors: List[float]
    slope: float


@dataclass
class ConvergenceReport:
    """harness.hpp:73-88, harness.cpp:272-316."""
    entries: List[ConvergenceEntry]

    def write(self, f) -> None:
        """harness.cpp:301-313."""
        for e in self.entries:
            f.write(f"{nls2d.method_name(e.method)}:\n")
            for h, err in zip(e.h_values, e.errors):
                f.write(f"  h = {h:<10.6g} error = {err:.6e}\n")
            f.write(f"  fitted order = {e.slope:.3f}\n")


def convergence_study(cfg: RunConfig, methods, h_list, device: int = 0) -> ConvergenceReport:
    """Errors against a run at h_min / 8 and the least-squares log-log slope."""
    if len(h_list) < 3:
        raise ConfigError("convergence_study: need at least 3 h values")
    for a, b in zip(h_list, h_list[1:]):
        if not b < a:
            raise ConfigError("convergence_study: h_list must descend")
    rep = ConvergenceReport([])
    for m in methods:
        base = replace(cfg, method=m, out_dir="", snapshot_times=[])
        ref = run(replace(base, dt=h_list[-1] / 8.0), device).final_state
        ref_norm = float(np.sqrt(np.sum(np.abs(ref) ** 2)))
        errs = []
        for h in h_list:
            uh = run(replace(base, dt=h), device).final_state
            errs.append(float(np.sqrt(np.sum(np.abs(uh - ref) ** 2))) / ref_norm)
        x, y = np.log(np.array(h_list)), np.log(np.array(errs))
        n = len(h_list)
        slope = (n * np.sum(x * y) - x.sum() * y.sum()) / (n * np.sum(x * x) - x.sum() ** 2)
        rep.entries.append(ConvergenceEntry(m, list(h_list), errs, float(slope)))
    return rep
