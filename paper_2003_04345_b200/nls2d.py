"""Python mirror of the reference's hot-path API (proj/include/nls2d), backed by
the C ABI of libmb4cu (include/mb4cu.h).

Names, argument meaning and error behaviour follow the reference so the parity
tests read like its own tests:

  GridSpec / GridModel          lattice.hpp:21-73
  Mb4Scheme                     mb4_scheme.hpp:26-64
  NewtonConfig / StepStats      mb4_integrator.hpp:25-35, 97-101
  NonConvergenceError           mb4_integrator.hpp:17-23
  Observables / observables()   lattice.hpp:78-88
  rhs(), GridModel.apply_kv     lattice.hpp:62-76
  eval_phi()                    mb4_integrator.hpp:79-83
  mb4_step()                    mb4_integrator.hpp:103-110
  StepDriver.advance()          integrators.hpp:46-66

A State is a complex128 numpy vector, site k = j*nx + i (lattice.hpp:13-14).
All arithmetic runs on the GPU; host arrays only cross the boundary.
`Session` is the device-resident form (state stays in HBM across steps).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import dptr

MB4 = "mb4"
# the reference's methods in MethodId order (integrators.hpp:12)
METHODS = ("rk4", "gauss2", "gauss4", "avf2", "avf4", "mb4")
_METHOD_NAMES = ("RK4", "GAUSS2", "GAUSS4", "AVF2", "AVF4", "MB4")


def parse_method(name: str) -> Optional[str]:
    """integrators.cpp:34-43 (case-insensitive); None when unknown."""
    n = name.lower()
    return n if n in METHODS else None


def method_name(method: str) -> str:
    """integrators.cpp:22-32."""
    return _METHOD_NAMES[METHODS.index(method)]


def method_order(method: str) -> int:
    """integrators.cpp:13-20."""
    return 2 if method in ("gauss2", "avf2") else 4


class NonConvergenceError(RuntimeError):
    """mb4_integrator.hpp:17-23."""

    def __init__(self, what: str, residual: float):
        super().__init__(what)
        self.last_residual = residual
        self.at_time = -1.0


class ComplexEigenvalueError(RuntimeError):
    """small_dense.hpp:43-46 (scheme validation failures map here or to ValueError)."""


class Mb4CudaError(RuntimeError):
    pass


def _raise_for(code: int, text: str, residual: float = float("nan")):
    if code == _lib.MB4CU_OK:
        return
    if code == _lib.MB4CU_NONCONVERGED:
        raise NonConvergenceError(text, residual)
    if code == _lib.MB4CU_INVALID:
        if text.startswith("eig3_real"):
            raise ComplexEigenvalueError(text)
        raise ValueError(text)
    if code == _lib.MB4CU_NUMERIC:
        raise RuntimeError(text)
    raise Mb4CudaError(f"mb4cu status {code}: {text}")


# --------------------------------------------------------------------------- lattice


@dataclass
class GridSpec:
    """Regular nx x ny periodic grid on [0,lx] x [0,ly] (lattice.hpp:21-33)."""

    nx: int
    ny: int
    lx: float
    ly: float

    def __post_init__(self):
        if self.nx < 2 or self.ny < 2:
            raise ValueError("GridSpec: nx and ny must be >= 2")
        if not (self.lx > 0.0) or not (self.ly > 0.0):
            raise ValueError("GridSpec: domain lengths must be positive")

    def hx(self) -> float:
        return self.lx / self.nx

    def hy(self) -> float:
        return self.ly / self.ny

    def points(self) -> int:
        return self.nx * self.ny

    def index(self, i: int, j: int) -> int:
        return j * self.nx + i


def build_delta_potential(grid: GridSpec, v0: float) -> np.ndarray:
    """lattice.hpp:40-41: v0 at grid point (0,0), zero elsewhere."""
    v = np.zeros(grid.points())
    v[grid.index(0, 0)] = v0
    return v


def initial_condition(grid: GridSpec) -> np.ndarray:
    """lattice.hpp:43-44: u = 1 + 2 cos x + 2 cos y."""
    x = np.arange(grid.nx) * grid.hx()
    y = np.arange(grid.ny) * grid.hy()
    u = 1.0 + 2.0 * np.cos(x)[None, :] + 2.0 * np.cos(y)[:, None]
    return u.reshape(-1).astype(np.complex128)


class GridModel:
    """i du/dt = K u - gamma |u|^2 u + V u with the periodic 5-point K (lattice.hpp:48-73).

    The custom-kinetic-matrix constructor (lattice.hpp:54) is out of scope for the
    GPU path: K is the hard-coded stencil with cx = 1/hx^2, cy = 1/hy^2.
    """

    def __init__(self, grid: GridSpec, gamma: float, potential: Optional[Sequence[float]] = None):
        self._grid = grid
        self._gamma = float(gamma)
        if potential is None:
            potential = np.zeros(grid.points())
        v = np.ascontiguousarray(potential, dtype=np.float64)
        if v.shape != (grid.points(),):
            raise ValueError("GridModel: potential length mismatch")
        self._v = v

    def grid(self) -> GridSpec:
        return self._grid

    def potential(self) -> np.ndarray:
        return self._v

    def gamma(self) -> float:
        return self._gamma

    def points(self) -> int:
        return self._grid.points()

    @property
    def cx(self) -> float:
        return 1.0 / (self._grid.hx() ** 2)

    @property
    def cy(self) -> float:
        return 1.0 / (self._grid.hy() ** 2)

    def apply_kv(self, u: np.ndarray) -> np.ndarray:
        """y = (K + V) u on the GPU (lattice.cpp:86-89)."""
        with _OpContext(self) as s:
            return s._unary("mb4cu_apply_kv", u)


# --------------------------------------------------------------------------- scheme


class Mb4Scheme:
    """Scheme constants (mb4_scheme.hpp:26-64), computed by libmb4cu on the host."""

    kAlpha1Bound = -300.0 * 0.7770503941

    def __init__(self, alpha1: float = -300.0 * 19.0 / 8.0, nodes=(1.0 / 3.0, 2.0 / 3.0, 1.0)):
        s = _lib.Scheme()
        L = _lib.lib()
        rc = L.mb4cu_scheme_init(alpha1, nodes[0], nodes[1], nodes[2], C.byref(s))
        _raise_for(rc, L.mb4cu_create_error().decode())
        self._s = s
        self._alpha1 = float(alpha1)

    @property
    def raw(self) -> _lib.Scheme:
        return self._s

    def alpha1(self) -> float:
        return self._alpha1

    def nodes(self):
        return tuple(self._s.nodes)

    def e_ext(self, i: int, j: int) -> float:
        return self._s.E[i - 1][j]

    def w(self, i: int, a: int, b: int, c: int) -> float:
        return self._s.W[i - 1][a][b][c]

    def eigenvalues(self):
        return tuple(self._s.lam)

    def t(self) -> np.ndarray:
        return np.array([[self._s.T[i][j] for j in range(3)] for i in range(3)])

    def t_inv(self) -> np.ndarray:
        return np.array([[self._s.Tinv[i][j] for j in range(3)] for i in range(3)])

    def E(self) -> np.ndarray:
        return np.array([[self._s.E[i][j] for j in range(4)] for i in range(3)])

    def W(self) -> np.ndarray:
        return np.array(self._s.W)

    def gl6_L(self) -> np.ndarray:
        return np.array([[self._s.L[q][a] for a in range(4)] for q in range(6)])

    def gl6_WA(self) -> np.ndarray:
        return np.array([[self._s.WA[i][q] for q in range(6)] for i in range(3)])


# --------------------------------------------------------------------------- integrator config


@dataclass
class NewtonConfig:
    """mb4_integrator.hpp:25-35.  On the GPU path max_iters caps the stage sweeps."""

    epsilon: float = 1e-13
    max_iters: int = 50
    max_step_halvings: int = 4

    def validate(self):
        if not (self.epsilon > 0.0):
            raise ValueError("NewtonConfig: epsilon must be > 0")
        if self.max_iters < 1:
            raise ValueError("NewtonConfig: max_iters must be >= 1")
        if self.max_step_halvings < 0:
            raise ValueError("NewtonConfig: negative halvings")


@dataclass
class StepStats:
    """mb4_integrator.hpp:97-101; newton_iters counts stage sweeps on the GPU path."""

    newton_iters: int = 0
    halvings: int = 0
    solve_seconds: float = 0.0
    last_residual: float = 0.0


@dataclass
class Observables:
    """lattice.hpp:78-86."""

    u_kinetic: float = 0.0
    u_nonlinear: float = 0.0
    u_external: float = 0.0
    total_energy: float = 0.0
    probability: float = 0.0
    participation: float = 0.0
    raw_quartic: float = 0.0

    @classmethod
    def from_row(cls, row) -> "Observables":
        return cls(*[float(x) for x in row[:7]])


OBS_FIELDS = ("u_kinetic", "u_nonlinear", "u_external", "total_energy", "probability",
              "participation", "raw_quartic")


# --------------------------------------------------------------------------- device session


class Session:
    """A device-resident MB4 stepping context (one mb4cu_ctx).

    Holds u0, V and the stage buffers in HBM; host arrays cross only in
    set_state / get_state.  neumann_terms selects the preconditioner depth m
    (None = library default); kernel 1 forces the tiled reference kernel.
    """

    def __init__(self, model: GridModel, scheme: Optional[Mb4Scheme] = None,
                 cfg: Optional[NewtonConfig] = None, neumann_terms: Optional[int] = None,
                 device: int = 0, kernel: int = 0, neumann_first: Optional[int] = None,
                 method: str = MB4, first_poly: int = 0):
        self._L = _lib.lib()
        if method not in METHODS:
            raise ValueError(f"StepDriver: unknown method {method!r}")
        self.method = method
        self._mid = METHODS.index(method)
        self.model = model
        self.scheme = scheme if scheme is not None else Mb4Scheme()
        self.cfg = cfg if cfg is not None else NewtonConfig()
        self.cfg.validate()
        p = _lib.Problem()
        p.nx, p.ny = model.grid().nx, model.grid().ny
        p.cx, p.cy = model.cx, model.cy
        p.gamma = model.gamma()
        self._v = model.potential()
        p.V = dptr(self._v)
        p.epsilon = self.cfg.epsilon
        p.max_iters = self.cfg.max_iters
        p.max_step_halvings = self.cfg.max_step_halvings
        p.neumann_terms = -1 if neumann_terms is None else int(neumann_terms)
        p.neumann_first = -1 if neumann_first is None else int(neumann_first)
        p.first_poly = int(first_poly)  # 0: Chebyshev first sweep when H is convex (mb4cu.h)
        p.ghost = 0
        p.device = device
        p.kernel = kernel
        self._ctx = C.c_void_p()
        rc = self._L.mb4cu_create(C.byref(p), C.byref(self.scheme.raw), C.byref(self._ctx))
        _raise_for(rc, self._L.mb4cu_create_error().decode())
        self.n = model.points()

    # lifecycle -------------------------------------------------------------
    def close(self):
        if getattr(self, "_ctx", None):
            self._L.mb4cu_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, rc: int, residual: float = float("nan")):
        if rc != _lib.MB4CU_OK:
            _raise_for(rc, self._L.mb4cu_last_error(self._ctx).decode(), residual)

    # state -----------------------------------------------------------------
    def set_state(self, u: np.ndarray):
        u = np.ascontiguousarray(u, dtype=np.complex128)
        if u.shape != (self.n,):
            raise ValueError("state length mismatch")
        self._check(self._L.mb4cu_set_state(self._ctx, dptr(u)))

    def get_state(self) -> np.ndarray:
        out = np.empty(self.n, dtype=np.complex128)
        self._check(self._L.mb4cu_get_state(self._ctx, dptr(out)))
        return out

    def set_stream(self, stream_ptr: int):
        self._check(self._L.mb4cu_set_stream(self._ctx, C.c_void_p(stream_ptr)))

    def set_state_device(self, ptr: int):
        self._check(self._L.mb4cu_set_state_device(self._ctx, C.c_void_p(ptr)))

    def get_state_device(self, ptr: int):
        self._check(self._L.mb4cu_get_state_device(self._ctx, C.c_void_p(ptr)))

    # stepping --------------------------------------------------------------
    def step(self, h: float, stats: Optional[StepStats] = None):
        st = _lib.Stats()
        rc = self._L.mb4cu_method_step(self._ctx, self._mid, float(h), C.byref(st))
        if stats is not None:
            stats.newton_iters += st.newton_iters
            stats.halvings += st.halvings
            stats.solve_seconds += st.solve_seconds
            stats.last_residual = st.last_residual
        self._check(rc, st.last_residual)

    def run(self, h: float, nsteps: int, record: bool = True, stats: Optional[StepStats] = None):
        """nsteps device-resident steps; returns (obs_series[(nsteps+1),7], iters[nsteps])."""
        obs = np.zeros((nsteps + 1, 7)) if record else None
        iters = np.zeros(nsteps, dtype=np.int32)
        st = _lib.Stats()
        rc = self._L.mb4cu_method_run(self._ctx, self._mid, float(h), int(nsteps),
                                      dptr(obs) if record else None,
                                      iters.ctypes.data_as(C.POINTER(C.c_int)), C.byref(st))
        if stats is not None:
            stats.newton_iters += st.newton_iters
            stats.halvings += st.halvings
            stats.solve_seconds += st.solve_seconds
            stats.last_residual = st.last_residual
        self._check(rc, st.last_residual)
        return obs, iters

    def spectral_bound(self) -> float:
        """The bound rho >= rho(J(u0)) placing the next step's Chebyshev polynomial (the
        context tracks max|u0|^2 per step through its first sweeps)."""
        rho = C.c_double(0.0)
        self._check(self._L.mb4cu_spectral_bound(self._ctx, C.byref(rho)))
        return rho.value

    def profile_enable(self, on: bool = True):
        self._check(self._L.mb4cu_profile_enable(self._ctx, int(on)))

    def profile_reset(self):
        self._check(self._L.mb4cu_profile_reset(self._ctx))

    def profile(self) -> dict:
        p = _lib.Profile()
        self._check(self._L.mb4cu_profile_get(self._ctx, C.byref(p)))
        out = {}
        for f, _ in _lib.Profile._fields_:
            v = getattr(p, f)
            out[f] = list(v) if hasattr(v, "__len__") else v
        return out

    def observables(self) -> Observables:
        o = _lib.Obs()
        self._check(self._L.mb4cu_observables(self._ctx, C.byref(o)))
        return Observables(*[getattr(o, f) for f in OBS_FIELDS])

    # parity operators on host arrays ----------------------------------------
    def _unary(self, fn: str, u: np.ndarray) -> np.ndarray:
        u = np.ascontiguousarray(u, dtype=np.complex128)
        y = np.empty_like(u)
        self._check(getattr(self._L, fn)(self._ctx, dptr(u), dptr(y)))
        return y

    def eval_phi(self, u0, stages, h):
        u0 = np.ascontiguousarray(u0, dtype=np.complex128)
        st = [np.ascontiguousarray(s, dtype=np.complex128) for s in stages]
        out = [np.empty_like(u0) for _ in range(3)]
        self._check(self._L.mb4cu_eval_phi(self._ctx, dptr(u0), dptr(st[0]), dptr(st[1]),
                                           dptr(st[2]), float(h), dptr(out[0]), dptr(out[1]),
                                           dptr(out[2])))
        return out


class _OpContext:
    """Short-lived session for the stateless operators (apply_kv, rhs, eval_phi, observables)."""

    def __init__(self, model: GridModel, scheme: Optional[Mb4Scheme] = None):
        self.model = model
        self.scheme = scheme

    def __enter__(self) -> Session:
        self.s = Session(self.model, self.scheme)
        return self.s

    def __exit__(self, *exc):
        self.s.close()


def rhs(model: GridModel, u: np.ndarray) -> np.ndarray:
    """f(u) = -i(Ku + Vu - gamma |u|^2 u) on the GPU (lattice.cpp:91-104)."""
    if len(u) != model.points():
        raise ValueError("rhs: state length mismatch")
    with _OpContext(model) as s:
        return s._unary("mb4cu_rhs", u)


def observables(model: GridModel, u: np.ndarray) -> Observables:
    """Energy monitor on the GPU (lattice.cpp:106-137)."""
    if len(u) != model.points():
        raise ValueError("observables: state length mismatch")
    with _OpContext(model) as s:
        s.set_state(u)
        return s.observables()


def eval_phi(model: GridModel, scheme: Mb4Scheme, u0: np.ndarray, stages, h: float):
    """Stage residuals (mb4_integrator.cpp:159-192) via the GL-6 quadrature form."""
    with _OpContext(model, scheme) as s:
        return s.eval_phi(u0, stages, h)


def _method_step(method: str, model: GridModel, u0: np.ndarray, h: float, cfg: Optional[NewtonConfig],
                 stats: Optional[StepStats]) -> np.ndarray:
    cfg = cfg if cfg is not None else NewtonConfig()
    cfg.validate()
    # a plain step: the free functions of integrators.hpp do not halve
    plain = NewtonConfig(cfg.epsilon, cfg.max_iters, 0)
    with Session(model, Mb4Scheme(), plain, method=method) as s:
        s.set_state(u0)
        s.step(h, stats)
        return s.get_state()


def rk4_step(model: GridModel, u0: np.ndarray, h: float) -> np.ndarray:
    """integrators.cpp:45-59 on the GPU."""
    return _method_step("rk4", model, u0, h, None, None)


def gauss_step(model: GridModel, u0: np.ndarray, h: float, stages: int, cfg: NewtonConfig,
               stats: Optional[StepStats] = None, solver=None, cached_order=None) -> np.ndarray:
    """integrators.cpp:103-208 (stages 1: implicit midpoint, 2: Gauss order 4)."""
    if stages not in (1, 2):
        raise ValueError("gauss_step: stages must be 1 or 2")
    return _method_step("gauss2" if stages == 1 else "gauss4", model, u0, h, cfg, stats)


def avf2_step(model: GridModel, u0: np.ndarray, h: float, cfg: NewtonConfig,
              stats: Optional[StepStats] = None, solver=None, cached_order=None) -> np.ndarray:
    """integrators.cpp:210-282."""
    return _method_step("avf2", model, u0, h, cfg, stats)


def avf4_step(model: GridModel, u0: np.ndarray, h: float, cfg: NewtonConfig,
              stats: Optional[StepStats] = None, solver=None, cached_order=None) -> np.ndarray:
    """integrators.cpp:284-395."""
    return _method_step("avf4", model, u0, h, cfg, stats)


def mb4_step(model: GridModel, scheme: Mb4Scheme, u0: np.ndarray, h: float, cfg: NewtonConfig,
             pool=None, stats: Optional[StepStats] = None, solver=None, cached_order=None,
             neumann_terms: Optional[int] = None) -> np.ndarray:
    """One MB4 step (mb4_integrator.cpp:275-316) through the C ABI with host buffers.

    pool / solver / cached_order are accepted for signature compatibility and
    ignored: the GPU path has no sparse factorization and no worker pool.
    """
    cfg.validate()
    if not (h > 0.0):
        raise ValueError("mb4_step: h must be positive")
    with Session(model, scheme, cfg, neumann_terms=neumann_terms) as s:
        s.set_state(u0)
        s.step(h, stats)
        return s.get_state()


class StepDriver:
    """integrators.hpp:46-66: any of the reference's methods on the GPU.

    Owns one device session for its model; each advance() uploads u0, steps,
    and downloads the result (the reference's host-vector contract).  MB4 runs the
    production stage solver; RK4 / GAUSS2 / GAUSS4 / AVF2 / AVF4 run methods.cu
    with the reference's halving-on-failure policy (RK4: none).
    """

    def __init__(self, model: GridModel, method: str = MB4, cfg: Optional[NewtonConfig] = None,
                 solver=None, pool=None, neumann_terms: Optional[int] = None, device: int = 0):
        method = method.lower() if isinstance(method, str) else method
        if method not in METHODS:
            raise ValueError(f"StepDriver: unknown method {method!r}")
        self.method = method
        self.cfg = cfg if cfg is not None else NewtonConfig()
        self.cfg.validate()
        self._scheme = Mb4Scheme()
        self._session = Session(model, self._scheme, self.cfg, neumann_terms=neumann_terms,
                                device=device, method=method)

    def scheme(self) -> Mb4Scheme:
        return self._scheme

    @property
    def session(self) -> Session:
        return self._session

    def advance(self, u0: np.ndarray, h: float, stats: Optional[StepStats] = None) -> np.ndarray:
        if not (h > 0.0):
            raise ValueError("advance: h must be positive")
        self._session.set_state(u0)
        self._session.step(h, stats)
        return self._session.get_state()

    def close(self):
        self._session.close()
