"""TEST INFRASTRUCTURE ONLY -- ctypes bindings of the CPU checkers.

  Restatement : oracle/liboracle.so        (oracle/mb4_oracle.c, plain C)
  Reference   : oracle/_ref/libnls2d_ref.so (the unmodified reference library
                compiled from /root/reference/proj/src + oracle/ref_driver.cpp)

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this module.  Nothing in the product package
(paper_2003_04345_b200/) imports it.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libnls2d_ref.so")

D = C.c_double
DP = C.POINTER(D)
IP = C.POINTER(C.c_int)


class OrcScheme(C.Structure):
    _fields_ = [
        ("alpha1", D), ("nodes", D * 4), ("E", (D * 4) * 3), ("W", (((D * 4) * 4) * 4) * 3),
        ("lam", D * 3), ("T", (D * 3) * 3), ("Tinv", (D * 3) * 3), ("zeta6", D * 6),
        ("w6", D * 6), ("L", (D * 4) * 6), ("WA", (D * 6) * 3),
    ]


class OrcModel(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("cx", D), ("cy", D), ("gamma", D), ("V", DP)]


class OrcNewton(C.Structure):
    _fields_ = [("epsilon", D), ("max_iters", C.c_int), ("max_step_halvings", C.c_int)]


class OrcObs(C.Structure):
    _fields_ = [(k, D) for k in ("u_kinetic", "u_nonlinear", "u_external", "total_energy",
                                 "probability", "participation", "raw_quartic")]


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"] and a.dtype in (np.float64, np.complex128)
    return a.ctypes.data_as(DP)


_olib = None
_rlib = None


def oracle_lib() -> C.CDLL:
    global _olib
    if _olib is None:
        L = C.CDLL(ORACLE_SO)
        L.orc_scheme_init.argtypes = [D, D, D, D, C.POINTER(OrcScheme)]
        L.orc_scheme_init.restype = C.c_int
        L.orc_apply_kv.argtypes = [C.POINTER(OrcModel), DP, DP]
        L.orc_rhs.argtypes = [C.POINTER(OrcModel), DP, DP]
        L.orc_observables.argtypes = [C.POINTER(OrcModel), DP, C.POINTER(OrcObs)]
        L.orc_observables.restype = C.c_int
        L.orc_eval_phi.argtypes = [C.POINTER(OrcModel), C.POINTER(OrcScheme), DP, C.POINTER(DP), D,
                                   C.POINTER(DP)]
        L.orc_newton_solve.argtypes = [C.POINTER(OrcModel), C.POINTER(OrcScheme), DP, D,
                                       C.POINTER(OrcNewton), C.POINTER(DP), IP, DP]
        L.orc_newton_solve.restype = C.c_int
        L.orc_mb4_step.argtypes = [C.POINTER(OrcModel), C.POINTER(OrcScheme), DP, D,
                                   C.POINTER(OrcNewton), DP, IP, IP, DP]
        L.orc_mb4_step.restype = C.c_int
        L.orc_run.argtypes = [C.POINTER(OrcModel), C.POINTER(OrcScheme), DP, D, C.c_int,
                              C.POINTER(OrcNewton), DP, IP]
        L.orc_run.restype = C.c_int
        _olib = L
    return _olib


INPUTS_SO = os.path.join(HERE, "libinputs.so")
_ilib = None


def inputs_generator():
    """(make_inputs, scale_state) of oracle/libinputs.so: the BASELINE input generator
    compiled host-only (g++), for bench.py's reference arm -- same source and arithmetic
    as the product library's mb4cu_make_inputs, without mapping libmb4cu.so.
    Pass it as configs.make_inputs(cfg, gen=...)."""
    global _ilib
    if _ilib is None:
        L = C.CDLL(INPUTS_SO)
        L.orc_make_inputs.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, DP, DP, DP]
        L.orc_make_inputs.restype = C.c_int
        L.orc_scale_state.argtypes = [DP, C.c_size_t, D, C.c_int]
        L.orc_scale_state.restype = C.c_int
        _ilib = L
    return _ilib.orc_make_inputs, _ilib.orc_scale_state


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib() -> C.CDLL:
    global _rlib
    if _rlib is None:
        L = C.CDLL(REF_SO)
        L.ref_scheme.argtypes = [DP, DP, DP, DP, DP]
        L.ref_scheme.restype = C.c_int
        L.ref_observables.argtypes = [C.c_int, C.c_int, D, D, D, DP, DP, DP]
        L.ref_observables.restype = C.c_int
        L.ref_eval_phi.argtypes = [C.c_int, C.c_int, D, D, D, DP, DP, DP, DP, DP, D, DP, DP, DP]
        L.ref_eval_phi.restype = C.c_int
        L.ref_mb4_run.argtypes = [C.c_int, C.c_int, D, D, D, DP, DP, D, C.c_int, D, C.c_int,
                                  C.c_int, C.c_int, C.c_int, DP, IP, DP]
        L.ref_mb4_run.restype = C.c_int
        L.ref_method_run.argtypes = [C.c_int] + L.ref_mb4_run.argtypes
        L.ref_method_run.restype = C.c_int
        _rlib = L
    return _rlib


# --------------------------------------------------------------------------- restatement


class Oracle:
    """The plain-C restatement bound to one lattice problem."""

    def __init__(self, nx: int, ny: int, gamma: float, V: np.ndarray, cx: float = 1.0,
                 cy: float = 1.0, alpha1: float = -712.5):
        self.L = oracle_lib()
        self.V = np.ascontiguousarray(V, dtype=np.float64)
        self.m = OrcModel(nx, ny, cx, cy, gamma, _p(self.V))
        self.s = OrcScheme()
        rc = self.L.orc_scheme_init(alpha1, 1.0 / 3.0, 2.0 / 3.0, 1.0, C.byref(self.s))
        if rc != 0:
            raise ValueError(f"orc_scheme_init failed ({rc})")
        self.n = nx * ny

    def apply_kv(self, u):
        u = np.ascontiguousarray(u, dtype=np.complex128)
        y = np.empty_like(u)
        self.L.orc_apply_kv(C.byref(self.m), _p(u), _p(y))
        return y

    def rhs(self, u):
        u = np.ascontiguousarray(u, dtype=np.complex128)
        y = np.empty_like(u)
        self.L.orc_rhs(C.byref(self.m), _p(u), _p(y))
        return y

    def observables(self, u):
        u = np.ascontiguousarray(u, dtype=np.complex128)
        o = OrcObs()
        rc = self.L.orc_observables(C.byref(self.m), _p(u), C.byref(o))
        if rc != 0:
            raise RuntimeError("orc_observables: non-real kinetic quadratic form")
        return o

    def eval_phi(self, u0, stages, h):
        u0 = np.ascontiguousarray(u0, dtype=np.complex128)
        st = [np.ascontiguousarray(s, dtype=np.complex128) for s in stages]
        out = [np.empty_like(u0) for _ in range(3)]
        sp = (DP * 3)(*[_p(s) for s in st])
        op = (DP * 3)(*[_p(o) for o in out])
        self.L.orc_eval_phi(C.byref(self.m), C.byref(self.s), _p(u0), sp, h, op)
        return out

    def newton_solve(self, u0, h, eps=1e-13, max_iters=50):
        u0 = np.ascontiguousarray(u0, dtype=np.complex128)
        out = [np.empty_like(u0) for _ in range(3)]
        op = (DP * 3)(*[_p(o) for o in out])
        it = C.c_int(0)
        res = D(0.0)
        cfg = OrcNewton(eps, max_iters, 0)
        rc = self.L.orc_newton_solve(C.byref(self.m), C.byref(self.s), _p(u0), h, C.byref(cfg), op,
                                     C.byref(it), C.byref(res))
        return rc, out, it.value, res.value

    def step(self, u0, h, eps=1e-13, max_iters=50, max_halvings=4):
        u0 = np.ascontiguousarray(u0, dtype=np.complex128)
        u1 = np.empty_like(u0)
        it, hv, res = C.c_int(0), C.c_int(0), D(0.0)
        cfg = OrcNewton(eps, max_iters, max_halvings)
        rc = self.L.orc_mb4_step(C.byref(self.m), C.byref(self.s), _p(u0), h, C.byref(cfg), _p(u1),
                                 C.byref(it), C.byref(hv), C.byref(res))
        return rc, u1, it.value, hv.value, res.value

    def run(self, u0, h, nsteps, eps=1e-14, max_iters=50, max_halvings=4):
        u = np.array(u0, dtype=np.complex128, copy=True)
        obs = np.zeros((nsteps + 1, 7))
        iters = np.zeros(nsteps, dtype=np.int32)
        cfg = OrcNewton(eps, max_iters, max_halvings)
        rc = self.L.orc_run(C.byref(self.m), C.byref(self.s), _p(u), h, nsteps, C.byref(cfg),
                            _p(obs), iters.ctypes.data_as(IP))
        if rc != 0:
            raise RuntimeError(f"orc_run failed with status {rc}")
        return u, obs, iters


# --------------------------------------------------------------------------- the reference itself


def ref_scheme():
    L = ref_lib()
    E = np.zeros(12)
    W = np.zeros(192)
    lam = np.zeros(3)
    T = np.zeros(9)
    Ti = np.zeros(9)
    if L.ref_scheme(_p(E), _p(W), _p(lam), _p(T), _p(Ti)) != 0:
        raise RuntimeError("ref_scheme failed")
    return E.reshape(3, 4), W.reshape(3, 4, 4, 4), lam, T.reshape(3, 3), Ti.reshape(3, 3)


def ref_observables(nx, ny, lx, ly, gamma, V, u):
    out = np.zeros(7)
    V = np.ascontiguousarray(V, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.complex128)
    if ref_lib().ref_observables(nx, ny, lx, ly, gamma, _p(V), _p(u), _p(out)) != 0:
        raise RuntimeError("ref_observables failed")
    return out


def ref_eval_phi(nx, ny, lx, ly, gamma, V, u0, stages, h):
    V = np.ascontiguousarray(V, dtype=np.float64)
    u0 = np.ascontiguousarray(u0, dtype=np.complex128)
    st = [np.ascontiguousarray(s, dtype=np.complex128) for s in stages]
    out = [np.empty_like(u0) for _ in range(3)]
    rc = ref_lib().ref_eval_phi(nx, ny, lx, ly, gamma, _p(V), _p(u0), _p(st[0]), _p(st[1]),
                                _p(st[2]), h, _p(out[0]), _p(out[1]), _p(out[2]))
    if rc != 0:
        raise RuntimeError("ref_eval_phi failed")
    return out


METHODS = ("rk4", "gauss2", "gauss4", "avf2", "avf4", "mb4")  # integrators.hpp:12 order


def ref_run(nx, ny, lx, ly, gamma, V, u0, h, nsteps, eps=1e-14, max_iters=50, max_halvings=4,
            solver: str = "direct", workers: int = 1, record: bool = True, method: str = "mb4"):
    """The reference stepping loop (StepDriver(method) -> advance) on the host cores.

    Returns (u_final, obs[(nsteps+1),7] or None, iters[nsteps], seconds)."""
    V = np.ascontiguousarray(V, dtype=np.float64)
    u = np.array(u0, dtype=np.complex128, copy=True)
    obs = np.zeros((nsteps + 1, 7)) if record else None
    iters = np.zeros(nsteps, dtype=np.int32)
    secs = D(0.0)
    rc = ref_lib().ref_method_run(METHODS.index(method.lower()), nx, ny, lx, ly, gamma, _p(V), _p(u), h,
                                  nsteps, eps, max_iters, max_halvings, 1 if solver == "gmres" else 0,
                                  workers, _p(obs) if record else None, iters.ctypes.data_as(IP),
                                  C.byref(secs))
    if rc != 0:
        raise RuntimeError(f"ref_method_run({method}) failed with status {rc}")
    return u, obs, iters, secs.value
