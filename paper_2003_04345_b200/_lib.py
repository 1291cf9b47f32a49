"""ctypes binding of the C ABI in include/mb4cu.h (libmb4cu.so, built in-tree).

The product path has no CPU fallback: if the shared library is missing or
fails to load, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MB4CU_LIB") or os.path.join(HERE, "libmb4cu.so")

MB4CU_OK = 0
MB4CU_INVALID = 1
MB4CU_NONCONVERGED = 2
MB4CU_CUDA_ERROR = 3
MB4CU_COMM_ERROR = 4
MB4CU_OOM = 5
MB4CU_NUMERIC = 6

D = C.c_double
I = C.c_int


class Scheme(C.Structure):
    _fields_ = [
        ("alpha1", D),
        ("nodes", D * 4),
        ("E", (D * 4) * 3),
        ("W", (((D * 4) * 4) * 4) * 3),
        ("lam", D * 3),
        ("T", (D * 3) * 3),
        ("Tinv", (D * 3) * 3),
        ("zeta6", D * 6),
        ("w6", D * 6),
        ("L", (D * 4) * 6),
        ("WA", (D * 6) * 3),
    ]


class Problem(C.Structure):
    _fields_ = [
        ("nx", I), ("ny", I),
        ("cx", D), ("cy", D),
        ("gamma", D),
        ("V", C.POINTER(D)),
        ("epsilon", D),
        ("max_iters", I),
        ("max_step_halvings", I),
        ("neumann_terms", I),
        ("device", I),
        ("kernel", I),
        ("ghost", I),
        ("neumann_first", I),
        ("first_poly", I),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("newton_iters", I),
        ("halvings", I),
        ("solve_seconds", D),
        ("last_residual", D),
    ]


class Obs(C.Structure):
    _fields_ = [(k, D) for k in (
        "u_kinetic", "u_nonlinear", "u_external", "total_energy", "probability",
        "participation", "raw_quartic")]


class Profile(C.Structure):
    _fields_ = [
        ("kernel_ms", D),
        ("launches", C.c_longlong),
        ("sweeps", C.c_longlong),
        ("alg_bytes", D),
        ("other_launches", C.c_longlong),
        ("sweep_ms", D * 8),
        ("sweep_n", C.c_longlong * 8),
        ("redone", C.c_longlong),
        ("krylov_iters", C.c_longlong),
    ]


class Inputs(C.Structure):
    _fields_ = [
        ("gnx", I), ("gny", I),
        ("defect_frac", D),
        ("defect_seed", C.c_uint64),
        ("vd_min", D), ("vd_max", D),
        ("npackets", I),
        ("sigma", D),
        ("x0", D), ("y0", D), ("kx", D), ("ky", D),
        ("random_packets", I),
        ("packet_seed", C.c_uint64),
        ("k_max", D),
        ("threads", I),
    ]


_lib = None
_load_error = None


def lib() -> C.CDLL:
    """Load libmb4cu.so (once). Raises if it is absent -- there is no fallback."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    L = C.CDLL(LIB_PATH)
    P = C.c_void_p
    DP = C.POINTER(D)
    IP = C.POINTER(I)
    sigs = {
        "mb4cu_scheme_init": (I, [D, D, D, D, C.POINTER(Scheme)]),
        "mb4cu_create": (I, [C.POINTER(Problem), C.POINTER(Scheme), C.POINTER(P)]),
        "mb4cu_destroy": (I, [P]),
        "mb4cu_last_error": (C.c_char_p, [P]),
        "mb4cu_create_error": (C.c_char_p, []),
        "mb4cu_set_state": (I, [P, DP]),
        "mb4cu_get_state": (I, [P, DP]),
        "mb4cu_set_state_device": (I, [P, P]),
        "mb4cu_get_state_device": (I, [P, P]),
        "mb4cu_step": (I, [P, D, C.POINTER(Stats)]),
        "mb4cu_run": (I, [P, D, I, DP, IP, C.POINTER(Stats)]),
        "mb4cu_method_step": (I, [P, I, D, C.POINTER(Stats)]),
        "mb4cu_method_run": (I, [P, I, D, I, DP, IP, C.POINTER(Stats)]),
        "mb4cu_observables": (I, [P, C.POINTER(Obs)]),
        "mb4cu_set_stream": (I, [P, P]),
        "mb4cu_spectral_bound": (I, [P, DP]),
        "mb4cu_set_spectral_bound": (I, [P, D]),
        "mb4cu_set_neumann_terms": (I, [P, I]),
        "mb4cu_apply_kv": (I, [P, DP, DP]),
        "mb4cu_rhs": (I, [P, DP, DP]),
        "mb4cu_eval_phi": (I, [P, DP, DP, DP, DP, D, DP, DP, DP]),
        "mb4cu_make_inputs": (I, [C.POINTER(Inputs), I, I, I, I, DP, DP, DP]),
        "mb4cu_scale_state": (I, [DP, C.c_size_t, D, I]),
        "mb4cu_version": (C.c_char_p, []),
        "mb4cu_profile_enable": (I, [P, I]),
        "mb4cu_profile_reset": (I, [P]),
        "mb4cu_profile_get": (I, [P, C.POINTER(Profile)]),
        "mb4cu_halo_count": (C.c_size_t, [P, I, I]),
        "mb4cu_halo_pack": (I, [P, I, I, P]),
        "mb4cu_halo_unpack": (I, [P, I, I, P]),
        "mb4cu_sweep": (I, [P, D, I, DP, DP]),
        "mb4cu_sweep_async": (I, [P, D, I, I, P]),
        "mb4cu_sweep_region": (I, [P, D, I, I, I, I, P]),
        "mb4cu_commit_step": (I, [P, I]),
        "mb4cu_observables_sums": (I, [P, DP]),
        "mb4cu_ns_begin": (I, [P, D]),
        "mb4cu_ns_phibar": (I, [P]),
        "mb4cu_ns_solve": (I, [P, I]),
        "mb4cu_ns_get_correction": (I, [P, I, P]),
        "mb4cu_ns_set_correction": (I, [P, I, P]),
        "mb4cu_ns_update": (I, [P, DP]),
        "mb4cu_ns_commit": (I, [P]),
        "mb4cu_ns_get_stages": (I, [P, DP, DP, DP]),
        "mb4cu_ns_abort": (I, [P]),
        "mb4cu_eval_a": (D, [D, D, D]),
        "mb4cu_lagrange_basis": (I, [DP, I, D, DP]),
        "mb4cu_scheme_integrate_e": (I, [D, DP, I, DP]),
        "mb4cu_set_amax2": (I, [P, D]),
        "mb4cu_nccl_unique_id": (I, [C.c_char_p, C.c_char_p]),
        "mb4cu_dist_attach": (I, [P, C.c_char_p, C.c_char_p, I, I, IP, I, I, I, I, I]),
        "mb4cu_dist_step": (I, [P, D, C.POINTER(Stats), DP]),
        "mb4cu_dist_observables": (I, [P, DP]),
        "mb4cu_dist_detach": (I, [P]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def dptr(a: np.ndarray):
    """Pointer to a C-contiguous float64 / complex128 array."""
    assert a.flags["C_CONTIGUOUS"] and a.dtype in (np.float64, np.complex128), a.dtype
    return a.ctypes.data_as(C.POINTER(D))


EXPORTED = [
    "mb4cu_scheme_init", "mb4cu_create", "mb4cu_destroy", "mb4cu_last_error",
    "mb4cu_create_error", "mb4cu_set_state", "mb4cu_get_state", "mb4cu_set_state_device",
    "mb4cu_get_state_device", "mb4cu_step", "mb4cu_run", "mb4cu_method_step", "mb4cu_method_run",
    "mb4cu_observables",
    "mb4cu_set_stream", "mb4cu_spectral_bound", "mb4cu_set_spectral_bound", "mb4cu_set_neumann_terms", "mb4cu_apply_kv", "mb4cu_rhs", "mb4cu_eval_phi",
    "mb4cu_make_inputs", "mb4cu_scale_state", "mb4cu_version", "mb4cu_profile_enable",
    "mb4cu_profile_reset", "mb4cu_profile_get", "mb4cu_halo_count", "mb4cu_halo_pack",
    "mb4cu_halo_unpack", "mb4cu_sweep", "mb4cu_sweep_async", "mb4cu_sweep_region", "mb4cu_commit_step", "mb4cu_observables_sums",
    "mb4cu_ns_begin", "mb4cu_ns_phibar", "mb4cu_ns_solve", "mb4cu_ns_get_correction", "mb4cu_ns_set_correction",
    "mb4cu_ns_update", "mb4cu_ns_commit", "mb4cu_ns_get_stages", "mb4cu_ns_abort",
    "mb4cu_eval_a", "mb4cu_lagrange_basis", "mb4cu_scheme_integrate_e", "mb4cu_set_amax2",
    "mb4cu_nccl_unique_id", "mb4cu_dist_attach", "mb4cu_dist_step", "mb4cu_dist_observables", "mb4cu_dist_detach",
]
