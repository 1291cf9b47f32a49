"""CPU tests of the drop-in boundary: libmb4cu.so loads and exports every symbol
include/mb4cu.h declares; host-side logic (scheme tables, input generator,
argument validation) behaves like the reference.  No GPU compute here."""
import ctypes as C
import json
import os
import re

import numpy as np
import pytest

from paper_2003_04345_b200 import _lib, configs, nls2d

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def declared_symbols():
    with open(os.path.join(ROOT, "include", "mb4cu.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(mb4cu_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert set(syms) == set(_lib.EXPORTED)


def test_library_is_sm100a():
    # the shipped fatbin is compiled for sm_100a only
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out


def test_scheme_tables_match_exact_rationals():
    with open(os.path.join(GOLD, "scheme_exact.json")) as f:
        ex = json.load(f)
    s = nls2d.Mb4Scheme()
    assert np.abs(s.E() - np.array(ex["E"]).reshape(3, 4)).max() <= 1e-14
    assert np.abs(s.W() - np.array(ex["W"]).reshape(3, 4, 4, 4)).max() <= 1e-14
    assert np.abs(np.array(s.eigenvalues()) - np.array(ex["eigenvalues"])).max() <= 1e-13
    W2 = np.einsum("iq,qa,qb,qc->iabc", s.gl6_WA(), s.gl6_L(), s.gl6_L(), s.gl6_L())
    assert np.abs(W2 - np.array(ex["W"]).reshape(3, 4, 4, 4)).max() <= 1e-14


def test_scheme_validation_matches_reference():
    # mb4_scheme.cpp:84-93
    with pytest.raises(ValueError):
        nls2d.Mb4Scheme(alpha1=-100.0)
    with pytest.raises(ValueError):
        nls2d.Mb4Scheme(nodes=(1 / 3, 2 / 3, 0.9))
    with pytest.raises(ValueError):
        nls2d.Mb4Scheme(nodes=(0.5, 0.5, 1.0))
    with pytest.raises(ValueError):
        nls2d.Mb4Scheme(nodes=(0.0, 0.5, 1.0))


def test_grid_and_newton_validation():
    with pytest.raises(ValueError):
        nls2d.GridSpec(1, 4, 1.0, 1.0)
    with pytest.raises(ValueError):
        nls2d.GridSpec(4, 4, 0.0, 1.0)
    for bad in (dict(epsilon=0.0), dict(max_iters=0), dict(max_step_halvings=-1)):
        with pytest.raises(ValueError):
            nls2d.NewtonConfig(**bad).validate()
    g = nls2d.GridSpec(4, 4, 1.0, 1.0)
    with pytest.raises(ValueError):
        nls2d.GridModel(g, 0.1, np.zeros(5))


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg4"])
def test_input_generator_block_equals_slice(name):
    cfg = configs.CONFIGS[name]
    if cfg.sites > 4096 * 4096:
        pytest.skip("too large")
    small = cfg if cfg.nx <= 256 else cfg.with_lattice(512, 512)
    V, psi, s = configs.make_block(small)
    Vb, pb, sb = configs.make_block(small, 3, 5, small.nx // 2, small.ny // 3)
    Vs = V.reshape(small.ny, small.nx)[5:5 + small.ny // 3, 3:3 + small.nx // 2]
    ps = psi.reshape(small.ny, small.nx)[5:5 + small.ny // 3, 3:3 + small.nx // 2]
    assert np.array_equal(Vb.reshape(Vs.shape), Vs)
    assert np.array_equal(pb.reshape(ps.shape), ps)


def test_input_generator_statistics_and_determinism():
    cfg = configs.CONFIGS["cfg2"]
    V1, p1 = configs.make_inputs(cfg)
    V2, p2 = configs.make_inputs(cfg, threads=3)
    assert np.array_equal(V1, V2) and np.array_equal(p1, p2)
    frac = (V1 > 0).mean()
    assert abs(frac - cfg.defect_frac) < 0.005
    assert set(np.unique(V1)) <= {0.0, cfg.vd_min}
    assert abs(np.vdot(p1, p1).real - 1.0) < 1e-14
    # packet centre at (64,128) with the stated momentum: |psi| peaks there
    k = int(np.argmax(np.abs(p1)))
    assert (k % cfg.nx, k // cfg.nx) == (64, 128)
    c4 = configs.CONFIGS["cfg4"].with_lattice(256, 256)
    V4, _ = configs.make_inputs(c4)
    d = V4[V4 > 0]
    assert d.min() >= 5.0 and d.max() < 50.0


def test_cfg5_weak_scaling_tiling():
    assert configs.cfg5_lattice(1) == (8192, 8192)
    assert configs.cfg5_lattice(8) == (16384, 32768)
    for n in (1, 2, 4, 8):
        nx, ny = configs.cfg5_lattice(n)
        assert nx * ny == n * 8192 * 8192


def test_create_rejects_bad_problems_before_touching_the_gpu():
    L = _lib.lib()
    s = nls2d.Mb4Scheme()
    V = np.zeros(16)
    for field, val in (("nx", 1), ("epsilon", 0.0), ("max_iters", 0), ("neumann_terms", 7), ("first_poly", 3),
                       ("first_poly", -1)):
        p = _lib.Problem()
        p.nx = p.ny = 4
        p.cx = p.cy = 1.0
        p.gamma = -1.0
        p.V = _lib.dptr(V)
        p.epsilon, p.max_iters, p.max_step_halvings, p.neumann_terms = 1e-14, 50, 4, 2
        setattr(p, field, val)
        ctx = C.c_void_p()
        rc = L.mb4cu_create(C.byref(p), C.byref(s.raw), C.byref(ctx))
        assert rc == _lib.MB4CU_INVALID
        assert L.mb4cu_create_error().decode()


def test_abi_null_and_range_checks_without_a_gpu():
    """Entry points validate their arguments before any device work (status codes of
    include/mb4cu.h); the spectral-bound setter rejects negative / non-finite bounds."""
    L = _lib.lib()
    assert L.mb4cu_spectral_bound(None, None) == _lib.MB4CU_INVALID
    assert L.mb4cu_set_spectral_bound(None, 1.0) == _lib.MB4CU_INVALID
    assert L.mb4cu_step(None, 0.01, None) == _lib.MB4CU_INVALID
    assert L.mb4cu_set_neumann_terms(None, 1) == _lib.MB4CU_INVALID
    assert L.mb4cu_ns_begin(None, 0.01) == _lib.MB4CU_INVALID
    assert L.mb4cu_ns_commit(None) == _lib.MB4CU_INVALID
