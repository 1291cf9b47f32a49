"""GPU parity tests: the CUDA path (through the C ABI) against the oracle.

Tolerances (written here, per BASELINE.json north_star):
  - state after 10 steps: relative L2 <= 1e-10 against the reference oracle;
  - relative energy drift |H(t)-H(0)|/|H(0)| <= 1e-13 over the run;
  - operators (Phi, (K+V)u, f(u), observables) <= 1e-12 / 1e-13 as the
    reference's own tests use (test_mb4_integrator.cpp:78-91, test_lattice.cpp:177-198).
"""
import numpy as np
import pytest

import sweep_model as SM
from oracle import oracle as O
from paper_2003_04345_b200 import configs, nls2d

pytestmark = pytest.mark.gpu

TWO_PI = 2.0 * np.pi


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def random_state(n, seed, amp=1.0):
    rng = np.random.default_rng(seed)
    return (rng.uniform(-amp, amp, n) + 1j * rng.uniform(-amp, amp, n)).astype(np.complex128)


# ----------------------------------------------------------------------------- operators


@pytest.mark.parametrize("nx,ny", [(4, 4), (5, 4), (2, 3), (64, 48)])
def test_apply_kv_and_rhs_match_oracle(nx, ny):
    g = nls2d.GridSpec(nx, ny, TWO_PI, 4.0)
    V = np.linspace(-2.0, 3.0, nx * ny)
    model = nls2d.GridModel(g, 0.3, V)
    o = O.Oracle(nx, ny, 0.3, V, cx=model.cx, cy=model.cy)
    u = random_state(nx * ny, 5)
    scale = np.abs(o.apply_kv(u)).max()
    assert np.abs(model.apply_kv(u) - o.apply_kv(u)).max() <= 1e-13 * scale
    assert np.abs(nls2d.rhs(model, u) - o.rhs(u)).max() <= 1e-13 * scale


@pytest.mark.parametrize("gamma", [0.0, 0.1, -2.0])
def test_eval_phi_matches_reference_w_form(gamma):
    # Phi via the GL-6 quadrature form vs the reference's W contraction
    # (mb4_integrator.cpp:159-192); tolerance of test_mb4_integrator.cpp:89.
    g = nls2d.GridSpec(4, 4, TWO_PI, TWO_PI)
    V = nls2d.build_delta_potential(g, 0.0 if gamma == 0.0 else -2.0)
    model = nls2d.GridModel(g, gamma, V)
    scheme = nls2d.Mb4Scheme()
    u0 = random_state(16, 31)
    st = [random_state(16, 40 + i) for i in range(3)]
    phi = nls2d.eval_phi(model, scheme, u0, st, 0.01)
    o = O.Oracle(4, 4, gamma, V, cx=model.cx, cy=model.cy)
    ref = o.eval_phi(u0, st, 0.01)
    assert max(np.abs(a - b).max() for a, b in zip(phi, ref)) <= 1e-12
    if O.ref_available():
        rr = O.ref_eval_phi(4, 4, TWO_PI, TWO_PI, gamma, V, u0, st, 0.01)
        assert max(np.abs(a - b).max() for a, b in zip(phi, rr)) <= 1e-12


def test_eval_phi_fixed_point_at_zero_step():
    # test_mb4_integrator.cpp:67-76
    g = nls2d.GridSpec(4, 4, TWO_PI, TWO_PI)
    model = nls2d.GridModel(g, 0.1)
    u0 = random_state(16, 9)
    phi = nls2d.eval_phi(model, nls2d.Mb4Scheme(), u0, [u0, u0, u0], 0.0)
    assert all(np.abs(p).max() == 0.0 for p in phi)


def test_observables_match_oracle():
    cfg = configs.CONFIGS["cfg2"]
    V, psi = configs.make_inputs(cfg)
    model = configs.model_for(cfg, V)
    got = nls2d.observables(model, psi)
    o = O.Oracle(cfg.nx, cfg.ny, cfg.gamma, V).observables(psi)
    for f in nls2d.OBS_FIELDS:
        a, b = getattr(got, f), getattr(o, f)
        assert abs(a - b) <= 1e-13 * max(1.0, abs(b)), (f, a, b)


# ----------------------------------------------------------------------------- single sweeps


@pytest.mark.parametrize("m", [0, 1, 2, 3])
@pytest.mark.parametrize("kernel", [0, 1, 2])
def test_first_step_sweep_count_and_state_match_numpy_model(m, kernel):
    cfg = configs.CONFIGS["cfg1"]
    V, psi = configs.make_inputs(cfg)
    model = configs.model_for(cfg, V)
    scheme = nls2d.Mb4Scheme()
    # default first-sweep depth: 6 on the production kernel, 2 on the tiled one, m on v1
    mf = m if (kernel == 2 or m > 2) else (6 if kernel == 0 else 2)
    ref, its = SM.step(psi, V, cfg.gamma, cfg.dt, scheme, m, cfg.nx, cfg.ny, cfg.epsilon, mf=mf,
                       first_poly=0 if (kernel == 0 and m <= 2) else 1)
    with nls2d.Session(model, scheme, configs.newton_for(cfg), neumann_terms=m, kernel=kernel) as s:
        s.set_state(psi)
        st = nls2d.StepStats()
        s.step(cfg.dt, st)
        got = s.get_state()
    assert st.newton_iters == its
    assert rel(got, ref) <= 1e-13


# ----------------------------------------------------------------------------- stepping parity


def _oracle_steps(cfg, V, psi, nsteps):
    if O.ref_available():
        solver = "direct" if cfg.sites <= 4096 else "gmres"
        u, obs, iters, _ = O.ref_run(cfg.nx, cfg.ny, float(cfg.nx), float(cfg.ny), cfg.gamma, V, psi,
                                     cfg.dt, nsteps, eps=cfg.epsilon, solver=solver)
        return u, obs
    u, obs, _ = O.Oracle(cfg.nx, cfg.ny, cfg.gamma, V).run(psi, cfg.dt, nsteps, eps=cfg.epsilon)
    return u, obs


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
@pytest.mark.parametrize("m", [None, 0, 1, 2, 3])  # None: default (deep first sweep, adaptive m)
def test_ten_steps_match_oracle(name, m):
    cfg = configs.CONFIGS[name]
    V, psi = configs.make_inputs(cfg)
    ref, ref_obs = _oracle_steps(cfg, V, psi, 10)
    model = configs.model_for(cfg, V)
    with nls2d.Session(model, nls2d.Mb4Scheme(), configs.newton_for(cfg), neumann_terms=m) as s:
        s.set_state(psi)
        obs, iters = s.run(cfg.dt, 10)
        got = s.get_state()
    assert rel(got, ref) <= 1e-10
    H0 = ref_obs[0, 3]
    assert np.abs(obs[:, 3] - ref_obs[:, 3]).max() <= 1e-13 * abs(H0)
    assert np.abs(obs[:, 3] - obs[0, 3]).max() <= 1e-13 * abs(obs[0, 3])


def test_mb4_step_drop_in_matches_oracle():
    cfg = configs.CONFIGS["cfg1"]
    V, psi = configs.make_inputs(cfg)
    model = configs.model_for(cfg, V)
    stats = nls2d.StepStats()
    u1 = nls2d.mb4_step(model, nls2d.Mb4Scheme(), psi, cfg.dt, configs.newton_for(cfg), stats=stats)
    ref, _ = _oracle_steps(cfg, V, psi, 1)
    assert rel(u1, ref) <= 1e-10
    assert stats.newton_iters > 0 and stats.halvings == 0


@pytest.mark.parametrize("alpha1", [-712.5, -800.0])
@pytest.mark.parametrize("m", [1, 2])
def test_scheme_tables_runtime_and_compiled(alpha1, m):
    """The production kernel uses compile-time tables only for the default scheme
    (alpha1 = -712.5); any other alpha1 runs on the runtime tables.  Both must
    match the oracle built with the same scheme."""
    cfg = configs.CONFIGS["cfg2"]
    V, psi = configs.make_inputs(cfg)
    o = O.Oracle(cfg.nx, cfg.ny, cfg.gamma, V, alpha1=alpha1)
    ref, ref_obs, _ = o.run(psi, cfg.dt, 5, eps=cfg.epsilon)
    model = configs.model_for(cfg, V)
    with nls2d.Session(model, nls2d.Mb4Scheme(alpha1), configs.newton_for(cfg), neumann_terms=m) as s:
        s.set_state(psi)
        obs, _ = s.run(cfg.dt, 5)
        got = s.get_state()
    assert rel(got, ref) <= 1e-10
    assert np.abs(obs[:, 3] - ref_obs[:, 3]).max() <= 1e-13 * abs(ref_obs[0, 3])


def _packet_lattice(nx, ny, lx, ly, seed=3):
    g = nls2d.GridSpec(nx, ny, lx, ly)
    rng = np.random.default_rng(seed)
    V = np.where(rng.uniform(size=nx * ny) < 0.02, 5.0, 0.0)
    x = (np.arange(nx) - nx / 3) / 9.0
    y = (np.arange(ny) - ny / 2) / 7.0
    psi = (np.exp(-(y[:, None] ** 2 + x[None, :] ** 2)) * np.exp(0.4j * np.arange(nx))[None, :]).reshape(-1)
    psi = (psi / np.linalg.norm(psi) * 3.0).astype(np.complex128)
    return g, V, psi


@pytest.mark.parametrize("first_poly", [0, 1, 2])
@pytest.mark.parametrize("mf,m", [(2, 1), (3, 1), (4, 1), (5, 1), (6, 1), (4, 2), (6, 2)])
@pytest.mark.parametrize("lattice", ["cfg1", "aniso_ragged"])
def test_deep_first_sweep_matches_numpy_model(mf, m, lattice, first_poly):
    """The specialised first sweep at depth mf (one J-chain instead of three stage
    recursions) gives the same sweep count and state as the numpy model, on an
    isotropic lattice (compiled scheme tables) and on an anisotropic one whose
    width is not a multiple of the band (runtime tables, partial bands)."""
    scheme = nls2d.Mb4Scheme()
    if lattice == "cfg1":
        cfg = configs.CONFIGS["cfg1"]
        V, psi = configs.make_inputs(cfg)
        model = configs.model_for(cfg, V)
        h, eps, nx, ny = cfg.dt, cfg.epsilon, cfg.nx, cfg.ny
        newton = configs.newton_for(cfg)
    else:
        nx, ny = 250, 70
        g, V, psi = _packet_lattice(nx, ny, 250.0, 84.0)
        model = nls2d.GridModel(g, 0.7, V)
        h, eps = 0.01, 1e-13
        newton = nls2d.NewtonConfig(eps, 50, 0)
    ref, its = SM.step(psi, V, model.gamma(), h, scheme, m, nx, ny, eps, mf=mf, cx=model.cx, cy=model.cy,
                       first_poly=first_poly)
    with nls2d.Session(model, scheme, newton, neumann_terms=m, neumann_first=mf, first_poly=first_poly) as s:
        s.set_state(psi)
        st = nls2d.StepStats()
        s.step(h, st)
        got = s.get_state()
    assert st.newton_iters == its
    assert rel(got, ref) <= 1e-13


@pytest.mark.parametrize("first_poly", [1, 2])
@pytest.mark.parametrize("mf", [4, 6])
def test_deep_first_sweep_ten_steps_match_oracle(mf, first_poly):
    cfg = configs.CONFIGS["cfg2"]
    V, psi = configs.make_inputs(cfg)
    ref, ref_obs = _oracle_steps(cfg, V, psi, 10)
    model = configs.model_for(cfg, V)
    with nls2d.Session(model, nls2d.Mb4Scheme(), configs.newton_for(cfg), neumann_terms=1, neumann_first=mf,
                       first_poly=first_poly) as s:
        s.set_state(psi)
        obs, _ = s.run(cfg.dt, 10)
        got = s.get_state()
    assert rel(got, ref) <= 1e-10
    assert np.abs(obs[:, 3] - ref_obs[:, 3]).max() <= 1e-13 * abs(ref_obs[0, 3])


def test_speculative_final_sweep_miss_is_redone_exactly():
    """The production kernel stores only U3 in the sweep the previous step's count
    predicts to be final; when the prediction misses (here: the second step is
    twice as long and needs more sweeps) the sweep is redone with all stages.  The
    result and the sweep counts equal the numpy model's (no speculation there)."""
    cfg = configs.CONFIGS["cfg2"]
    V, psi = configs.make_inputs(cfg)
    model = configs.model_for(cfg, V)
    scheme = nls2d.Mb4Scheme()
    rho = SM.spectral_bound(psi, V, cfg.gamma)  # the library's bound is that of the set state
    u1, it1 = SM.step(psi, V, cfg.gamma, cfg.dt, scheme, 1, cfg.nx, cfg.ny, cfg.epsilon, mf=6, rho=rho)
    u2, it2 = SM.step(u1, V, cfg.gamma, 2 * cfg.dt, scheme, 1, cfg.nx, cfg.ny, cfg.epsilon, mf=6, rho=rho)
    u3, it3 = SM.step(u2, V, cfg.gamma, cfg.dt, scheme, 1, cfg.nx, cfg.ny, cfg.epsilon, mf=6, rho=rho)
    assert it2 > it1
    with nls2d.Session(model, scheme, configs.newton_for(cfg), neumann_terms=1, neumann_first=6) as s:
        s.set_state(psi)
        s.profile_enable(True)
        got = []
        for h in (cfg.dt, 2 * cfg.dt, cfg.dt):
            st = nls2d.StepStats()
            s.step(h, st)
            got.append((s.get_state(), st.newton_iters))
        prof = s.profile()
    assert [g[1] for g in got] == [it1, it2, it3]
    for (u, _), ref in zip(got, (u1, u2, u3)):
        assert rel(u, ref) <= 1e-13
    assert prof["redone"] >= 1


@pytest.mark.parametrize("nx,ny,lx,ly", [(2, 3, 2.0, 3.0), (5, 4, 5.0, 4.0), (7, 130, 7.0, 130.0),
                                         (130, 7, 130.0, 7.0), (255, 33, 255.0, 40.0), (129, 129, 129.0, 129.0)])
def test_ragged_lattices_default_path_match_oracle(nx, ny, lx, ly):
    """Edge shapes through the default production path (deep first sweep,
    speculative final sweep, isotropic and anisotropic, widths below / just above
    one column band, the smallest lattices): 4 steps against the oracle."""
    g = nls2d.GridSpec(nx, ny, lx, ly)
    rng = np.random.default_rng(nx * 1000 + ny)
    V = np.where(rng.uniform(size=nx * ny) < 0.1, 3.0, 0.0)
    model = nls2d.GridModel(g, -1.0, V)
    psi = random_state(nx * ny, nx + ny, 0.2)
    h = 0.01
    o = O.Oracle(nx, ny, -1.0, V, cx=model.cx, cy=model.cy)
    ref, ref_obs, _ = o.run(psi, h, 4, eps=1e-14)
    with nls2d.Session(model, nls2d.Mb4Scheme(), nls2d.NewtonConfig(1e-14, 50, 4)) as s:
        s.set_state(psi)
        obs, iters = s.run(h, 4)
        got = s.get_state()
    assert rel(got, ref) <= 1e-10
    assert np.abs(obs[:, 3] - ref_obs[:, 3]).max() <= 1e-13 * max(1.0, abs(ref_obs[0, 3]))


def test_spectral_bound_abi():
    """mb4cu_spectral_bound is the Gershgorin bound of the resident state rounded up to a
    power of 2^(1/16) (the numpy model's value); an agreed bound set by the caller changes
    the first sweep's polynomial but not the converged step (within the stopping rule)."""
    import ctypes as C

    from paper_2003_04345_b200 import _lib

    cfg = configs.CONFIGS["cfg2"]
    V, psi = configs.make_inputs(cfg)
    model = configs.model_for(cfg, V)
    L = _lib.lib()
    with nls2d.Session(model, nls2d.Mb4Scheme(), configs.newton_for(cfg)) as s:
        s.set_state(psi)
        rho = C.c_double(0.0)
        assert L.mb4cu_spectral_bound(s._ctx, C.byref(rho)) == 0
        assert rho.value == pytest.approx(SM.spectral_bound(psi, V, cfg.gamma), rel=1e-14)
        assert L.mb4cu_set_spectral_bound(s._ctx, -1.0) == _lib.MB4CU_INVALID
        assert L.mb4cu_set_spectral_bound(s._ctx, float("nan")) == _lib.MB4CU_INVALID
        s.step(cfg.dt)
        u_own = s.get_state()
        s.set_state(psi)
        assert L.mb4cu_set_spectral_bound(s._ctx, 2.0 * rho.value) == 0
        s.step(cfg.dt)
        u_wide = s.get_state()
    assert rel(u_own, u_wide) <= 1e-13
