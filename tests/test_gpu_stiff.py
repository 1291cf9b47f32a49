"""GPU tests of the stiff-regime stage solver (kernel = 3, Newton-Krylov):
the reference's own paper-scale test cases (test_mb4_integrator.cpp), which the
matrix-free sweep cannot converge at full step (h*lambda*rho(J) ~ 15)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2003_04345_b200 import nls2d

pytestmark = pytest.mark.gpu
TWO_PI = 2.0 * np.pi
NEWTON_KRYLOV = 3


def paper_model(n=70, gamma=0.1, v0=0.0):
    g = nls2d.GridSpec(n, n, TWO_PI, TWO_PI)
    V = nls2d.build_delta_potential(g, v0) if v0 else None
    return g, nls2d.GridModel(g, gamma, V)


def test_paper_scale_newton_iterations_single_digit():
    # test_mb4_integrator.cpp:176-187
    g, model = paper_model()
    u0 = nls2d.initial_condition(g)
    st = nls2d.StepStats()
    with nls2d.Session(model, nls2d.Mb4Scheme(), nls2d.NewtonConfig(), kernel=NEWTON_KRYLOV) as s:
        s.set_state(u0)
        s.step(0.01, st)
    assert st.halvings == 0
    assert st.newton_iters <= 9


def test_paper_scale_one_step_energy():
    # test_mb4_integrator.cpp:300-309
    g, model = paper_model()
    u0 = nls2d.initial_condition(g)
    with nls2d.Session(model, nls2d.Mb4Scheme(), nls2d.NewtonConfig(), kernel=NEWTON_KRYLOV) as s:
        s.set_state(u0)
        h0 = s.observables().total_energy
        s.step(0.01)
        h1 = s.observables().total_energy
    assert abs(h1 - h0) <= 1e-12 * abs(h0)


def test_single_mode_phase_rotation_at_reference_steps():
    # test_mb4_integrator.cpp:238-265 at h = 0.4 / 0.2 (stiff for the matrix-free sweep)
    g = nls2d.GridSpec(8, 8, TWO_PI, TWO_PI)
    model = nls2d.GridModel(g, 0.0)
    x = np.arange(8) * g.hx()
    u0 = np.tile(np.exp(1j * x), 8).astype(np.complex128)
    mu = (2 - 2 * np.cos(g.hx())) / g.hx() ** 2

    def err(h):
        with nls2d.Session(model, nls2d.Mb4Scheme(), nls2d.NewtonConfig(), kernel=NEWTON_KRYLOV) as s:
            s.set_state(u0)
            s.step(h)
            u1 = s.get_state()
        return np.abs(u1 - np.exp(-1j * mu * h) * u0).max()

    ratio = err(0.4) / err(0.2)
    assert 24.0 <= ratio <= 40.0


def test_paper_baseline_config_matches_reference():
    # configs/baseline.cfg (70x70, lx = 2 pi, gamma = -0.1, dt = 0.01): 5 steps vs the
    # reference's direct-LU path; same simplified-Newton iteration counts
    g, model = paper_model(gamma=-0.1)
    u0 = nls2d.initial_condition(g)
    with nls2d.Session(model, nls2d.Mb4Scheme(), nls2d.NewtonConfig(1e-13, 50, 4), kernel=NEWTON_KRYLOV) as s:
        s.set_state(u0)
        obs, iters = s.run(0.01, 5)
        u = s.get_state()
    ref, robs, riters, _ = O.ref_run(70, 70, TWO_PI, TWO_PI, -0.1, np.zeros(4900), u0, 0.01, 5, eps=1e-13,
                                     solver="direct")
    assert np.linalg.norm(u - ref) / np.linalg.norm(ref) <= 1e-10
    assert list(iters) == list(riters)
    assert np.abs(obs[:, 3] - robs[:, 3]).max() <= 1e-12 * abs(robs[0, 3])


def test_delta_potential_config_one_step():
    # configs/delta_short.cfg style: 100x100, delta potential V0 = -50 at (0,0)
    g, model = paper_model(n=100, gamma=0.1, v0=-50.0)
    u0 = np.full(g.points(), 1.0 / np.sqrt(g.points()), dtype=np.complex128)
    with nls2d.Session(model, nls2d.Mb4Scheme(), nls2d.NewtonConfig(1e-13, 50, 4), kernel=NEWTON_KRYLOV) as s:
        s.set_state(u0)
        s.step(0.002)
        u = s.get_state()
    ref, _, _, _ = O.ref_run(100, 100, TWO_PI, TWO_PI, 0.1, model.potential(), u0, 0.002, 1, eps=1e-13,
                             solver="gmres", record=False)
    assert np.linalg.norm(u - ref) / np.linalg.norm(ref) <= 1e-10


def test_newton_krylov_nonconvergence_semantics():
    # test_mb4_integrator.cpp:336-345
    g = nls2d.GridSpec(6, 6, TWO_PI, TWO_PI)
    model = nls2d.GridModel(g, 0.5)
    u0 = nls2d.initial_condition(g)
    with nls2d.Session(model, nls2d.Mb4Scheme(), nls2d.NewtonConfig(1e-13, 1, 0), kernel=NEWTON_KRYLOV) as s:
        s.set_state(u0)
        with pytest.raises(nls2d.NonConvergenceError):
            s.step(0.5)
        assert np.array_equal(s.get_state(), u0)


@pytest.mark.parametrize("v0", [0.0, -50.0])
def test_batched_stage_solves_equal_sequential(monkeypatch, v0):
    """The three stage systems of a Newton iteration solved together (one stream per
    system, lockstep GMRES, one host round trip per Arnoldi step) give the same iterates
    bit for bit as solving them one after the other (MB4CU_KR_BATCH=0)."""
    g, model = paper_model(n=70 if v0 == 0.0 else 100, v0=v0)
    u0 = nls2d.initial_condition(g)
    out = {}
    for batch in ("1", "0"):
        monkeypatch.setenv("MB4CU_KR_BATCH", batch)
        st = nls2d.StepStats()
        with nls2d.Session(model, nls2d.Mb4Scheme(), nls2d.NewtonConfig(), kernel=NEWTON_KRYLOV) as s:
            s.set_state(u0)
            for _ in range(2):
                s.step(0.01 if v0 == 0.0 else 0.002, st)
            out[batch] = (s.get_state(), st.newton_iters)
    assert out["1"][1] == out["0"][1]
    assert np.array_equal(out["1"][0], out["0"][0])
