"""CPU tests: pin the oracle restatement (oracle/mb4_oracle.c) before trusting it.

Pins:
  - exact-rational scheme tables from the reference's own generator (scheme_exact.json),
    tolerances of test_mb4_scheme.cpp:68-176 (1e-14 E, W; 1e-13 eigenvalues);
  - Phi against a 64-node quadrature of the stage residual (test_mb4_integrator.cpp:29-55,78-91), 1e-12;
  - one simplified-Newton correction against the dense coupled 6N solve
    (test_mb4_integrator.cpp:189-236), 1e-11;
  - h = 0 Newton fixed point (test_mb4_integrator.cpp:147-159);
  - golden states / energy records produced by the reference library itself (ref_*.npz).
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2003_04345_b200 import configs

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TWO_PI = 2.0 * np.pi


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def random_state(n, seed, amp=1.0):
    rng = np.random.default_rng(seed)
    return (rng.uniform(-amp, amp, n) + 1j * rng.uniform(-amp, amp, n)).astype(np.complex128)


@pytest.fixture(scope="module")
def exact():
    with open(os.path.join(GOLD, "scheme_exact.json")) as f:
        return json.load(f)


def test_oracle_scheme_matches_exact_tables(exact):
    o = O.Oracle(4, 4, 0.1, np.zeros(16))
    E = np.array(o.s.E)
    W = np.array(o.s.W)
    assert np.abs(E - np.array(exact["E"]).reshape(3, 4)).max() <= 1e-14
    assert np.abs(W - np.array(exact["W"]).reshape(3, 4, 4, 4)).max() <= 1e-14
    assert np.abs(np.array(o.s.lam) - np.array(exact["eigenvalues"])).max() <= 1e-13
    # T diagonalises the core: E T = T diag(lambda)
    core = E[:, 1:]
    T, Ti = np.array(o.s.T), np.array(o.s.Tinv)
    assert np.abs(core @ T - T @ np.diag(o.s.lam)).max() <= 1e-12 * np.abs(core).sum(1).max()
    assert np.abs(T @ Ti - np.eye(3)).max() <= 1e-14


def test_gl6_tables_reproduce_w_and_e(exact):
    o = O.Oracle(4, 4, 0.1, np.zeros(16))
    L, WA = np.array(o.s.L), np.array(o.s.WA)
    W = np.einsum("iq,qa,qb,qc->iabc", WA, L, L, L)
    E = np.einsum("iq,qa->ia", WA, L)
    assert np.abs(W - np.array(exact["W"]).reshape(3, 4, 4, 4)).max() <= 1e-14
    assert np.abs(E - np.array(exact["E"]).reshape(3, 4)).max() <= 1e-14
    # Lagrange basis value pinned by the reference tables: l_3(1/2) over {0,1/3,2/3,1}
    nodes = np.array([0, 1 / 3, 2 / 3, 1.0])
    l3 = np.prod([(0.5 - nodes[b]) / (nodes[3] - nodes[b]) for b in range(3)])
    assert abs(l3 - exact["l3_half"]) <= 1e-16


def _gauss_legendre_01(n):
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


def _eval_a(alpha, tau, zeta):
    base = tau * (4 - 6 * zeta) + tau * tau * (6 * zeta - 3)
    return base + alpha * tau * (1 - tau) * (1 - 2 * tau) * (1 - 6 * zeta * (1 - zeta))


def _phi_quadrature(o, u0, stages, h, alpha=-712.5):
    # 64-node quadrature of Phi_i = U_i - u0 - h int_0^1 A(c_i,z) f(U_z) dz
    nodes = np.array([0, 1 / 3, 2 / 3, 1.0])
    zq, wq = _gauss_legendre_01(64)
    integ = [np.zeros_like(u0) for _ in range(3)]
    for z, w in zip(zq, wq):
        l = [np.prod([(z - nodes[b]) / (nodes[a] - nodes[b]) for b in range(4) if b != a]) for a in range(4)]
        uz = l[0] * u0 + l[1] * stages[0] + l[2] * stages[1] + l[3] * stages[2]
        f = o.rhs(uz)
        for i in range(3):
            integ[i] += w * _eval_a(alpha, nodes[i + 1], z) * f
    return [stages[i] - u0 - h * integ[i] for i in range(3)]


@pytest.mark.parametrize("gamma", [0.0, 0.1])
def test_oracle_phi_matches_64_node_quadrature(gamma):
    V = np.zeros(16)
    V[0] = 0.0 if gamma == 0.0 else -2.0
    cx = 1.0 / (TWO_PI / 4) ** 2
    o = O.Oracle(4, 4, gamma, V, cx=cx, cy=cx)
    u0 = random_state(16, 31)
    st = [random_state(16, 40 + i) for i in range(3)]
    phi = o.eval_phi(u0, st, 0.01)
    q = _phi_quadrature(o, u0, st, 0.01)
    assert max(np.abs(a - b).max() for a, b in zip(phi, q)) <= 1e-12


def test_oracle_newton_h0_is_fixed_point():
    o = O.Oracle(4, 4, 0.1, np.zeros(16), cx=0.4, cy=0.4)
    u0 = random_state(16, 3)
    rc, st, it, _ = o.newton_solve(u0, 0.0)
    assert rc == 0 and it == 1
    assert all(np.array_equal(s, u0) for s in st)


def _jacobian_dense(o, u0):
    """Real-split J (mb4_integrator.hpp:52-55) as a dense 2N x 2N matrix, columnwise."""
    n = o.n
    J = np.zeros((2 * n, 2 * n))
    g = o.m.gamma
    p, q = u0.real, u0.imag
    for c in range(2 * n):
        e = np.zeros(n, dtype=np.complex128)
        if c < n:
            e[c] = 1.0
        else:
            e[c - n] = 1.0j
        kv = o.apply_kv(e)  # (K+V) e
        tp, tq = e.real, e.imag
        jp = -2 * g * p * q * tp + kv.imag - g * (p * p + 3 * q * q) * tq
        jq = -kv.real + g * (3 * p * p + q * q) * tp + 2 * g * p * q * tq
        J[:n, c] = jp
        J[n:, c] = jq
    return J


def test_oracle_one_correction_matches_dense_coupled_solve():
    # test_mb4_integrator.cpp:189-236: (I - h E (x) J) r = -Phi vs the eigendecomposed path
    V = np.zeros(16)
    V[0] = -1.0
    cx = 1.0 / (TWO_PI / 4) ** 2
    o = O.Oracle(4, 4, 0.1, V, cx=cx, cy=cx)
    u0 = random_state(16, 8)
    h = 0.02
    n2 = 32
    phi = o.eval_phi(u0, [u0, u0, u0], h)
    J = _jacobian_dense(o, u0)
    e3 = np.array(o.s.E)[:, 1:]
    big = np.eye(3 * n2) - h * np.kron(e3, J)
    rhs = np.concatenate([-np.concatenate([p.real, p.imag]) for p in phi])
    r_dense = np.linalg.solve(big, rhs)
    rc, st, it, _ = o.newton_solve(u0, h, eps=1e300, max_iters=1)
    assert rc == 0
    scale = max(1.0, np.abs(r_dense).max())
    for i in range(3):
        d = st[i] - u0
        r_eig = np.concatenate([d.real, d.imag])
        assert np.abs(r_eig - r_dense[i * n2:(i + 1) * n2]).max() <= 1e-11 * scale


def test_oracle_matches_reference_golden_cfg1():
    g = np.load(os.path.join(GOLD, "ref_cfg1_10.npz"))
    cfg = configs.CONFIGS["cfg1"]
    V, psi = configs.make_inputs(cfg)
    import hashlib

    h = hashlib.sha256()
    h.update(V.tobytes())
    h.update(psi.tobytes())
    assert h.hexdigest() == str(g["input_sha256"]), "input generator drifted from the golden inputs"
    o = O.Oracle(cfg.nx, cfg.ny, cfg.gamma, V)
    u1, obs1, it1 = o.run(psi, cfg.dt, 1, eps=cfg.epsilon)
    assert rel(u1, g["state_1"]) <= 1e-12
    u10, obs10, it10 = o.run(u1, cfg.dt, 9, eps=cfg.epsilon)
    assert rel(u10, g["state_10"]) <= 1e-12
    assert list(it1) + list(it10) == list(g["iters"])  # same simplified-Newton iteration counts
    H = np.concatenate([obs1[:, 3], obs10[1:, 3]])
    assert np.abs(H - g["obs"][:, 3]).max() <= 1e-13 * abs(g["obs"][0, 3])


def test_reference_golden_energy_record_is_conservative():
    g = np.load(os.path.join(GOLD, "ref_cfg1_full.npz"))
    H = g["obs"][:, 3]
    assert len(H) == 1001
    assert np.abs(H - H[0]).max() / abs(H[0]) <= 1e-13


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_restatement_matches_reference_library_eval_phi():
    V = np.linspace(0, 3, 30)
    u0 = random_state(30, 1)
    st = [random_state(30, 2 + i) for i in range(3)]
    cx, cy = 1.0 / (TWO_PI / 6) ** 2, 1.0 / (2.0 / 5) ** 2
    o = O.Oracle(6, 5, -0.7, V, cx=cx, cy=cy)
    a = o.eval_phi(u0, st, 0.03)
    b = O.ref_eval_phi(6, 5, TWO_PI, 2.0, -0.7, V, u0, st, 0.03)
    assert max(np.abs(x - y).max() for x, y in zip(a, b)) <= 1e-13


def test_methods_golden_fixture_pinned():
    """The other integrators' fixture (reference StepDriver, 5 cfg1 steps) belongs to
    the current inputs; with the reference built here it is reproduced bit for bit,
    and its conservation classes hold (AVF energy, Gauss probability)."""
    g = np.load(os.path.join(GOLD, "ref_methods_cfg1_5.npz"))
    cfg = configs.CONFIGS["cfg1"]
    V, psi = configs.make_inputs(cfg)
    import hashlib

    h = hashlib.sha256()
    h.update(V.tobytes())
    h.update(psi.tobytes())
    assert h.hexdigest() == str(g["input_sha256"])
    for m in ("avf2", "avf4"):
        H = g[f"{m}_obs"][:, 3]
        assert np.abs(H - H[0]).max() <= 1e-13 * abs(H[0])
    for m in ("gauss2", "gauss4"):
        P = g[f"{m}_obs"][:, 4]
        assert np.abs(P - P[0]).max() <= 1e-13 * P[0]
    assert list(g["rk4_iters"]) == [0] * 5
    if O.ref_available():
        u, _, _, _ = O.ref_run(cfg.nx, cfg.ny, float(cfg.nx), float(cfg.ny), cfg.gamma, V, psi, cfg.dt, 5,
                               eps=cfg.epsilon, solver="direct", method="avf2")
        assert np.array_equal(u, g["avf2_state"])


def test_host_only_input_generator_is_bit_identical():
    """oracle/libinputs.so (g++ only; bench.py's reference arm) produces the product
    library's BASELINE inputs bit for bit -- whole lattices and a cfg5 sub-block."""
    from paper_2003_04345_b200 import configs

    gen = O.inputs_generator()
    for name in ("cfg1", "cfg2", "cfg4"):
        cfg = configs.CONFIGS[name]
        Va, pa = configs.make_inputs(cfg)
        Vb, pb = configs.make_inputs(cfg, gen=gen)
        assert np.array_equal(Va.view(np.uint64), Vb.view(np.uint64))
        assert np.array_equal(pa.view(np.uint64), pb.view(np.uint64))
    cfg = configs.CONFIGS["cfg5"]
    a = configs.make_block(cfg, 4096, 1024, 300, 200)
    b = configs.make_block(cfg, 4096, 1024, 300, 200, gen=gen)
    assert all(np.array_equal(np.asarray(x).view(np.uint64), np.asarray(y).view(np.uint64)) for x, y in zip(a, b))
