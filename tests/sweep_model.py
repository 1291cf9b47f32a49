"""TEST INFRASTRUCTURE: numpy model of one matrix-free stage sweep (the GPU algorithm).

Used to check single GPU sweeps and sweep counts; it is not the oracle (the
oracle restates the reference's simplified Newton, oracle/mb4_oracle.c).
"""
import numpy as np


def kv(u, V, nx, ny, cx=1.0, cy=1.0):
    U = u.reshape(ny, nx)
    y = (2 * cx + 2 * cy) * U - cx * (np.roll(U, 1, 1) + np.roll(U, -1, 1)) \
        - cy * (np.roll(U, 1, 0) + np.roll(U, -1, 0)) + V.reshape(ny, nx) * U
    return y.reshape(-1)


def jac(t, u0, V, gamma, nx, ny, cx=1.0, cy=1.0):
    a = kv(t, V, nx, ny, cx, cy)
    nl = 2 * np.abs(u0) ** 2 * t + u0 ** 2 * np.conj(t)
    return -1j * a + 1j * gamma * nl


def spectral_bound(u0, V, gamma, cx=1.0, cy=1.0):
    """The library's first-sweep bound: Gershgorin 4cx + 4cy + max|V| + 3|gamma| max|u0|^2,
    rounded up to a power of 2^(1/16) (mb4cu_api.cu own_first_rho)."""
    rho = 4.0 * cx + 4.0 * cy + np.abs(V).max() + 3.0 * abs(gamma) * (np.abs(u0) ** 2).max()
    return float(2.0 ** (np.ceil(16.0 * np.log2(rho)) / 16.0))


def cheb_coeffs(beta, rho, deg):
    """Monomial coefficients of the polynomial p(x) ~ 1/(1 - beta x) interpolating at the
    deg + 1 Chebyshev points of the segment i[-rho, rho] (mb4cu_api.cu cheb_first_poly)."""
    n = deg + 1
    t = np.cos((2 * np.arange(n) + 1) * np.pi / (2 * n))
    e = np.linalg.solve(np.vander(t, n, increasing=True).astype(complex), 1.0 / (1.0 - 1j * beta * rho * t))
    return np.array([(e[q] * (-1j) ** q).real / rho ** q for q in range(n)])


def first_poly_default(V, gamma):
    """first_poly 0 resolves to Chebyshev (2) when H is convex, else Neumann (1)."""
    return 2 if (np.min(V) >= 0.0 and gamma <= 0.0) else 1


def sweep(u0, U, V, gamma, h, scheme, m, nx, ny, cx=1.0, cy=1.0, coeffs=None):
    """One stage iteration; returns (U_new, ||r||_inf over split reals).  coeffs[k][n]:
    the stage-k polynomial of (I - h lam_k J)^-1 (default: the m-term Neumann series)."""
    E, L, WA = scheme.E(), scheme.gl6_L(), scheme.gl6_WA()
    T, Ti, lam = scheme.t(), scheme.t_inv(), np.array(scheme.eigenvalues())
    if U is None:
        U = [u0, u0, u0]
    z = [u0] + list(U)
    w = [kv(zj, V, nx, ny, cx, cy) for zj in z]
    Uq = [sum(L[q, a] * z[a] for a in range(4)) for q in range(6)]
    gq = [np.abs(x) ** 2 * x for x in Uq]
    phi = []
    for i in range(3):
        kc = sum(E[i, j] * w[j] for j in range(4))
        cub = sum(WA[i, q] * gq[q] for q in range(6))
        R = -1j * kc + 1j * gamma * cub
        phi.append(U[i] - u0 - h * R)
    if m == 0:
        r = [-p for p in phi]
    else:
        pb = [sum(Ti[k, i] * phi[i] for i in range(3)) for k in range(3)]
        if coeffs is None:
            b = list(pb)
            for _ in range(m):
                b = [pb[k] + h * lam[k] * jac(b[k], u0, V, gamma, nx, ny, cx, cy) for k in range(3)]
        else:  # Horner in J
            b = [coeffs[k][m] * pb[k] for k in range(3)]
            for n in range(m - 1, -1, -1):
                b = [coeffs[k][n] * pb[k] + jac(b[k], u0, V, gamma, nx, ny, cx, cy) for k in range(3)]
        rb = [-x for x in b]
        r = [sum(T[i, k] * rb[k] for k in range(3)) for i in range(3)]
    Un = [U[i] + r[i] for i in range(3)]
    rmax = max(max(np.abs(x.real).max(), np.abs(x.imag).max()) for x in r)
    return Un, rmax


def step(u0, V, gamma, h, scheme, m, nx, ny, eps, max_iters=50, mf=None, cx=1.0, cy=1.0, first_poly=0,
         rho=None):
    """One step; the first sweep uses depth mf (default m), the others m.  first_poly:
    the first sweep's polynomial as in mb4cu_problem (0 = default, 1 = Neumann, 2 =
    Chebyshev on i[-rho, rho], rho default: spectral_bound of u0); it applies to the
    production kernel's deep first sweep (mf >= 1) and its depth-2 later sweeps."""
    from paper_2003_04345_b200.dist import stage_converged, widen_residual

    if first_poly == 0:
        first_poly = first_poly_default(V, gamma)
    d1 = m if mf is None else mf
    coeffs = None
    if first_poly == 2 and d1 >= 1:
        rho = spectral_bound(u0, V, gamma, cx, cy) if rho is None else rho
        lam = np.array(scheme.eigenvalues())
        coeffs = [cheb_coeffs(h * lam[k], rho, d1) for k in range(3)]
    later = None
    if first_poly == 2 and m == 2:  # depth-2 later sweeps: Chebyshev multipliers (mb4cu_api.cu hlam2)
        rho = spectral_bound(u0, V, gamma, cx, cy) if rho is None else rho
        lam = np.array(scheme.eigenvalues())
        later = [cheb_coeffs(h * lam[k], rho, 2) for k in range(3)]
    U = None
    r_prev = float("nan")
    for it in range(1, max_iters + 1):
        U, r = sweep(u0, U, V, gamma, h, scheme, m if (it > 1 or mf is None) else mf, nx, ny, cx, cy,
                     coeffs if it == 1 else later)
        r = widen_residual(r)
        if stage_converged(r, r_prev, it - 1, eps):
            return U[2], it
        r_prev = r
    raise RuntimeError("no convergence")
