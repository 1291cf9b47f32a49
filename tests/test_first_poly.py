"""CPU tests of the first sweep's stage polynomial (host logic; no GPU).

The first sweep of a step approximates (I - h lam_k J)^-1 by a polynomial p_k(J) of
degree mf.  The Neumann series is the Taylor polynomial; the Chebyshev choice
(mb4cu_problem.first_poly = 2, the default for convex H) interpolates 1/(1 - beta x) at
the Chebyshev points of the spectral segment i[-rho, rho] of J = S H(u0)
(mb4cu_api.cu cheb_first_poly, restated in tests/sweep_model.py)."""
import numpy as np
import pytest

import sweep_model as SM


def _residual(coeffs, beta, rho, npts=20001):
    y = np.linspace(-rho, rho, npts)
    x = 1j * y
    p = sum(c * x ** n for n, c in enumerate(coeffs))
    return np.abs(1.0 - (1.0 - beta * x) * p).max()


@pytest.mark.parametrize("deg", [1, 2, 4, 5, 6])
@pytest.mark.parametrize("beta_rho", [0.02, 0.083, 0.3])
@pytest.mark.parametrize("sign", [1.0, -1.0])
def test_chebyshev_residual_is_the_scaled_chebyshev_bound(deg, beta_rho, sign):
    """max |1 - (1 - beta x) p(x)| over the segment equals 1/|T_{d+1}(i/(beta rho))|
    (the optimum over degree-d polynomials), ~2 (beta rho / 2)^(d+1), below the Neumann
    series' (beta rho)^(d+1) / (1 + ...) -- by 2^d."""
    rho = 18.0
    beta = sign * beta_rho / rho
    c = SM.cheb_coeffs(beta, rho, deg)
    s = 1.0 / beta_rho
    n = deg + 1  # |T_n(i s)| = cosh(n asinh s) for even n, sinh(n asinh s) for odd n
    t_im = abs(np.cosh(n * np.arcsinh(s)) if n % 2 == 0 else np.sinh(n * np.arcsinh(s)))
    got = _residual(c, beta, rho)
    assert got == pytest.approx(1.0 / t_im, rel=1e-6)
    taylor = _residual([beta ** n for n in range(deg + 1)], beta, rho)
    assert got < taylor
    if deg >= 2:
        assert got < 0.6 * taylor * 2.0 ** (1 - deg)


def test_chebyshev_coefficients_are_real_and_tend_to_taylor():
    """p has real coefficients (the spectrum is symmetric under conjugation) and tends to
    the Neumann series as the segment shrinks."""
    beta = 0.002 * 1.5206207261596576
    for rho in (1e-3, 1e-2):
        c = SM.cheb_coeffs(beta, rho, 6)
        t = np.array([beta ** n for n in range(7)])
        assert np.all(np.isfinite(c))
        assert np.abs(c[:3] - t[:3]).max() <= 1e-6 * np.abs(t[:3]).max()


def test_spectral_bound_is_gershgorin_rounded_up():
    V = np.array([0.0, 10.0, 3.0])
    u = np.array([0.1, 0.2j, -0.05])
    rho = SM.spectral_bound(u, V, -1.5)
    exact = 8.0 + 10.0 + 3 * 1.5 * 0.04
    assert exact <= rho <= exact * 2 ** (1 / 16)
    assert np.log2(rho) * 16 == pytest.approx(round(np.log2(rho) * 16), abs=1e-9)


def test_default_resolution_follows_convexity():
    assert SM.first_poly_default(np.array([0.0, 5.0]), -1.0) == 2
    assert SM.first_poly_default(np.array([-1.0, 5.0]), -1.0) == 1
    assert SM.first_poly_default(np.array([0.0, 5.0]), 0.7) == 1
