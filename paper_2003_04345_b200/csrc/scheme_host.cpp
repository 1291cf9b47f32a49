// Host-side scheme constants for the MB4 sweep kernels.
//
// Replaces Mb4Scheme::Mb4Scheme (reference mb4_scheme.cpp:83-125) and
// eig3_real / SmallMat::inverse (small_dense.cpp:27-174).  Everything is
// computed once per context in long double and rounded to FP64, then handed
// to the device as kernel-parameter constants.  Beyond the reference's E, W,
// lambda, T, T^-1 this also emits the Gauss-Legendre-6 tables L and WA of the
// quadrature form of the cubic term, which the reference does not expose.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <string>

#include "mb4cu.h"
#include "mb4cu_internal.hpp"

namespace mb4cu {
namespace {

using ld = long double;

// A(tau, zeta): the alpha1 block of the coefficient matrix is rank one, which
// gives the cancellation-free form of mb4_scheme.cpp:17-27.
ld coeff_a(ld alpha, ld tau, ld zeta) {
    const ld lin = tau * (4.0L - 6.0L * zeta) + tau * tau * (6.0L * zeta - 3.0L);
    return lin + alpha * (tau * (1.0L - tau) * (1.0L - 2.0L * tau)) *
                     (1.0L - 6.0L * zeta * (1.0L - zeta));
}

// n-point Gauss-Legendre rule on [0, 1] (nodes ascending), Newton on P_n.
void gl_rule(int n, ld* nodes, ld* weights) {
    const ld pi = 3.141592653589793238462643383279502884L;
    for (int r = 0; r < n; ++r) {
        ld x = std::cos(pi * (r + 0.75L) / (n + 0.5L));
        ld deriv = 0.0L;
        for (int it = 0; it < 200; ++it) {
            ld pm = 1.0L, pc = x;
            for (int k = 2; k <= n; ++k) {
                const ld pn = ((2.0L * k - 1.0L) * x * pc - (k - 1.0L) * pm) / k;
                pm = pc;
                pc = pn;
            }
            deriv = n * (x * pc - pm) / (x * x - 1.0L);
            const ld step = pc / deriv;
            x -= step;
            if (std::fabs(step) < 1e-20L) break;
        }
        nodes[n - 1 - r] = 0.5L * (x + 1.0L);
        weights[n - 1 - r] = 1.0L / ((1.0L - x * x) * deriv * deriv);
    }
}

ld lagrange(const std::array<ld, 4>& c, int a, ld z) {
    ld v = 1.0L;
    for (int b = 0; b < 4; ++b)
        if (b != a) v *= (z - c[b]) / (c[a] - c[b]);
    return v;
}

using Mat3 = std::array<std::array<double, 3>, 3>;

bool invert3(const Mat3& m, Mat3& inv) {
    Mat3 a = m;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) inv[i][j] = (i == j);
    for (int k = 0; k < 3; ++k) {
        int piv = k;
        for (int i = k + 1; i < 3; ++i)
            if (std::fabs(a[i][k]) > std::fabs(a[piv][k])) piv = i;
        if (a[piv][k] == 0.0) return false;
        std::swap(a[k], a[piv]);
        std::swap(inv[k], inv[piv]);
        const double d = a[k][k];
        for (int j = 0; j < 3; ++j) {
            a[k][j] /= d;
            inv[k][j] /= d;
        }
        for (int i = 0; i < 3; ++i) {
            if (i == k || a[i][k] == 0.0) continue;
            const double f = a[i][k];
            for (int j = 0; j < 3; ++j) {
                a[i][j] -= f * a[k][j];
                inv[i][j] -= f * inv[k][j];
            }
        }
    }
    return true;
}

// Three distinct real eigenvalues (ascending) and unit eigenvectors with a
// deterministic sign, following the method of small_dense.cpp:83-174.
bool real_eig3(const Mat3& e, std::array<double, 3>& lam, Mat3& t, Mat3& tinv,
               std::string& why) {
    double scale = 0.0;
    for (const auto& row : e)
        scale = std::max(scale, std::fabs(row[0]) + std::fabs(row[1]) + std::fabs(row[2]));
    scale = std::max(scale, 1e-300);
    const double tr = e[0][0] + e[1][1] + e[2][2];
    const double m2 = e[0][0] * e[1][1] - e[0][1] * e[1][0] + e[0][0] * e[2][2] -
                      e[0][2] * e[2][0] + e[1][1] * e[2][2] - e[1][2] * e[2][1];
    const double det = e[0][0] * (e[1][1] * e[2][2] - e[1][2] * e[2][1]) -
                       e[0][1] * (e[1][0] * e[2][2] - e[1][2] * e[2][0]) +
                       e[0][2] * (e[1][0] * e[2][1] - e[1][1] * e[2][0]);
    const double shift = tr / 3.0;
    const double p = m2 - tr * tr / 3.0;
    const double q = -det + m2 * shift - 2.0 * tr * tr * tr / 27.0;
    if (q * q / 4.0 + p * p * p / 27.0 > 1e-14 * std::pow(scale, 6.0) || p >= 0.0) {
        why = "complex eigenvalue pair detected";
        return false;
    }
    const double rho = 2.0 * std::sqrt(-p / 3.0);
    const double theta = std::acos(std::clamp(3.0 * q / (p * rho), -1.0, 1.0)) / 3.0;
    for (int k = 0; k < 3; ++k) lam[k] = rho * std::cos(theta - 2.0 * M_PI * k / 3.0) + shift;
    std::sort(lam.begin(), lam.end());
    for (double& l : lam)
        for (int it = 0; it < 3; ++it) {
            const double f = ((l - tr) * l + m2) * l - det;
            const double fp = (3.0 * l - 2.0 * tr) * l + m2;
            if (fp == 0.0) break;
            const double step = f / fp;
            l -= step;
            if (std::fabs(step) <= 1e-18 * std::max(1.0, std::fabs(l))) break;
        }
    std::sort(lam.begin(), lam.end());
    if (std::min(lam[1] - lam[0], lam[2] - lam[1]) < 1e-12 * std::max(1.0, std::fabs(lam[2]))) {
        why = "eigenvalues not separated";
        return false;
    }
    const int rows[3][2] = {{0, 1}, {0, 2}, {1, 2}};
    for (int k = 0; k < 3; ++k) {
        Mat3 s = e;
        for (int i = 0; i < 3; ++i) s[i][i] -= lam[k];
        std::array<double, 3> v{}, best{};
        double best_nn = -1.0;
        for (const auto& pr : rows) {
            const auto& a = s[pr[0]];
            const auto& b = s[pr[1]];
            v = {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
            const double nn = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
            if (nn > best_nn) {
                best_nn = nn;
                best = v;
            }
        }
        if (best_nn <= 0.0) {
            why = "defective eigenvector";
            return false;
        }
        int imax = 0;
        for (int i = 1; i < 3; ++i)
            if (std::fabs(best[i]) > std::fabs(best[imax])) imax = i;
        const double nrm = best[imax] < 0.0 ? -std::sqrt(best_nn) : std::sqrt(best_nn);
        for (int i = 0; i < 3; ++i) t[i][k] = best[i] / nrm;
    }
    if (!invert3(t, tinv)) {
        why = "singular eigenvector matrix";
        return false;
    }
    double resid = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double acc = 0.0;
            for (int k = 0; k < 3; ++k) acc += e[i][k] * t[k][j];
            resid = std::max(resid, std::fabs(acc - t[i][j] * lam[j]));
        }
    if (resid > 1e-12 * scale) {
        why = "eigendecomposition residual too large";
        return false;
    }
    return true;
}

}  // namespace

int scheme_init(double alpha1, double c1, double c2, double c3, mb4cu_scheme* out,
                std::string& why) {
    if (!out) {
        why = "null output";
        return MB4CU_INVALID;
    }
    if (!(alpha1 < -300.0 * 0.7770503941)) {
        why = "Mb4Scheme: alpha1 must be < -300*0.7770503941";
        return MB4CU_INVALID;
    }
    if (c3 != 1.0) {
        why = "Mb4Scheme: c3 must be 1";
        return MB4CU_INVALID;
    }
    const double cd[4] = {0.0, c1, c2, c3};
    for (int i = 1; i < 4; ++i) {
        if (!(cd[i] > 0.0) || cd[i] > 1.0) {
            why = "Mb4Scheme: nodes must lie in (0,1]";
            return MB4CU_INVALID;
        }
        for (int j = 0; j < i; ++j)
            if (cd[i] == cd[j]) {
                why = "Mb4Scheme: nodes must be distinct";
                return MB4CU_INVALID;
            }
    }
    mb4cu_scheme s;
    std::memset(&s, 0, sizeof(s));
    s.alpha1 = alpha1;
    std::array<ld, 4> c{};
    for (int i = 0; i < 4; ++i) {
        s.nodes[i] = cd[i];
        c[i] = cd[i];
    }
    const ld a1 = alpha1;

    ld z4[4], w4[4], z6[6], w6[6];
    gl_rule(4, z4, w4);
    gl_rule(6, z6, w6);
    // E: integrand degree 5, exact with 4 nodes.
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 4; ++j) {
            ld acc = 0.0L;
            for (int q = 0; q < 4; ++q) acc += w4[q] * coeff_a(a1, c[i + 1], z4[q]) * lagrange(c, j, z4[q]);
            s.E[i][j] = static_cast<double>(acc);
        }
    // W: integrand degree 11, exact with 6 nodes; symmetric in the last two slots.
    for (int i = 0; i < 3; ++i)
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b)
                for (int d = b; d < 4; ++d) {
                    ld acc = 0.0L;
                    for (int q = 0; q < 6; ++q)
                        acc += w6[q] * coeff_a(a1, c[i + 1], z6[q]) * lagrange(c, a, z6[q]) *
                               lagrange(c, b, z6[q]) * lagrange(c, d, z6[q]);
                    s.W[i][a][b][d] = s.W[i][a][d][b] = static_cast<double>(acc);
                }
    for (int q = 0; q < 6; ++q) {
        s.zeta6[q] = static_cast<double>(z6[q]);
        s.w6[q] = static_cast<double>(w6[q]);
        for (int a = 0; a < 4; ++a) s.L[q][a] = static_cast<double>(lagrange(c, a, z6[q]));
        for (int i = 0; i < 3; ++i) s.WA[i][q] = static_cast<double>(w6[q] * coeff_a(a1, c[i + 1], z6[q]));
    }
    Mat3 core, t, tinv;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) core[i][j] = s.E[i][j + 1];
    std::array<double, 3> lam{};
    if (!real_eig3(core, lam, t, tinv, why)) {
        why = "eig3_real: " + why;
        return MB4CU_INVALID;
    }
    for (int i = 0; i < 3; ++i) {
        s.lam[i] = lam[i];
        for (int j = 0; j < 3; ++j) {
            s.T[i][j] = t[i][j];
            s.Tinv[i][j] = tinv[i][j];
        }
    }
    *out = s;
    return MB4CU_OK;
}

// ---- scheme helpers of the reference API (mb4_scheme.hpp:14-20, 53-58) ----------

double eval_a_double(double alpha1, double tau, double zeta) {
    // the rank-one form of coeff_a above, in double as the reference's free eval_A
    const double lin = tau * (4.0 - 6.0 * zeta) + tau * tau * (6.0 * zeta - 3.0);
    const double t3 = tau * (1.0 - tau) * (1.0 - 2.0 * tau);
    const double z2 = 1.0 - 6.0 * zeta * (1.0 - zeta);
    return lin + alpha1 * t3 * z2;
}

int lagrange_basis_double(const double nodes[4], int i, double zeta, double* out, std::string& why) {
    if (!nodes || !out || i < 0 || i > 3) {
        why = "lagrange_basis: index out of range";
        return MB4CU_INVALID;
    }
    double v = 1.0;
    for (int b = 0; b < 4; ++b) {
        if (b == i) continue;
        const double den = nodes[i] - nodes[b];
        if (den == 0.0) {
            why = "lagrange_basis: coincident nodes";
            return MB4CU_INVALID;
        }
        v *= (zeta - nodes[b]) / den;
    }
    *out = v;
    return MB4CU_OK;
}

int integrate_e(double alpha1, const double nodes[4], int points, double out[12], std::string& why) {
    if (!nodes || !out || points < 1 || points > 64) {
        why = "integrate_e: points must be in 1..64";
        return MB4CU_INVALID;
    }
    std::array<ld, 4> c{};
    for (int i = 0; i < 4; ++i) c[i] = nodes[i];
    ld z[64], w[64];
    gl_rule(points, z, w);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 4; ++j) {
            ld acc = 0.0L;
            for (int q = 0; q < points; ++q) acc += w[q] * coeff_a(alpha1, c[i + 1], z[q]) * lagrange(c, j, z[q]);
            out[i * 4 + j] = static_cast<double>(acc);
        }
    return MB4CU_OK;
}

// ---- tables of the other integrators -----------------------------------------
// The reference builds them in double at first use from its Gauss-Legendre rule
// (quadrature.cpp:9-36: Newton iteration on P_n from the Chebyshev guess); the
// same rule and summation order are restated here so the GPU methods consume the
// same constants.
namespace {

void gauss_legendre_01_d(int n, double* nodes, double* weights) {
    const double pi = 3.14159265358979323846;
    for (int i = 0; i < n; ++i) {
        double x = std::cos(pi * (i + 0.75) / (n + 0.5));
        double dp = 0.0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = x;
            for (int k = 2; k <= n; ++k) {
                const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            dp = n * (x * p1 - p0) / (x * x - 1.0);
            const double dx = p1 / dp;
            x -= dx;
            if (std::abs(dx) < 1e-16) break;
        }
        const double w = 2.0 / ((1.0 - x * x) * dp * dp);
        nodes[n - 1 - i] = 0.5 * (x + 1.0);
        weights[n - 1 - i] = 0.5 * w;
    }
}

}  // namespace

void method_tables(MethodConsts* t) {
    // AVF2: B2[a][b][c] = int_0^1 m_a m_b m_c, m0 = 1 - x, m1 = x (2-node rule, exact)
    double x2[2], w2[2], x4[4], w4[4];
    gauss_legendre_01_d(2, x2, w2);
    gauss_legendre_01_d(4, x4, w4);
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            for (int c = 0; c < 2; ++c) {
                double s = 0.0;
                for (int g = 0; g < 2; ++g) {
                    const double m[2] = {1.0 - x2[g], x2[g]};
                    s += w2[g] * m[a] * m[b] * m[c];
                }
                t->b2[a][b][c] = s;
            }
    // AVF4 (integrators.cpp:301-335): Lagrange basis on the 2 Gauss nodes
    const double r3 = std::sqrt(3.0);
    const double c1 = 0.5 - r3 / 6.0, c2 = 0.5 + r3 / 6.0;
    const double bw[2] = {0.5, 0.5};
    auto ell = [&](int i, double x) { return i == 0 ? (x - c2) / (c1 - c2) : (x - c1) / (c2 - c1); };
    auto bigl = [&](int j, double x) {
        return j == 0 ? (0.5 * x * x - c2 * x) / (c1 - c2) : (0.5 * x * x - c1 * x) / (c2 - c1);
    };
    auto phi = [&](int a, double x) { return a == 0 ? 1.0 : bigl(a - 1, x); };
    for (int i = 0; i < 2; ++i)
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b)
                for (int c = 0; c < 3; ++c) {
                    double s = 0.0;
                    for (int g = 0; g < 4; ++g)
                        s += w4[g] * ell(i, x4[g]) * phi(a, x4[g]) * phi(b, x4[g]) * phi(c, x4[g]);
                    t->wt[i][a][b][c] = s / bw[i];
                }
    (void)x2;
}

// AVF4's Newton coupling mt[i][j] = (1/b_i) int l_i L_j (2-node rule)
void avf4_coupling(double mt[2][2]) {
    double x2[2], w2[2];
    gauss_legendre_01_d(2, x2, w2);
    const double r3 = std::sqrt(3.0);
    const double c1 = 0.5 - r3 / 6.0, c2 = 0.5 + r3 / 6.0;
    auto ell = [&](int i, double x) { return i == 0 ? (x - c2) / (c1 - c2) : (x - c1) / (c2 - c1); };
    auto bigl = [&](int j, double x) {
        return j == 0 ? (0.5 * x * x - c2 * x) / (c1 - c2) : (0.5 * x * x - c1 * x) / (c2 - c1);
    };
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) {
            double s = 0.0;
            for (int g = 0; g < 2; ++g) s += w2[g] * ell(i, x2[g]) * bigl(j, x2[g]);
            mt[i][j] = s / 0.5;
        }
}

}  // namespace mb4cu
