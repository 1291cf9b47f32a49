/*
 * oracle/mb4_oracle.c -- TEST INFRASTRUCTURE ONLY (see mb4_oracle.h).
 *
 * Plain-C restatement of the reference MB4 path.  Each function names the
 * reference file:line it restates (paths relative to /root/reference/proj).
 * The one deliberate difference from the reference is the stage linear
 * solver: the reference factorizes I - h*lambda_i*J with a sparse LU (or
 * ILU(0)+GMRES(50), mb4_integrator.cpp:19-34); this restatement solves the
 * same systems matrix-free with unpreconditioned restarted GMRES(50)
 * (iterative.cpp:68-153 with the identity preconditioner) to a relative
 * residual of 1e-13.  The converged stage root does not depend on the linear
 * solver (simplified Newton only changes its path), which the golden tests
 * against oracle/_ref (the reference itself) confirm.
 */
#include "mb4_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef long double ld;

/* ------------------------------------------------------------------------- */
/* Scheme constants: mb4_scheme.cpp:17-125, small_dense.cpp:27-174            */
/* ------------------------------------------------------------------------- */

/* A(tau, zeta) in the cancellation-free form of mb4_scheme.cpp:17-27. */
static ld eval_a_ld(ld a, ld tau, ld zeta) {
    const ld base = tau * (4.0L - 6.0L * zeta) + tau * tau * (6.0L * zeta - 3.0L);
    const ld tfac = tau * (1.0L - tau) * (1.0L - 2.0L * tau);
    const ld zfac = 1.0L - 6.0L * zeta * (1.0L - zeta);
    return base + a * tfac * zfac;
}

/* Gauss-Legendre rule on [0,1] in long double (mb4_scheme.cpp:30-50):
 * Newton iteration on P_n from the Chebyshev-like initial guess. Nodes ascending. */
static void gauss_legendre_ld(int n, ld* x01, ld* w01) {
    const ld pi = 3.14159265358979323846264338327950288L;
    for (int i = 0; i < n; ++i) {
        ld x = cosl(pi * (i + 0.75L) / (n + 0.5L));
        ld dp = 0.0L;
        for (int it = 0; it < 200; ++it) {
            ld p0 = 1.0L, p1 = x;
            for (int k = 2; k <= n; ++k) {
                const ld p2 = ((2.0L * k - 1.0L) * x * p1 - (k - 1.0L) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            dp = n * (x * p1 - p0) / (x * x - 1.0L);
            const ld dx = p1 / dp;
            x -= dx;
            if (fabsl(dx) < 1e-20L) break;
        }
        x01[n - 1 - i] = 0.5L * (x + 1.0L);
        w01[n - 1 - i] = 1.0L / ((1.0L - x * x) * dp * dp);
    }
}

/* Cubic Lagrange basis over 4 nodes (mb4_scheme.cpp:52-58). */
static ld lagrange_ld(const ld* nodes, int i, ld z) {
    ld v = 1.0L;
    for (int j = 0; j < 4; ++j)
        if (j != i) v *= (z - nodes[j]) / (nodes[i] - nodes[j]);
    return v;
}

/* 3x3 Gauss-Jordan inverse with partial pivoting (small_dense.cpp:27-58). */
static int inverse3(const double m[3][3], double inv[3][3]) {
    double a[3][3];
    memcpy(a, m, sizeof(a));
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) inv[i][j] = (i == j) ? 1.0 : 0.0;
    for (int k = 0; k < 3; ++k) {
        int piv = k;
        for (int i = k + 1; i < 3; ++i)
            if (fabs(a[i][k]) > fabs(a[piv][k])) piv = i;
        if (a[piv][k] == 0.0) return ORC_ERROR;
        if (piv != k)
            for (int j = 0; j < 3; ++j) {
                double t = a[k][j]; a[k][j] = a[piv][j]; a[piv][j] = t;
                t = inv[k][j]; inv[k][j] = inv[piv][j]; inv[piv][j] = t;
            }
        const double d = a[k][k];
        for (int j = 0; j < 3; ++j) {
            a[k][j] /= d;
            inv[k][j] /= d;
        }
        for (int i = 0; i < 3; ++i) {
            if (i == k) continue;
            const double f = a[i][k];
            if (f == 0.0) continue;
            for (int j = 0; j < 3; ++j) {
                a[i][j] -= f * a[k][j];
                inv[i][j] -= f * inv[k][j];
            }
        }
    }
    return ORC_OK;
}

static double inf_norm3(const double e[3][3]) {
    double best = 0.0;
    for (int i = 0; i < 3; ++i) {
        double s = fabs(e[i][0]) + fabs(e[i][1]) + fabs(e[i][2]);
        if (s > best) best = s;
    }
    return best;
}

static void sort3(double* v) {
    for (int i = 0; i < 3; ++i)
        for (int j = i + 1; j < 3; ++j)
            if (v[j] < v[i]) { double t = v[i]; v[i] = v[j]; v[j] = t; }
}

/* Real eigendecomposition of a 3x3 matrix with distinct real eigenvalues
 * (small_dense.cpp:83-174): trigonometric roots of the characteristic cubic,
 * Newton polish, eigenvectors from the best-conditioned cross product of rows
 * of (E - lambda I), deterministic sign (largest component positive). */
static int eig3_real(const double e[3][3], double lam[3], double t[3][3], double tinv[3][3]) {
    const double scale = fmax(inf_norm3(e), 1e-300);
    const double c2 = e[0][0] + e[1][1] + e[2][2];
    const double c1 = e[0][0] * e[1][1] - e[0][1] * e[1][0] + e[0][0] * e[2][2] -
                      e[0][2] * e[2][0] + e[1][1] * e[2][2] - e[1][2] * e[2][1];
    const double c0 = e[0][0] * (e[1][1] * e[2][2] - e[1][2] * e[2][1]) -
                      e[0][1] * (e[1][0] * e[2][2] - e[1][2] * e[2][0]) +
                      e[0][2] * (e[1][0] * e[2][1] - e[1][1] * e[2][0]);
    const double shift = c2 / 3.0;
    const double p = c1 - c2 * c2 / 3.0;
    const double q = -c0 + c1 * shift - 2.0 * c2 * c2 * c2 / 27.0;
    const double disc = q * q / 4.0 + p * p * p / 27.0;
    if (disc > 1e-14 * pow(scale, 6.0) || p >= 0.0) return ORC_ERROR;
    const double rho = 2.0 * sqrt(-p / 3.0);
    double arg = 3.0 * q / (p * rho);
    if (arg < -1.0) arg = -1.0;
    if (arg > 1.0) arg = 1.0;
    const double theta = acos(arg) / 3.0;
    const double pi = 3.14159265358979323846;
    for (int k = 0; k < 3; ++k) lam[k] = rho * cos(theta - 2.0 * pi * k / 3.0) + shift;
    sort3(lam);
    for (int k = 0; k < 3; ++k) {
        double l = lam[k];
        for (int it = 0; it < 3; ++it) {
            const double f = ((l - c2) * l + c1) * l - c0;
            const double fp = (3.0 * l - 2.0 * c2) * l + c1;
            if (fp == 0.0) break;
            const double step = f / fp;
            l -= step;
            if (fabs(step) <= 1e-18 * fmax(1.0, fabs(l))) break;
        }
        lam[k] = l;
    }
    sort3(lam);
    const double sep = fmin(lam[1] - lam[0], lam[2] - lam[1]);
    if (sep < 1e-12 * fmax(1.0, fabs(lam[2]))) return ORC_ERROR;

    static const int pairs[3][2] = {{0, 1}, {0, 2}, {1, 2}};
    for (int k = 0; k < 3; ++k) {
        double m[3][3];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) m[i][j] = e[i][j] - (i == j ? lam[k] : 0.0);
        double best[3] = {0, 0, 0}, best_norm = -1.0;
        for (int pi_ = 0; pi_ < 3; ++pi_) {
            const double* a = m[pairs[pi_][0]];
            const double* b = m[pairs[pi_][1]];
            const double v[3] = {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2],
                                 a[0] * b[1] - a[1] * b[0]};
            const double nn = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
            if (nn > best_norm) {
                best_norm = nn;
                best[0] = v[0]; best[1] = v[1]; best[2] = v[2];
            }
        }
        if (best_norm <= 0.0) return ORC_ERROR;
        double nrm = sqrt(best_norm);
        int imax = 0;
        for (int i = 1; i < 3; ++i)
            if (fabs(best[i]) > fabs(best[imax])) imax = i;
        if (best[imax] < 0.0) nrm = -nrm;
        for (int i = 0; i < 3; ++i) t[i][k] = best[i] / nrm;
    }
    if (inverse3(t, tinv) != ORC_OK) return ORC_ERROR;
    /* residual health check E T = T diag(lambda) */
    double resid = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double lhs = 0.0;
            for (int k = 0; k < 3; ++k) lhs += e[i][k] * t[k][j];
            const double r = fabs(lhs - t[i][j] * lam[j]);
            if (r > resid) resid = r;
        }
    if (resid > 1e-12 * scale) return ORC_ERROR;
    return ORC_OK;
}

int orc_scheme_init(double alpha1, double c1, double c2, double c3, orc_scheme_t* s) {
    /* validation: mb4_scheme.cpp:84-93 */
    if (!(alpha1 < -300.0 * 0.7770503941)) return ORC_INVALID;
    if (c3 != 1.0) return ORC_INVALID;
    const double nd[4] = {0.0, c1, c2, c3};
    for (int i = 1; i < 4; ++i) {
        if (!(nd[i] > 0.0) || nd[i] > 1.0) return ORC_INVALID;
        for (int j = 0; j < i; ++j)
            if (nd[i] == nd[j]) return ORC_INVALID;
    }
    memset(s, 0, sizeof(*s));
    s->alpha1 = alpha1;
    for (int i = 0; i < 4; ++i) s->nodes[i] = nd[i];
    const ld nl[4] = {nd[0], nd[1], nd[2], nd[3]};
    const ld al = alpha1;

    /* E with the 4-point rule (mb4_scheme.cpp:101-102,142-157) */
    ld x4[4], w4[4];
    gauss_legendre_ld(4, x4, w4);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 4; ++j) {
            ld acc = 0.0L;
            for (int q = 0; q < 4; ++q)
                acc += w4[q] * eval_a_ld(al, nl[i + 1], x4[q]) * lagrange_ld(nl, j, x4[q]);
            s->E[i][j] = (double)acc;
        }
    /* W with the 6-point rule, b <= c then mirrored (mb4_scheme.cpp:104-119) */
    ld x6[6], w6[6];
    gauss_legendre_ld(6, x6, w6);
    for (int i = 0; i < 3; ++i)
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b)
                for (int c = b; c < 4; ++c) {
                    ld acc = 0.0L;
                    for (int q = 0; q < 6; ++q)
                        acc += w6[q] * eval_a_ld(al, nl[i + 1], x6[q]) * lagrange_ld(nl, a, x6[q]) *
                               lagrange_ld(nl, b, x6[q]) * lagrange_ld(nl, c, x6[q]);
                    s->W[i][a][b][c] = (double)acc;
                    s->W[i][a][c][b] = (double)acc;
                }
    /* GL-6 tables for the quadrature form of the cubic term */
    for (int q = 0; q < 6; ++q) {
        s->zeta6[q] = (double)x6[q];
        s->w6[q] = (double)w6[q];
        for (int a = 0; a < 4; ++a) s->L[q][a] = (double)lagrange_ld(nl, a, x6[q]);
        for (int i = 0; i < 3; ++i) s->WA[i][q] = (double)(w6[q] * eval_a_ld(al, nl[i + 1], x6[q]));
    }
    /* eigendecomposition of the 3x3 core (mb4_scheme.cpp:121-124) */
    double core[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) core[i][j] = s->E[i][j + 1];
    return eig3_real(core, s->lam, s->T, s->Tinv);
}

/* ------------------------------------------------------------------------- */
/* Lattice: lattice.cpp:33-49 (K), :86-89 (apply_kv), :91-104 (rhs),           */
/* :106-137 (observables)                                                      */
/* ------------------------------------------------------------------------- */

/* y = K x for one complex component pair (interleaved), periodic 5-point stencil
 * with diagonal 2cx+2cy and off-diagonals -cx, -cy; for nx or ny = 2 both
 * wraparound neighbours coincide and are summed, as csr_from_triplets does. */
static void apply_k(const orc_model_t* m, const double* x, double* y) {
    const int nx = m->nx, ny = m->ny;
    const double d = 2.0 * m->cx + 2.0 * m->cy;
    for (int j = 0; j < ny; ++j) {
        const int jm = (j - 1 + ny) % ny, jp = (j + 1) % ny;
        for (int i = 0; i < nx; ++i) {
            const int im = (i - 1 + nx) % nx, ip = (i + 1) % nx;
            const long k = (long)j * nx + i;
            for (int c = 0; c < 2; ++c) {
                const double xl = x[2 * ((long)j * nx + im) + c], xr = x[2 * ((long)j * nx + ip) + c];
                const double xd = x[2 * ((long)jm * nx + i) + c], xu = x[2 * ((long)jp * nx + i) + c];
                y[2 * k + c] = d * x[2 * k + c] - m->cx * (xl + xr) - m->cy * (xd + xu);
            }
        }
    }
}

void orc_apply_kv(const orc_model_t* m, const double* u, double* y) {
    apply_k(m, u, y);
    const long n = (long)m->nx * m->ny;
    for (long k = 0; k < n; ++k) {
        y[2 * k] += m->V[k] * u[2 * k];
        y[2 * k + 1] += m->V[k] * u[2 * k + 1];
    }
}

void orc_rhs(const orc_model_t* m, const double* u, double* y) {
    apply_k(m, u, y);
    const long n = (long)m->nx * m->ny;
    for (long k = 0; k < n; ++k) {
        const double p = u[2 * k], q = u[2 * k + 1];
        const double n2 = p * p + q * q;
        const double ar = y[2 * k] + m->V[k] * p - m->gamma * n2 * p;
        const double ai = y[2 * k + 1] + m->V[k] * q - m->gamma * n2 * q;
        y[2 * k] = ai;    /* -i (ar + i ai) = ai - i ar */
        y[2 * k + 1] = -ar;
    }
}

int orc_observables(const orc_model_t* m, const double* u, orc_obs_t* out) {
    const long n = (long)m->nx * m->ny;
    double* ku = (double*)malloc(sizeof(double) * 2 * n);
    if (!ku) return ORC_ERROR;
    apply_k(m, u, ku);
    double qr = 0.0, qi = 0.0, prob = 0.0, quart = 0.0, ext = 0.0;
    for (long k = 0; k < n; ++k) {
        const double p = u[2 * k], q = u[2 * k + 1];
        /* conj(u) * ku */
        qr += p * ku[2 * k] + q * ku[2 * k + 1];
        qi += p * ku[2 * k + 1] - q * ku[2 * k];
        const double n2 = p * p + q * q;
        prob += n2;
        quart += n2 * n2;
        ext += m->V[k] * n2;
    }
    free(ku);
    const double kinf = 4.0 * m->cx + 4.0 * m->cy; /* max row sum of |K| */
    const double imag_scale = fmax(fabs(qr), kinf * prob);
    if (fabs(qi) > 1e-12 * imag_scale && imag_scale > 0.0) return ORC_ERROR;
    out->u_kinetic = qr;
    out->u_nonlinear = -0.5 * m->gamma * quart;
    out->u_external = ext;
    out->total_energy = out->u_kinetic + out->u_nonlinear + out->u_external;
    out->probability = prob;
    out->raw_quartic = quart;
    out->participation = prob > 0.0 ? quart / (prob * prob) : 0.0;
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Stage residual: mb4_integrator.cpp:159-192 (W contraction, b<=c folding)   */
/* ------------------------------------------------------------------------- */

void orc_eval_phi(const orc_model_t* m, const orc_scheme_t* s, const double* u0,
                  const double* const stages[3], double h, double* const phi[3]) {
    const long n = (long)m->nx * m->ny;
    const double g = m->gamma;
    double* combo = (double*)malloc(sizeof(double) * 2 * n);
    double* kv = (double*)malloc(sizeof(double) * 2 * n);
    for (int i = 0; i < 3; ++i) {
        for (long k = 0; k < 2 * n; ++k)
            combo[k] = s->E[i][0] * u0[k] + s->E[i][1] * stages[0][k] + s->E[i][2] * stages[1][k] +
                       s->E[i][3] * stages[2][k];
        orc_apply_kv(m, combo, kv);
        for (long k = 0; k < n; ++k) {
            const double zr[4] = {u0[2 * k], stages[0][2 * k], stages[1][2 * k], stages[2][2 * k]};
            const double zi[4] = {u0[2 * k + 1], stages[0][2 * k + 1], stages[1][2 * k + 1],
                                  stages[2][2 * k + 1]};
            double cr = 0.0, ci = 0.0;
            for (int a = 0; a < 4; ++a) {
                double ir = 0.0, ii = 0.0;
                for (int b = 0; b < 4; ++b) {
                    const double wbb = s->W[i][a][b][b];
                    ir += wbb * (zr[b] * zr[b] - zi[b] * zi[b]);
                    ii += wbb * (2.0 * zr[b] * zi[b]);
                    for (int c = b + 1; c < 4; ++c) {
                        const double w2 = 2.0 * s->W[i][a][b][c];
                        ir += w2 * (zr[b] * zr[c] - zi[b] * zi[c]);
                        ii += w2 * (zr[b] * zi[c] + zi[b] * zr[c]);
                    }
                }
                /* conj(z_a) * inner */
                cr += zr[a] * ir + zi[a] * ii;
                ci += zr[a] * ii - zi[a] * ir;
            }
            /* -i kv + i g cubic */
            const double fr = kv[2 * k + 1] - g * ci;
            const double fi = -kv[2 * k] + g * cr;
            phi[i][2 * k] = stages[i][2 * k] - u0[2 * k] - h * fr;
            phi[i][2 * k + 1] = stages[i][2 * k + 1] - u0[2 * k + 1] - h * fi;
        }
    }
    free(combo);
    free(kv);
}

/* ------------------------------------------------------------------------- */
/* Stage systems (I - h lambda J) in split form, applied matrix-free.          */
/* J as assembled in mb4_integrator.cpp:36-107 (hpp:52-55):                   */
/*   [ -2g p q            (K+V) - g(p^2+3q^2) ]                                */
/*   [ -(K+V) + g(3p^2+q^2)         2g p q     ]                               */
/* ------------------------------------------------------------------------- */

typedef struct {
    const orc_model_t* m;
    const double* u0;
    double hl;       /* h * lambda_i */
    double* tmp_c;   /* 2N scratch: interleaved complex */
    double* tmp_kv;  /* 2N scratch */
} stage_op_t;

/* y = (I - hl J) x, x and y split [p; q] of length 2N */
static void stage_apply(const stage_op_t* op, const double* x, double* y) {
    const orc_model_t* m = op->m;
    const long n = (long)m->nx * m->ny;
    const double g = m->gamma;
    for (long k = 0; k < n; ++k) {
        op->tmp_c[2 * k] = x[k];
        op->tmp_c[2 * k + 1] = x[n + k];
    }
    orc_apply_kv(m, op->tmp_c, op->tmp_kv); /* (K+V) tp, (K+V) tq interleaved */
    for (long k = 0; k < n; ++k) {
        const double p = op->u0[2 * k], q = op->u0[2 * k + 1];
        const double tp = x[k], tq = x[n + k];
        const double jp = -2.0 * g * p * q * tp + op->tmp_kv[2 * k + 1] - g * (p * p + 3.0 * q * q) * tq;
        const double jq = -op->tmp_kv[2 * k] + g * (3.0 * p * p + q * q) * tp + 2.0 * g * p * q * tq;
        y[k] = tp - op->hl * jp;
        y[n + k] = tq - op->hl * jq;
    }
}

static double norm2(const double* v, long n) {
    double s = 0.0;
    for (long i = 0; i < n; ++i) s += v[i] * v[i];
    return sqrt(s);
}

/* Restarted GMRES(50), unpreconditioned restatement of iterative.cpp:68-153. */
static int gmres_solve(const stage_op_t* op, const double* b, double* x, double tol) {
    const long n = 2L * op->m->nx * op->m->ny;
    const int restart = 50, max_iters = 2000;
    const int mr = (long)restart < n ? restart : (int)n;
    const double bnorm = norm2(b, n);
    memset(x, 0, sizeof(double) * n);
    if (bnorm == 0.0) return ORC_OK;
    double* v = (double*)malloc(sizeof(double) * n * (mr + 1));
    double* hmat = (double*)calloc((size_t)(mr + 1) * mr, sizeof(double));
    double* cs = (double*)calloc(mr, sizeof(double));
    double* sn = (double*)calloc(mr, sizeof(double));
    double* gv = (double*)calloc(mr + 1, sizeof(double));
    double* yv = (double*)calloc(mr, sizeof(double));
    double* r = (double*)malloc(sizeof(double) * n);
    double* w = (double*)malloc(sizeof(double) * n);
#define H(i, j) hmat[(size_t)(i) * mr + (j)]
    int status = ORC_OK;
    for (int iter = 0; iter < max_iters;) {
        stage_apply(op, x, r);
        for (long i = 0; i < n; ++i) r[i] = b[i] - r[i];
        const double beta = norm2(r, n);
        if (beta / bnorm <= tol) break;
        for (long i = 0; i < n; ++i) v[i] = r[i] / beta;
        memset(gv, 0, sizeof(double) * (mr + 1));
        gv[0] = beta;
        int j = 0;
        for (; j < mr && iter < max_iters; ++j, ++iter) {
            stage_apply(op, v + (size_t)j * n, w);
            for (int i = 0; i <= j; ++i) {
                double dot = 0.0;
                const double* vi = v + (size_t)i * n;
                for (long k = 0; k < n; ++k) dot += w[k] * vi[k];
                H(i, j) = dot;
                for (long k = 0; k < n; ++k) w[k] -= dot * vi[k];
            }
            H(j + 1, j) = norm2(w, n);
            if (H(j + 1, j) > 0.0) {
                double* vj1 = v + (size_t)(j + 1) * n;
                for (long k = 0; k < n; ++k) vj1[k] = w[k] / H(j + 1, j);
            }
            for (int i = 0; i < j; ++i) {
                const double t = cs[i] * H(i, j) + sn[i] * H(i + 1, j);
                H(i + 1, j) = -sn[i] * H(i, j) + cs[i] * H(i + 1, j);
                H(i, j) = t;
            }
            const double denom = hypot(H(j, j), H(j + 1, j));
            if (denom == 0.0) { status = ORC_ERROR; goto done; }
            cs[j] = H(j, j) / denom;
            sn[j] = H(j + 1, j) / denom;
            H(j, j) = denom;
            H(j + 1, j) = 0.0;
            gv[j + 1] = -sn[j] * gv[j];
            gv[j] = cs[j] * gv[j];
            if (fabs(gv[j + 1]) / bnorm <= tol) { ++j; break; }
        }
        for (int i = j - 1; i >= 0; --i) {
            double sacc = gv[i];
            for (int kk = i + 1; kk < j; ++kk) sacc -= H(i, kk) * yv[kk];
            yv[i] = sacc / H(i, i);
        }
        for (int kk = 0; kk < j; ++kk) {
            const double* vk = v + (size_t)kk * n;
            for (long i = 0; i < n; ++i) x[i] += vk[i] * yv[kk];
        }
        stage_apply(op, x, r);
        for (long i = 0; i < n; ++i) r[i] = b[i] - r[i];
        if (norm2(r, n) / bnorm <= tol) break;
    }
done:
#undef H
    free(v); free(hmat); free(cs); free(sn); free(gv); free(yv); free(r); free(w);
    return status;
}

/* ------------------------------------------------------------------------- */
/* Simplified Newton: mb4_integrator.cpp:194-255                               */
/* ------------------------------------------------------------------------- */

int orc_newton_solve(const orc_model_t* m, const orc_scheme_t* s, const double* u0, double h,
                     const orc_newton_t* cfg, double* const st[3], int* iters,
                     double* last_residual) {
    if (!(cfg->epsilon > 0.0) || cfg->max_iters < 1 || cfg->max_step_halvings < 0)
        return ORC_INVALID;
    const long n = (long)m->nx * m->ny;
    for (int i = 0; i < 3; ++i) memcpy(st[i], u0, sizeof(double) * 2 * n);
    double* phi[3];
    double* rhs[3];
    double* sol[3];
    for (int i = 0; i < 3; ++i) {
        phi[i] = (double*)malloc(sizeof(double) * 2 * n);
        rhs[i] = (double*)malloc(sizeof(double) * 2 * n);
        sol[i] = (double*)malloc(sizeof(double) * 2 * n);
    }
    stage_op_t op = {m, u0, 0.0, (double*)malloc(sizeof(double) * 2 * n),
                     (double*)malloc(sizeof(double) * 2 * n)};
    int status = ORC_NONCONVERGED;
    double rnorm = 0.0;
    *iters = 0;
    for (int iter = 1; iter <= cfg->max_iters; ++iter) {
        orc_eval_phi(m, s, u0, (const double* const*)st, h, phi);
        /* rhs_i = -(T^{-1} (x) I) Phi in split form (:212-219) */
        for (int i = 0; i < 3; ++i)
            for (long k = 0; k < n; ++k) {
                const double sr = s->Tinv[i][0] * phi[0][2 * k] + s->Tinv[i][1] * phi[1][2 * k] +
                                  s->Tinv[i][2] * phi[2][2 * k];
                const double si = s->Tinv[i][0] * phi[0][2 * k + 1] +
                                  s->Tinv[i][1] * phi[1][2 * k + 1] +
                                  s->Tinv[i][2] * phi[2][2 * k + 1];
                rhs[i][k] = -sr;
                rhs[i][n + k] = -si;
            }
        /* three independent stage solves (:221-229) */
        for (int i = 0; i < 3; ++i) {
            op.hl = h * s->lam[i];
            if (gmres_solve(&op, rhs[i], sol[i], 1e-13) != ORC_OK) {
                status = ORC_ERROR;
                goto out;
            }
        }
        /* r = (T (x) I) rbar, update, ||r||_inf, finite check (:231-250) */
        rnorm = 0.0;
        int finite = 1;
        for (int i = 0; i < 3; ++i)
            for (long k = 0; k < n; ++k) {
                const double rp = s->T[i][0] * sol[0][k] + s->T[i][1] * sol[1][k] + s->T[i][2] * sol[2][k];
                const double rq = s->T[i][0] * sol[0][n + k] + s->T[i][1] * sol[1][n + k] +
                                  s->T[i][2] * sol[2][n + k];
                st[i][2 * k] += rp;
                st[i][2 * k + 1] += rq;
                const double a = fmax(fabs(rp), fabs(rq));
                if (a > rnorm) rnorm = a;
                finite = finite && isfinite(rp) && isfinite(rq);
            }
        *iters = iter;
        if (!finite) {
            rnorm = INFINITY;
            status = ORC_NONCONVERGED;
            goto out;
        }
        if (rnorm <= cfg->epsilon) {
            status = ORC_OK;
            goto out;
        }
    }
out:
    if (last_residual) *last_residual = rnorm;
    for (int i = 0; i < 3; ++i) { free(phi[i]); free(rhs[i]); free(sol[i]); }
    free(op.tmp_c);
    free(op.tmp_kv);
    return status;
}

/* ------------------------------------------------------------------------- */
/* mb4_step with the halving policy: mb4_integrator.cpp:259-316               */
/* ------------------------------------------------------------------------- */

int orc_mb4_step(const orc_model_t* m, const orc_scheme_t* s, const double* u0, double h,
                 const orc_newton_t* cfg, double* u1, int* newton_iters, int* halvings,
                 double* last_residual) {
    if (!(h > 0.0)) return ORC_INVALID;
    if (!(cfg->epsilon > 0.0) || cfg->max_iters < 1 || cfg->max_step_halvings < 0)
        return ORC_INVALID;
    const long n = (long)m->nx * m->ny;
    double* u = (double*)malloc(sizeof(double) * 2 * n);
    double* st[3];
    for (int i = 0; i < 3; ++i) st[i] = (double*)malloc(sizeof(double) * 2 * n);
    double last = 0.0;
    int status = ORC_NONCONVERGED;
    for (int hv = 0; hv <= cfg->max_step_halvings; ++hv) {
        const int sub = 1 << hv;
        const double hs = h / sub;
        memcpy(u, u0, sizeof(double) * 2 * n);
        int ok = 1, attempt_iters = 0;
        for (int k = 0; k < sub; ++k) {
            int it = 0;
            const int rc = orc_newton_solve(m, s, u, hs, cfg, st, &it, &last);
            attempt_iters += it;
            if (rc == ORC_ERROR) { status = ORC_ERROR; goto out; }
            if (rc != ORC_OK) { ok = 0; break; }
            memcpy(u, st[2], sizeof(double) * 2 * n); /* c3 = 1: u1 = U_{c3} */
        }
        if (ok) {
            memcpy(u1, u, sizeof(double) * 2 * n);
            if (newton_iters) *newton_iters = attempt_iters;
            if (halvings) *halvings = hv;
            status = ORC_OK;
            break;
        }
    }
out:
    if (last_residual) *last_residual = last;
    free(u);
    for (int i = 0; i < 3; ++i) free(st[i]);
    return status;
}

static void put_obs(double* row, const orc_obs_t* o) {
    row[0] = o->u_kinetic; row[1] = o->u_nonlinear; row[2] = o->u_external;
    row[3] = o->total_energy; row[4] = o->probability; row[5] = o->participation;
    row[6] = o->raw_quartic;
}

/* run(): stepping loop with per-step observables (harness.cpp:64-133). */
int orc_run(const orc_model_t* m, const orc_scheme_t* s, double* u, double h, int nsteps,
            const orc_newton_t* cfg, double* obs_series, int* iters_series) {
    orc_obs_t o;
    if (obs_series) {
        if (orc_observables(m, u, &o) != ORC_OK) return ORC_ERROR;
        put_obs(obs_series, &o);
    }
    for (int st = 1; st <= nsteps; ++st) {
        int it = 0, hv = 0;
        double last = 0.0;
        const int rc = orc_mb4_step(m, s, u, h, cfg, u, &it, &hv, &last);
        if (rc != ORC_OK) return rc;
        if (iters_series) iters_series[st - 1] = it;
        if (obs_series) {
            if (orc_observables(m, u, &o) != ORC_OK) return ORC_ERROR;
            put_obs(obs_series + 7 * st, &o);
        }
    }
    return ORC_OK;
}
