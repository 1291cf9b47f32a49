/*
 * oracle/mb4_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C99, long double where the reference uses it) of the
 * reference MB4 time-stepping path of arxiv/paper_2003_04345
 * (/root/reference/proj).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library, and only as the
 * checker or the timed CPU baseline -- never as part of the product path.
 *
 * Pinning: the restatement is checked (tests/test_oracle_pins.py) against
 *   - the exact-rational scheme tables the reference's own generator produces
 *     (tools/exact_scheme_tables.py -> tests/golden/scheme_exact.json),
 *   - the 64-node quadrature oracle of Phi (test_mb4_integrator.cpp:29-55,78-91),
 *   - golden states/energy series produced by the reference library itself
 *     (oracle/_ref, tests/golden/make_golden.py).
 *
 * State layout: interleaved complex doubles (re, im) per site, site k = j*nx + i
 * (lattice.hpp:13-14,32), i.e. exactly std::vector<std::complex<double>> memory.
 */
#ifndef MB4_ORACLE_H
#define MB4_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    double alpha1;
    double nodes[4];          /* {0, c1, c2, c3} */
    double E[3][4];           /* e_ext(i+1, j)                     mb4_scheme.hpp:271 */
    double W[3][4][4][4];     /* w(i+1, a, b, c)                   mb4_scheme.hpp:272 */
    double lam[3];            /* eigenvalues of the 3x3 core, ascending */
    double T[3][3];           /* columns = eigenvectors             small_dense.hpp:213-217 */
    double Tinv[3][3];
    /* GL-6 tables (not exposed by the reference; used by the matrix-free form)
     * L[q][a] = l_a(zeta_q), WA[i][q] = w_q * A(c_{i+1}, zeta_q). */
    double zeta6[6], w6[6];
    double L[6][4];
    double WA[3][6];
} orc_scheme_t;

typedef struct {
    int nx, ny;
    double cx, cy;            /* 1/hx^2, 1/hy^2 (lattice.cpp:33-49) */
    double gamma;             /* reference gamma: i du/dt = Ku - gamma|u|^2u + Vu */
    const double* V;          /* N potential values */
} orc_model_t;

typedef struct {
    double epsilon;
    int max_iters;
    int max_step_halvings;
} orc_newton_t;

typedef struct {
    double u_kinetic, u_nonlinear, u_external, total_energy, probability, participation,
        raw_quartic;
} orc_obs_t;

/* status codes */
enum { ORC_OK = 0, ORC_INVALID = 1, ORC_NONCONVERGED = 2, ORC_ERROR = 3 };

int orc_scheme_init(double alpha1, double c1, double c2, double c3, orc_scheme_t* s);

void orc_apply_kv(const orc_model_t* m, const double* u, double* y);
void orc_rhs(const orc_model_t* m, const double* u, double* y);
int orc_observables(const orc_model_t* m, const double* u, orc_obs_t* out);

/* phi: 3 stage residuals, each 2N doubles, stages = 3 arrays of 2N doubles */
void orc_eval_phi(const orc_model_t* m, const orc_scheme_t* s, const double* u0,
                  const double* const stages[3], double h, double* const phi[3]);

/* Simplified Newton (mb4_integrator.cpp:194-255); stages out = 3 x 2N.
 * Returns ORC_OK / ORC_NONCONVERGED; *iters and *last_residual filled. */
int orc_newton_solve(const orc_model_t* m, const orc_scheme_t* s, const double* u0, double h,
                     const orc_newton_t* cfg, double* const stages_out[3], int* iters,
                     double* last_residual);

/* One MB4 step with the halving policy (mb4_integrator.cpp:275-316). u1 may alias u0. */
int orc_mb4_step(const orc_model_t* m, const orc_scheme_t* s, const double* u0, double h,
                 const orc_newton_t* cfg, double* u1, int* newton_iters, int* halvings,
                 double* last_residual);

/* nsteps steps; obs_series gets (nsteps+1) rows of 7 doubles (may be NULL),
 * iters_series nsteps ints (may be NULL). u is updated in place. */
int orc_run(const orc_model_t* m, const orc_scheme_t* s, double* u, double h, int nsteps,
            const orc_newton_t* cfg, double* obs_series, int* iters_series);

#ifdef __cplusplus
}
#endif
#endif
