/*
 * mb4cu.h -- C ABI of the B200-native MB4 time-stepping core.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj/include/nls2d/mb4_integrator.hpp:107-110 `mb4_step`,
 *  integrators.hpp:51 `StepDriver::advance`, lattice.hpp:88 `observables`).
 * The reference has no FFI layer; its boundary is the C++ API in
 * proj/include/nls2d.  The C++ mirror of that API (the headers in include/nls2d/) calls
 * these entry points, and so do the Python tests (ctypes) and bench.py.
 *
 * Conventions
 *  - plain pointers and sizes only; no exceptions cross this boundary;
 *  - every call returns an int status (MB4CU_*); mb4cu_last_error(ctx) has text;
 *  - a state is N interleaved complex doubles (re, im), site k = j*nx + i
 *    (lattice.hpp:13-14,32) -- byte-identical to std::vector<std::complex<double>>;
 *  - the context owns all device memory and its CUDA stream; the caller owns
 *    host buffers.  One host thread per context at a time.
 *
 * FP64 throughout.  The per-step implicit stage solve is a matrix-free,
 * stage-decoupled (T / T^-1) Neumann-preconditioned fixed-point iteration of
 * fused sm_100a stencil kernels; see DESIGN.md.
 */
#ifndef MB4CU_H
#define MB4CU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. */
enum {
    MB4CU_OK = 0,
    MB4CU_INVALID = 1,        /* invalid argument (reference: std::invalid_argument)      */
    MB4CU_NONCONVERGED = 2,   /* reference: NonConvergenceError (mb4_integrator.hpp:17-23) */
    MB4CU_CUDA_ERROR = 3,
    MB4CU_COMM_ERROR = 4,
    MB4CU_OOM = 5,
    MB4CU_NUMERIC = 6         /* observables health check (lattice.cpp:123-126)           */
};

/* Scheme constants (reference Mb4Scheme, mb4_scheme.hpp:26-64), computed on the
 * host in long double and rounded, plus the Gauss-Legendre-6 tables of the
 * quadrature form of the cubic term (not exposed by the reference):
 *   L[q][a]  = l_a(zeta_q)            (Lagrange basis over {0, c1, c2, c3})
 *   WA[i][q] = w_q * A(c_{i+1}, zeta_q)
 * so that W[i][a][b][c] = sum_q WA[i][q] L[q][a] L[q][b] L[q][c] and
 *         E[i][j]       = sum_q WA[i][q] L[q][j]. */
typedef struct {
    double alpha1;
    double nodes[4];
    double E[3][4];
    double W[3][4][4][4];
    double lam[3];
    double T[3][3];
    double Tinv[3][3];
    double zeta6[6];
    double w6[6];
    double L[6][4];
    double WA[3][6];
} mb4cu_scheme;

/* Replaces Mb4Scheme::Mb4Scheme(alpha1, nodes) (mb4_scheme.cpp:83-125).
 * Returns MB4CU_INVALID for the reference's validation failures and for
 * ComplexEigenvalueError (small_dense.cpp:100-101,127-128,151-152,171-172). */
int mb4cu_scheme_init(double alpha1, double c1, double c2, double c3, mb4cu_scheme* out);

/* Scheme helpers of the reference API (host arithmetic, no device):
 *   mb4cu_eval_a             eval_A(alpha1, tau, zeta)          mb4_scheme.hpp:14, mb4_scheme.cpp:66-68
 *   mb4cu_lagrange_basis     lagrange_basis(nodes, i, zeta)     mb4_scheme.hpp:17, mb4_scheme.cpp:70-80
 *                            (MB4CU_INVALID: index out of range / coincident nodes)
 *   mb4cu_scheme_integrate_e Mb4Scheme::integrate_e(alpha1, nodes, points)
 *                            mb4_scheme.hpp:55-58, mb4_scheme.cpp:141-157; out[i*4+j] = E_{i+1,j} */
double mb4cu_eval_a(double alpha1, double tau, double zeta);
int mb4cu_lagrange_basis(const double nodes[4], int i, double zeta, double* out);
int mb4cu_scheme_integrate_e(double alpha1, const double nodes[4], int points, double out[12]);

/* Problem description (replaces GridModel + NewtonConfig, lattice.hpp:49-73,
 * mb4_integrator.hpp:25-35). */
typedef struct {
    int nx, ny;               /* lattice (>= 2 each; lattice.cpp:117-121)               */
    double cx, cy;            /* 1/hx^2, 1/hy^2 of the periodic 5-point K (lattice.cpp:33-49) */
    double gamma;             /* reference gamma: i du/dt = K u - gamma |u|^2 u + V u   */
    const double* V;          /* host, nx*ny potential values (copied at create)        */
    double epsilon;           /* stop when ||r||_inf <= epsilon (split reals)          */
    int max_iters;            /* cap on stage sweeps per (sub)step                      */
    int max_step_halvings;    /* halving-on-failure policy (mb4_integrator.cpp:287-315) */
    int neumann_terms;        /* m in 0..3: preconditioner sum_{k<=m} (h lam J)^k; -1 = default
                                 (kernel 0: adaptive 1/2 from the sweep counts; else 1)    */
    int device;               /* CUDA device ordinal                                    */
    int kernel;               /* stage solver: 0 = default (persistent matrix-free sweeps),
                                 1 = tiled sweep kernel, 2 = march v1, 3 = Newton-Krylov
                                 (the reference's simplified Newton with matrix-free
                                 GMRES stage solves, for stiff h*lambda*rho(J) >~ 1)    */
    int ghost;                /* 0: one periodic domain.  > 0: this context is a sub-domain
                                 of a decomposed lattice (multi-GPU): arrays carry `ghost`
                                 halo layers (>= neumann_terms + 1) filled by the caller via
                                 mb4cu_halo_pack / _unpack, and steps are driven sweep by
                                 sweep (mb4cu_sweep / mb4cu_commit_step).                 */
    int neumann_first;        /* Neumann depth of the FIRST sweep of a step (its Phi is the
                                 cheap closed form, so the recursion is one J-chain);
                                 -1 = default (kernel 0: 6; sub-domain mode / tiled: 2).
                                 Kernel 0 pairs (first, terms): (0,0) (1,1) (2,0..2)
                                 (3,1) (4,1..2) (5,1..2) (6,0..2); tiled: equal or (2, <=2). */
    int first_poly;           /* polynomial p_k(J) ~ (I - h lam_k J)^-1 of that first sweep:
                                 0 = default (2 when H is convex -- V >= 0 and gamma <= 0 --,
                                 else 1); 1 = the Neumann (Taylor) series; 2 = the Chebyshev
                                 interpolant on the Gershgorin segment i[-rho, rho] of the
                                 spectrum of J (residual 2 (|h lam| rho / 2)^(d+1) instead of
                                 (|h lam| rho)^(d+1)).  With 2 the depth-2 later
                                 sweeps use the Chebyshev interpolant too (4x the contraction
                                 of the Neumann series, same cost).  Only the split of work
                                 between sweeps changes: the converged result does not.
                                 Kernels 1 / 2 always run the Neumann series.             */
} mb4cu_problem;

typedef struct {
    int newton_iters;         /* stage sweeps executed (all sub-steps)  (StepStats)      */
    int halvings;             /* halvings applied                                        */
    double solve_seconds;     /* device time of the stage solve (CUDA events)            */
    double last_residual;     /* ||r||_inf of the last sweep                             */
} mb4cu_stats;

typedef struct {
    double u_kinetic, u_nonlinear, u_external, total_energy, probability, participation,
        raw_quartic;          /* lattice.hpp:78-86 */
} mb4cu_obs;

typedef struct mb4cu_ctx mb4cu_ctx;

int mb4cu_create(const mb4cu_problem* prob, const mb4cu_scheme* scheme, mb4cu_ctx** out);
int mb4cu_destroy(mb4cu_ctx* ctx);
const char* mb4cu_last_error(const mb4cu_ctx* ctx);
/* text of the last failed mb4cu_create / mb4cu_scheme_init in this thread */
const char* mb4cu_create_error(void);

/* State transfer (host buffers: 2*nx*ny doubles). */
int mb4cu_set_state(mb4cu_ctx* ctx, const double* u_host);
int mb4cu_get_state(mb4cu_ctx* ctx, double* u_host);
/* Device-resident transfer (device pointers, async on the context stream). */
int mb4cu_set_state_device(mb4cu_ctx* ctx, const double* u_dev);
int mb4cu_get_state_device(mb4cu_ctx* ctx, double* u_dev);

/* One MB4 step of size h on the resident state (mb4_step, mb4_integrator.cpp:275-316).
 * On MB4CU_NONCONVERGED the state is unchanged. */
int mb4cu_step(mb4cu_ctx* ctx, double h, mb4cu_stats* stats);

/* nsteps steps; obs_series (may be NULL) receives (nsteps+1) rows of 7 doubles
 * (mb4cu_obs order), the t=0 row first (harness.cpp:105-122).  iters_series (may
 * be NULL) receives the sweeps of each step. */
int mb4cu_run(mb4cu_ctx* ctx, double h, int nsteps, double* obs_series, int* iters_series,
              mb4cu_stats* stats);

/* The reference's other integrators on the resident state (StepDriver::advance,
 * integrators.cpp:425-455; methods integrators.cpp:45-395), for the harness's
 * method comparison / convergence studies.  method = the reference's MethodId
 * order: */
#define MB4CU_METHOD_RK4 0    /* rk4_step, explicit, no halving                  */
#define MB4CU_METHOD_GAUSS2 1 /* gauss_step(1): implicit midpoint               */
#define MB4CU_METHOD_GAUSS4 2 /* gauss_step(2): 2-stage Gauss, coupled system   */
#define MB4CU_METHOD_AVF2 3   /* avf2_step                                      */
#define MB4CU_METHOD_AVF4 4   /* avf4_step, coupled system                      */
#define MB4CU_METHOD_MB4 5    /* = mb4cu_step / mb4cu_run                        */
/* Implicit methods: the reference's simplified Newton iteration (J at u0, stop on
 * ||delta||_inf <= epsilon) with the linear systems solved matrix-free by GMRES
 * on the GPU; halving on failure as the reference.  stats->newton_iters counts
 * Newton iterations.  Not available in sub-domain mode. */
int mb4cu_method_step(mb4cu_ctx* ctx, int method, double h, mb4cu_stats* stats);
/* mb4cu_run for any method (energy record from a separate monitor pass). */
int mb4cu_method_run(mb4cu_ctx* ctx, int method, double h, int nsteps, double* obs_series, int* iters_series,
                     mb4cu_stats* stats);

/* Energy monitor of the resident state (observables, lattice.cpp:106-137). */
int mb4cu_observables(mb4cu_ctx* ctx, mb4cu_obs* out);

/* Bind the context to an external CUDA stream (e.g. torch's current stream);
 * NULL restores the context's own (non-blocking) stream.  For the legacy default
 * stream (torch's default stream reports handle 0) pass cudaStreamLegacy. */
int mb4cu_set_stream(mb4cu_ctx* ctx, void* cuda_stream);

/* Spectral bound rho >= rho(J(u0)) that places the first sweep's Chebyshev polynomial
 * (first_poly 2): the Gershgorin bound 4cx + 4cy + max|V| + 3|gamma| max|u0|^2 of this
 * context's owned sites and resident state, rounded up to a power of 2^(1/16).  The
 * ranks of a decomposed lattice must agree on one bound: all-reduce (max) their
 * mb4cu_spectral_bound and pass the result to mb4cu_set_spectral_bound (0 restores
 * the context's own bound). */
int mb4cu_spectral_bound(mb4cu_ctx* ctx, double* rho);
/* Neumann depth m of the later sweeps from now on (production kernel; m + 1 <= ghost for a
 * sub-domain context).  A decomposed lattice applies the single-domain adaptive policy
 * (m = 2 once a step needs >= 4 sweeps at m = 1, back to 1 after 64 steps) through it. */
int mb4cu_set_neumann_terms(mb4cu_ctx* ctx, int m);
int mb4cu_set_spectral_bound(mb4cu_ctx* ctx, double rho);
/* max|u0|^2 the context's spectral bound and stiffness test use from now on.  A whole
 * lattice tracks it itself (every step's first sweep measures its entry state, and the
 * next step uses it); a decomposed lattice passes the all-reduced (max) value of the
 * last step's dev_out7[6] to every rank, then agrees on the bound as above. */
int mb4cu_set_amax2(mb4cu_ctx* ctx, double amax2);

/* ---- Sub-domain (multi-GPU) stepping, ghost > 0 ---------------------------------
 * The caller owns the decomposition and the exchange (paper_2003_04345_b200/dist.py
 * does it over torch.distributed / NCCL).  One MB4 step is:
 *   exchange u0 halos;  for s = 0, 1, ...: (s > 0: exchange halos of stage set
 *   (s-1) & 1);  mb4cu_sweep(ctx, h, s, &r, sums);  r = allreduce_max(r);
 *   stop when r <= eps;  mb4cu_commit_step(ctx, s + 1).
 * Fields: 0 = u0, 1 = V, 2 = stage set 0 (U1..U3), 3 = stage set 1 (sets m + 1 wide;
 * u0 / V ghost wide); 4, 5 = stage set 0 / 1 ghost wide (halo-overlap mode, where the
 * last sweep's U3 halos become the next step's u0 halos).
 * Sides: 0 = west (x low), 1 = east, 2 = south (y low), 3 = north.  Pack reads the
 * ghost-wide strip of owned sites adjacent to the side; unpack writes the ghost strip
 * on that side.  x sides cover the owned rows; y sides the full padded width, so an
 * x exchange followed by a y exchange also fills the corners.  Counts are in doubles. */
size_t mb4cu_halo_count(const mb4cu_ctx* ctx, int field, int side);
int mb4cu_halo_pack(mb4cu_ctx* ctx, int field, int side, double* dev_buf);
int mb4cu_halo_unpack(mb4cu_ctx* ctx, int field, int side, const double* dev_buf);
/* One stage sweep (sweep index s; s == 0 starts from U = (u0,u0,u0) and also returns
 * the local energy sums of u0: Re u^H K u, Im u^H K u, sum|u|^2, sum|u|^4, sum V|u|^2).
 * *local_rmax = max over owned sites of the split-real update. */
int mb4cu_sweep(mb4cu_ctx* ctx, double h, int s, double* local_rmax, double* local_sums5);
/* Accept the iterate after `sweeps` sweeps as the step result (u0 <- U3). */
/* Asynchronous sweep for device-side collectives: enqueues sweep s on the context
 * stream and a copy of [local ||r||_inf, 5 local energy sums of u0, local max|u0|^2
 * (the last six for s = 0 only)] into dev_out7 (device memory; 7 doubles; a non-finite
 * residual is reported as +inf), without a host synchronisation, so the caller
 * can all-reduce the buffer on the same stream (NCCL) and read it once.
 * final_guess != 0 (s > 0): the sweep is predicted to be the last, only U3 (the
 * step result) is stored; if the reduced residual does not converge the caller
 * repeats the same sweep with final_guess = 0 before going on. */
int mb4cu_sweep_async(mb4cu_ctx* ctx, double h, int s, int final_guess, double* dev_out7);
/* Halo-exchange overlap: sweep s in two launches.  region 1 = the boundary frame
 * (the `ghost`-wide strips the neighbours' halos need; run it first, then start
 * exchanging them), region 2 = the interior (needs no halo; launched with at most
 * grid_cap CTAs -- 0 = all, < 0 = all but those of -grid_cap SMs -- to leave SMs to the
 * concurrent NCCL kernels) which then
 * leaves [||r||_inf over both, energy sums, max|u0|^2] in dev_out7 like mb4cu_sweep_async.
 * region 0 = the whole sub-domain (= mb4cu_sweep_async). */
int mb4cu_sweep_region(mb4cu_ctx* ctx, double h, int s, int final_guess, int region, int grid_cap,
                       double* dev_out7);
int mb4cu_commit_step(mb4cu_ctx* ctx, int sweeps);

/* ---- Native multi-GPU stepping over NCCL (optional; libnccl is dlopen'ed) ---------
 * The decomposed step without the host in the sweep loop: per sweep the boundary frame,
 * its halo exchange (NCCL send / recv on the context's communication stream) concurrently
 * with the interior, the all-reduce of [||r||_inf, energy sums, max|u0|^2] and the stopping
 * test (mb4_integrator.cpp:250 with the margin) on the device; the sweeps the previous
 * step's count predicts are enqueued at once and the host reads once per step.  Halving as
 * mb4cu_step.  The whole lattice's max|V| / min V are all-reduced at attach, so every rank
 * places the single domain's Chebyshev polynomial (bit-identical to one GPU).
 *   mb4cu_nccl_unique_id   rank 0: a communicator id (128 bytes) to broadcast to the ranks
 *   mb4cu_dist_attach      every rank, after mb4cu_set_state: neighbours = ranks west,
 *                          east, south, north on the px x py torus; grid_cap as
 *                          mb4cu_sweep_region; force_p2p: exchange through NCCL even with
 *                          oneself (1-GPU tests); adaptive_m: the single-domain depth policy
 *   mb4cu_dist_step        one MB4 step; entry_sums5 = the entry state's global energy sums
 *   mb4cu_dist_observables global energy sums of the resident state
 * libnccl: path of the process's libnccl.so.2 (NULL: the loader's). */
int mb4cu_nccl_unique_id(const char* libnccl, unsigned char id[128]);
int mb4cu_dist_attach(mb4cu_ctx* ctx, const char* libnccl, const unsigned char id[128], int nranks, int rank,
                      const int neighbours[4], int px, int py, int grid_cap, int force_p2p, int adaptive_m);
int mb4cu_dist_step(mb4cu_ctx* ctx, double h, mb4cu_stats* stats, double* entry_sums5);
int mb4cu_dist_observables(mb4cu_ctx* ctx, double* sums5);
int mb4cu_dist_detach(mb4cu_ctx* ctx);

/* ---- Stage-split Newton-Krylov (the paper's 3-way stage partition) ---------------
 * The simplified Newton iteration of the stiff-regime solver (mb4_integrator.cpp:194-255
 * with matrix-free, Fourier-preconditioned GMRES stage solves), opened up so that the
 * three decoupled stage systems (I - h lam_k J) x_k = b_k of an iteration can be solved
 * on different GPUs -- the partition the paper parallelises over nodes
 * (paper_2003_04345_b200/dist.py StageSplitSession).  Every rank holds the whole lattice:
 *   mb4cu_ns_begin(ctx, h);
 *   repeat: mb4cu_ns_phibar(ctx);  mb4cu_ns_solve(ctx, k) for the owned k;
 *           exchange x_k (mb4cu_ns_get_correction / mb4cu_ns_set_correction, 2N doubles
 *           of device memory);  mb4cu_ns_update(ctx, &r);  until r <= epsilon;
 *   mb4cu_ns_commit(ctx);
 * A context that solves all three systems reproduces kernel 3's step bit for bit. */
int mb4cu_ns_begin(mb4cu_ctx* ctx, double h);
int mb4cu_ns_phibar(mb4cu_ctx* ctx);
int mb4cu_ns_solve(mb4cu_ctx* ctx, int k);
int mb4cu_ns_get_correction(mb4cu_ctx* ctx, int k, double* dev_out);
int mb4cu_ns_set_correction(mb4cu_ctx* ctx, int k, const double* dev_in);
int mb4cu_ns_update(mb4cu_ctx* ctx, double* rmax);
int mb4cu_ns_commit(mb4cu_ctx* ctx);
/* The three stage values U_1..U_3 of the open step (host buffers, 2N doubles each):
 * NewtonResult::stages of newton_solve (mb4_integrator.hpp:85-95). */
int mb4cu_ns_get_stages(mb4cu_ctx* ctx, double* u1_host, double* u2_host, double* u3_host);
/* Close an open step without committing (the resident state is unchanged). */
int mb4cu_ns_abort(mb4cu_ctx* ctx);
/* Local energy sums of the resident state (ghosts of u0 must be current). */
int mb4cu_observables_sums(mb4cu_ctx* ctx, double* local_sums5);

/* ---- Lattice operators on caller-supplied host arrays (device-computed) -------
 * Used by the parity tests for the vector-field evaluator rows of SURVEY 8a. */
/* y = (K + V) u   (GridModel::apply_kv, lattice.cpp:86-89) */
int mb4cu_apply_kv(mb4cu_ctx* ctx, const double* u_host, double* y_host);
/* y = f(u) = -i(Ku + Vu - gamma|u|^2 u)   (rhs, lattice.cpp:91-104) */
int mb4cu_rhs(mb4cu_ctx* ctx, const double* u_host, double* y_host);
/* Stage residuals Phi_1..3 (eval_phi, mb4_integrator.cpp:159-192), evaluated
 * with the GL-6 quadrature form the sweep kernels use. */
int mb4cu_eval_phi(mb4cu_ctx* ctx, const double* u0, const double* s1, const double* s2,
                   const double* s3, double h, double* p1, double* p2, double* p3);

/* ---- BASELINE input generator (host, deterministic, counter-based RNG) --------
 * Seeded delta-defect potential and Gaussian wave packets.  Fills
 * the sub-block [x0, x0+lnx) x [y0, y0+lny) of the global gnx x gny lattice.
 * psi is NOT normalised; *psum receives sum |psi|^2 over the block so callers
 * can normalise globally (mb4cu_scale_state). */
typedef struct {
    int gnx, gny;             /* global lattice                                        */
    double defect_frac;       /* Bernoulli(frac) per site                              */
    uint64_t defect_seed;
    double vd_min, vd_max;    /* V at defects: vd_min if vd_max <= vd_min, else U[vd_min, vd_max) */
    int npackets;             /* Gaussian packets                                      */
    double sigma;
    /* explicit packet (used when random_packets == 0 and npackets == 1) */
    double x0, y0, kx, ky;
    int random_packets;       /* 1: centres, momenta, phases drawn from packet_seed    */
    uint64_t packet_seed;
    double k_max;             /* random momenta uniform in [-k_max, k_max]^2           */
    int threads;              /* host threads (<= 0: hardware concurrency)             */
} mb4cu_inputs;

int mb4cu_make_inputs(const mb4cu_inputs* spec, int x0, int y0, int lnx, int lny, double* V,
                      double* psi, double* psum);
/* psi *= s  (host, multithreaded) */
int mb4cu_scale_state(double* psi, size_t nsites, double s, int threads);

/* Kernel-level profiling of the stage sweeps (CUDA events around every sweep
 * launch, on the context stream).  alg_bytes counts the algorithmic HBM bytes
 * of the sweeps: 72 B/site for the first sweep of a step (u0, V in; U out) and
 * 120 B/site for the others (u0, V, U in; U out), 88 B/site for a final sweep
 * that stored U3 only (speculative final sweep) -- see DESIGN.md. */
typedef struct {
    double kernel_ms;         /* summed device time of the sweep launches            */
    long long launches;       /* sweep-kernel launches                                */
    long long sweeps;         /* stage sweeps executed                                */
    double alg_bytes;         /* algorithmic bytes of those sweeps                    */
    long long other_launches; /* energy-monitor / helper kernels                      */
    double sweep_ms[8];       /* device time by sweep index within a step (0 = first),
                                 persistent kernel only (%globaltimer at grid barriers) */
    long long sweep_n[8];     /* samples accumulated in sweep_ms                      */
    long long redone;         /* speculative final sweeps that missed and were redone */
    long long krylov_iters;   /* GMRES inner iterations (Newton-Krylov / other methods) */
} mb4cu_profile;

int mb4cu_profile_enable(mb4cu_ctx* ctx, int on);
int mb4cu_profile_reset(mb4cu_ctx* ctx);
int mb4cu_profile_get(mb4cu_ctx* ctx, mb4cu_profile* out);

/* Library version / build string. */
const char* mb4cu_version(void);

#ifdef __cplusplus
}
#endif
#endif
