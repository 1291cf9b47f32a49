// C ABI of libmb4cu: context management, the per-step stage-iteration driver
// with the reference's halving policy, the energy monitor, and the parity
// entry points.  See include/mb4cu.h for the contract and the reference
// interfaces each entry point replaces.
#include <cuda_runtime.h>
#include <cufft.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstddef>
#include <cstdlib>
#include <dlfcn.h>

#include <type_traits>

#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "mb4cu.h"
#include "mb4cu_internal.hpp"

using mb4cu::SweepArgs;
using mb4cu::SweepConsts;

struct mb4cu_ctx {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    int nx = 0, ny = 0;
    size_t n = 0;
    double cx = 0, cy = 0, gamma = 0, eps = 0;
    double vmax = 0;    // max |V| (host, at create)
    double amax2 = 0;   // max |u|^2 of the last set state (stiffness estimate)
    bool amax2_valid = false;  // recomputed on the device after every state set
    int max_iters = 0, max_halvings = 0, m = 2, mf = 2, kernel = 0;
    bool m_auto = false;  // neumann_terms = -1 on the production kernel: m adapts in {1, 2}
    int auto_steps = 0;
    int last_sweeps = 0;  // sweeps of the last converged step (predicts the final sweep)
    int first_poly = 1;   // first-sweep polynomial (resolved): 1 = Neumann (Taylor), 2 = Chebyshev
    bool kr_batch = true; // Newton-Krylov: the three stage solves in flight together (krb)
    // stage-split Newton-Krylov (mb4cu_ns_*): the step size and constants of the open step
    bool ns_open = false;
    double ns_h = 0.0;
    SweepConsts ns_c{};
    double vmin = 0;      // min V (host, at create)
    double rho_override = 0;  // > 0: spectral bound set by the caller (decomposed lattices)
    int ghost = 0, pitch = 0;  // sub-domain mode: halo width and padded row pitch
    size_t alloc_n = 0;        // elements per array (padded in sub-domain mode)
    mb4cu_scheme scheme{};
    double2* u0 = nullptr;
    double* V = nullptr;
    double2* U[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};
    double2* ubak = nullptr;
    unsigned long long* d_rmax = nullptr;
    unsigned long long* h_rmax = nullptr;  // pinned
    double* d_obs_partial = nullptr;
    double* d_obs5 = nullptr;
    double* h_obs5 = nullptr;  // pinned
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t pev0 = nullptr, pev1 = nullptr;
    // persistent-kernel path
    unsigned long long* d_rmax_arr = nullptr;  // [max_iters + 1]: residual bits per sweep, max |u0|^2
    unsigned* d_work = nullptr;                // [kWorkCounters]: chunk counters of the later sweeps
    int work_seq = 0;                          // sub-domain sweep launches so far (rotating counter index)
    double* d_obs_march = nullptr;             // [grid][kObsFields]
    mb4cu::StepStatus* d_status = nullptr;
    mb4cu::StepStatus* h_status = nullptr;     // pinned
    bool batched = true;                       // mb4cu_run enqueues steps device-resident
    struct DistNative* dn = nullptr;           // native NCCL stepping of a sub-domain (mb4cu_dist_*)
    bool first_poly_auto = false;
    int obs_grid = 0;                          // CTAs d_obs_march holds partial sums for
    // batched stepping (mb4cu_run): per-step status and residual slots, the abort flag and
    // per-step events, allocated on first use
    mb4cu::StepStatus* d_bstatus = nullptr;
    mb4cu::StepStatus* h_bstatus = nullptr;   // pinned
    unsigned long long* d_brmax = nullptr;     // [kBatch][max_iters]
    int* d_babort = nullptr;
    cudaEvent_t bev[65] = {};
    bool obs_cached = false;                   // energy sums of the current u0 known
    double obs_cache[mb4cu::kObsFields] = {0, 0, 0, 0, 0};
    double entry_obs[mb4cu::kObsFields] = {0, 0, 0, 0, 0};
    // Newton-Krylov path (kernel = 3), allocated on first use
    struct {
        int m = 0;                  // GMRES restart length
        int nblk = 0;
        size_t len = 0;             // complex entries per vector (N, or 2N for coupled systems)
        double2* mem = nullptr;     // basis (m+1) + b[3] + x[3] + w + y vectors
        double2** v_dev = nullptr;  // device array of basis pointers
        double* partial = nullptr;  // [m+1][nblk]
        double* h_partial = nullptr;  // pinned copy
        double* coef = nullptr;     // device coefficients [m+1]
        double* h_coef = nullptr;   // pinned
        double* hcol = nullptr;     // device Hessenberg column [m+2] (kr_arnoldi)
        double* h_hcol = nullptr;   // pinned
        long long gmres_iters = 0;  // total inner iterations (stats)
    } kr;
    // Fourier preconditioner of the Krylov solves (fft_precond.cu), created on first use
    struct {
        cufftHandle plan1 = 0, plan2 = 0;  // N-point 2-D Z2Z; batch of 2 (coupled systems)
        bool have1 = false, have2 = false;
        double* partial = nullptr;         // shift partial sums [blocks][2]
        double* h_partial = nullptr;
        double shift = 0.0;                // mean(V) - 2 gamma mean(|u0|^2) of the current u0
        double* shift_dev = nullptr;       // its device copy (read by graph-captured steps)
        double* h_shift = nullptr;         // pinned staging
    } fft;
    // The three decoupled stage solves of a Newton-Krylov iteration in flight at once
    // (the paper's stage parallelism, on one GPU): one stream, Krylov basis, FFT plan and
    // reduction buffers per stage system; used while 3 (m + 4) vectors fit kKrBatchBytes.
    struct {
        size_t len = 0;
        int m = 0, nblk = 0;
        double2* mem = nullptr;  // per system: basis (m + 1), w, y, preconditioner scratch
        double2** v_dev[3] = {nullptr, nullptr, nullptr};
        double* partial[3] = {nullptr, nullptr, nullptr};
        double* h_partial[3] = {nullptr, nullptr, nullptr};
        double* coef[3] = {nullptr, nullptr, nullptr};
        double* h_coef[3] = {nullptr, nullptr, nullptr};
        double* hcol[3] = {nullptr, nullptr, nullptr};
        double* h_hcol[3] = {nullptr, nullptr, nullptr};
        cudaStream_t st[3] = {nullptr, nullptr, nullptr};
        cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
        cufftHandle plan[3] = {0, 0, 0};
        bool ready = false;
        // one Arnoldi step of system q as a CUDA graph (gather v_j, preconditioner, matvec,
        // CGS2, Hessenberg column to the host), j in device memory (jd[q]); captured once per
        // (u0, h, shift) and relaunched for every step of every cycle
        int* jd = nullptr;
        struct Slot {
            const void* u0 = nullptr;  // the Newton-Krylov commit alternates u0 between two buffers
            double h = 0.0;
            cudaGraphExec_t g[3] = {nullptr, nullptr, nullptr};
        } slot[2];
        int next_slot = 0;
        bool use_graphs = true;
    } krb;
    bool profiling = false;
    mb4cu_profile prof{};
    std::string err;
};

namespace {

// Default Neumann depth m of the stage preconditioner (fastest measured on B200 at
// the BASELINE sizes, profiles/); on the production kernel m adapts between 1 and 2
// (adapt_neumann), and the first sweep of a step runs at depth kDefaultFirst.
constexpr int kDefaultNeumann = 1;
constexpr int kDefaultFirst = 6;

// Adaptive m (production kernel, neumann_terms = -1).  A later sweep at m = 2 costs
// ~1.28x one at m = 1 and contracts ~1.5x as much (kappa^3 vs kappa^2), so m = 2
// pays once a step needs >= 3 later sweeps at m = 1; it is re-probed every 64 steps.
// The choice depends only on sweep counts: reruns stay bit-identical.
void adapt_neumann(mb4cu_ctx* ctx, int sweeps) {
    if (!ctx->m_auto) return;
    if (ctx->m == 1 && sweeps >= 4) {
        ctx->m = 2;
        ctx->auto_steps = 0;
        ctx->last_sweeps = 0;
    } else if (ctx->m == 2 && ++ctx->auto_steps >= 64) {
        ctx->m = 1;
        ctx->auto_steps = 0;
        ctx->last_sweeps = 0;
    }
}

thread_local std::string g_create_error;

int fail(mb4cu_ctx* ctx, int code, const std::string& what) {
    if (ctx) ctx->err = what;
    return code;
}

int cuda_fail(mb4cu_ctx* ctx, cudaError_t e, const char* where) {
    const int code = e == cudaErrorMemoryAllocation ? MB4CU_OOM : MB4CU_CUDA_ERROR;
    return fail(ctx, code, std::string(where) + ": " + cudaGetErrorString(e));
}

#define MB4_CUDA(ctx, call)                                  \
    do {                                                     \
        cudaError_t e_ = (call);                             \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
    } while (0)

// Host copy of the generated default-scheme tables (build/gen/defscheme.inc).
namespace defscheme_host {
#define MB4_DS_QUAL static constexpr
#include "defscheme.inc"
#undef MB4_DS_QUAL
}  // namespace defscheme_host

// 1 if the context's scheme is bit-identical to the compiled-in default tables,
// so the production kernel may use them as immediates.
int is_default_scheme(const mb4cu_scheme& s) {
    namespace d = defscheme_host;
    return std::memcmp(s.L, d::L, sizeof(d::L)) == 0 && std::memcmp(s.WA, d::WA, sizeof(d::WA)) == 0 &&
                   std::memcmp(s.E, d::E, sizeof(d::E)) == 0 && std::memcmp(s.T, d::T, sizeof(d::T)) == 0 &&
                   std::memcmp(s.Tinv, d::Tinv, sizeof(d::Tinv)) == 0
               ? 1
               : 0;
}

// Gershgorin bound of the spectral radius of J(u0): rho <= 4cx + 4cy + max|V| + 3|gamma| max|u0|^2.
double spectral_bound(const mb4cu_ctx* ctx) {
    return 4.0 * ctx->cx + 4.0 * ctx->cy + ctx->vmax + 3.0 * std::fabs(ctx->gamma) * ctx->amax2;
}

// The bound that places the first sweep's Chebyshev polynomial: the context's own
// Gershgorin bound rounded up to a power of 2^(1/16) (so that last-bit differences of
// max|u0|^2 between a lattice and its decomposition pick the same polynomial), or
// the bound a decomposed lattice agreed on (mb4cu_set_spectral_bound).
double own_first_rho(const mb4cu_ctx* ctx) {
    const double rho = spectral_bound(ctx);
    return rho > 0.0 ? std::exp2(std::ceil(16.0 * std::log2(rho)) / 16.0) : 0.0;
}
double first_rho(const mb4cu_ctx* ctx) { return ctx->rho_override > 0.0 ? ctx->rho_override : own_first_rho(ctx); }

// Degree-`deg` polynomial p(x) = sum_n out[n] x^n approximating 1/(1 - beta x) on the
// spectrum of J.  With H(u0) positive semidefinite (K >= 0, V >= 0, defocusing) J = S H
// has its spectrum on i[-rho, rho]; p interpolates 1/(1 - beta x) at the deg + 1
// Chebyshev points of that segment, so the residual polynomial 1 - (1 - beta x) p(x)
// is the scaled Chebyshev polynomial T_{deg+1}: max residual ~ 2 (|beta| rho / 2)^(deg+1)
// instead of (|beta| rho)^(deg+1) for the Taylor (Neumann) series.  The iteration's
// fixed point does not depend on p; only how much the first sweep leaves for the next.
// In t = y / rho, G(t) = 1/(1 - i a t), a = beta rho: Re G = 1/(1 + a^2 t^2) (even),
// Im G = a t / (1 + a^2 t^2) (odd); interpolated in long double, then mapped back
// through y = -i x.
void cheb_first_poly(double beta, double rho, int deg, double* out) {
    const int n = deg + 1;
    long double A[8][8], bre[8], bim[8];
    const long double a = static_cast<long double>(beta) * rho;
    for (int j = 0; j < n; ++j) {
        const long double t = std::cos((2.0L * j + 1.0L) * 3.14159265358979323846264338327950288L / (2.0L * n));
        long double tp = 1.0L;
        for (int q = 0; q < n; ++q) {
            A[j][q] = tp;
            tp *= t;
        }
        const long double den = 1.0L + a * a * t * t;
        bre[j] = 1.0L / den;
        bim[j] = a * t / den;
    }
    // Gaussian elimination with partial pivoting, two right-hand sides
    for (int col = 0; col < n; ++col) {
        int piv = col;
        for (int r = col + 1; r < n; ++r)
            if (std::fabs(A[r][col]) > std::fabs(A[piv][col])) piv = r;
        for (int q = 0; q < n; ++q) std::swap(A[col][q], A[piv][q]);
        std::swap(bre[col], bre[piv]);
        std::swap(bim[col], bim[piv]);
        for (int r = col + 1; r < n; ++r) {
            const long double f = A[r][col] / A[col][col];
            for (int q = col; q < n; ++q) A[r][q] -= f * A[col][q];
            bre[r] -= f * bre[col];
            bim[r] -= f * bim[col];
        }
    }
    for (int r = n - 1; r >= 0; --r) {
        for (int q = r + 1; q < n; ++q) {
            bre[r] -= A[r][q] * bre[q];
            bim[r] -= A[r][q] * bim[q];
        }
        bre[r] /= A[r][r];
        bim[r] /= A[r][r];
    }
    // sum_q e_q t^q with t = y / rho and y = -i x: coefficient of x^q is e_q (-i)^q / rho^q,
    // real by the parity of G (even q: Re part, odd q: Im part)
    long double rp = 1.0L;
    for (int q = 0; q <= mb4cu::kMaxNeumannFirst; ++q) {
        long double v = 0.0L;
        if (q < n) v = (q % 2 == 0 ? bre[q] : bim[q]) * (((q / 2) % 2) ? -1.0L : 1.0L) / rp;
        out[q] = static_cast<double>(v);
        rp *= rho;
    }
}

SweepConsts make_consts(const mb4cu_ctx* ctx, double h) {
    SweepConsts c{};
    const mb4cu_scheme& s = ctx->scheme;
    std::memcpy(c.E, s.E, sizeof(c.E));
    std::memcpy(c.L, s.L, sizeof(c.L));
    std::memcpy(c.WA, s.WA, sizeof(c.WA));
    std::memcpy(c.T, s.T, sizeof(c.T));
    std::memcpy(c.Tinv, s.Tinv, sizeof(c.Tinv));
    for (int k = 0; k < 3; ++k) c.hlam[k] = h * s.lam[k];
    // First sweep from U = (u0, u0, u0): Phi_i = -h c_i f(u0) with c_i = sum_j E[i][j]
    // (the Lagrange basis sums to one), so phibar_k = -h (T^-1 c)_k f(u0).
    double csum[3];
    for (int i = 0; i < 3; ++i) csum[i] = s.E[i][0] + s.E[i][1] + s.E[i][2] + s.E[i][3];
    for (int k = 0; k < 3; ++k) {
        c.first_s[k] = -h * (s.Tinv[k][0] * csum[0] + s.Tinv[k][1] * csum[1] + s.Tinv[k][2] * csum[2]);
        c.first_c[k] = h * csum[k];
    }
    c.h = h;
    c.gamma = ctx->gamma;
    c.cx = ctx->cx;
    c.cy = ctx->cy;
    c.diag = 2.0 * ctx->cx + 2.0 * ctx->cy;
    c.iso = ctx->cx == ctx->cy ? 1 : 0;
    const double cc = ctx->cx;
    c.inv_c = 1.0 / cc;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 4; ++j) c.Es[i][j] = cc * s.E[i][j];
    c.gs = ctx->gamma / cc;
    c.hs = cc * h;
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 4; ++j) {
            c.hE[i][j] = h * s.E[i][j];
            c.hEs[i][j] = (cc * h) * s.E[i][j];
        }
        for (int q = 0; q < 6; ++q) {
            c.hgW[i][q] = (h * ctx->gamma) * s.WA[i][q];
            c.hgW8[i][q] = 0.125 * c.hgW[i][q];
        }
    }
    c.def = is_default_scheme(s);
    for (int k = 0; k < 3; ++k) {
        c.hls[k] = cc * c.hlam[k];
        c.first_ss[k] = cc * c.first_s[k];
        c.first_cs[k] = cc * c.first_c[k];
    }
    // per-stage polynomial p_k(x) ~ 1/(1 - h lam_k x) of the first sweep, monomial coefficients
    double pc[3][mb4cu::kMaxNeumannFirst + 1] = {};
    const double rho = first_rho(ctx);
    for (int k = 0; k < 3; ++k) {
        if (ctx->first_poly == 2 && rho > 0.0)
            cheb_first_poly(c.hlam[k], rho, ctx->mf, pc[k]);
        else
            for (int n = 0; n <= mb4cu::kMaxNeumannFirst; ++n) pc[k][n] = std::pow(c.hlam[k], n);
    }
    // depth-2 later sweeps: the Chebyshev interpolant at the nodes 0, +-(sqrt(3)/2) rho is
    // 1 + s (b x + b^2 x^2) -- the Neumann Horner form with the second multiplier scaled
    // by s (residual (|b| rho)^3 / 4 instead of (|b| rho)^3), at no extra cost
    for (int k = 0; k < 3; ++k) {
        const double br = c.hlam[k] * rho;
        c.hlam2[k] = ctx->first_poly == 2 && rho > 0.0 ? c.hlam[k] / (1.0 + 0.75 * br * br) : c.hlam[k];
        c.hls2[k] = cc * c.hlam2[k];
    }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            long double a = 0.0L;
            for (int k = 0; k < 3; ++k)
                a += static_cast<long double>(s.T[i][k]) * s.lam[k] * static_cast<long double>(s.Tinv[k][j]);
            c.hA[i][j] = static_cast<double>(h * a);
            c.hAs[i][j] = static_cast<double>(cc * (h * a));
        }
    for (int i = 0; i < 3; ++i)
        for (int n = 0; n <= mb4cu::kMaxNeumannFirst; ++n) {
            double acc = 0.0;
            for (int k = 0; k < 3; ++k) acc += s.T[i][k] * c.first_s[k] * pc[k][n];
            c.fco[i][n] = -acc * (c.iso ? std::pow(cc, n + 1) : 1.0);
        }
    return c;
}

double decode_bits(unsigned long long b) {
    double d;
    std::memcpy(&d, &b, sizeof(d));
    return d;
}

// Persistent path: the whole stage iteration of one sub-step in one cooperative
// launch (sweep_march.cu); the host reads back a 80-byte status block.
// Per-step spectral bound: the first sweep of every (sub)step measures max|u0|^2 of its
// entry state in its energy monitor (no extra pass); the next (sub)step's Chebyshev
// interval and stiffness test use it.  Only a newly set state pays a separate pass
// (refresh_amax2), as does the step after a Newton-Krylov step (no sweep measured it).
void track_amax2(mb4cu_ctx* ctx, double amax2) {
    ctx->amax2 = amax2;
    ctx->amax2_valid = true;
}

int substep_march(mb4cu_ctx* ctx, double h, int* sweeps, double* last_res) {
    const SweepConsts c = make_consts(ctx, h);
    MB4_CUDA(ctx, cudaMemsetAsync(ctx->d_rmax_arr, 0, sizeof(unsigned long long) * (ctx->max_iters + 1),
                                  ctx->stream));
    if (ctx->profiling) MB4_CUDA(ctx, cudaEventRecord(ctx->pev0, ctx->stream));
    // the step is predicted to converge at the previous step's sweep count: that
    // sweep stores U3 only (redone in-kernel with all stages if the guess fails)
    const int spec = ctx->last_sweeps >= 2 ? ctx->last_sweeps - 1 : -1;
    if (ctx->kernel == 0 && mb4cu::march2_supported(ctx->mf, ctx->m)) {
        MB4_CUDA(ctx, mb4cu::launch_step_march2(ctx->mf, ctx->m, ctx->nx, ctx->ny, ctx->u0, ctx->V, ctx->U,
                                                ctx->d_rmax_arr, ctx->d_obs_march, ctx->d_status,
                                                ctx->max_iters, ctx->eps, 1, c, ctx->device,
                                                ctx->stream, 0, 0, spec, 0, nullptr, 0, 0, nullptr, 0, ctx->d_work,
                                                ctx->obs_grid * mb4cu::kObsSlotsPerCta));
    } else {
        MB4_CUDA(ctx, mb4cu::launch_step_march(ctx->m, ctx->nx, ctx->ny, ctx->u0, ctx->V, ctx->U,
                                               ctx->d_rmax_arr, ctx->d_obs_march, ctx->d_status,
                                               ctx->max_iters, ctx->eps, 1, c, ctx->device,
                                               ctx->stream));
    }
    if (ctx->profiling) MB4_CUDA(ctx, cudaEventRecord(ctx->pev1, ctx->stream));
    MB4_CUDA(ctx, cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(mb4cu::StepStatus),
                                  cudaMemcpyDeviceToHost, ctx->stream));
    MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    const mb4cu::StepStatus st = *ctx->h_status;
    if (ctx->profiling) {
        float ms = 0.f;
        MB4_CUDA(ctx, cudaEventElapsedTime(&ms, ctx->pev0, ctx->pev1));
        ctx->prof.kernel_ms += ms;
        const bool m2 = ctx->kernel == 0 && mb4cu::march2_supported(ctx->mf, ctx->m);
        ctx->prof.launches += m2 ? mb4cu::march2_launches(ctx->mf, 0, 0, ctx->max_iters) : 1;
        ctx->prof.sweeps += st.sweeps;
        // U3-only final sweep: 88 instead of 120 B/site (a redone guess is overhead, not counted)
        const bool spec_hit = st.converged && st.sweeps - 1 == spec && spec >= 1;
        ctx->prof.alg_bytes += static_cast<double>(ctx->n) * (72.0 + 120.0 * (st.sweeps - 1) - (spec_hit ? 32.0 : 0.0));
        ctx->prof.redone += st.redone;
        if (ctx->kernel == 0 && mb4cu::march2_supported(ctx->mf, ctx->m)) {
            for (int k = 0; k < st.sweeps && k < 8; ++k) {
                ctx->prof.sweep_ms[k] += 1e-6 * static_cast<double>(st.t[k + 1] - st.t[k]);
                ctx->prof.sweep_n[k] += 1;
            }
        }
    }
    // the first sweep evaluated the energy sums of the entry state
    for (int f = 0; f < mb4cu::kObsFields; ++f) ctx->obs_cache[f] = st.obs[f];
    ctx->obs_cached = true;
    *sweeps = st.sweeps;
    *last_res = st.rlast;
    if (!std::isfinite(st.rlast)) {
        *last_res = INFINITY;
        return fail(ctx, MB4CU_NONCONVERGED, "stage iteration diverged (non-finite update)");
    }
    if (st.converged) {
        std::swap(ctx->u0, ctx->U[st.set][2]);
        ctx->obs_cached = false;
        const bool prod = mb4cu::march2_supported(ctx->mf, ctx->m) && ctx->kernel == 0;
        ctx->last_sweeps = prod ? st.sweeps : 0;
        if (prod) track_amax2(ctx, st.amax2);
        adapt_neumann(ctx, st.sweeps);
        return MB4CU_OK;
    }
    return fail(ctx, MB4CU_NONCONVERGED,
                "stage iteration: no convergence after " + std::to_string(ctx->max_iters) + " sweeps");
}

// Stiffness of a (sub)step: kappa = h max|lambda| rho(J(u0)) with the Gershgorin
// bound rho(J) <= 4cx + 4cy + max|V| + 3|gamma| max|u0|^2.  The m-term Neumann
// sweep contracts by ~kappa^(m+1) and is the fast path only well below kappa = 1.
constexpr double kStiffKappa = 0.5;

// max |u0|^2 of a newly set state, on the device (one read of u0 + 8 B back).
// Refreshed lazily when a state is set, not per step: the amplitude of a
// Hamiltonian run drifts slowly and the policy falls back to Newton-Krylov on any
// sweep failure, so the estimate only steers the choice of the fast path.
int refresh_amax2(mb4cu_ctx* ctx) {
    if (ctx->amax2_valid) return MB4CU_OK;
    const size_t off = static_cast<size_t>(ctx->ghost) * ctx->pitch + ctx->ghost;  // owned sites only
    MB4_CUDA(ctx, mb4cu::launch_amax2_2d(ctx->u0 + off, ctx->nx, ctx->ny, ctx->pitch, ctx->d_rmax, ctx->stream));
    ctx->prof.other_launches += 1;
    MB4_CUDA(ctx, cudaMemcpyAsync(ctx->h_rmax, ctx->d_rmax, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                  ctx->stream));
    MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    ctx->amax2 = decode_bits(*ctx->h_rmax);
    ctx->amax2_valid = true;
    return MB4CU_OK;
}

bool stiff_step(const mb4cu_ctx* ctx, double h) {
    const double lam = std::max({std::fabs(ctx->scheme.lam[0]), std::fabs(ctx->scheme.lam[1]),
                                 std::fabs(ctx->scheme.lam[2])});
    return h * lam * spectral_bound(ctx) > kStiffKappa;
}

// ---- Newton-Krylov stage solver (kernel = 3) --------------------------------
// The reference's simplified Newton iteration (mb4_integrator.cpp:194-255) with
// matrix-free GMRES(m) stage solves (restating iterative.cpp:68-153 without the
// ILU(0) preconditioner); O(N) work on the device, Hessenberg on the host.

constexpr int kKrylovRestart = 30;  // the Fourier-preconditioned solves converge in < 10 iterations
constexpr int kKrylovMaxIters = 2000;
constexpr double kKrylovTol = 1e-13;

void kr_free(mb4cu_ctx* ctx) {
    auto& k = ctx->kr;
    cudaFree(k.mem);
    cudaFree(k.v_dev);
    cudaFree(k.partial);
    cudaFreeHost(k.h_partial);
    cudaFree(k.coef);
    cudaFreeHost(k.h_coef);
    cudaFree(k.hcol);
    cudaFreeHost(k.h_hcol);
    k.hcol = nullptr;
    k.h_hcol = nullptr;
    k.mem = nullptr;
    k.v_dev = nullptr;
    k.partial = nullptr;
    k.h_partial = nullptr;
    k.coef = nullptr;
    k.h_coef = nullptr;
    k.len = 0;
}

// Krylov arena for vectors of len complex entries: basis (m+1), then 8 work
// vectors (b, x, ... of the callers; w, y of kr_gmres).
int kr_alloc(mb4cu_ctx* ctx, size_t len) {
    auto& k = ctx->kr;
    if (k.mem && k.len == len) return MB4CU_OK;
    if (k.mem) {
        MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        kr_free(ctx);
    }
    k.m = kKrylovRestart;
    k.len = len;
    k.nblk = mb4cu::krylov_blocks(len);
    const size_t nvec = static_cast<size_t>(k.m + 1) + 3 + 3 + 2 + 1;  // + preconditioner scratch
    MB4_CUDA(ctx, cudaMalloc(&k.mem, nvec * len * sizeof(double2)));
    MB4_CUDA(ctx, cudaMalloc(&k.v_dev, sizeof(double2*) * (k.m + 1)));
    std::vector<double2*> ptrs(k.m + 1);
    for (int i = 0; i <= k.m; ++i) ptrs[i] = k.mem + static_cast<size_t>(i) * len;
    // on the context stream (a legacy-stream copy does not order against it)
    MB4_CUDA(ctx, cudaMemcpyAsync(k.v_dev, ptrs.data(), sizeof(double2*) * (k.m + 1), cudaMemcpyHostToDevice,
                                  ctx->stream));
    MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    MB4_CUDA(ctx, cudaMalloc(&k.partial, sizeof(double) * (k.m + 1) * k.nblk));
    MB4_CUDA(ctx, cudaMallocHost(&k.h_partial, sizeof(double) * (k.m + 1) * k.nblk));
    MB4_CUDA(ctx, cudaMalloc(&k.coef, sizeof(double) * (k.m + 1)));
    MB4_CUDA(ctx, cudaMallocHost(&k.h_coef, sizeof(double) * (k.m + 1)));
    MB4_CUDA(ctx, cudaMalloc(&k.hcol, sizeof(double) * (k.m + 2)));
    MB4_CUDA(ctx, cudaMallocHost(&k.h_hcol, sizeof(double) * (k.m + 2)));
    return MB4CU_OK;
}

double2* kr_vec(mb4cu_ctx* ctx, size_t idx) { return ctx->kr.mem + idx * ctx->kr.len; }

// fixed-order host sum of nv rows of block partials
int kr_fetch(mb4cu_ctx* ctx, int nv, double* out) {
    auto& k = ctx->kr;
    MB4_CUDA(ctx, cudaMemcpyAsync(k.h_partial, k.partial, sizeof(double) * nv * k.nblk, cudaMemcpyDeviceToHost,
                                  ctx->stream));
    MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < nv; ++i) {
        double s = 0.0;
        for (int b = 0; b < k.nblk; ++b) s += k.h_partial[static_cast<size_t>(i) * k.nblk + b];
        out[i] = s;
    }
    return MB4CU_OK;
}

// Solve A x = b by restarted GMRES(m), x initialised to zero; A applied by
// matvec(x, y) over vectors of the arena length (N, or 2N for coupled systems).
template <class MatVec>
int kr_gmres(mb4cu_ctx* ctx, const MatVec& matvec, const double2* b, double2* x) {
    auto& k = ctx->kr;
    const size_t n = k.len;
    const int m = k.m;
    double2* w = kr_vec(ctx, m + 1 + 6);
    double2* y = kr_vec(ctx, m + 1 + 7);
    std::vector<double> H(static_cast<size_t>(m + 1) * m, 0.0), cs(m, 0.0), sn(m, 0.0), g(m + 1, 0.0),
        yv(m, 0.0), tmp(m + 1, 0.0);
    auto Hat = [&](int i, int j) -> double& { return H[static_cast<size_t>(i) * m + j]; };
    MB4_CUDA(ctx, cudaMemsetAsync(x, 0, n * sizeof(double2), ctx->stream));
    // v_0 <- b and ||b||^2 (residual of x = 0)
    MB4_CUDA(ctx, cudaMemsetAsync(y, 0, n * sizeof(double2), ctx->stream));
    MB4_CUDA(ctx, mb4cu::kr_residual(b, y, kr_vec(ctx, 0), n, k.partial, ctx->stream));
    double bn2 = 0.0;
    if (int rc = kr_fetch(ctx, 1, &bn2)) return rc;
    const double bnorm = std::sqrt(bn2);
    if (bnorm == 0.0) return MB4CU_OK;
    if (!std::isfinite(bnorm)) return fail(ctx, MB4CU_NONCONVERGED, "gmres: non-finite right-hand side");
    bool first = true;
    for (int iter = 0; iter < kKrylovMaxIters;) {
        double beta;
        if (first) {
            beta = bnorm;  // r = b already in v_0 (unscaled)
            first = false;
        } else {
            MB4_CUDA(ctx, matvec(x, y));
            MB4_CUDA(ctx, mb4cu::kr_residual(b, y, kr_vec(ctx, 0), n, k.partial, ctx->stream));
            double r2 = 0.0;
            if (int rc = kr_fetch(ctx, 1, &r2)) return rc;
            beta = std::sqrt(r2);
        }
        if (beta / bnorm <= kKrylovTol) return MB4CU_OK;
        MB4_CUDA(ctx, mb4cu::kr_scale(kr_vec(ctx, 0), kr_vec(ctx, 0), 1.0 / beta, n, ctx->stream));
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = beta;
        int j = 0;
        bool done = false;
        for (; j < m && iter < kKrylovMaxIters; ++j, ++iter) {
            MB4_CUDA(ctx, matvec(kr_vec(ctx, j), w));
            // classical Gram-Schmidt twice + normalisation, one cooperative launch
            MB4_CUDA(ctx, mb4cu::kr_arnoldi(w, k.v_dev, j, n, k.partial, k.coef, k.hcol, ctx->stream));
            MB4_CUDA(ctx, cudaMemcpyAsync(k.h_hcol, k.hcol, sizeof(double) * (j + 2), cudaMemcpyDeviceToHost,
                                          ctx->stream));
            MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
            for (int i = 0; i <= j; ++i) Hat(i, j) = k.h_hcol[i];
            const double hn = k.h_hcol[j + 1];
            Hat(j + 1, j) = hn;
            for (int i = 0; i < j; ++i) {
                const double t = cs[i] * Hat(i, j) + sn[i] * Hat(i + 1, j);
                Hat(i + 1, j) = -sn[i] * Hat(i, j) + cs[i] * Hat(i + 1, j);
                Hat(i, j) = t;
            }
            const double den = std::hypot(Hat(j, j), Hat(j + 1, j));
            if (den == 0.0) return fail(ctx, MB4CU_NONCONVERGED, "gmres: breakdown");
            cs[j] = Hat(j, j) / den;
            sn[j] = Hat(j + 1, j) / den;
            Hat(j, j) = den;
            Hat(j + 1, j) = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            if (std::fabs(g[j + 1]) / bnorm <= kKrylovTol || hn == 0.0) {
                ++j;
                ++iter;
                done = true;
                break;
            }
        }
        k.gmres_iters += j;
        ctx->prof.krylov_iters += j;
        for (int i = j - 1; i >= 0; --i) {
            double s = g[i];
            for (int q = i + 1; q < j; ++q) s -= Hat(i, q) * yv[q];
            yv[i] = s / Hat(i, i);
        }
        for (int i = 0; i < j; ++i) k.h_coef[i] = yv[i];
        MB4_CUDA(ctx, cudaMemcpyAsync(k.coef, k.h_coef, sizeof(double) * j, cudaMemcpyHostToDevice, ctx->stream));
        MB4_CUDA(ctx, mb4cu::kr_combine(x, k.v_dev, k.coef, j, n, ctx->stream));
        if (done) return MB4CU_OK;
    }
    return MB4CU_OK;  // best effort after the iteration cap, as the reference (iterative.cpp:152)
}

// ---- Fourier preconditioner (fft_precond.cu) ---------------------------------

int fft_fail(mb4cu_ctx* ctx, cufftResult r, const char* where) {
    return fail(ctx, MB4CU_CUDA_ERROR, std::string("cufft ") + where + ": error " + std::to_string(static_cast<int>(r)));
}

// plans (on first use) and the diagonal shift of the current u0
int fft_prepare(mb4cu_ctx* ctx, int stages) {
    auto& f = ctx->fft;
    cufftResult r;
    if (stages == 1 && !f.have1) {
        if ((r = cufftPlan2d(&f.plan1, ctx->ny, ctx->nx, CUFFT_Z2Z)) != CUFFT_SUCCESS) return fft_fail(ctx, r, "plan");
        f.have1 = true;
    }
    if (stages == 2 && !f.have2) {
        int dims[2] = {ctx->ny, ctx->nx};
        if ((r = cufftPlanMany(&f.plan2, 2, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2Z, 2)) != CUFFT_SUCCESS)
            return fft_fail(ctx, r, "plan");
        f.have2 = true;
    }
    const int nb = mb4cu::fft_shift_blocks(ctx->n);
    if (!f.partial) {
        MB4_CUDA(ctx, cudaMalloc(&f.partial, sizeof(double) * 2 * nb));
        MB4_CUDA(ctx, cudaMallocHost(&f.h_partial, sizeof(double) * 2 * nb));
    }
    MB4_CUDA(ctx, mb4cu::launch_fft_shift_partials(ctx->u0, ctx->V, ctx->n, f.partial, ctx->stream));
    MB4_CUDA(ctx, cudaMemcpyAsync(f.h_partial, f.partial, sizeof(double) * 2 * nb, cudaMemcpyDeviceToHost,
                                  ctx->stream));
    MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    double sv = 0.0, su = 0.0;
    for (int b = 0; b < nb; ++b) {
        sv += f.h_partial[2 * b];
        su += f.h_partial[2 * b + 1];
    }
    const double n = static_cast<double>(ctx->n);
    f.shift = sv / n - 2.0 * ctx->gamma * (su / n);
    if (!f.shift_dev) {
        MB4_CUDA(ctx, cudaMalloc(&f.shift_dev, sizeof(double)));
        MB4_CUDA(ctx, cudaMallocHost(&f.h_shift, sizeof(double)));
    }
    *f.h_shift = f.shift;
    MB4_CUDA(ctx, cudaMemcpyAsync(f.shift_dev, f.h_shift, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));  // the pinned staging is reused
    return MB4CU_OK;
}

// y <- P^-1 y in place (len = stages * N).  stages 1: P = I + i sigma (K + shift);
// stages 2: P = I + i h C (x) (K + shift).
int fft_apply(mb4cu_ctx* ctx, int stages, double sigma_or_h, const double C[2][2], double2* y) {
    auto& f = ctx->fft;
    const cufftHandle plan = stages == 1 ? f.plan1 : f.plan2;
    cufftResult r;
    if ((r = cufftSetStream(plan, ctx->stream)) != CUFFT_SUCCESS) return fft_fail(ctx, r, "stream");
    auto* z = reinterpret_cast<cufftDoubleComplex*>(y);
    if ((r = cufftExecZ2Z(plan, z, z, CUFFT_FORWARD)) != CUFFT_SUCCESS) return fft_fail(ctx, r, "forward");
    if (stages == 1)
        MB4_CUDA(ctx, mb4cu::launch_fft_scale1(y, ctx->nx, ctx->ny, ctx->cx, ctx->cy, f.shift, sigma_or_h, ctx->stream));
    else
        MB4_CUDA(ctx, mb4cu::launch_fft_scale2(y, y + ctx->n, ctx->nx, ctx->ny, ctx->cx, ctx->cy, f.shift, sigma_or_h,
                                               C, ctx->stream));
    if ((r = cufftExecZ2Z(plan, z, z, CUFFT_INVERSE)) != CUFFT_SUCCESS) return fft_fail(ctx, r, "inverse");
    ctx->prof.other_launches += 3;
    return MB4CU_OK;
}

// Right-preconditioned GMRES: solve (A P^-1) x' = b, x = P^-1 x'; A applied by
// amul(x, y) over len = stages * N.
template <class AMul>
int kr_gmres_fft(mb4cu_ctx* ctx, int stages, double sigma_or_h, const double C[2][2], const AMul& amul,
                 const double2* b, double2* x) {
    const size_t len = ctx->kr.len;
    double2* tmp = kr_vec(ctx, ctx->kr.m + 9);
    int prc = MB4CU_OK;
    auto mv = [&](const double2* xin, double2* yout) -> cudaError_t {
        cudaError_t e = cudaMemcpyAsync(tmp, xin, len * sizeof(double2), cudaMemcpyDeviceToDevice, ctx->stream);
        if (e != cudaSuccess) return e;
        if ((prc = fft_apply(ctx, stages, sigma_or_h, C, tmp)) != MB4CU_OK) return cudaErrorUnknown;
        return amul(tmp, yout);
    };
    if (int rc = kr_gmres(ctx, mv, b, x)) return prc ? prc : rc;
    if (prc) return prc;
    return fft_apply(ctx, stages, sigma_or_h, C, x);
}

constexpr size_t kKrBatchBytes = size_t(1) << 31;

void krb_free(mb4cu_ctx* ctx) {
    auto& B = ctx->krb;
    for (int q = 0; q < 3; ++q) {
        cudaFree(B.v_dev[q]);
        cudaFree(B.partial[q]);
        cudaFreeHost(B.h_partial[q]);
        cudaFree(B.coef[q]);
        cudaFreeHost(B.h_coef[q]);
        cudaFree(B.hcol[q]);
        cudaFreeHost(B.h_hcol[q]);
        if (B.st[q]) cudaStreamDestroy(B.st[q]);
        if (B.plan[q]) cufftDestroy(B.plan[q]);
        B.v_dev[q] = nullptr;
        B.partial[q] = B.h_partial[q] = B.coef[q] = B.h_coef[q] = B.hcol[q] = B.h_hcol[q] = nullptr;
        B.st[q] = nullptr;
        B.plan[q] = 0;
    }
    for (auto& e : B.ev) {
        if (e) cudaEventDestroy(e);
        e = nullptr;
    }
    for (auto& sl : B.slot) {
        for (auto& g : sl.g) {
            if (g) cudaGraphExecDestroy(g);
            g = nullptr;
        }
        sl.u0 = nullptr;
    }
    cudaFree(B.jd);
    B.jd = nullptr;
    cudaFree(B.mem);
    B.mem = nullptr;
    B.ready = false;
    B.len = 0;
}

// 1 if the batched stage solves are set up for vectors of len entries
int krb_alloc(mb4cu_ctx* ctx, size_t len) {
    auto& B = ctx->krb;
    if (B.ready && B.len == len) return 1;
    const int m = kKrylovRestart;
    const size_t per = static_cast<size_t>(m + 4);
    // concurrent cooperative Arnoldi launches must fit the device together
    const int cap = mb4cu::arnoldi_capacity();
    if (3 * per * len * sizeof(double2) > kKrBatchBytes || 3 * mb4cu::krylov_blocks(len) > cap) return 0;
    if (B.mem) {
        if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return 0;
        krb_free(ctx);
    }
    B.m = m;
    B.len = len;
    B.nblk = mb4cu::krylov_blocks(len);
    bool ok = cudaMalloc(&B.mem, 3 * per * len * sizeof(double2)) == cudaSuccess;
    for (int q = 0; q < 3 && ok; ++q) {
        ok = cudaStreamCreateWithFlags(&B.st[q], cudaStreamNonBlocking) == cudaSuccess &&
             cudaMalloc(&B.v_dev[q], sizeof(double2*) * (m + 1)) == cudaSuccess &&
             cudaMalloc(&B.partial[q], sizeof(double) * (m + 1) * B.nblk) == cudaSuccess &&
             cudaMallocHost(&B.h_partial[q], sizeof(double) * (m + 1) * B.nblk) == cudaSuccess &&
             cudaMalloc(&B.coef[q], sizeof(double) * (m + 1)) == cudaSuccess &&
             cudaMallocHost(&B.h_coef[q], sizeof(double) * (m + 1)) == cudaSuccess &&
             cudaMalloc(&B.hcol[q], sizeof(double) * (m + 2)) == cudaSuccess &&
             cudaMallocHost(&B.h_hcol[q], sizeof(double) * (m + 2)) == cudaSuccess &&
             cufftPlan2d(&B.plan[q], ctx->ny, ctx->nx, CUFFT_Z2Z) == CUFFT_SUCCESS &&
             cufftSetStream(B.plan[q], B.st[q]) == CUFFT_SUCCESS;
        if (ok) {
            std::vector<double2*> ptrs(m + 1);
            for (int i = 0; i <= m; ++i) ptrs[i] = B.mem + (q * per + i) * len;
            ok = cudaMemcpy(B.v_dev[q], ptrs.data(), sizeof(double2*) * (m + 1), cudaMemcpyHostToDevice) ==
                 cudaSuccess;
        }
    }
    for (auto& e : B.ev) ok = ok && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaMalloc(&B.jd, 3 * sizeof(int)) == cudaSuccess;
    if (!ok) {
        krb_free(ctx);
        cudaGetLastError();
        return 0;
    }
    B.ready = true;
    return 1;
}

// The three stage systems (I - h lam_k J) x_k = b_k of one Newton iteration, solved
// together: the same right-preconditioned restarted GMRES(m) as kr_gmres_fft per
// system (identical arithmetic: the same kernels, host Givens updates and stopping
// tests), advanced in lockstep, system q on its own stream, so one host round trip
// per Arnoldi step serves all three and their small kernels run concurrently.
int kr_gmres_stages_impl(mb4cu_ctx* ctx, const SweepConsts& c, const double2* const b[3], double2* const x[3]);

int kr_gmres_stages(mb4cu_ctx* ctx, const SweepConsts& c, const double2* const b[3], double2* const x[3]) {
    const int rc = kr_gmres_stages_impl(ctx, c, b, x);
    if (rc != MB4CU_OK)  // no stage-stream work may outlive a failed solve (the buffers are reused)
        for (int q = 0; q < 3; ++q) cudaStreamSynchronize(ctx->krb.st[q]);
    return rc;
}

int kr_gmres_stages_impl(mb4cu_ctx* ctx, const SweepConsts& c, const double2* const b[3], double2* const x[3]) {
    auto& B = ctx->krb;
    const size_t n = B.len;
    const int m = B.m;
    const size_t per = static_cast<size_t>(m + 4);
    auto V = [&](int q, int i) { return B.mem + (q * per + i) * n; };
    auto W = [&](int q) { return V(q, m + 1); };
    auto Y = [&](int q) { return V(q, m + 2); };
    auto T = [&](int q) { return V(q, m + 3); };
    auto& f = ctx->fft;
    // y = A P^-1 v for system q
    auto mv = [&](int q, const double2* in, double2* out) -> int {
        MB4_CUDA(ctx, cudaMemcpyAsync(T(q), in, n * sizeof(double2), cudaMemcpyDeviceToDevice, B.st[q]));
        auto* z = reinterpret_cast<cufftDoubleComplex*>(T(q));
        if (cufftExecZ2Z(B.plan[q], z, z, CUFFT_FORWARD) != CUFFT_SUCCESS) return fail(ctx, MB4CU_CUDA_ERROR, "cufft");
        MB4_CUDA(ctx, mb4cu::launch_fft_scale1(T(q), ctx->nx, ctx->ny, ctx->cx, ctx->cy, f.shift, c.hlam[q], B.st[q]));
        if (cufftExecZ2Z(B.plan[q], z, z, CUFFT_INVERSE) != CUFFT_SUCCESS) return fail(ctx, MB4CU_CUDA_ERROR, "cufft");
        MB4_CUDA(ctx, mb4cu::kr_matvec(T(q), out, ctx->u0, ctx->V, ctx->nx, ctx->ny, c.hlam[q], c, B.st[q]));
        ctx->prof.other_launches += 3;
        return MB4CU_OK;
    };
    // one Arnoldi step of system q on its stream (the body of the captured graph)
    auto arnoldi_step = [&](int q) -> int {
        MB4_CUDA(ctx, mb4cu::kr_gather_basis(T(q), B.v_dev[q], B.jd + q, n, B.st[q]));
        auto* z = reinterpret_cast<cufftDoubleComplex*>(T(q));
        if (cufftExecZ2Z(B.plan[q], z, z, CUFFT_FORWARD) != CUFFT_SUCCESS) return fail(ctx, MB4CU_CUDA_ERROR, "cufft");
        MB4_CUDA(ctx, mb4cu::launch_fft_scale1(T(q), ctx->nx, ctx->ny, ctx->cx, ctx->cy, f.shift, c.hlam[q], B.st[q],
                                               f.shift_dev));
        if (cufftExecZ2Z(B.plan[q], z, z, CUFFT_INVERSE) != CUFFT_SUCCESS) return fail(ctx, MB4CU_CUDA_ERROR, "cufft");
        MB4_CUDA(ctx, mb4cu::kr_matvec(T(q), W(q), ctx->u0, ctx->V, ctx->nx, ctx->ny, c.hlam[q], c, B.st[q]));
        MB4_CUDA(ctx, mb4cu::kr_arnoldi(W(q), B.v_dev[q], 0, n, B.partial[q], B.coef[q], B.hcol[q], B.st[q],
                                        B.jd + q));
        MB4_CUDA(ctx, cudaMemcpyAsync(B.h_hcol[q], B.hcol[q], sizeof(double) * (m + 2), cudaMemcpyDeviceToHost,
                                      B.st[q]));
        return MB4CU_OK;
    };
    // the three step graphs for this (u0, h): cached in two slots (the commit alternates u0
    // between two buffers; the preconditioner shift is read from device memory)
    cudaGraphExec_t* gx = nullptr;
    if (B.use_graphs) {
        for (auto& sl : B.slot)
            if (sl.u0 == ctx->u0 && sl.h == c.h && sl.g[0]) gx = sl.g;
        if (!gx) {
            auto& sl = B.slot[B.next_slot];
            B.next_slot ^= 1;
            for (auto& g : sl.g) {
                if (g) cudaGraphExecDestroy(g);
                g = nullptr;
            }
            sl.u0 = nullptr;
            bool ok = true;
            for (int q = 0; q < 3 && ok; ++q) {
                cudaGraph_t graph = nullptr;
                ok = cudaStreamBeginCapture(B.st[q], cudaStreamCaptureModeThreadLocal) == cudaSuccess;
                const int rc = ok ? arnoldi_step(q) : MB4CU_CUDA_ERROR;
                ok = cudaStreamEndCapture(B.st[q], &graph) == cudaSuccess && ok && rc == MB4CU_OK;
                ok = ok && cudaGraphInstantiate(&sl.g[q], graph, 0) == cudaSuccess;
                if (graph) cudaGraphDestroy(graph);
            }
            if (ok) {
                sl.u0 = ctx->u0;
                sl.h = c.h;
                gx = sl.g;
            } else {  // capture unsupported here: launch the steps one by one
                cudaGetLastError();
                for (auto& g : sl.g) {
                    if (g) cudaGraphExecDestroy(g);
                    g = nullptr;
                }
                B.use_graphs = false;
            }
        }
    }
    auto fetch_sum = [&](int q, int nv, double* out) {
        for (int i = 0; i < nv; ++i) {
            double sum = 0.0;
            for (int blk = 0; blk < B.nblk; ++blk) sum += B.h_partial[q][static_cast<size_t>(i) * B.nblk + blk];
            out[i] = sum;
        }
    };
    auto sync_all = [&](const bool* which) -> int {
        for (int q = 0; q < 3; ++q)
            if (which[q]) MB4_CUDA(ctx, cudaStreamSynchronize(B.st[q]));
        return MB4CU_OK;
    };
    // the stage streams start after the right-hand sides (context stream)
    MB4_CUDA(ctx, cudaEventRecord(B.ev[3], ctx->stream));
    for (int q = 0; q < 3; ++q) MB4_CUDA(ctx, cudaStreamWaitEvent(B.st[q], B.ev[3], 0));

    std::vector<double> H[3], cs[3], sn[3], g[3], yv[3];
    double bnorm[3] = {0, 0, 0}, beta[3] = {0, 0, 0};
    bool active[3] = {true, true, true}, first[3] = {true, true, true}, inner[3] = {false, false, false};
    int j[3] = {0, 0, 0}, iters[3] = {0, 0, 0};
    for (int q = 0; q < 3; ++q) {
        H[q].assign(static_cast<size_t>(m + 1) * m, 0.0);
        cs[q].assign(m, 0.0);
        sn[q].assign(m, 0.0);
        g[q].assign(m + 1, 0.0);
        yv[q].assign(m, 0.0);
        MB4_CUDA(ctx, cudaMemsetAsync(x[q], 0, n * sizeof(double2), B.st[q]));
        MB4_CUDA(ctx, cudaMemsetAsync(Y(q), 0, n * sizeof(double2), B.st[q]));
        MB4_CUDA(ctx, mb4cu::kr_residual(b[q], Y(q), V(q, 0), n, B.partial[q], B.st[q]));
        MB4_CUDA(ctx, cudaMemcpyAsync(B.h_partial[q], B.partial[q], sizeof(double) * B.nblk, cudaMemcpyDeviceToHost,
                                      B.st[q]));
    }
    if (int rc = sync_all(active)) return rc;
    for (int q = 0; q < 3; ++q) {
        double b2 = 0.0;
        fetch_sum(q, 1, &b2);
        bnorm[q] = std::sqrt(b2);
        if (bnorm[q] == 0.0) active[q] = false;
        if (!std::isfinite(bnorm[q])) return fail(ctx, MB4CU_NONCONVERGED, "gmres: non-finite right-hand side");
    }
    auto Hat = [&](int q, int i, int jj) -> double& { return H[q][static_cast<size_t>(i) * m + jj]; };
    for (;;) {
        bool any = false, need[3] = {false, false, false};
        // restart: residual of the current x (not for the first cycle: r = b is in v_0)
        for (int q = 0; q < 3; ++q) {
            if (!active[q]) continue;
            any = true;
            if (first[q]) continue;
            if (iters[q] >= kKrylovMaxIters) {  // best effort after the cap (iterative.cpp:152)
                active[q] = false;
                continue;
            }
            need[q] = true;
            if (int rc = mv(q, x[q], Y(q))) return rc;
            MB4_CUDA(ctx, mb4cu::kr_residual(b[q], Y(q), V(q, 0), n, B.partial[q], B.st[q]));
            MB4_CUDA(ctx, cudaMemcpyAsync(B.h_partial[q], B.partial[q], sizeof(double) * B.nblk,
                                          cudaMemcpyDeviceToHost, B.st[q]));
        }
        if (!any) break;
        if (int rc = sync_all(need)) return rc;
        for (int q = 0; q < 3; ++q) {
            if (!active[q]) continue;
            if (first[q]) {
                beta[q] = bnorm[q];
                first[q] = false;
            } else {
                double r2 = 0.0;
                fetch_sum(q, 1, &r2);
                beta[q] = std::sqrt(r2);
            }
            if (beta[q] / bnorm[q] <= kKrylovTol) {
                active[q] = false;
                continue;
            }
            MB4_CUDA(ctx, mb4cu::kr_scale(V(q, 0), V(q, 0), 1.0 / beta[q], n, B.st[q]));
            MB4_CUDA(ctx, cudaMemsetAsync(B.jd + q, 0, sizeof(int), B.st[q]));  // step index of the cycle
            std::fill(g[q].begin(), g[q].end(), 0.0);
            g[q][0] = beta[q];
            j[q] = 0;
            inner[q] = true;
        }
        // Arnoldi steps of all systems in the inner cycle, one host round trip each
        for (;;) {
            bool step[3] = {false, false, false}, anyin = false;
            for (int q = 0; q < 3; ++q) {
                if (!inner[q]) continue;
                anyin = step[q] = true;
                if (gx) {
                    MB4_CUDA(ctx, cudaGraphLaunch(gx[q], B.st[q]));
                    ctx->prof.other_launches += 6;
                } else if (int rc = arnoldi_step(q)) {
                    return rc;
                }
            }
            if (!anyin) break;
            if (int rc = sync_all(step)) return rc;
            for (int q = 0; q < 3; ++q) {
                if (!step[q]) continue;
                const int jj = j[q];
                for (int i = 0; i <= jj; ++i) Hat(q, i, jj) = B.h_hcol[q][i];
                const double hn = B.h_hcol[q][jj + 1];
                Hat(q, jj + 1, jj) = hn;
                for (int i = 0; i < jj; ++i) {
                    const double t = cs[q][i] * Hat(q, i, jj) + sn[q][i] * Hat(q, i + 1, jj);
                    Hat(q, i + 1, jj) = -sn[q][i] * Hat(q, i, jj) + cs[q][i] * Hat(q, i + 1, jj);
                    Hat(q, i, jj) = t;
                }
                const double den = std::hypot(Hat(q, jj, jj), Hat(q, jj + 1, jj));
                if (den == 0.0) return fail(ctx, MB4CU_NONCONVERGED, "gmres: breakdown");
                cs[q][jj] = Hat(q, jj, jj) / den;
                sn[q][jj] = Hat(q, jj + 1, jj) / den;
                Hat(q, jj, jj) = den;
                Hat(q, jj + 1, jj) = 0.0;
                g[q][jj + 1] = -sn[q][jj] * g[q][jj];
                g[q][jj] = cs[q][jj] * g[q][jj];
                ++iters[q];
                j[q] = jj + 1;
                const bool conv = std::fabs(g[q][jj + 1]) / bnorm[q] <= kKrylovTol || hn == 0.0;
                if (conv || j[q] == m || iters[q] >= kKrylovMaxIters) {
                    inner[q] = false;
                    const int nj = j[q];
                    ctx->kr.gmres_iters += nj;
                    ctx->prof.krylov_iters += nj;
                    for (int i = nj - 1; i >= 0; --i) {
                        double sum = g[q][i];
                        for (int k2 = i + 1; k2 < nj; ++k2) sum -= Hat(q, i, k2) * yv[q][k2];
                        yv[q][i] = sum / Hat(q, i, i);
                    }
                    for (int i = 0; i < nj; ++i) B.h_coef[q][i] = yv[q][i];
                    MB4_CUDA(ctx, cudaMemcpyAsync(B.coef[q], B.h_coef[q], sizeof(double) * nj, cudaMemcpyHostToDevice,
                                                  B.st[q]));
                    MB4_CUDA(ctx, mb4cu::kr_combine(x[q], B.v_dev[q], B.coef[q], nj, n, B.st[q]));
                    if (conv) active[q] = false;
                }
            }
        }
    }
    // x = P^-1 x' (right preconditioning), then join the context stream
    for (int q = 0; q < 3; ++q) {
        auto* z = reinterpret_cast<cufftDoubleComplex*>(x[q]);
        if (cufftExecZ2Z(B.plan[q], z, z, CUFFT_FORWARD) != CUFFT_SUCCESS) return fail(ctx, MB4CU_CUDA_ERROR, "cufft");
        MB4_CUDA(ctx, mb4cu::launch_fft_scale1(x[q], ctx->nx, ctx->ny, ctx->cx, ctx->cy, f.shift, c.hlam[q], B.st[q]));
        if (cufftExecZ2Z(B.plan[q], z, z, CUFFT_INVERSE) != CUFFT_SUCCESS) return fail(ctx, MB4CU_CUDA_ERROR, "cufft");
        MB4_CUDA(ctx, cudaEventRecord(B.ev[q], B.st[q]));
        MB4_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, B.ev[q], 0));
    }
    return MB4CU_OK;
}

int substep_krylov(mb4cu_ctx* ctx, double h, int* iters, double* last_res) {
    if (int rc = kr_alloc(ctx, ctx->n)) return rc;
    const SweepConsts c = make_consts(ctx, h);
    const size_t sb = ctx->n * sizeof(double2);
    double2* st[3] = {ctx->U[0][0], ctx->U[0][1], ctx->U[0][2]};
    for (int i = 0; i < 3; ++i)
        MB4_CUDA(ctx, cudaMemcpyAsync(st[i], ctx->u0, sb, cudaMemcpyDeviceToDevice, ctx->stream));
    const int m = ctx->kr.m;
    // vectors 0..m: Krylov basis; m+1..m+3: b; m+4..m+6: x; m+7, m+8: work (kr_gmres)
    double2* b[3] = {kr_vec(ctx, m + 1), kr_vec(ctx, m + 2), kr_vec(ctx, m + 3)};
    double2* x[3] = {kr_vec(ctx, m + 4), kr_vec(ctx, m + 5), kr_vec(ctx, m + 6)};
    *iters = 0;
    if (int rc = fft_prepare(ctx, 1)) return rc;
    // the three stage solves in flight together while their Krylov storage is small
    const bool batch = ctx->kr_batch && krb_alloc(ctx, ctx->n) == 1;
    for (int it = 1; it <= ctx->max_iters; ++it) {
        const double2* cst[3] = {st[0], st[1], st[2]};
        MB4_CUDA(ctx, mb4cu::kr_phibar(ctx->nx, ctx->ny, ctx->u0, cst, ctx->V, b, c, ctx->stream));
        if (batch) {
            if (int rc = kr_gmres_stages(ctx, c, b, x)) return rc;
        } else {
            for (int k = 0; k < 3; ++k) {
                const double hl = c.hlam[k];
                auto mv = [&](const double2* xin, double2* yout) {
                    return mb4cu::kr_matvec(xin, yout, ctx->u0, ctx->V, ctx->nx, ctx->ny, hl, c, ctx->stream);
                };
                if (int rc = kr_gmres_fft(ctx, 1, hl, nullptr, mv, b[k], x[k])) return rc;
            }
        }
        MB4_CUDA(ctx, cudaMemsetAsync(ctx->d_rmax, 0, sizeof(unsigned long long), ctx->stream));
        const double2* cx[3] = {x[0], x[1], x[2]};
        MB4_CUDA(ctx, mb4cu::kr_update(st, cx, ctx->n, ctx->d_rmax, c, ctx->stream));
        MB4_CUDA(ctx, cudaMemcpyAsync(ctx->h_rmax, ctx->d_rmax, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                      ctx->stream));
        MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        *iters = it;
        const double r = decode_bits(*ctx->h_rmax);
        *last_res = r;
        if (!std::isfinite(r)) {
            *last_res = INFINITY;
            return fail(ctx, MB4CU_NONCONVERGED, "newton_solve: iteration diverged (non-finite update)");
        }
        if (r <= ctx->eps) {  // the reference test (:250); Newton's remaining error is << eps
            std::swap(ctx->u0, ctx->U[0][2]);
            return MB4CU_OK;
        }
    }
    return fail(ctx, MB4CU_NONCONVERGED,
                "newton_solve: no convergence after " + std::to_string(ctx->max_iters) + " iterations");
}

// One MB4 sub-step of size h on ctx->u0: sweeps until ||r||_inf <= eps
// (newton_solve, mb4_integrator.cpp:194-255).  On success u0 <- U3 (c3 = 1).
int substep(mb4cu_ctx* ctx, double h, int* sweeps, double* last_res) {
    if (ctx->kernel == 3) return substep_krylov(ctx, h, sweeps, last_res);
    if (ctx->kernel == 0) {
        // default policy: matrix-free sweeps unless the step is stiff; a sweep
        // iteration that fails falls back to Newton-Krylov at the same step size
        // (the reference would not halve there), then the halving policy applies.
        if (stiff_step(ctx, h)) {
            const int rck = substep_krylov(ctx, h, sweeps, last_res);
            if (rck == MB4CU_OK) ctx->amax2_valid = false;  // no sweep measured the new state
            return rck;
        }
        int sw = 0;
        const int rc = substep_march(ctx, h, &sw, last_res);
        if (rc != MB4CU_NONCONVERGED) {
            *sweeps = sw;
            return rc;
        }
        int it = 0;
        const int rc2 = substep_krylov(ctx, h, &it, last_res);
        if (rc2 == MB4CU_OK) ctx->amax2_valid = false;
        *sweeps = sw + it;
        return rc2;
    }
    if (ctx->kernel != 1) return substep_march(ctx, h, sweeps, last_res);
    const SweepConsts c = make_consts(ctx, h);
    int cur = -1;
    *sweeps = 0;
    for (int it = 1; it <= ctx->max_iters; ++it) {
        const int nxt = cur < 0 ? 0 : 1 - cur;
        SweepArgs a{};
        a.nx = ctx->nx;
        a.ny = ctx->ny;
        a.u0 = ctx->u0;
        a.V = ctx->V;
        for (int i = 0; i < 3; ++i) {
            a.uin[i] = cur < 0 ? ctx->u0 : ctx->U[cur][i];
            a.uout[i] = ctx->U[nxt][i];
        }
        a.rmax = ctx->d_rmax;
        MB4_CUDA(ctx, cudaMemsetAsync(ctx->d_rmax, 0, sizeof(unsigned long long), ctx->stream));
        if (ctx->profiling) MB4_CUDA(ctx, cudaEventRecord(ctx->pev0, ctx->stream));
        MB4_CUDA(ctx, mb4cu::launch_sweep_tiled(cur < 0 ? ctx->mf : ctx->m, cur < 0, a, c, ctx->stream));
        if (ctx->profiling) MB4_CUDA(ctx, cudaEventRecord(ctx->pev1, ctx->stream));
        MB4_CUDA(ctx, cudaMemcpyAsync(ctx->h_rmax, ctx->d_rmax, sizeof(unsigned long long),
                                      cudaMemcpyDeviceToHost, ctx->stream));
        MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        if (ctx->profiling) {
            float ms = 0.f;
            MB4_CUDA(ctx, cudaEventElapsedTime(&ms, ctx->pev0, ctx->pev1));
            ctx->prof.kernel_ms += ms;
            ctx->prof.launches += 1;
            ctx->prof.sweeps += 1;
            ctx->prof.alg_bytes += static_cast<double>(ctx->n) * (cur < 0 ? 72.0 : 120.0);
        }
        *sweeps = it;
        unsigned long long bits = *ctx->h_rmax;
        // same widened high-word residual as the production kernel
        if (bits >> 32) bits = (bits & 0xFFFFFFFF00000000ull) | 0xFFFFFFFFull;
        const double r = decode_bits(bits);
        const double r_prev = *last_res;
        *last_res = r;
        cur = nxt;
        if (!std::isfinite(r)) {
            *last_res = INFINITY;
            return fail(ctx, MB4CU_NONCONVERGED, "stage iteration diverged (non-finite update)");
        }
        if (mb4cu::stage_converged(r, r_prev, it - 1, ctx->eps)) {
            std::swap(ctx->u0, ctx->U[cur][2]);
            return MB4CU_OK;
        }
    }
    return fail(ctx, MB4CU_NONCONVERGED,
                "stage iteration: no convergence after " + std::to_string(ctx->max_iters) + " sweeps");
}

}  // namespace

extern "C" {

const char* mb4cu_version(void) { return "mb4cu 0.1 (sm_100a, FP64)"; }

const char* mb4cu_create_error(void) { return g_create_error.c_str(); }

int mb4cu_scheme_init(double alpha1, double c1, double c2, double c3, mb4cu_scheme* out) {
    g_create_error.clear();
    return mb4cu::scheme_init(alpha1, c1, c2, c3, out, g_create_error);
}

double mb4cu_eval_a(double alpha1, double tau, double zeta) { return mb4cu::eval_a_double(alpha1, tau, zeta); }

int mb4cu_lagrange_basis(const double nodes[4], int i, double zeta, double* out) {
    g_create_error.clear();
    return mb4cu::lagrange_basis_double(nodes, i, zeta, out, g_create_error);
}

int mb4cu_scheme_integrate_e(double alpha1, const double nodes[4], int points, double out[12]) {
    g_create_error.clear();
    return mb4cu::integrate_e(alpha1, nodes, points, out, g_create_error);
}

int mb4cu_make_inputs(const mb4cu_inputs* spec, int x0, int y0, int lnx, int lny, double* V,
                      double* psi, double* psum) {
    g_create_error.clear();
    return mb4cu::make_inputs(spec, x0, y0, lnx, lny, V, psi, psum, g_create_error);
}

int mb4cu_scale_state(double* psi, size_t nsites, double s, int threads) {
    return mb4cu::scale_state(psi, nsites, s, threads);
}

int mb4cu_create(const mb4cu_problem* p, const mb4cu_scheme* scheme, mb4cu_ctx** out) {
    g_create_error.clear();
    if (!p || !scheme || !out) {
        g_create_error = "mb4cu_create: null argument";
        return MB4CU_INVALID;
    }
    *out = nullptr;
    if (p->nx < 2 || p->ny < 2) {
        g_create_error = "GridSpec: nx and ny must be >= 2";
        return MB4CU_INVALID;
    }
    if (!(p->cx > 0.0) || !(p->cy > 0.0) || !std::isfinite(p->gamma) || !p->V) {
        g_create_error = "mb4cu_create: bad stencil / potential";
        return MB4CU_INVALID;
    }
    if (!(p->epsilon > 0.0)) {
        g_create_error = "NewtonConfig: epsilon must be > 0";
        return MB4CU_INVALID;
    }
    if (p->max_iters < 1) {
        g_create_error = "NewtonConfig: max_iters must be >= 1";
        return MB4CU_INVALID;
    }
    if (p->max_step_halvings < 0) {
        g_create_error = "NewtonConfig: negative halvings";
        return MB4CU_INVALID;
    }
    const int m = p->neumann_terms < 0 ? kDefaultNeumann : p->neumann_terms;
    if (m > 3) {
        g_create_error = "mb4cu_create: neumann_terms must be in 0..3";
        return MB4CU_INVALID;
    }
    auto* ctx = new mb4cu_ctx();
    ctx->device = p->device;
    ctx->nx = p->nx;
    ctx->ny = p->ny;
    ctx->n = static_cast<size_t>(p->nx) * p->ny;
    ctx->cx = p->cx;
    ctx->cy = p->cy;
    ctx->gamma = p->gamma;
    ctx->eps = p->epsilon;
    ctx->max_iters = p->max_iters;
    ctx->max_halvings = p->max_step_halvings;
    ctx->m = m;
    ctx->kernel = p->kernel;
    ctx->batched = std::getenv("MB4CU_NO_BATCH") == nullptr;  // A/B switch for the bench
    ctx->ghost = p->ghost;
    if (p->kernel < 0 || p->kernel > 3) {
        g_create_error = "mb4cu_create: kernel must be 0 (default), 1 (tiled), 2 (march v1) or 3 (Newton-Krylov)";
        delete ctx;
        return MB4CU_INVALID;
    }
    // first-sweep depth: default kDefaultFirst on the production kernel (2 in
    // sub-domain mode, 2 on the tiled kernel; v1 march: same as m)
    ctx->m_auto = p->neumann_terms < 0 && p->kernel == 0 && p->ghost == 0;
    if (p->neumann_first >= 0)
        ctx->mf = p->neumann_first;
    else if (p->kernel == 0 && p->ghost == 0 && mb4cu::march2_supported(kDefaultFirst, m))
        ctx->mf = kDefaultFirst;
    else
        ctx->mf = p->kernel == 2 || m > 2 ? m : 2;
    if (p->kernel == 2) ctx->mf = m;
    if (ctx->m_auto && !mb4cu::march2_supported(ctx->mf, 2)) ctx->m_auto = false;
    if (ctx->mf != m && !(p->kernel == 0 && mb4cu::march2_supported(ctx->mf, m)) &&
        !(p->kernel != 2 && ctx->mf == 2 && m <= 2)) {
        g_create_error = "mb4cu_create: unsupported (neumann_first, neumann_terms) pair for this kernel";
        delete ctx;
        return MB4CU_INVALID;
    }
    const int mmax = ctx->mf > m ? ctx->mf : m;
    if (p->ghost < 0 || (p->ghost > 0 && (p->ghost < mmax + 1 || m > 2 || p->kernel != 0 ||
                                          p->ghost > p->nx || p->ghost > p->ny))) {
        g_create_error = "mb4cu_create: sub-domain mode needs neumann_first + 1 <= ghost <= block size, "
                         "neumann_terms + 1 <= ghost, m <= 2, kernel 0";
        delete ctx;
        return MB4CU_INVALID;
    }
    // sub-domain rows padded to a multiple of 8 sites (128 B): every row of a band then
    // has one alignment, which the sweeps' cp.async ring placement relies on
    ctx->pitch = p->ghost > 0 ? (p->nx + 2 * p->ghost + 7) / 8 * 8 : p->nx;
    ctx->alloc_n = static_cast<size_t>(ctx->pitch) * (p->ny + 2 * p->ghost);
    ctx->scheme = *scheme;
    for (size_t k = 0; k < ctx->n; ++k) ctx->vmax = std::max(ctx->vmax, std::fabs(p->V[k]));
    ctx->vmin = ctx->n ? p->V[0] : 0.0;
    for (size_t k = 0; k < ctx->n; ++k) ctx->vmin = std::min(ctx->vmin, p->V[k]);
    // Chebyshev placement needs the spectrum of J = S H(u0) on the imaginary axis, i.e.
    // H(u0) positive semidefinite: K >= 0 always, V >= 0 and a defocusing cubic term
    if (p->first_poly < 0 || p->first_poly > 2) {
        g_create_error = "mb4cu_create: first_poly must be 0 (default), 1 (Neumann) or 2 (Chebyshev)";
        delete ctx;
        return MB4CU_INVALID;
    }
    // cross-check knob: MB4CU_KR_BATCH=0 solves the stage systems one after the other
    if (const char* kb = std::getenv("MB4CU_KR_BATCH")) ctx->kr_batch = std::atoi(kb) != 0;
    ctx->first_poly = p->first_poly != 0 ? p->first_poly : (ctx->vmin >= 0.0 && ctx->gamma <= 0.0 ? 2 : 1);
    ctx->first_poly_auto = p->first_poly == 0;
    // the cross-check kernels (and the v1 march the production kernel falls back to for
    // pairs it does not compile) run the per-stage Neumann recursion
    if (p->kernel != 0 || !mb4cu::march2_supported(ctx->mf, m)) ctx->first_poly = 1;

    auto bail = [&](cudaError_t e, const char* where) {
        g_create_error = std::string(where) + ": " + cudaGetErrorString(e);
        const int code = e == cudaErrorMemoryAllocation ? MB4CU_OOM : MB4CU_CUDA_ERROR;
        mb4cu_destroy(ctx);
        return code;
    };
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return bail(e, "cudaSetDevice");
    if ((e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking)) != cudaSuccess)
        return bail(e, "cudaStreamCreate");
    ctx->stream = ctx->own_stream;
    const size_t sb = ctx->alloc_n * sizeof(double2);
    if ((e = cudaMalloc(&ctx->u0, sb)) != cudaSuccess) return bail(e, "cudaMalloc(u0)");
    if ((e = cudaMalloc(&ctx->V, ctx->alloc_n * sizeof(double))) != cudaSuccess) return bail(e, "cudaMalloc(V)");
    for (int b = 0; b < 2; ++b)
        for (int i = 0; i < 3; ++i)
            if ((e = cudaMalloc(&ctx->U[b][i], sb)) != cudaSuccess) return bail(e, "cudaMalloc(U)");
    if ((e = cudaMalloc(&ctx->d_rmax, 64)) != cudaSuccess) return bail(e, "cudaMalloc(rmax)");
    if ((e = cudaMallocHost(&ctx->h_rmax, 64)) != cudaSuccess) return bail(e, "cudaMallocHost");
    const int nb = mb4cu::obs_blocks(ctx->nx, ctx->ny);
    if ((e = cudaMalloc(&ctx->d_obs_partial, sizeof(double) * mb4cu::kObsFields * nb)) != cudaSuccess)
        return bail(e, "cudaMalloc(obs)");
    if ((e = cudaMalloc(&ctx->d_obs5, sizeof(double) * 8)) != cudaSuccess) return bail(e, "cudaMalloc(obs5)");
    if ((e = cudaMallocHost(&ctx->h_obs5, sizeof(double) * 8)) != cudaSuccess) return bail(e, "cudaMallocHost");
    if ((e = cudaEventCreate(&ctx->ev0)) != cudaSuccess) return bail(e, "cudaEventCreate");
    if ((e = cudaEventCreate(&ctx->ev1)) != cudaSuccess) return bail(e, "cudaEventCreate");
    if (ctx->kernel != 1) {
        int grid = std::max(mb4cu::march_grid_size(ctx->m, ctx->device),
                            mb4cu::march2_supported(ctx->mf, ctx->m)
                                ? mb4cu::march2_grid_size(ctx->mf, ctx->m, ctx->device)
                                : 0);
        if (ctx->m_auto) grid = std::max(grid, mb4cu::march2_grid_size(ctx->mf, 2, ctx->device));
        if (grid <= 0) return bail(cudaErrorLaunchOutOfResources, "march_grid_size");
        if ((e = cudaMalloc(&ctx->d_rmax_arr, sizeof(unsigned long long) * (ctx->max_iters + 1))) != cudaSuccess)
            return bail(e, "cudaMalloc(rmax_arr)");
        // chunk counters of the later sweeps (MB4CU_FIXED_SHARES: A/B switch for the tests --
        // without counters every launch uses the fixed even split)
        if (std::getenv("MB4CU_FIXED_SHARES") == nullptr) {
            if ((e = cudaMalloc(&ctx->d_work, sizeof(unsigned) * mb4cu::kWorkCounters)) != cudaSuccess)
                return bail(e, "cudaMalloc(work)");
            if ((e = cudaMemset(ctx->d_work, 0, sizeof(unsigned) * mb4cu::kWorkCounters)) != cudaSuccess)
                return bail(e, "cudaMemset(work)");
        }
        if ((e = cudaMalloc(&ctx->d_obs_march, sizeof(double) * mb4cu::kObsFields * mb4cu::kObsSlotsPerCta * grid)) !=
            cudaSuccess)
            return bail(e, "cudaMalloc(obs_march)");
        ctx->obs_grid = grid;
        if ((e = cudaMalloc(&ctx->d_status, sizeof(mb4cu::StepStatus))) != cudaSuccess)
            return bail(e, "cudaMalloc(status)");
        if ((e = cudaMallocHost(&ctx->h_status, sizeof(mb4cu::StepStatus))) != cudaSuccess)
            return bail(e, "cudaMallocHost(status)");
    }
    if ((e = cudaEventCreate(&ctx->pev0)) != cudaSuccess) return bail(e, "cudaEventCreate");
    if ((e = cudaEventCreate(&ctx->pev1)) != cudaSuccess) return bail(e, "cudaEventCreate");
    if (ctx->ghost > 0) {
        for (auto& set : ctx->U)
            for (auto* q : set)
                if ((e = cudaMemset(q, 0, sb)) != cudaSuccess) return bail(e, "cudaMemset(U)");
        if ((e = cudaMemset(ctx->V, 0, ctx->alloc_n * sizeof(double))) != cudaSuccess) return bail(e, "cudaMemset(V)");
        e = cudaMemcpy2D(ctx->V + static_cast<size_t>(ctx->ghost) * ctx->pitch + ctx->ghost,
                         sizeof(double) * ctx->pitch, p->V, sizeof(double) * ctx->nx, sizeof(double) * ctx->nx,
                         ctx->ny, cudaMemcpyHostToDevice);
    } else {
        e = cudaMemcpy(ctx->V, p->V, ctx->n * sizeof(double), cudaMemcpyHostToDevice);
    }
    if (e != cudaSuccess)
        return bail(e, "cudaMemcpy(V)");
    if ((e = cudaMemset(ctx->u0, 0, sb)) != cudaSuccess) return bail(e, "cudaMemset(u0)");
    // cudaMemset is asynchronous and runs on the legacy stream, which does not order
    // against the non-blocking context stream: finish the initialisation here, or a
    // late zero-fill can overwrite the first set_state copy.
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return bail(e, "cudaDeviceSynchronize(create)");
    *out = ctx;
    return MB4CU_OK;
}

namespace {
void dn_free(mb4cu_ctx* ctx);
void dn_state_set(mb4cu_ctx* ctx);  // a new resident state: its halos are not exchanged yet
}  // namespace

int mb4cu_destroy(mb4cu_ctx* ctx) {
    if (!ctx) return MB4CU_OK;
    cudaSetDevice(ctx->device);
    if (ctx->own_stream) cudaStreamSynchronize(ctx->own_stream);
    cudaFree(ctx->u0);
    cudaFree(ctx->V);
    for (auto& set : ctx->U)
        for (auto* p : set) cudaFree(p);
    cudaFree(ctx->ubak);
    cudaFree(ctx->d_rmax);
    cudaFreeHost(ctx->h_rmax);
    cudaFree(ctx->d_obs_partial);
    cudaFree(ctx->d_obs5);
    cudaFreeHost(ctx->h_obs5);
    cudaFree(ctx->d_rmax_arr);
    cudaFree(ctx->d_work);
    cudaFree(ctx->d_obs_march);
    cudaFree(ctx->d_status);
    cudaFreeHost(ctx->h_status);
    dn_free(ctx);
    cudaFree(ctx->d_bstatus);
    cudaFreeHost(ctx->h_bstatus);
    cudaFree(ctx->d_brmax);
    cudaFree(ctx->d_babort);
    for (auto& ev : ctx->bev)
        if (ev) cudaEventDestroy(ev);
    kr_free(ctx);
    krb_free(ctx);
    if (ctx->fft.have1) cufftDestroy(ctx->fft.plan1);
    if (ctx->fft.have2) cufftDestroy(ctx->fft.plan2);
    cudaFree(ctx->fft.partial);
    cudaFreeHost(ctx->fft.h_partial);
    cudaFree(ctx->fft.shift_dev);
    cudaFreeHost(ctx->fft.h_shift);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->pev0) cudaEventDestroy(ctx->pev0);
    if (ctx->pev1) cudaEventDestroy(ctx->pev1);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
    return MB4CU_OK;
}

const char* mb4cu_last_error(const mb4cu_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

// Test hook (not part of the boundary, tests/test_chunks.py): chunk c of the chunked later
// sweeps' split of `total` band-rows over G CTAs -> [*p0, *p1), 0 past the last chunk; c < 0
// returns the number of chunks.
extern "C" long long mb4cu_debug_chunk(long long c, long long total, long long G, long long* p0, long long* p1) {
    if (total <= 0 || G <= 0) return -1;
    if (c < 0) return mb4cu::march2_chunk_count(total, G);
    if (!p0 || !p1) return -1;
    return mb4cu::march2_chunk_range(c, total, G, p0, p1) ? 1 : 0;
}

int mb4cu_set_neumann_terms(mb4cu_ctx* ctx, int m) {
    if (!ctx) return MB4CU_INVALID;
    if (ctx->kernel != 0 || m < 0 || m > 2 || !mb4cu::march2_supported(ctx->mf, m) ||
        (ctx->ghost > 0 && m + 1 > ctx->ghost))
        return fail(ctx, MB4CU_INVALID, "set_neumann_terms: production kernel, m in 0..2 with a compiled "
                                        "(neumann_first, m) pair and m + 1 <= ghost");
    // the first sweeps write one energy partial per CTA: the grid of the new (mf, m)
    // pair must fit the buffer sized at create time (reallocate if it does not)
    const int grid = mb4cu::march2_grid_size(ctx->mf, m, ctx->device);
    if (grid > ctx->obs_grid) {
        MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        double* fresh = nullptr;
        MB4_CUDA(ctx, cudaMalloc(&fresh, sizeof(double) * mb4cu::kObsFields * mb4cu::kObsSlotsPerCta * grid));
        cudaFree(ctx->d_obs_march);
        ctx->d_obs_march = fresh;
        ctx->obs_grid = grid;
    }
    if (m != ctx->m) ctx->last_sweeps = 0;  // as adapt_neumann: no speculative sweep right after a switch
    ctx->m = m;
    ctx->m_auto = false;  // the caller drives the depth from now on
    return MB4CU_OK;
}

int mb4cu_spectral_bound(mb4cu_ctx* ctx, double* rho) {
    if (!ctx || !rho) return fail(ctx, MB4CU_INVALID, "spectral_bound: null argument");
    MB4_CUDA(ctx, cudaSetDevice(ctx->device));
    const int rc = refresh_amax2(ctx);
    if (rc) return rc;
    *rho = own_first_rho(ctx);
    return MB4CU_OK;
}

int mb4cu_set_spectral_bound(mb4cu_ctx* ctx, double rho) {
    if (!ctx) return MB4CU_INVALID;
    if (!(rho >= 0.0) || !std::isfinite(rho)) return fail(ctx, MB4CU_INVALID, "set_spectral_bound: rho must be >= 0");
    ctx->rho_override = rho;
    return MB4CU_OK;
}

int mb4cu_set_amax2(mb4cu_ctx* ctx, double amax2) {
    if (!ctx) return MB4CU_INVALID;
    if (!(amax2 >= 0.0) || !std::isfinite(amax2)) return fail(ctx, MB4CU_INVALID, "set_amax2: amax2 must be >= 0");
    track_amax2(ctx, amax2);
    return MB4CU_OK;
}

int mb4cu_set_stream(mb4cu_ctx* ctx, void* s) {
    if (!ctx) return MB4CU_INVALID;
    ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own_stream;
    return MB4CU_OK;
}

// Copy between a contiguous nx*ny state and the (possibly padded) device u0.
static cudaError_t copy_state(mb4cu_ctx* ctx, void* dst, const void* src, bool to_device, cudaMemcpyKind kind) {
    if (ctx->ghost == 0) return cudaMemcpyAsync(dst, src, ctx->n * sizeof(double2), kind, ctx->stream);
    const size_t off = static_cast<size_t>(ctx->ghost) * ctx->pitch + ctx->ghost;
    const size_t row = sizeof(double2) * ctx->nx, dpitch = sizeof(double2) * ctx->pitch;
    if (to_device)
        return cudaMemcpy2DAsync(static_cast<double2*>(dst) + off, dpitch, src, row, row, ctx->ny, kind, ctx->stream);
    return cudaMemcpy2DAsync(dst, row, static_cast<const double2*>(src) + off, dpitch, row, ctx->ny, kind, ctx->stream);
}

int mb4cu_set_state(mb4cu_ctx* ctx, const double* u) {
    if (!ctx || !u) return fail(ctx, MB4CU_INVALID, "set_state: null argument");
    MB4_CUDA(ctx, cudaSetDevice(ctx->device));
    MB4_CUDA(ctx, copy_state(ctx, ctx->u0, u, true, cudaMemcpyHostToDevice));
    MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    ctx->obs_cached = false;
    ctx->amax2_valid = false;
    dn_state_set(ctx);
    return MB4CU_OK;
}

int mb4cu_get_state(mb4cu_ctx* ctx, double* u) {
    if (!ctx || !u) return fail(ctx, MB4CU_INVALID, "get_state: null argument");
    MB4_CUDA(ctx, cudaSetDevice(ctx->device));
    MB4_CUDA(ctx, copy_state(ctx, u, ctx->u0, false, cudaMemcpyDeviceToHost));
    MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return MB4CU_OK;
}

int mb4cu_set_state_device(mb4cu_ctx* ctx, const double* u) {
    if (!ctx || !u) return fail(ctx, MB4CU_INVALID, "set_state_device: null argument");
    MB4_CUDA(ctx, copy_state(ctx, ctx->u0, u, true, cudaMemcpyDeviceToDevice));
    ctx->obs_cached = false;
    ctx->amax2_valid = false;
    dn_state_set(ctx);
    return MB4CU_OK;
}

int mb4cu_get_state_device(mb4cu_ctx* ctx, double* u) {
    if (!ctx || !u) return fail(ctx, MB4CU_INVALID, "get_state_device: null argument");
    MB4_CUDA(ctx, copy_state(ctx, u, ctx->u0, false, cudaMemcpyDeviceToDevice));
    return MB4CU_OK;
}

int mb4cu_step(mb4cu_ctx* ctx, double h, mb4cu_stats* stats) {
    if (!ctx) return MB4CU_INVALID;
    if (!(h > 0.0)) return fail(ctx, MB4CU_INVALID, "mb4_step: h must be positive");
    if (ctx->ghost > 0)
        return fail(ctx, MB4CU_INVALID, "mb4_step: sub-domain contexts step through mb4cu_sweep");
    MB4_CUDA(ctx, cudaSetDevice(ctx->device));
    if (ctx->kernel == 0) {
        const int rca = refresh_amax2(ctx);
        if (rca) return rca;
    }
    MB4_CUDA(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
    double last = 0.0;
    int rc = MB4CU_NONCONVERGED;
    int used_halvings = 0, sweeps_total = 0;
    for (int hv = 0; hv <= ctx->max_halvings; ++hv) {
        const int sub = 1 << hv;
        const double hs = h / sub;
        if (hv == 1) {
            if (!ctx->ubak) MB4_CUDA(ctx, cudaMalloc(&ctx->ubak, ctx->n * sizeof(double2)));
            MB4_CUDA(ctx, cudaMemcpyAsync(ctx->ubak, ctx->u0, ctx->n * sizeof(double2),
                                          cudaMemcpyDeviceToDevice, ctx->stream));
        } else if (hv > 1) {
            MB4_CUDA(ctx, cudaMemcpyAsync(ctx->u0, ctx->ubak, ctx->n * sizeof(double2),
                                          cudaMemcpyDeviceToDevice, ctx->stream));
        }
        bool ok = true;
        int attempt = 0;
        for (int s = 0; s < sub; ++s) {
            int sw = 0;
            rc = substep(ctx, hs, &sw, &last);
            if (hv == 0 && s == 0)  // energy sums of the step's entry state (fused path)
                std::memcpy(ctx->entry_obs, ctx->obs_cache, sizeof(ctx->entry_obs));
            attempt += sw;
            if (rc == MB4CU_NONCONVERGED) {
                ok = false;
                break;
            }
            if (rc != MB4CU_OK) return rc;
        }
        if (ok) {
            used_halvings = hv;
            sweeps_total = attempt;
            rc = MB4CU_OK;
            break;
        }
    }
    if (rc != MB4CU_OK) {
        if (ctx->max_halvings >= 1)
            MB4_CUDA(ctx, cudaMemcpyAsync(ctx->u0, ctx->ubak, ctx->n * sizeof(double2),
                                          cudaMemcpyDeviceToDevice, ctx->stream));
        MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        if (stats) stats->last_residual = last;
        return fail(ctx, MB4CU_NONCONVERGED,
                    "mb4_step: no convergence after " + std::to_string(ctx->max_halvings) +
                        " step halvings");
    }
    MB4_CUDA(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
    MB4_CUDA(ctx, cudaEventSynchronize(ctx->ev1));
    float ms = 0.f;
    MB4_CUDA(ctx, cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    if (stats) {
        stats->newton_iters += sweeps_total;
        stats->halvings += used_halvings;
        stats->solve_seconds += 1e-3 * ms;
        stats->last_residual = last;
    }
    return MB4CU_OK;
}

int mb4cu_profile_enable(mb4cu_ctx* ctx, int on) {
    if (!ctx) return MB4CU_INVALID;
    ctx->profiling = on != 0;
    return MB4CU_OK;
}

int mb4cu_profile_reset(mb4cu_ctx* ctx) {
    if (!ctx) return MB4CU_INVALID;
    ctx->prof = mb4cu_profile{};
    return MB4CU_OK;
}

int mb4cu_profile_get(mb4cu_ctx* ctx, mb4cu_profile* out) {
    if (!ctx || !out) return MB4CU_INVALID;
    *out = ctx->prof;
    return MB4CU_OK;
}

// Energy sums -> Observables with the reference's health check (lattice.cpp:113-127).
static int finish_obs(mb4cu_ctx* ctx, const double* sums, mb4cu_obs* out) {
    const double qr = sums[0], qi = sums[1], prob = sums[2], quart = sums[3], ext = sums[4];
    // u^H K u is real for symmetric K; imaginary residue is a health check (lattice.cpp:123-126)
    const double imag_scale = std::max(std::fabs(qr), (4.0 * ctx->cx + 4.0 * ctx->cy) * prob);
    if (std::fabs(qi) > 1e-12 * imag_scale && imag_scale > 0.0)
        return fail(ctx, MB4CU_NUMERIC, "observables: non-real kinetic quadratic form");
    out->u_kinetic = qr;
    out->u_nonlinear = -0.5 * ctx->gamma * quart;
    out->u_external = ext;
    out->total_energy = out->u_kinetic + out->u_nonlinear + out->u_external;
    out->probability = prob;
    out->raw_quartic = quart;
    out->participation = prob > 0.0 ? quart / (prob * prob) : 0.0;
    return MB4CU_OK;
}

int mb4cu_observables(mb4cu_ctx* ctx, mb4cu_obs* out) {
    if (!ctx || !out) return fail(ctx, MB4CU_INVALID, "observables: null argument");
    MB4_CUDA(ctx, cudaSetDevice(ctx->device));
    mb4cu::ObsArgs a{};
    a.nx = ctx->nx;
    a.ny = ctx->ny;
    a.cx = ctx->cx;
    a.cy = ctx->cy;
    a.diag = 2.0 * ctx->cx + 2.0 * ctx->cy;
    a.u = ctx->u0;
    a.V = ctx->V;
    a.partial = ctx->d_obs_partial;
    if (ctx->ghost > 0)
        MB4_CUDA(ctx, mb4cu::launch_observables_ghost(a, ctx->ghost, ctx->pitch, ctx->d_obs5, ctx->stream));
    else
        MB4_CUDA(ctx, mb4cu::launch_observables(a, ctx->d_obs5, ctx->stream));
    ctx->prof.other_launches += 2;
    MB4_CUDA(ctx, cudaMemcpyAsync(ctx->h_obs5, ctx->d_obs5, sizeof(double) * mb4cu::kObsFields,
                                  cudaMemcpyDeviceToHost, ctx->stream));
    MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return finish_obs(ctx, ctx->h_obs5, out);
}

static void put_obs(double* row, const mb4cu_obs& o) {
    row[0] = o.u_kinetic;
    row[1] = o.u_nonlinear;
    row[2] = o.u_external;
    row[3] = o.total_energy;
    row[4] = o.probability;
    row[5] = o.participation;
    row[6] = o.raw_quartic;
}

namespace {

constexpr int kBatch = 64;  // steps enqueued per host round trip (mb4cu_run)

// Steps mb4cu_run may enqueue without waiting: the production sweep path of a whole
// lattice, non-stiff, with a known sweep count to predict from.
bool batchable(const mb4cu_ctx* ctx, double h) {
    return ctx->kernel == 0 && ctx->ghost == 0 && ctx->last_sweeps >= 1 && mb4cu::march2_supported(ctx->mf, ctx->m) &&
           !stiff_step(ctx, h);
}

// The max|u0|^2 values for which the step constants of h stay what they are for the
// current ctx->amax2: the same power-of-2^(1/16) Chebyshev interval (first_poly = 2)
// and a non-stiff step.  Shrunk by a relative 1e-9 so that the device's test never
// disagrees with the host's rounding at a boundary (a step ending there just ends the
// batch; the host then takes the next step on the one-step path).
void amax2_interval(const mb4cu_ctx* ctx, double h, double* lo, double* hi) {
    *lo = -1.0;
    *hi = HUGE_VAL;
    const double g3 = 3.0 * std::fabs(ctx->gamma);
    if (g3 == 0.0) return;
    const double base = 4.0 * ctx->cx + 4.0 * ctx->cy + ctx->vmax;
    if (ctx->first_poly == 2 && ctx->rho_override <= 0.0) {
        const double L = std::ceil(16.0 * std::log2(spectral_bound(ctx)));
        *lo = (std::exp2((L - 1.0) / 16.0) - base) / g3;
        *hi = (std::exp2(L / 16.0) - base) / g3;
    }
    const double lam = std::max({std::fabs(ctx->scheme.lam[0]), std::fabs(ctx->scheme.lam[1]),
                                 std::fabs(ctx->scheme.lam[2])});
    *hi = std::min(*hi, (kStiffKappa / (h * lam) - base) / g3);
    *lo += 1e-9 * std::fabs(*lo);
    *hi -= 1e-9 * std::fabs(*hi);
}

int batch_alloc(mb4cu_ctx* ctx) {
    if (ctx->d_bstatus) return MB4CU_OK;
    MB4_CUDA(ctx, cudaMalloc(&ctx->d_bstatus, sizeof(mb4cu::StepStatus) * kBatch));
    MB4_CUDA(ctx, cudaMallocHost(&ctx->h_bstatus, sizeof(mb4cu::StepStatus) * kBatch));
    MB4_CUDA(ctx, cudaMalloc(&ctx->d_brmax, sizeof(unsigned long long) * kBatch * (ctx->max_iters + 1)));
    MB4_CUDA(ctx, cudaMalloc(&ctx->d_babort, sizeof(int)));
    for (auto& ev : ctx->bev) MB4_CUDA(ctx, cudaEventCreate(&ev));
    return MB4CU_OK;
}

// Device-resident stepping: up to kBatch steps of size h enqueued back to back, with
// one host round trip at the end.  Each step is launched on the buffers of the sweep
// count of the step before it (the same prediction substep_march makes for its
// speculative final sweep); the step's last launch ends the batch on the device (the
// later launches return at once) when the step did not converge, took another sweep
// count, or made the adaptive depth switch.  The host then commits the steps that ran,
// in order, exactly as the one-step path does -- the results are bit-identical to
// stepping one at a time -- and the caller steps the rest (a failed step goes through
// mb4cu_step's fallbacks).  Returns the steps committed in *done.
int run_batch(mb4cu_ctx* ctx, double h, int nmax, double* obs_rows, int* iters, mb4cu_stats* stats, int* done) {
    *done = 0;
    if (int rc = batch_alloc(ctx)) return rc;
    int B = std::min(nmax, kBatch);
    if (ctx->m_auto && ctx->m == 2) B = std::min(B, std::max(1, 64 - ctx->auto_steps));
    const int expect = ctx->last_sweeps;
    const int spec = expect >= 2 ? expect - 1 : -1;
    mb4cu::BatchCtl ctl{ctx->d_babort, expect, ctx->m_auto && ctx->m == 1 ? 4 : 0, 0.0, 0.0};
    amax2_interval(ctx, h, &ctl.amax2_lo, &ctl.amax2_hi);
    const SweepConsts c = make_consts(ctx, h);
    MB4_CUDA(ctx, cudaMemsetAsync(ctx->d_babort, 0, sizeof(int), ctx->stream));
    MB4_CUDA(ctx, cudaMemsetAsync(ctx->d_bstatus, 0, sizeof(mb4cu::StepStatus) * B, ctx->stream));
    const size_t rstride = static_cast<size_t>(ctx->max_iters) + 1;
    MB4_CUDA(ctx, cudaMemsetAsync(ctx->d_brmax, 0, sizeof(unsigned long long) * B * rstride, ctx->stream));
    const double2* u0p = ctx->u0;
    double2* Up[2][3];
    std::memcpy(Up, ctx->U, sizeof(Up));
    const int set = (expect - 1) & 1;
    MB4_CUDA(ctx, cudaEventRecord(ctx->bev[0], ctx->stream));
    for (int k = 0; k < B; ++k) {
        MB4_CUDA(ctx, mb4cu::launch_step_march2(ctx->mf, ctx->m, ctx->nx, ctx->ny, u0p, ctx->V, Up,
                                                ctx->d_brmax + static_cast<size_t>(k) * rstride,
                                                ctx->d_obs_march, ctx->d_bstatus + k, ctx->max_iters, ctx->eps, 1, c,
                                                ctx->device, ctx->stream, 0, 0, spec, 0, nullptr, 0, 0, &ctl, 0,
                                                ctx->d_work, ctx->obs_grid * mb4cu::kObsSlotsPerCta));
        MB4_CUDA(ctx, cudaEventRecord(ctx->bev[k + 1], ctx->stream));
        // the predicted commit: u0 <-> U[set][2]
        double2* nu0 = Up[set][2];
        Up[set][2] = const_cast<double2*>(u0p);
        u0p = nu0;
    }
    MB4_CUDA(ctx, cudaMemcpyAsync(ctx->h_bstatus, ctx->d_bstatus, sizeof(mb4cu::StepStatus) * B,
                                  cudaMemcpyDeviceToHost, ctx->stream));
    MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    const int launches = mb4cu::march2_launches(ctx->mf, 0, 0, ctx->max_iters);
    if (ctx->profiling) ctx->prof.launches += launches * B;
    for (int k = 0; k < B; ++k) {
        const mb4cu::StepStatus& st = ctx->h_bstatus[k];
        if (st.sweeps == 0 || !st.converged || !std::isfinite(st.rlast)) break;  // not run, or failed
        float ms = 0.f;
        MB4_CUDA(ctx, cudaEventElapsedTime(&ms, ctx->bev[k], ctx->bev[k + 1]));
        if (ctx->profiling) {
            ctx->prof.kernel_ms += ms;
            ctx->prof.sweeps += st.sweeps;
            const bool spec_hit = st.sweeps - 1 == spec && spec >= 1;
            ctx->prof.alg_bytes += static_cast<double>(ctx->n) * (72.0 + 120.0 * (st.sweeps - 1) - (spec_hit ? 32.0 : 0.0));
            ctx->prof.redone += st.redone;
            for (int q = 0; q < st.sweeps && q < 8; ++q) {
                ctx->prof.sweep_ms[q] += 1e-6 * static_cast<double>(st.t[q + 1] - st.t[q]);
                ctx->prof.sweep_n[q] += 1;
            }
        }
        std::swap(ctx->u0, ctx->U[st.set][2]);
        ctx->obs_cached = false;
        ctx->last_sweeps = st.sweeps;
        track_amax2(ctx, st.amax2);
        adapt_neumann(ctx, st.sweeps);
        std::memcpy(ctx->entry_obs, st.obs, sizeof(ctx->entry_obs));
        if (obs_rows) {
            mb4cu_obs o{};
            if (int rc = finish_obs(ctx, st.obs, &o)) return rc;
            put_obs(obs_rows + 7 * k, o);
        }
        if (iters) iters[k] = st.sweeps;
        if (stats) {
            stats->newton_iters += st.sweeps;
            stats->solve_seconds += 1e-3 * ms;
            stats->last_residual = st.rlast;
        }
        ++*done;
    }
    return MB4CU_OK;
}

}  // namespace

int mb4cu_run(mb4cu_ctx* ctx, double h, int nsteps, double* obs_series, int* iters_series,
              mb4cu_stats* stats) {
    if (!ctx) return MB4CU_INVALID;
    if (nsteps < 0) return fail(ctx, MB4CU_INVALID, "run: nsteps must be >= 0");
    mb4cu_obs o{};
    if (ctx->kernel == 0) {
        const int rca = refresh_amax2(ctx);
        if (rca) return rca;
    }
    // With the persistent kernel the energy monitor of each step's entry state is
    // fused into that step's first sweep; only the final state needs its own pass.
    MB4_CUDA(ctx, cudaSetDevice(ctx->device));
    for (int s = 1; s <= nsteps; ++s) {
        if (ctx->kernel == 0) {
            if (int rca = refresh_amax2(ctx)) return rca;  // (a no-op unless a Newton-Krylov step ran)
        }
        if (ctx->batched && batchable(ctx, h)) {
            int done = 0;
            if (int rc = run_batch(ctx, h, nsteps - s + 1, obs_series ? obs_series + 7 * (s - 1) : nullptr,
                                   iters_series ? iters_series + (s - 1) : nullptr, stats, &done))
                return rc;
            if (done > 0) {
                s += done - 1;  // (the loop advances past the last committed step)
                continue;
            }
            // the batch's first step failed: it goes through the one-step path below
        }
        // the step's energy sums come from its first sweep's fused monitor, unless the
        // step goes straight to the Newton-Krylov solver (stiff) or the kernel has none
        const bool fused = (ctx->kernel == 0 && !stiff_step(ctx, h)) || ctx->kernel == 2;
        if (obs_series && !fused) {
            const int rc0 = mb4cu_observables(ctx, &o);
            if (rc0) return rc0;
            put_obs(obs_series + 7 * (s - 1), o);
        }
        mb4cu_stats st{};
        const int rc = mb4cu_step(ctx, h, &st);
        if (stats) {
            stats->newton_iters += st.newton_iters;
            stats->halvings += st.halvings;
            stats->solve_seconds += st.solve_seconds;
            stats->last_residual = st.last_residual;
        }
        if (rc) return rc;
        if (iters_series) iters_series[s - 1] = st.newton_iters;
        if (obs_series && fused) {
            const int rc1 = finish_obs(ctx, ctx->entry_obs, &o);
            if (rc1) return rc1;
            put_obs(obs_series + 7 * (s - 1), o);
        }
    }
    if (obs_series) {
        const int rc2 = mb4cu_observables(ctx, &o);
        if (rc2) return rc2;
        put_obs(obs_series + 7 * nsteps, o);
    }
    return MB4CU_OK;
}

// ---- the other integrators (integrators.cpp:45-455) ---------------------------

namespace {

const char* method_label(int method) {
    static const char* names[] = {"rk4_step", "gauss_step(1)", "gauss_step(2)", "avf2_step", "avf4_step", "mb4_step"};
    return method >= 0 && method <= 5 ? names[method] : "?";
}

mb4cu::MethodConsts method_consts(const mb4cu_ctx* ctx, int method, double h) {
    mb4cu::MethodConsts c{};
    c.h = h;
    c.gamma = ctx->gamma;
    c.cx = ctx->cx;
    c.cy = ctx->cy;
    c.diag = 2.0 * ctx->cx + 2.0 * ctx->cy;
    mb4cu::method_tables(&c);
    if (method == mb4cu::kMethodGauss4) {
        // 2-stage Gauss A (integrators.cpp:160-161)
        const double r3 = std::sqrt(3.0);
        c.a[0][0] = 0.25;
        c.a[0][1] = 0.25 - r3 / 6.0;
        c.a[1][0] = 0.25 + r3 / 6.0;
        c.a[1][1] = 0.25;
    } else if (method == mb4cu::kMethodAvf4) {
        mb4cu::avf4_coupling(c.a);
    } else {
        c.a[0][0] = 0.5;  // stage_matrix(j, h / 2)
    }
    return c;
}

int method_stages(int method) {
    return method == mb4cu::kMethodGauss4 || method == mb4cu::kMethodAvf4 ? 2 : 1;
}

// One plain step of RK4 / an implicit method on ctx->u0 (u0 <- u1 on success;
// unchanged otherwise).  Implicit methods: the reference's simplified Newton
// iteration, the linear systems by matrix-free GMRES.
int method_plain_step(mb4cu_ctx* ctx, int method, double h, int* iters, double* last_res) {
    const mb4cu::MethodConsts c = method_consts(ctx, method, h);
    const size_t n = ctx->n;
    *iters = 0;
    *last_res = 0.0;
    if (method == mb4cu::kMethodRk4) {
        double2* acc = ctx->U[0][0];
        double2* t1 = ctx->U[0][1];
        double2* t2 = ctx->U[0][2];
        double2* out = ctx->U[1][0];
        MB4_CUDA(ctx, mb4cu::launch_rk4_stage(1, ctx->nx, ctx->ny, ctx->u0, ctx->u0, ctx->V, acc, t1, c, ctx->stream));
        MB4_CUDA(ctx, mb4cu::launch_rk4_stage(2, ctx->nx, ctx->ny, t1, ctx->u0, ctx->V, acc, t2, c, ctx->stream));
        MB4_CUDA(ctx, mb4cu::launch_rk4_stage(3, ctx->nx, ctx->ny, t2, ctx->u0, ctx->V, acc, t1, c, ctx->stream));
        MB4_CUDA(ctx, mb4cu::launch_rk4_stage(4, ctx->nx, ctx->ny, t1, ctx->u0, ctx->V, acc, out, c, ctx->stream));
        ctx->prof.other_launches += 4;
        std::swap(ctx->u0, ctx->U[1][0]);
        return MB4CU_OK;
    }
    const int st = method_stages(method);
    const size_t len = static_cast<size_t>(st) * n;
    if (int rc = kr_alloc(ctx, len)) return rc;
    const int m = ctx->kr.m;
    double2* b = kr_vec(ctx, m + 1);
    double2* x = kr_vec(ctx, m + 2);
    double2* unk = kr_vec(ctx, m + 3);
    if (method == mb4cu::kMethodAvf4) {
        MB4_CUDA(ctx, mb4cu::launch_avf4_init(ctx->nx, ctx->ny, ctx->u0, ctx->V, unk, c, ctx->stream));
    } else {
        for (int i = 0; i < st; ++i)
            MB4_CUDA(ctx, cudaMemcpyAsync(unk + i * n, ctx->u0, n * sizeof(double2), cudaMemcpyDeviceToDevice,
                                          ctx->stream));
    }
    auto mv = [&](const double2* xin, double2* yout) {
        return mb4cu::launch_method_matvec(st, ctx->nx, ctx->ny, xin, yout, ctx->u0, ctx->V, c, ctx->stream);
    };
    if (int rc = fft_prepare(ctx, st)) return rc;
    for (int it = 1; it <= ctx->max_iters; ++it) {
        MB4_CUDA(ctx, mb4cu::launch_method_residual(method, ctx->nx, ctx->ny, ctx->u0, ctx->V, unk, b, c,
                                                    ctx->stream));
        if (int rc = st == 1 ? kr_gmres_fft(ctx, 1, 0.5 * h, nullptr, mv, b, x)
                             : kr_gmres_fft(ctx, 2, h, c.a, mv, b, x))
            return rc;
        MB4_CUDA(ctx, mb4cu::launch_newton_add(unk, x, len, ctx->d_rmax, ctx->stream));
        MB4_CUDA(ctx, cudaMemcpyAsync(ctx->h_rmax, ctx->d_rmax, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                      ctx->stream));
        MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        *iters = it;
        const double r = decode_bits(*ctx->h_rmax);
        *last_res = r;
        if (!std::isfinite(r)) {
            *last_res = INFINITY;
            return fail(ctx, MB4CU_NONCONVERGED, std::string(method_label(method)) + ": iteration diverged");
        }
        if (r <= ctx->eps) {
            MB4_CUDA(ctx, mb4cu::launch_method_final(method, ctx->nx, ctx->ny, ctx->u0, ctx->V, unk, ctx->U[1][0], c,
                                                     ctx->stream));
            std::swap(ctx->u0, ctx->U[1][0]);
            return MB4CU_OK;
        }
    }
    return fail(ctx, MB4CU_NONCONVERGED, std::string(method_label(method)) + ": no convergence");
}

}  // namespace

int mb4cu_method_step(mb4cu_ctx* ctx, int method, double h, mb4cu_stats* stats) {
    if (!ctx) return MB4CU_INVALID;
    if (method < 0 || method > 5) return fail(ctx, MB4CU_INVALID, "StepDriver: unknown method");
    if (method == mb4cu::kMethodMb4) return mb4cu_step(ctx, h, stats);
    if (!(h > 0.0)) return fail(ctx, MB4CU_INVALID, "advance: h must be positive");
    if (ctx->ghost > 0) return fail(ctx, MB4CU_INVALID, "methods: sub-domain contexts are MB4-only");
    MB4_CUDA(ctx, cudaSetDevice(ctx->device));
    ctx->obs_cached = false;
    ctx->amax2_valid = false;
    int it = 0;
    double last = 0.0;
    if (method == mb4cu::kMethodRk4) return method_plain_step(ctx, method, h, &it, &last);  // no halving (:427)
    // halving-on-failure of StepDriver::advance (integrators.cpp:430-455)
    MB4_CUDA(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
    if (!ctx->ubak) MB4_CUDA(ctx, cudaMalloc(&ctx->ubak, ctx->n * sizeof(double2)));
    MB4_CUDA(ctx, cudaMemcpyAsync(ctx->ubak, ctx->u0, ctx->n * sizeof(double2), cudaMemcpyDeviceToDevice,
                                  ctx->stream));
    for (int hv = 0; hv <= ctx->max_halvings; ++hv) {
        const int sub = 1 << hv;
        const double hs = h / sub;
        if (hv > 0)
            MB4_CUDA(ctx, cudaMemcpyAsync(ctx->u0, ctx->ubak, ctx->n * sizeof(double2), cudaMemcpyDeviceToDevice,
                                          ctx->stream));
        bool ok = true;
        int attempt = 0;
        for (int s = 0; s < sub && ok; ++s) {
            const int rc = method_plain_step(ctx, method, hs, &it, &last);
            attempt += it;
            if (rc == MB4CU_NONCONVERGED)
                ok = false;
            else if (rc != MB4CU_OK)
                return rc;
        }
        if (ok) {
            MB4_CUDA(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
            MB4_CUDA(ctx, cudaEventSynchronize(ctx->ev1));
            float ms = 0.f;
            MB4_CUDA(ctx, cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
            if (stats) {
                stats->newton_iters += attempt;
                stats->halvings += hv;
                stats->solve_seconds += 1e-3 * ms;
                stats->last_residual = last;
            }
            return MB4CU_OK;
        }
    }
    MB4_CUDA(ctx, cudaMemcpyAsync(ctx->u0, ctx->ubak, ctx->n * sizeof(double2), cudaMemcpyDeviceToDevice,
                                  ctx->stream));
    MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (stats) stats->last_residual = last;
    return fail(ctx, MB4CU_NONCONVERGED,
                "advance: no convergence after " + std::to_string(ctx->max_halvings) + " step halvings");
}

int mb4cu_method_run(mb4cu_ctx* ctx, int method, double h, int nsteps, double* obs_series, int* iters_series,
                     mb4cu_stats* stats) {
    if (!ctx) return MB4CU_INVALID;
    if (method == mb4cu::kMethodMb4) return mb4cu_run(ctx, h, nsteps, obs_series, iters_series, stats);
    if (nsteps < 0) return fail(ctx, MB4CU_INVALID, "run: nsteps must be >= 0");
    mb4cu_obs o{};
    for (int s = 1; s <= nsteps; ++s) {
        if (obs_series) {
            const int rc0 = mb4cu_observables(ctx, &o);
            if (rc0) return rc0;
            put_obs(obs_series + 7 * (s - 1), o);
        }
        mb4cu_stats st{};
        const int rc = mb4cu_method_step(ctx, method, h, &st);
        if (stats) {
            stats->newton_iters += st.newton_iters;
            stats->halvings += st.halvings;
            stats->solve_seconds += st.solve_seconds;
            stats->last_residual = st.last_residual;
        }
        if (rc) return rc;
        if (iters_series) iters_series[s - 1] = st.newton_iters;
    }
    if (obs_series) {
        const int rc2 = mb4cu_observables(ctx, &o);
        if (rc2) return rc2;
        put_obs(obs_series + 7 * nsteps, o);
    }
    return MB4CU_OK;
}

// ---- sub-domain (multi-GPU) stepping ------------------------------------------

namespace {

// Halo width of a field: u0 and V feed the first sweep (depth mf -> mf + 1 layers);
// the stage sets (fields 2, 3) only the later sweeps (m + 1 layers); fields 4, 5 are
// the stage sets at the full ghost width (halo-overlap mode: U3 of the last sweep
// becomes u0 of the next step, halos included).
int halo_width(const mb4cu_ctx* ctx, int field) {
    return field <= 1 || field >= 4 ? ctx->ghost : std::min(ctx->ghost, ctx->m + 1);
}

// rectangle (x0, y0, w, h) of a halo side; pack == owned strip, unpack == ghost strip
void halo_rect(const mb4cu_ctx* ctx, int field, int side, bool pack, int* x0, int* y0, int* w, int* h) {
    const int g = halo_width(ctx, field), nx = ctx->nx, ny = ctx->ny;
    switch (side) {
        case 0: *x0 = pack ? 0 : -g; *y0 = 0; *w = g; *h = ny; break;            // west
        case 1: *x0 = pack ? nx - g : nx; *y0 = 0; *w = g; *h = ny; break;       // east
        case 2: *x0 = -g; *y0 = pack ? 0 : -g; *w = nx + 2 * g; *h = g; break;   // south
        default: *x0 = -g; *y0 = pack ? ny - g : ny; *w = nx + 2 * g; *h = g; break;  // north
    }
}

int halo_xfer(mb4cu_ctx* ctx, int field, int side, double* buf, bool pack) {
    if (!ctx || ctx->ghost <= 0 || field < 0 || field > 5 || side < 0 || side > 3 || !buf)
        return fail(ctx, MB4CU_INVALID, "halo: bad context / field / side / buffer");
    int x0, y0, w, h;
    halo_rect(ctx, field, side, pack, &x0, &y0, &w, &h);
    if (field == 1) {
        MB4_CUDA(ctx, mb4cu::launch_halo_copy1(ctx->V, ctx->pitch, ctx->ghost, x0, y0, w, h, buf, pack, ctx->stream));
    } else {
        double2* arr[3];
        int narr = 1;
        if (field == 0) {
            arr[0] = ctx->u0;
        } else {
            narr = 3;
            for (int q = 0; q < 3; ++q) arr[q] = ctx->U[(field - 2) & 1][q];
        }
        MB4_CUDA(ctx, mb4cu::launch_halo_copy2(arr, narr, ctx->pitch, ctx->ghost, x0, y0, w, h,
                                               reinterpret_cast<double2*>(buf), pack, ctx->stream));
    }
    return MB4CU_OK;
}

}  // namespace

size_t mb4cu_halo_count(const mb4cu_ctx* ctx, int field, int side) {
    if (!ctx || ctx->ghost <= 0 || field < 0 || field > 5 || side < 0 || side > 3) return 0;
    int x0, y0, w, h;
    halo_rect(ctx, field, side, true, &x0, &y0, &w, &h);
    const size_t sites = static_cast<size_t>(w) * h;
    return field == 1 ? sites : (field == 0 ? 2 * sites : 6 * sites);
}

int mb4cu_halo_pack(mb4cu_ctx* ctx, int field, int side, double* dev_buf) {
    return halo_xfer(ctx, field, side, dev_buf, true);
}

int mb4cu_halo_unpack(mb4cu_ctx* ctx, int field, int side, const double* dev_buf) {
    return halo_xfer(ctx, field, side, const_cast<double*>(dev_buf), false);
}

int mb4cu_sweep(mb4cu_ctx* ctx, double h, int s, double* local_rmax, double* local_sums5) {
    if (!ctx || ctx->ghost <= 0) return fail(ctx, MB4CU_INVALID, "sweep: sub-domain contexts only");
    if (!(h > 0.0) || s < 0) return fail(ctx, MB4CU_INVALID, "sweep: h must be positive, s >= 0");
    MB4_CUDA(ctx, cudaSetDevice(ctx->device));
    const SweepConsts c = make_consts(ctx, h);
    MB4_CUDA(ctx, cudaMemsetAsync(ctx->d_rmax_arr, 0, 2 * sizeof(unsigned long long), ctx->stream));
    if (ctx->profiling) MB4_CUDA(ctx, cudaEventRecord(ctx->pev0, ctx->stream));
    MB4_CUDA(ctx, mb4cu::launch_step_march2(ctx->mf, ctx->m, ctx->nx, ctx->ny, ctx->u0, ctx->V, ctx->U, ctx->d_rmax_arr,
                                            ctx->d_obs_march, ctx->d_status, 1, -1.0, s == 0 ? 1 : 0, c,
                                            ctx->device, ctx->stream, ctx->ghost, s, -1, 0, nullptr, 0, 0, nullptr,
                                            ctx->pitch));
    if (ctx->profiling) MB4_CUDA(ctx, cudaEventRecord(ctx->pev1, ctx->stream));
    MB4_CUDA(ctx, cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(mb4cu::StepStatus), cudaMemcpyDeviceToHost,
                                  ctx->stream));
    MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (ctx->profiling) {
        float ms = 0.f;
        MB4_CUDA(ctx, cudaEventElapsedTime(&ms, ctx->pev0, ctx->pev1));
        ctx->prof.kernel_ms += ms;
        ctx->prof.launches += 1;
        ctx->prof.sweeps += 1;
        ctx->prof.alg_bytes += static_cast<double>(ctx->n) * (s == 0 ? 72.0 : 120.0);
    }
    if (local_rmax) *local_rmax = ctx->h_status->rlast;
    if (local_sums5 && s == 0)
        for (int f = 0; f < mb4cu::kObsFields; ++f) local_sums5[f] = ctx->h_status->obs[f];
    return MB4CU_OK;
}

namespace {

// Output rectangles of a region of the sub-domain: 0 all, 1 the boundary frame of
// width ghost (the sites the neighbours' halos need), 2 the interior (needs no halo).
int region_rects(const mb4cu_ctx* ctx, int region, int rects[4][4], int s) {
    const int w = ctx->ghost, nx = ctx->nx, ny = ctx->ny;
    const bool thin = nx <= 2 * w || ny <= 2 * w;  // no interior: the frame is everything
    // west / east frame strips one sweep band wide (not `ghost` columns): a band computes
    // its full width anyway, so a ghost-wide strip would redo ~(band - ghost) columns per
    // row; large sub-domains only (small ones keep the ghost-wide frame and an interior)
    const int tx = mb4cu::march2_band_width(ctx->mf, ctx->m, s == 0);
    const int wx = tx > w && nx >= 4 * tx ? tx : w;
    if (region == 0 || (region == 1 && thin)) {
        const int r[4] = {0, 0, nx, ny};
        std::memcpy(rects[0], r, sizeof(r));
        return 1;
    }
    if (region == 2) {
        if (thin) return 0;
        const int r[4] = {wx, w, nx - 2 * wx, ny - 2 * w};
        std::memcpy(rects[0], r, sizeof(r));
        return 1;
    }
    const int f[4][4] = {{0, 0, nx, w}, {0, ny - w, nx, w}, {0, w, wx, ny - 2 * w}, {nx - wx, w, wx, ny - 2 * w}};
    std::memcpy(rects, f, sizeof(f));
    return 4;
}

}  // namespace

namespace {
int sweep_region_impl(mb4cu_ctx* ctx, double h, int s, int final_guess, int region, int grid_cap, double* dev_out7,
                      const int* skip, bool count);
}  // namespace

int mb4cu_sweep_region(mb4cu_ctx* ctx, double h, int s, int final_guess, int region, int grid_cap,
                       double* dev_out7) {
    return sweep_region_impl(ctx, h, s, final_guess, region, grid_cap, dev_out7, nullptr, true);
}

namespace {
int sweep_region_impl(mb4cu_ctx* ctx, double h, int s, int final_guess, int region, int grid_cap, double* dev_out7,
                      const int* skip, bool count) {
    if (!ctx || ctx->ghost <= 0) return fail(ctx, MB4CU_INVALID, "sweep: sub-domain contexts only");
    if (!(h > 0.0) || s < 0 || region < 0 || region > 2 || (region != 1 && !dev_out7))
        return fail(ctx, MB4CU_INVALID, "sweep: h > 0, s >= 0, region 0..2, output buffer");
    MB4_CUDA(ctx, cudaSetDevice(ctx->device));
    const SweepConsts c = make_consts(ctx, h);
    int rects[4][4];
    const int nrect = region_rects(ctx, region, rects, s);
    mb4cu::BatchCtl skipctl{};
    skipctl.skip = skip;
    // the frame (or the whole domain) starts the residual max; the interior adds to it
    if (region != 2) MB4_CUDA(ctx, cudaMemsetAsync(ctx->d_rmax_arr, 0, 2 * sizeof(unsigned long long), ctx->stream));
    if (nrect > 0) {
        MB4_CUDA(ctx, mb4cu::launch_step_march2(ctx->mf, ctx->m, ctx->nx, ctx->ny, ctx->u0, ctx->V, ctx->U,
                                                ctx->d_rmax_arr, ctx->d_obs_march, ctx->d_status, 1, -1.0,
                                                s == 0 ? 1 : 0, c, ctx->device, ctx->stream, ctx->ghost, s,
                                                final_guess && s > 0 ? s : -1, nrect, rects, region == 2 ? 1 : 0,
                                                region == 2 ? grid_cap : 0, skip ? &skipctl : nullptr, ctx->pitch,
                                                ctx->d_work, 0,
                                                s > 0 ? ctx->work_seq++ % mb4cu::kWorkCounters : -1));
        if (ctx->profiling) ctx->prof.launches += 1;
    }
    if (region != 1) {
        // [local ||r||_inf, the 5 energy sums of u0, max|u0|^2 (s = 0)] -> the caller's device buffer
        static_assert(offsetof(mb4cu::StepStatus, obs) == offsetof(mb4cu::StepStatus, rlast) + sizeof(double) &&
                          offsetof(mb4cu::StepStatus, amax2) ==
                              offsetof(mb4cu::StepStatus, obs) + sizeof(double) * mb4cu::kObsFields,
                      "rlast, obs and amax2 are contiguous");
        MB4_CUDA(ctx, cudaMemcpyAsync(dev_out7, reinterpret_cast<const char*>(ctx->d_status) +
                                                    offsetof(mb4cu::StepStatus, rlast),
                                      sizeof(double) * (2 + mb4cu::kObsFields), cudaMemcpyDeviceToDevice, ctx->stream));
        if (ctx->profiling && count) {
            ctx->prof.sweeps += 1;
            ctx->prof.alg_bytes += static_cast<double>(ctx->n) * (s == 0 ? 72.0 : (final_guess ? 88.0 : 120.0));
        }
    }
    return MB4CU_OK;
}
}  // namespace

int mb4cu_sweep_async(mb4cu_ctx* ctx, double h, int s, int final_guess, double* dev_out7) {
    return mb4cu_sweep_region(ctx, h, s, final_guess, 0, 0, dev_out7);
}

int mb4cu_commit_step(mb4cu_ctx* ctx, int sweeps) {
    if (!ctx || sweeps < 1) return fail(ctx, MB4CU_INVALID, "commit_step: sweeps must be >= 1");
    std::swap(ctx->u0, ctx->U[(sweeps - 1) & 1][2]);
    ctx->obs_cached = false;
    return MB4CU_OK;
}

int mb4cu_observables_sums(mb4cu_ctx* ctx, double* sums) {
    if (!ctx || !sums) return fail(ctx, MB4CU_INVALID, "observables_sums: null argument");
    mb4cu_obs tmp{};
    const int rc = mb4cu_observables(ctx, &tmp);
    // the raw sums are left in h_obs5 by mb4cu_observables (also on health-check failure)
    for (int f = 0; f < mb4cu::kObsFields; ++f) sums[f] = ctx->h_obs5[f];
    return rc == MB4CU_NUMERIC ? MB4CU_OK : rc;
}

// ---- parity entry points on host arrays -------------------------------------

namespace {

struct DevBuf {
    void* p = nullptr;
    ~DevBuf() { cudaFree(p); }
};

}  // namespace

static int kv_common(mb4cu_ctx* ctx, const double* u, double* y, bool rhs) {
    if (!ctx || !u || !y) return fail(ctx, MB4CU_INVALID, "apply_kv: null argument");
    MB4_CUDA(ctx, cudaSetDevice(ctx->device));
    DevBuf du, dy;
    const size_t sb = ctx->n * sizeof(double2);
    MB4_CUDA(ctx, cudaMalloc(&du.p, sb));
    MB4_CUDA(ctx, cudaMalloc(&dy.p, sb));
    MB4_CUDA(ctx, cudaMemcpyAsync(du.p, u, sb, cudaMemcpyHostToDevice, ctx->stream));
    MB4_CUDA(ctx, mb4cu::launch_apply_kv(ctx->nx, ctx->ny, ctx->cx, ctx->cy,
                                         static_cast<const double2*>(du.p), ctx->V, ctx->gamma, rhs,
                                         static_cast<double2*>(dy.p), ctx->stream));
    MB4_CUDA(ctx, cudaMemcpyAsync(y, dy.p, sb, cudaMemcpyDeviceToHost, ctx->stream));
    MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return MB4CU_OK;
}

int mb4cu_apply_kv(mb4cu_ctx* ctx, const double* u, double* y) { return kv_common(ctx, u, y, false); }

int mb4cu_rhs(mb4cu_ctx* ctx, const double* u, double* y) { return kv_common(ctx, u, y, true); }

int mb4cu_eval_phi(mb4cu_ctx* ctx, const double* u0, const double* s1, const double* s2,
                   const double* s3, double h, double* p1, double* p2, double* p3) {
    if (!ctx || !u0 || !s1 || !s2 || !s3 || !p1 || !p2 || !p3)
        return fail(ctx, MB4CU_INVALID, "eval_phi: null argument");
    MB4_CUDA(ctx, cudaSetDevice(ctx->device));
    const size_t sb = ctx->n * sizeof(double2);
    DevBuf bufs[7];
    for (auto& b : bufs) MB4_CUDA(ctx, cudaMalloc(&b.p, sb));
    const double* hin[4] = {u0, s1, s2, s3};
    for (int i = 0; i < 4; ++i)
        MB4_CUDA(ctx, cudaMemcpyAsync(bufs[i].p, hin[i], sb, cudaMemcpyHostToDevice, ctx->stream));
    const double2* st[3] = {static_cast<const double2*>(bufs[1].p), static_cast<const double2*>(bufs[2].p),
                            static_cast<const double2*>(bufs[3].p)};
    double2* ph[3] = {static_cast<double2*>(bufs[4].p), static_cast<double2*>(bufs[5].p),
                      static_cast<double2*>(bufs[6].p)};
    const SweepConsts c = make_consts(ctx, h);
    MB4_CUDA(ctx, mb4cu::launch_eval_phi(ctx->nx, ctx->ny, static_cast<const double2*>(bufs[0].p),
                                         ctx->V, st, ph, c, ctx->stream));
    double* hout[3] = {p1, p2, p3};
    for (int i = 0; i < 3; ++i)
        MB4_CUDA(ctx, cudaMemcpyAsync(hout[i], ph[i], sb, cudaMemcpyDeviceToHost, ctx->stream));
    MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return MB4CU_OK;
}


// ---- Stage-split Newton-Krylov (the paper's 3-way stage partition) --------------
// The simplified Newton iteration of substep_krylov, opened up so that the three
// decoupled stage solves of an iteration can run on different devices / processes:
//   ns_begin(h); repeat { ns_phibar; ns_solve(k) for the owned k; exchange the
//   corrections (ns_get/set_correction); ns_update -> ||r||_inf } until r <= eps;
//   ns_commit.  The same kernels and GMRES as substep_krylov: a context that solves all
//   three systems itself reproduces it bit for bit.
static double2* ns_b(mb4cu_ctx* ctx, int k) { return kr_vec(ctx, ctx->kr.m + 1 + k); }
static double2* ns_x(mb4cu_ctx* ctx, int k) { return kr_vec(ctx, ctx->kr.m + 4 + k); }

int mb4cu_ns_begin(mb4cu_ctx* ctx, double h) {
    if (!ctx) return MB4CU_INVALID;
    if (!(h > 0.0)) return fail(ctx, MB4CU_INVALID, "ns_begin: h must be positive");
    if (ctx->ghost > 0) return fail(ctx, MB4CU_INVALID, "ns_begin: needs a whole-lattice context");
    MB4_CUDA(ctx, cudaSetDevice(ctx->device));
    if (int rc = refresh_amax2(ctx)) return rc;
    if (int rc = kr_alloc(ctx, ctx->n)) return rc;
    ctx->ns_c = make_consts(ctx, h);
    ctx->ns_h = h;
    const size_t sb = ctx->n * sizeof(double2);
    for (int i = 0; i < 3; ++i)
        MB4_CUDA(ctx, cudaMemcpyAsync(ctx->U[0][i], ctx->u0, sb, cudaMemcpyDeviceToDevice, ctx->stream));
    if (int rc = fft_prepare(ctx, 1)) return rc;
    ctx->ns_open = true;
    return MB4CU_OK;
}

int mb4cu_ns_phibar(mb4cu_ctx* ctx) {
    if (!ctx || !ctx->ns_open) return fail(ctx, MB4CU_INVALID, "ns_phibar: no open step (ns_begin)");
    const double2* cst[3] = {ctx->U[0][0], ctx->U[0][1], ctx->U[0][2]};
    double2* b[3] = {ns_b(ctx, 0), ns_b(ctx, 1), ns_b(ctx, 2)};
    MB4_CUDA(ctx, mb4cu::kr_phibar(ctx->nx, ctx->ny, ctx->u0, cst, ctx->V, b, ctx->ns_c, ctx->stream));
    return MB4CU_OK;
}

int mb4cu_ns_solve(mb4cu_ctx* ctx, int k) {
    if (!ctx || !ctx->ns_open || k < 0 || k > 2) return fail(ctx, MB4CU_INVALID, "ns_solve: open step, k in 0..2");
    const SweepConsts& c = ctx->ns_c;
    const double hl = c.hlam[k];
    auto mv = [&](const double2* xin, double2* yout) {
        return mb4cu::kr_matvec(xin, yout, ctx->u0, ctx->V, ctx->nx, ctx->ny, hl, c, ctx->stream);
    };
    return kr_gmres_fft(ctx, 1, hl, nullptr, mv, ns_b(ctx, k), ns_x(ctx, k));
}

int mb4cu_ns_get_correction(mb4cu_ctx* ctx, int k, double* dev_out) {
    if (!ctx || !ctx->ns_open || k < 0 || k > 2 || !dev_out)
        return fail(ctx, MB4CU_INVALID, "ns_get_correction: open step, k in 0..2, buffer");
    MB4_CUDA(ctx, cudaMemcpyAsync(dev_out, ns_x(ctx, k), ctx->n * sizeof(double2), cudaMemcpyDeviceToDevice,
                                  ctx->stream));
    return MB4CU_OK;
}

int mb4cu_ns_set_correction(mb4cu_ctx* ctx, int k, const double* dev_in) {
    if (!ctx || !ctx->ns_open || k < 0 || k > 2 || !dev_in)
        return fail(ctx, MB4CU_INVALID, "ns_set_correction: open step, k in 0..2, buffer");
    MB4_CUDA(ctx, cudaMemcpyAsync(ns_x(ctx, k), dev_in, ctx->n * sizeof(double2), cudaMemcpyDeviceToDevice,
                                  ctx->stream));
    return MB4CU_OK;
}

int mb4cu_ns_update(mb4cu_ctx* ctx, double* rmax) {
    if (!ctx || !ctx->ns_open || !rmax) return fail(ctx, MB4CU_INVALID, "ns_update: open step, output");
    double2* st[3] = {ctx->U[0][0], ctx->U[0][1], ctx->U[0][2]};
    const double2* cx[3] = {ns_x(ctx, 0), ns_x(ctx, 1), ns_x(ctx, 2)};
    MB4_CUDA(ctx, cudaMemsetAsync(ctx->d_rmax, 0, sizeof(unsigned long long), ctx->stream));
    MB4_CUDA(ctx, mb4cu::kr_update(st, cx, ctx->n, ctx->d_rmax, ctx->ns_c, ctx->stream));
    MB4_CUDA(ctx, cudaMemcpyAsync(ctx->h_rmax, ctx->d_rmax, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                  ctx->stream));
    MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    *rmax = decode_bits(*ctx->h_rmax);
    return MB4CU_OK;
}

int mb4cu_ns_get_stages(mb4cu_ctx* ctx, double* u1, double* u2, double* u3) {
    if (!ctx || !ctx->ns_open || !u1 || !u2 || !u3)
        return fail(ctx, MB4CU_INVALID, "ns_get_stages: open step, three host buffers");
    double* out[3] = {u1, u2, u3};
    for (int i = 0; i < 3; ++i)
        MB4_CUDA(ctx, cudaMemcpyAsync(out[i], ctx->U[0][i], ctx->n * sizeof(double2), cudaMemcpyDeviceToHost,
                                      ctx->stream));
    MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return MB4CU_OK;
}

int mb4cu_ns_abort(mb4cu_ctx* ctx) {
    if (!ctx || !ctx->ns_open) return fail(ctx, MB4CU_INVALID, "ns_abort: no open step");
    ctx->ns_open = false;
    return MB4CU_OK;
}

int mb4cu_ns_commit(mb4cu_ctx* ctx) {
    if (!ctx || !ctx->ns_open) return fail(ctx, MB4CU_INVALID, "ns_commit: no open step");
    std::swap(ctx->u0, ctx->U[0][2]);
    ctx->obs_cached = false;
    ctx->ns_open = false;
    return MB4CU_OK;
}

// ---- Native multi-GPU stepping over NCCL (mb4cu_dist_*) -----------------------------
// The decomposed step without the host in the sweep loop: per sweep the boundary frame,
// its ghost-wide halo exchange (NCCL send / recv on a communication stream) concurrently
// with the interior, the all-reduce of [||r||_inf, energy sums, max|u0|^2] and the
// convergence test on the device (dist_converge_kernel), whose flag turns the sweeps
// enqueued ahead into no-ops.  The host enqueues the sweeps the previous step's count
// predicts and reads once per step when the prediction holds (dist.py's Python loop reads
// once per sweep).  Every NCCL call of a communicator goes through its one stream, in
// the same order on every rank.  libnccl is opened at run time (the process's own, e.g.
// torch's), so single-GPU users do not depend on it.

struct NcclApi {
    void* so = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
};

namespace {

bool nccl_open(NcclApi& api, const char* path, std::string& why) {
    const char* name = path && *path ? path : "libnccl.so.2";
    api.so = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
    if (!api.so) {
        why = std::string("dlopen(") + name + "): " + dlerror();
        return false;
    }
    bool ok = true;
    auto sym = [&](auto& fn, const char* s) {
        fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(api.so, s));
        if (!fn) {
            ok = false;
            why = std::string("libnccl lacks ") + s;
        }
    };
    sym(api.getUniqueId, "ncclGetUniqueId");
    sym(api.commInitRank, "ncclCommInitRank");
    sym(api.commDestroy, "ncclCommDestroy");
    sym(api.groupStart, "ncclGroupStart");
    sym(api.groupEnd, "ncclGroupEnd");
    sym(api.send, "ncclSend");
    sym(api.recv, "ncclRecv");
    sym(api.allReduce, "ncclAllReduce");
    sym(api.errorString, "ncclGetErrorString");
    return ok;
}

constexpr int kOutStride = 8;  // doubles per sweep row of the reduction buffer (7 used)

}  // namespace

struct DistNative {
    NcclApi api;
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0, px = 1, py = 1;
    int nbr[4] = {0, 0, 0, 0};    // west, east, south, north neighbour ranks
    bool force_p2p = false;       // exchange through NCCL even with oneself (tests on one GPU)
    int grid_cap = 0;             // interior launches leave SMs to NCCL's kernels
    cudaStream_t comms = nullptr;
    cudaEvent_t ev_frame = nullptr, ev_int = nullptr, ev_x = nullptr;
    double* d_out = nullptr;      // [max_iters][kOutStride]
    double* h_out = nullptr;      // pinned
    int* d_state = nullptr;       // [4]: done, sweeps, diverged
    int* h_state = nullptr;       // pinned
    double* sbuf[4] = {nullptr, nullptr, nullptr, nullptr};
    double* rbuf[4] = {nullptr, nullptr, nullptr, nullptr};
    size_t cap = 0;               // doubles per halo buffer
    double2* u0bak = nullptr;     // halving backup (padded array)
    bool u0_halo_ok = false;
};

namespace {

#define MB4_NCCL(ctx, call)                                                                       \
    do {                                                                                          \
        const ncclResult_t r_ = (call);                                                           \
        if (r_ != ncclSuccess)                                                                    \
            return fail(ctx, MB4CU_COMM_ERROR,                                                    \
                        std::string("NCCL: ") + (ctx)->dn->api.errorString(r_) + " at " #call);  \
    } while (0)

int dn_exchange(mb4cu_ctx* ctx, int field) {
    DistNative& D = *ctx->dn;
    const struct {
        int lo, hi, extent;
    } phases[2] = {{0, 1, D.px}, {2, 3, D.py}};
    for (const auto& ph : phases) {
        if (ph.extent == 1 && !D.force_p2p) {
            // this rank is its own neighbour: owned strips straight into the opposite ghosts
            double2* arr[3] = {ctx->u0, nullptr, nullptr};
            int narr = 1;
            if (field >= 2) {
                narr = 3;
                for (int q = 0; q < 3; ++q) arr[q] = ctx->U[(field - 2) & 1][q];
            }
            MB4_CUDA(ctx, mb4cu::launch_halo_wrap(field == 1 ? nullptr : arr, field == 1 ? ctx->V : nullptr, narr,
                                                  ctx->pitch, ctx->ghost, ctx->nx, ctx->ny, halo_width(ctx, field),
                                                  &ph == &phases[0] ? 0 : 1, D.comms));
            ctx->prof.other_launches += 1;
            continue;
        }
        const size_t n = mb4cu_halo_count(ctx, field, ph.lo);
        const int sides[2] = {ph.lo, ph.hi};
        for (int side : sides) {
            int x0, y0, w, h;
            halo_rect(ctx, field, side, true, &x0, &y0, &w, &h);
            if (field == 1) {
                MB4_CUDA(ctx, mb4cu::launch_halo_copy1(ctx->V, ctx->pitch, ctx->ghost, x0, y0, w, h, D.sbuf[side],
                                                       true, D.comms));
            } else {
                double2* arr[3] = {ctx->u0, nullptr, nullptr};
                int narr = 1;
                if (field != 0) {
                    narr = 3;
                    for (int q = 0; q < 3; ++q) arr[q] = ctx->U[(field - 2) & 1][q];
                }
                MB4_CUDA(ctx, mb4cu::launch_halo_copy2(arr, narr, ctx->pitch, ctx->ghost, x0, y0, w, h,
                                                       reinterpret_cast<double2*>(D.sbuf[side]), true, D.comms));
            }
        }
        double* src_for_hi = D.sbuf[ph.lo];  // periodic wrap onto this rank: my low strip is my high ghost
        double* src_for_lo = D.sbuf[ph.hi];
        if (ph.extent > 1 || D.force_p2p) {
            // sends [low strip -> low neighbour, high strip -> high neighbour], receives
            // [high ghost <- high neighbour, low ghost <- low neighbour] (dist.HaloExchange's
            // order: correct when both neighbours are the same rank, or this rank)
            MB4_NCCL(ctx, D.api.groupStart());
            MB4_NCCL(ctx, D.api.send(D.sbuf[ph.lo], n, ncclDouble, D.nbr[ph.lo], D.comm, D.comms));
            MB4_NCCL(ctx, D.api.send(D.sbuf[ph.hi], n, ncclDouble, D.nbr[ph.hi], D.comm, D.comms));
            MB4_NCCL(ctx, D.api.recv(D.rbuf[ph.hi], n, ncclDouble, D.nbr[ph.hi], D.comm, D.comms));
            MB4_NCCL(ctx, D.api.recv(D.rbuf[ph.lo], n, ncclDouble, D.nbr[ph.lo], D.comm, D.comms));
            MB4_NCCL(ctx, D.api.groupEnd());
            src_for_hi = D.rbuf[ph.hi];
            src_for_lo = D.rbuf[ph.lo];
        }
        const int dst[2] = {ph.hi, ph.lo};
        double* src[2] = {src_for_hi, src_for_lo};
        for (int k = 0; k < 2; ++k) {
            int x0, y0, w, h;
            halo_rect(ctx, field, dst[k], false, &x0, &y0, &w, &h);
            if (field == 1) {
                MB4_CUDA(ctx, mb4cu::launch_halo_copy1(ctx->V, ctx->pitch, ctx->ghost, x0, y0, w, h, src[k], false,
                                                       D.comms));
            } else {
                double2* arr[3] = {ctx->u0, nullptr, nullptr};
                int narr = 1;
                if (field != 0) {
                    narr = 3;
                    for (int q = 0; q < 3; ++q) arr[q] = ctx->U[(field - 2) & 1][q];
                }
                MB4_CUDA(ctx, mb4cu::launch_halo_copy2(arr, narr, ctx->pitch, ctx->ghost, x0, y0, w, h,
                                                       reinterpret_cast<double2*>(src[k]), false, D.comms));
            }
        }
        ctx->prof.other_launches += 4;
    }
    return MB4CU_OK;
}

// comms stream after everything enqueued so far on the compute stream, and vice versa
int dn_comms_after_compute(mb4cu_ctx* ctx) {
    MB4_CUDA(ctx, cudaEventRecord(ctx->dn->ev_int, ctx->stream));
    MB4_CUDA(ctx, cudaStreamWaitEvent(ctx->dn->comms, ctx->dn->ev_int, 0));
    return MB4CU_OK;
}
int dn_compute_after_comms(mb4cu_ctx* ctx) {
    MB4_CUDA(ctx, cudaEventRecord(ctx->dn->ev_x, ctx->dn->comms));
    MB4_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->dn->ev_x, 0));
    return MB4CU_OK;
}

// Sweep s of a decomposed sub-step, fully enqueued (no host wait): frame -> its exchange
// (comms) || interior -> all-reduce -> device convergence test (comms).
int dn_launch_sweep(mb4cu_ctx* ctx, double h, int s, bool final_guess) {
    DistNative& D = *ctx->dn;
    double* out = D.d_out + static_cast<size_t>(s) * kOutStride;
    MB4_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, D.ev_x, 0));  // input halos and the convergence flag
    if (int rc = sweep_region_impl(ctx, h, s, final_guess, 1, 0, nullptr, D.d_state, false)) return rc;
    MB4_CUDA(ctx, cudaEventRecord(D.ev_frame, ctx->stream));
    MB4_CUDA(ctx, cudaStreamWaitEvent(D.comms, D.ev_frame, 0));
    if (int rc = dn_exchange(ctx, 4 + (s & 1))) return rc;  // the frame's stage set, ghost wide
    if (int rc = sweep_region_impl(ctx, h, s, final_guess, 2, D.grid_cap, out, D.d_state, false)) return rc;
    if (int rc = dn_comms_after_compute(ctx)) return rc;
    MB4_NCCL(ctx, D.api.allReduce(out, out, 1, ncclDouble, ncclMax, D.comm, D.comms));
    if (s == 0) {
        MB4_NCCL(ctx, D.api.allReduce(out + 1, out + 1, mb4cu::kObsFields, ncclDouble, ncclSum, D.comm, D.comms));
        MB4_NCCL(ctx, D.api.allReduce(out + 6, out + 6, 1, ncclDouble, ncclMax, D.comm, D.comms));
    }
    MB4_CUDA(ctx, mb4cu::launch_dist_converge(D.d_out, kOutStride, s, ctx->eps, D.d_state, D.comms));
    MB4_CUDA(ctx, cudaEventRecord(D.ev_x, D.comms));
    ctx->prof.other_launches += 1;
    return MB4CU_OK;
}

int dn_read(mb4cu_ctx* ctx, int rows) {
    DistNative& D = *ctx->dn;
    MB4_CUDA(ctx, cudaMemcpyAsync(D.h_state, D.d_state, 4 * sizeof(int), cudaMemcpyDeviceToHost, D.comms));
    MB4_CUDA(ctx, cudaMemcpyAsync(D.h_out, D.d_out, sizeof(double) * kOutStride * rows, cudaMemcpyDeviceToHost,
                                  D.comms));
    MB4_CUDA(ctx, cudaStreamSynchronize(D.comms));
    return MB4CU_OK;
}

// global max|u0|^2 of a newly set state (all ranks), once per set_state
int dn_refresh_amax2(mb4cu_ctx* ctx) {
    if (ctx->amax2_valid) return MB4CU_OK;
    DistNative& D = *ctx->dn;
    if (int rc = dn_comms_after_compute(ctx)) return rc;  // (after the set_state copy)
    const size_t off = static_cast<size_t>(ctx->ghost) * ctx->pitch + ctx->ghost;
    MB4_CUDA(ctx, cudaMemsetAsync(ctx->d_rmax, 0, sizeof(unsigned long long), D.comms));
    MB4_CUDA(ctx, mb4cu::launch_amax2_2d(ctx->u0 + off, ctx->nx, ctx->ny, ctx->pitch, ctx->d_rmax, D.comms));
    // non-negative doubles: max of the bit patterns == max of the values; reduce as doubles
    MB4_NCCL(ctx, D.api.allReduce(ctx->d_rmax, ctx->d_rmax, 1, ncclDouble, ncclMax, D.comm, D.comms));
    MB4_CUDA(ctx, cudaMemcpyAsync(ctx->h_rmax, ctx->d_rmax, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                  D.comms));
    MB4_CUDA(ctx, cudaStreamSynchronize(D.comms));
    track_amax2(ctx, decode_bits(*ctx->h_rmax));
    return MB4CU_OK;
}

// One decomposed sub-step of size h: *sweeps, *last_res, entry sums5 + amax2 in out7.
int dn_substep(mb4cu_ctx* ctx, double h, int* sweeps, double* last_res, double* entry7) {
    DistNative& D = *ctx->dn;
    MB4_CUDA(ctx, cudaMemsetAsync(D.d_state, 0, 4 * sizeof(int), D.comms));
    if (!D.u0_halo_ok) {
        if (int rc = dn_comms_after_compute(ctx)) return rc;
        if (int rc = dn_exchange(ctx, 0)) return rc;
    }
    MB4_CUDA(ctx, cudaEventRecord(D.ev_x, D.comms));
    D.u0_halo_ok = false;
    const int guess = ctx->last_sweeps;  // the previous sub-step's count (0: none)
    const int ahead = std::min(std::max(guess, 1), ctx->max_iters);
    for (int s = 0; s < ahead; ++s)
        if (int rc = dn_launch_sweep(ctx, h, s, s > 0 && s == guess - 1)) return rc;
    int launched = ahead - 1;
    bool last_was_final = launched > 0 && launched == guess - 1;
    bool redone = false;
    for (;;) {
        if (int rc = dn_read(ctx, launched + 1)) return rc;
        std::memcpy(entry7, D.h_out + 1, sizeof(double) * 6);  // sweep 0: the entry state's sums, max|u0|^2
        const int done = D.h_state[0], diverged = D.h_state[2];
        if (diverged) {
            *last_res = INFINITY;
            ctx->last_sweeps = 0;
            return fail(ctx, MB4CU_NONCONVERGED, "stage iteration diverged (non-finite update)");
        }
        if (done) {
            const int sw = D.h_state[1];
            *sweeps = sw;
            *last_res = D.h_out[static_cast<size_t>(sw - 1) * kOutStride];
            mb4cu_commit_step(ctx, sw);
            D.u0_halo_ok = true;  // the last sweep's exchange carried U3 ghost wide
            ctx->last_sweeps = sw;
            track_amax2(ctx, D.h_out[6]);
            adapt_neumann(ctx, sw);
            if (ctx->profiling) {
                ctx->prof.sweeps += sw;
                const bool spec_hit = sw >= 2 && sw == guess && !redone;  // the U3-only final sweep converged
                ctx->prof.alg_bytes += static_cast<double>(ctx->n) * (72.0 + 120.0 * (sw - 1) - (spec_hit ? 32.0 : 0.0));
            }
            return MB4CU_OK;
        }
        *last_res = D.h_out[static_cast<size_t>(launched) * kOutStride];
        if (last_was_final) {
            // the predicted final sweep stored U3 only and did not converge: repeat it with all stages
            if (int rc = dn_launch_sweep(ctx, h, launched, false)) return rc;
            last_was_final = false;
            redone = true;
            ctx->prof.redone += 1;
            continue;
        }
        if (launched + 1 >= ctx->max_iters) break;
        ++launched;
        if (int rc = dn_launch_sweep(ctx, h, launched, false)) return rc;
    }
    ctx->last_sweeps = 0;
    return fail(ctx, MB4CU_NONCONVERGED,
                "stage iteration: no convergence after " + std::to_string(ctx->max_iters) + " sweeps");
}

void dn_state_set(mb4cu_ctx* ctx) {
    if (ctx->dn) ctx->dn->u0_halo_ok = false;
}

void dn_free(mb4cu_ctx* ctx) {
    DistNative* D = ctx->dn;
    if (!D) return;
    if (D->comms) cudaStreamSynchronize(D->comms);
    if (D->comm && D->api.commDestroy) D->api.commDestroy(D->comm);
    for (int k = 0; k < 4; ++k) {
        cudaFree(D->sbuf[k]);
        cudaFree(D->rbuf[k]);
    }
    cudaFree(D->d_out);
    cudaFreeHost(D->h_out);
    cudaFree(D->d_state);
    cudaFreeHost(D->h_state);
    cudaFree(D->u0bak);
    if (D->ev_frame) cudaEventDestroy(D->ev_frame);
    if (D->ev_int) cudaEventDestroy(D->ev_int);
    if (D->ev_x) cudaEventDestroy(D->ev_x);
    if (D->comms) cudaStreamDestroy(D->comms);
    delete D;
    ctx->dn = nullptr;
}

}  // namespace

int mb4cu_nccl_unique_id(const char* libnccl, unsigned char id[128]) {
    g_create_error.clear();
    if (!id) return MB4CU_INVALID;
    NcclApi api;
    if (!nccl_open(api, libnccl, g_create_error)) return MB4CU_COMM_ERROR;
    ncclUniqueId u;
    const ncclResult_t r = api.getUniqueId(&u);
    if (r != ncclSuccess) {
        g_create_error = std::string("ncclGetUniqueId: ") + api.errorString(r);
        return MB4CU_COMM_ERROR;
    }
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId layout");
    std::memcpy(id, &u, 128);
    return MB4CU_OK;
}

int mb4cu_dist_attach(mb4cu_ctx* ctx, const char* libnccl, const unsigned char id[128], int nranks, int rank,
                      const int neighbours[4], int px, int py, int grid_cap, int force_p2p, int adaptive_m) {
    if (!ctx || ctx->ghost <= 0 || !id || !neighbours || nranks < 1 || rank < 0 || rank >= nranks || px < 1 ||
        py < 1 || px * py != nranks)
        return fail(ctx, MB4CU_INVALID, "dist_attach: sub-domain context, id, neighbours, px * py == nranks");
    if (ctx->kernel != 0 || !mb4cu::march2_supported(ctx->mf, ctx->m) || ctx->mf < 4)
        return fail(ctx, MB4CU_INVALID, "dist_attach: the production sweep kernels (neumann_first >= 4)");
    if (ctx->dn) return fail(ctx, MB4CU_INVALID, "dist_attach: already attached");
    MB4_CUDA(ctx, cudaSetDevice(ctx->device));
    ctx->dn = new DistNative();
    DistNative& D = *ctx->dn;
    std::string why;
    if (!nccl_open(D.api, libnccl, why)) {
        dn_free(ctx);
        return fail(ctx, MB4CU_COMM_ERROR, why);
    }
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    D.nranks = nranks;
    D.rank = rank;
    D.px = px;
    D.py = py;
    for (int k = 0; k < 4; ++k) D.nbr[k] = neighbours[k];
    D.force_p2p = force_p2p != 0;
    D.grid_cap = grid_cap;
    auto bail = [&](int rc) {
        dn_free(ctx);
        return rc;
    };
    const ncclResult_t r = D.api.commInitRank(&D.comm, nranks, u, rank);
    if (r != ncclSuccess) {
        const std::string e = std::string("ncclCommInitRank: ") + D.api.errorString(r);
        dn_free(ctx);
        return fail(ctx, MB4CU_COMM_ERROR, e);
    }
    cudaError_t e;
    if ((e = cudaStreamCreateWithFlags(&D.comms, cudaStreamNonBlocking)) != cudaSuccess) return bail(cuda_fail(ctx, e, "stream"));
    if ((e = cudaEventCreateWithFlags(&D.ev_frame, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&D.ev_int, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&D.ev_x, cudaEventDisableTiming)) != cudaSuccess)
        return bail(cuda_fail(ctx, e, "event"));
    for (int f = 0; f < 6; ++f)
        for (int side = 0; side < 4; ++side) D.cap = std::max(D.cap, mb4cu_halo_count(ctx, f, side));
    for (int k = 0; k < 4; ++k)
        if ((e = cudaMalloc(&D.sbuf[k], D.cap * sizeof(double))) != cudaSuccess ||
            (e = cudaMalloc(&D.rbuf[k], D.cap * sizeof(double))) != cudaSuccess)
            return bail(cuda_fail(ctx, e, "cudaMalloc(halo)"));
    if ((e = cudaMalloc(&D.d_out, sizeof(double) * kOutStride * (ctx->max_iters + 1))) != cudaSuccess ||
        (e = cudaMallocHost(&D.h_out, sizeof(double) * kOutStride * (ctx->max_iters + 1))) != cudaSuccess ||
        (e = cudaMalloc(&D.d_state, 4 * sizeof(int))) != cudaSuccess ||
        (e = cudaMallocHost(&D.h_state, 4 * sizeof(int))) != cudaSuccess)
        return bail(cuda_fail(ctx, e, "cudaMalloc(dist)"));
    // the whole lattice's max|V| and min V: every rank then places the same Chebyshev
    // polynomial (and the same later-sweep depth policy) as the single domain would
    double* d2 = nullptr;
    if ((e = cudaMalloc(&d2, 2 * sizeof(double))) != cudaSuccess) return bail(cuda_fail(ctx, e, "cudaMalloc"));
    const double h2[2] = {ctx->vmax, -ctx->vmin};
    cudaMemcpy(d2, h2, sizeof(h2), cudaMemcpyHostToDevice);
    const ncclResult_t r2 = D.api.allReduce(d2, d2, 2, ncclDouble, ncclMax, D.comm, D.comms);
    double g2[2] = {0.0, 0.0};
    cudaStreamSynchronize(D.comms);
    cudaMemcpy(g2, d2, sizeof(g2), cudaMemcpyDeviceToHost);
    cudaFree(d2);
    if (r2 != ncclSuccess) return bail(fail(ctx, MB4CU_COMM_ERROR, "NCCL all-reduce of max|V|"));
    ctx->vmax = g2[0];
    ctx->vmin = -g2[1];
    if (ctx->first_poly_auto) ctx->first_poly = ctx->vmin >= 0.0 && ctx->gamma <= 0.0 ? 2 : 1;
    ctx->rho_override = 0.0;
    ctx->m_auto = adaptive_m != 0 && mb4cu::march2_supported(ctx->mf, 2) && ctx->ghost >= 3;
    ctx->last_sweeps = 0;
    // V halos once (stream-ordered after set_state / create)
    if (int rc = dn_comms_after_compute(ctx)) return bail(rc);
    if (int rc = dn_exchange(ctx, 1)) return bail(rc);
    if ((e = cudaStreamSynchronize(D.comms)) != cudaSuccess) return bail(cuda_fail(ctx, e, "exchange(V)"));
    return MB4CU_OK;
}

int mb4cu_dist_step(mb4cu_ctx* ctx, double h, mb4cu_stats* stats, double* entry_sums5) {
    if (!ctx || !ctx->dn) return fail(ctx, MB4CU_INVALID, "dist_step: no NCCL transport (mb4cu_dist_attach)");
    if (!(h > 0.0)) return fail(ctx, MB4CU_INVALID, "mb4_step: h must be positive");
    MB4_CUDA(ctx, cudaSetDevice(ctx->device));
    DistNative& D = *ctx->dn;
    if (int rc = dn_refresh_amax2(ctx)) return rc;
    double last = 0.0, entry7[6] = {0, 0, 0, 0, 0, 0};
    int rc = MB4CU_NONCONVERGED, used = 0, total = 0;
    const size_t pb = ctx->alloc_n * sizeof(double2);
    for (int hv = 0; hv <= ctx->max_halvings; ++hv) {
        const int sub = 1 << hv;
        if (hv == 1) {
            if (!D.u0bak) MB4_CUDA(ctx, cudaMalloc(&D.u0bak, pb));
            // (the first attempt left u0 untouched: only commits move it)
            MB4_CUDA(ctx, cudaMemcpyAsync(D.u0bak, ctx->u0, pb, cudaMemcpyDeviceToDevice, ctx->stream));
        } else if (hv > 1) {
            MB4_CUDA(ctx, cudaMemcpyAsync(ctx->u0, D.u0bak, pb, cudaMemcpyDeviceToDevice, ctx->stream));
            D.u0_halo_ok = false;
        }
        bool ok = true;
        int attempt = 0;
        for (int k = 0; k < sub; ++k) {
            int sw = 0;
            double e7[6] = {0, 0, 0, 0, 0, 0};
            rc = dn_substep(ctx, h / sub, &sw, &last, e7);
            if (hv == 0 && k == 0) std::memcpy(entry7, e7, sizeof(e7));  // the step's entry state
            attempt += sw;
            if (rc == MB4CU_NONCONVERGED) {
                ok = false;
                break;
            }
            if (rc != MB4CU_OK) return rc;
        }
        if (ok) {
            used = hv;
            total = attempt;
            rc = MB4CU_OK;
            break;
        }
    }
    if (rc != MB4CU_OK) {
        if (ctx->max_halvings >= 1 && D.u0bak) {
            MB4_CUDA(ctx, cudaMemcpyAsync(ctx->u0, D.u0bak, pb, cudaMemcpyDeviceToDevice, ctx->stream));
            D.u0_halo_ok = false;
        }
        MB4_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        if (stats) stats->last_residual = last;
        return fail(ctx, MB4CU_NONCONVERGED,
                    "mb4_step: no convergence after " + std::to_string(ctx->max_halvings) + " step halvings");
    }
    if (entry_sums5) std::memcpy(entry_sums5, entry7, sizeof(double) * mb4cu::kObsFields);
    if (stats) {
        stats->newton_iters += total;
        stats->halvings += used;
        stats->last_residual = last;
    }
    return MB4CU_OK;
}

int mb4cu_dist_observables(mb4cu_ctx* ctx, double* sums5) {
    if (!ctx || !ctx->dn || !sums5) return fail(ctx, MB4CU_INVALID, "dist_observables: attached context, output");
    DistNative& D = *ctx->dn;
    MB4_CUDA(ctx, cudaSetDevice(ctx->device));
    if (!D.u0_halo_ok) {
        if (int rc = dn_comms_after_compute(ctx)) return rc;
        if (int rc = dn_exchange(ctx, 0)) return rc;
        D.u0_halo_ok = true;
    }
    if (int rc = dn_compute_after_comms(ctx)) return rc;
    mb4cu::ObsArgs a{};
    a.nx = ctx->nx;
    a.ny = ctx->ny;
    a.cx = ctx->cx;
    a.cy = ctx->cy;
    a.diag = 2.0 * ctx->cx + 2.0 * ctx->cy;
    a.u = ctx->u0;
    a.V = ctx->V;
    a.partial = ctx->d_obs_partial;
    MB4_CUDA(ctx, mb4cu::launch_observables_ghost(a, ctx->ghost, ctx->pitch, ctx->d_obs5, ctx->stream));
    if (int rc = dn_comms_after_compute(ctx)) return rc;
    MB4_NCCL(ctx, D.api.allReduce(ctx->d_obs5, ctx->d_obs5, mb4cu::kObsFields, ncclDouble, ncclSum, D.comm, D.comms));
    MB4_CUDA(ctx, cudaMemcpyAsync(ctx->h_obs5, ctx->d_obs5, sizeof(double) * mb4cu::kObsFields,
                                  cudaMemcpyDeviceToHost, D.comms));
    MB4_CUDA(ctx, cudaStreamSynchronize(D.comms));
    std::memcpy(sums5, ctx->h_obs5, sizeof(double) * mb4cu::kObsFields);
    return MB4CU_OK;
}

int mb4cu_dist_detach(mb4cu_ctx* ctx) {
    if (!ctx) return MB4CU_INVALID;
    dn_free(ctx);
    return MB4CU_OK;
}
}  // extern "C"
