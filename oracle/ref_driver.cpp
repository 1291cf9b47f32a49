// oracle/ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference library (compiled by
// oracle/Makefile from /root/reference/proj/src into oracle/_ref/).  It lets
// the Python tests and bench.py's reference arm drive the reference's own
// public API (proj/include/nls2d) with BASELINE inputs:
//   GridModel(GridSpec(nx,ny,lx,ly), gamma, V)                lattice.hpp:52
//   StepDriver(model, MethodId::Mb4, NewtonConfig, solver, pool) integrators.hpp:48-51
//   advance(u, h, &stats) per step, observables(model, u)       integrators.hpp:51, lattice.hpp:88
// Nothing here re-implements the algorithm; it only marshals plain arrays.
#include <chrono>
#include <complex>
#include <cstring>
#include <exception>
#include <vector>

#include "nls2d/harness.hpp"
#include "nls2d/integrators.hpp"
#include "nls2d/lattice.hpp"
#include "nls2d/mb4_integrator.hpp"
#include "nls2d/mb4_scheme.hpp"
#include "nls2d/worker_pool.hpp"

using namespace nls2d;

namespace {

State to_state(const double* u, int n) {
    State s(n);
    std::memcpy(static_cast<void*>(s.data()), u, sizeof(double) * 2 * n);
    return s;
}

void put_obs(double* row, const Observables& o) {
    row[0] = o.u_kinetic;
    row[1] = o.u_nonlinear;
    row[2] = o.u_external;
    row[3] = o.total_energy;
    row[4] = o.probability;
    row[5] = o.participation;
    row[6] = o.raw_quartic;
}

}  // namespace

extern "C" {

// Scheme constants exactly as the reference computes them (mb4_scheme.cpp:83-125).
int ref_scheme(double* e /*12*/, double* w /*192*/, double* lam /*3*/, double* t /*9*/,
               double* tinv /*9*/) {
    try {
        const Mb4Scheme s;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 4; ++j) e[i * 4 + j] = s.e_ext(i + 1, j);
        for (int i = 0; i < 3; ++i)
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < 4; ++b)
                    for (int c = 0; c < 4; ++c) w[((i * 4 + a) * 4 + b) * 4 + c] = s.w(i + 1, a, b, c);
        for (int i = 0; i < 3; ++i) {
            lam[i] = s.eigenvalues()[i];
            for (int j = 0; j < 3; ++j) {
                t[i * 3 + j] = s.t()(i, j);
                tinv[i * 3 + j] = s.t_inv()(i, j);
            }
        }
        return 0;
    } catch (...) {
        return 3;
    }
}

int ref_observables(int nx, int ny, double lx, double ly, double gamma, const double* v,
                    const double* u, double* out7) {
    try {
        const GridModel model(GridSpec(nx, ny, lx, ly), gamma,
                              std::vector<double>(v, v + static_cast<size_t>(nx) * ny));
        put_obs(out7, observables(model, to_state(u, nx * ny)));
        return 0;
    } catch (...) {
        return 3;
    }
}

int ref_eval_phi(int nx, int ny, double lx, double ly, double gamma, const double* v,
                 const double* u0, const double* s1, const double* s2, const double* s3, double h,
                 double* p1, double* p2, double* p3) {
    try {
        const int n = nx * ny;
        const GridModel model(GridSpec(nx, ny, lx, ly), gamma,
                              std::vector<double>(v, v + static_cast<size_t>(n)));
        const Mb4Scheme scheme;
        const std::array<State, 3> st = {to_state(s1, n), to_state(s2, n), to_state(s3, n)};
        const auto phi = eval_phi(model, scheme, to_state(u0, n), st, h);
        std::memcpy(p1, phi[0].data(), sizeof(double) * 2 * n);
        std::memcpy(p2, phi[1].data(), sizeof(double) * 2 * n);
        std::memcpy(p3, phi[2].data(), sizeof(double) * 2 * n);
        return 0;
    } catch (...) {
        return 3;
    }
}

// The reference stepping loop: StepDriver(MB4) -> mb4_step per step, with
// observables recorded per step as run() does (harness.cpp:105-122).
// solver: 0 = Direct (default), 1 = Gmres.  obs: (nsteps+1)*7 or NULL.
// Returns 0 ok, 2 non-convergence, 1 invalid argument, 3 other error.
int ref_method_run(int method, int nx, int ny, double lx, double ly, double gamma, const double* v,
                   double* u, double h, int nsteps, double eps, int max_iters, int max_halvings, int solver,
                   int workers, double* obs, int* iters, double* seconds);

int ref_mb4_run(int nx, int ny, double lx, double ly, double gamma, const double* v, double* u,
                double h, int nsteps, double eps, int max_iters, int max_halvings, int solver,
                int workers, double* obs, int* iters, double* seconds) {
    return ref_method_run(static_cast<int>(MethodId::Mb4), nx, ny, lx, ly, gamma, v, u, h, nsteps, eps,
                          max_iters, max_halvings, solver, workers, obs, iters, seconds);
}

// StepDriver(model, method, ...) stepping loop; method = the reference's MethodId
// order (Rk4, Gauss2, Gauss4, Avf2, Avf4, Mb4), integrators.hpp:12.
int ref_method_run(int method, int nx, int ny, double lx, double ly, double gamma, const double* v,
                   double* u, double h, int nsteps, double eps, int max_iters, int max_halvings, int solver,
                   int workers, double* obs, int* iters, double* seconds) {
    if (method < 0 || method > 5) return 1;
    try {
        const int n = nx * ny;
        const GridModel model(GridSpec(nx, ny, lx, ly), gamma,
                              std::vector<double>(v, v + static_cast<size_t>(n)));
        WorkerPool pool(workers);
        StepDriver driver(model, static_cast<MethodId>(method), NewtonConfig{eps, max_iters, max_halvings},
                          solver == 1 ? SolverKind::Gmres : SolverKind::Direct, &pool);
        State s = to_state(u, n);
        if (obs) put_obs(obs, observables(model, s));
        double secs = 0.0;
        for (int k = 1; k <= nsteps; ++k) {
            StepStats stats;
            const auto t0 = std::chrono::steady_clock::now();
            s = driver.advance(s, h, &stats);
            secs += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (iters) iters[k - 1] = stats.newton_iters;
            if (obs) put_obs(obs + 7 * k, observables(model, s));
        }
        std::memcpy(u, s.data(), sizeof(double) * 2 * n);
        if (seconds) *seconds = secs;
        return 0;
    } catch (const NonConvergenceError&) {
        return 2;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (...) {
        return 3;
    }
}

}  // extern "C"
