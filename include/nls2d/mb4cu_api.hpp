// C++ mirror of the reference's hot-path API (proj/include/nls2d), implemented
// header-only on top of the C ABI in mb4cu.h (link with libmb4cu.so).
//
// Declarations follow the reference so existing callers compile unchanged:
//   GridSpec / GridModel / rhs / observables      lattice.hpp:21-88
//   split_state / join_state                      lattice.hpp:17-18
//   SmallMat / Eig3                               small_dense.hpp:11-41
//   eval_A / lagrange_basis / Mb4Scheme           mb4_scheme.hpp:14-64
//   StageSystem / NewtonResult / newton_solve     mb4_integrator.hpp:76-95
//   NewtonConfig / StepStats / NonConvergenceError / eval_phi / mb4_step
//                                                 mb4_integrator.hpp:17-110
//   MethodId / StepDriver                         integrators.hpp:11-66
// Differences (documented in INTEGRATION.md):
//   - the kinetic operator is the periodic 5-point stencil (the custom-K ctor,
//     lattice.hpp:54, is not offered);
//   - WorkerPool / SolverKind / cached_order are accepted and ignored (no sparse
//     factorization, no CPU threads on this path);
//   - for MB4, StepStats::newton_iters counts stage sweeps; solve_seconds is device time;
//   - every MethodId runs on the GPU (RK4 / GAUSS / AVF: methods.cu, their linear
//     systems by matrix-free GMRES instead of sparse LU).
#pragma once

#include <array>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <cctype>
#include <chrono>
#include <limits>
#include <functional>
#include <memory>
#include <optional>
#include <ostream>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "mb4cu.h"

namespace nls2d {

using Complex = std::complex<double>;
using State = std::vector<Complex>;

class NonConvergenceError : public std::runtime_error {
public:
    NonConvergenceError(const std::string& what, double residual)
        : std::runtime_error(what), last_residual(residual) {}
    double last_residual;
    double at_time = -1.0;
};

class ComplexEigenvalueError : public std::runtime_error {
public:
    explicit ComplexEigenvalueError(const std::string& what) : std::runtime_error(what) {}
};

namespace detail {
inline void throw_status(int rc, const std::string& text, double residual = 0.0) {
    switch (rc) {
        case MB4CU_OK: return;
        case MB4CU_NONCONVERGED: throw NonConvergenceError(text, residual);
        case MB4CU_INVALID:
            if (text.rfind("eig3_real", 0) == 0) throw ComplexEigenvalueError(text);
            throw std::invalid_argument(text);
        default: throw std::runtime_error("mb4cu status " + std::to_string(rc) + ": " + text);
    }
}
}  // namespace detail

/// Split view [p; q] of a state (lattice.hpp:17-18): real parts, then imaginary parts.
inline std::vector<double> split_state(const State& u) {
    const std::size_t n = u.size();
    std::vector<double> v(2 * n);
    for (std::size_t k = 0; k < n; ++k) {
        v[k] = u[k].real();
        v[n + k] = u[k].imag();
    }
    return v;
}
inline State join_state(std::span<const double> v) {
    if (v.size() % 2 != 0) throw std::invalid_argument("join_state: odd length");
    const std::size_t n = v.size() / 2;
    State u(n);
    for (std::size_t k = 0; k < n; ++k) u[k] = Complex(v[k], v[n + k]);
    return u;
}

/// Small row-major dense matrix (small_dense.hpp:11-34): the scheme-side 3x3 work.
class SmallMat {
public:
    static constexpr int kMax = 8;
    SmallMat() = default;
    SmallMat(int rows, int cols) : rows_(rows), cols_(cols) {
        if (rows < 0 || cols < 0 || rows > kMax || cols > kMax)
            throw std::invalid_argument("SmallMat: dimension out of range");
    }
    static SmallMat identity(int n) {
        SmallMat m(n, n);
        for (int i = 0; i < n; ++i) m(i, i) = 1.0;
        return m;
    }
    int rows() const { return rows_; }
    int cols() const { return cols_; }
    double& operator()(int r, int c) { return a_[static_cast<std::size_t>(r) * kMax + c]; }
    double operator()(int r, int c) const { return a_[static_cast<std::size_t>(r) * kMax + c]; }
    SmallMat operator*(const SmallMat& b) const {
        if (cols_ != b.rows_) throw std::invalid_argument("SmallMat: dimension mismatch");
        SmallMat p(rows_, b.cols_);
        for (int i = 0; i < rows_; ++i)
            for (int j = 0; j < b.cols_; ++j) {
                double acc = 0.0;
                for (int k = 0; k < cols_; ++k) acc += (*this)(i, k) * b(k, j);
                p(i, j) = acc;
            }
        return p;
    }
    /// Gauss-Jordan elimination with partial pivoting on an augmented copy.
    SmallMat inverse() const {
        if (rows_ != cols_) throw std::invalid_argument("SmallMat: inverse of a non-square matrix");
        const int n = rows_;
        SmallMat w = *this, inv = identity(n);
        for (int c = 0; c < n; ++c) {
            int piv = c;
            for (int r = c + 1; r < n; ++r)
                if (std::abs(w(r, c)) > std::abs(w(piv, c))) piv = r;
            if (w(piv, c) == 0.0) throw std::runtime_error("SmallMat: singular matrix");
            for (int k = 0; k < n; ++k) {
                std::swap(w(c, k), w(piv, k));
                std::swap(inv(c, k), inv(piv, k));
            }
            const double d = w(c, c);
            for (int k = 0; k < n; ++k) {
                w(c, k) /= d;
                inv(c, k) /= d;
            }
            for (int r = 0; r < n; ++r) {
                if (r == c || w(r, c) == 0.0) continue;
                const double f = w(r, c);
                for (int k = 0; k < n; ++k) {
                    w(r, k) -= f * w(c, k);
                    inv(r, k) -= f * inv(c, k);
                }
            }
        }
        return inv;
    }
    double inf_norm() const {
        double m = 0.0;
        for (int i = 0; i < rows_; ++i) {
            double s = 0.0;
            for (int j = 0; j < cols_; ++j) s += std::abs((*this)(i, j));
            m = std::max(m, s);
        }
        return m;
    }

private:
    int rows_ = 0, cols_ = 0;
    std::array<double, kMax * kMax> a_{};
};

struct Eig3 {
    std::array<double, 3> values{};  // ascending
    SmallMat t;                      // columns are eigenvectors
    SmallMat t_inv;
};

/// A(tau, zeta) of the scheme (mb4_scheme.hpp:14), computed by the library.
inline double eval_A(double alpha1, double tau, double zeta) { return mb4cu_eval_a(alpha1, tau, zeta); }

/// Cubic Lagrange basis over {0, c1, c2, c3} (mb4_scheme.hpp:17).
inline double lagrange_basis(const std::array<double, 4>& nodes, int i, double zeta) {
    double v = 0.0;
    detail::throw_status(mb4cu_lagrange_basis(nodes.data(), i, zeta, &v), mb4cu_create_error());
    return v;
}

struct GridSpec {
    int nx = 0, ny = 0;
    double lx = 0.0, ly = 0.0;
    GridSpec(int nx_, int ny_, double lx_, double ly_) : nx(nx_), ny(ny_), lx(lx_), ly(ly_) {
        if (nx < 2 || ny < 2) throw std::invalid_argument("GridSpec: nx and ny must be >= 2");
        if (!(lx > 0.0) || !(ly > 0.0))
            throw std::invalid_argument("GridSpec: domain lengths must be positive");
    }
    double hx() const { return lx / nx; }
    double hy() const { return ly / ny; }
    int points() const { return nx * ny; }
    int index(int i, int j) const { return j * nx + i; }
};

inline std::vector<double> build_delta_potential(const GridSpec& g, double v0) {
    std::vector<double> v(g.points(), 0.0);
    v[g.index(0, 0)] = v0;
    return v;
}

inline State initial_condition(const GridSpec& g) {
    State u(g.points());
    for (int j = 0; j < g.ny; ++j)
        for (int i = 0; i < g.nx; ++i)
            u[g.index(i, j)] = Complex(1.0 + 2.0 * std::cos(i * g.hx()) + 2.0 * std::cos(j * g.hy()), 0.0);
    return u;
}

struct NewtonConfig {
    double epsilon = 1e-13;
    int max_iters = 50;
    int max_step_halvings = 4;
    void validate() const {
        if (!(epsilon > 0.0)) throw std::invalid_argument("NewtonConfig: epsilon must be > 0");
        if (max_iters < 1) throw std::invalid_argument("NewtonConfig: max_iters must be >= 1");
        if (max_step_halvings < 0) throw std::invalid_argument("NewtonConfig: negative halvings");
    }
};

enum class SolverKind { Direct, Gmres };

struct StepStats {
    int newton_iters = 0;
    int halvings = 0;
    double solve_seconds = 0.0;
};

struct Observables {
    double u_kinetic = 0.0, u_nonlinear = 0.0, u_external = 0.0, total_energy = 0.0,
           probability = 0.0, participation = 0.0, raw_quartic = 0.0;
};

class WorkerPool {  // accepted for signature compatibility; the GPU path has no CPU workers
public:
    explicit WorkerPool(int workers = 1) : workers_(workers) {}
    int workers() const { return workers_; }

private:
    int workers_;
};

class Mb4Scheme {
public:
    static constexpr double kAlpha1Bound = -300.0 * 0.7770503941;
    explicit Mb4Scheme(double alpha1 = -300.0 * 19.0 / 8.0,
                       std::array<double, 3> nodes = {1.0 / 3.0, 2.0 / 3.0, 1.0}) {
        const int rc = mb4cu_scheme_init(alpha1, nodes[0], nodes[1], nodes[2], &s_);
        detail::throw_status(rc, mb4cu_create_error());
        fill_eig();
    }
    double alpha1() const { return s_.alpha1; }
    std::array<double, 4> nodes() const { return {s_.nodes[0], s_.nodes[1], s_.nodes[2], s_.nodes[3]}; }
    double e_ext(int i, int j) const { return s_.E[i - 1][j]; }
    double w(int i, int a, int b, int c) const { return s_.W[i - 1][a][b][c]; }
    std::array<double, 3> eigenvalues() const { return {s_.lam[0], s_.lam[1], s_.lam[2]}; }
    /// E_core = T diag(lambda) T^{-1} (mb4_scheme.hpp:45-47)
    const SmallMat& t() const { return eig_.t; }
    const SmallMat& t_inv() const { return eig_.t_inv; }
    double t(int r, int c) const { return s_.T[r][c]; }
    double t_inv(int r, int c) const { return s_.Tinv[r][c]; }
    double eval_A(double tau, double zeta) const { return nls2d::eval_A(s_.alpha1, tau, zeta); }
    double lagrange(int i, double zeta) const { return lagrange_basis(nodes(), i, zeta); }

    /// The 3x3 matrix M of A(tau,zeta) = [tau, tau^2/2, tau^3/3] M [1, zeta, zeta^2]^T
    /// (mb4_scheme.hpp:36-38): the alpha1-free part plus alpha1 times the rank-one
    /// block (1, -6, 6)^T (1, -6, 6) of the cancellation-free form.
    SmallMat a_coeff() const {
        const double a = s_.alpha1;
        static const double base[3][3] = {{4.0, -6.0, 0.0}, {-6.0, 12.0, 0.0}, {0.0, 0.0, 0.0}};
        static const double r1[3] = {1.0, -6.0, 6.0};
        SmallMat m(3, 3);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) m(i, j) = base[i][j] + a * r1[i] * r1[j];
        return m;
    }

    /// Plain-text key = value table of every constant, 17 significant digits
    /// (mb4_scheme.hpp:50-51; same keys and order).
    void dump(std::ostream& os) const {
        char buf[96];
        auto put = [&](const char* key, double v) {
            std::snprintf(buf, sizeof(buf), "%s = %.17g\n", key, v);
            os << buf;
        };
        put("alpha1", s_.alpha1);
        char key[32];
        for (int i = 1; i <= 3; ++i) {
            std::snprintf(key, sizeof(key), "c%d", i);
            put(key, s_.nodes[i]);
        }
        for (int i = 1; i <= 3; ++i)
            for (int j = 0; j < 4; ++j) {
                std::snprintf(key, sizeof(key), "E_%d_%d", i, j);
                put(key, e_ext(i, j));
            }
        for (int i = 0; i < 3; ++i) {
            std::snprintf(key, sizeof(key), "lambda%d", i + 1);
            put(key, s_.lam[i]);
        }
        for (int i = 1; i <= 3; ++i)
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < 4; ++b)
                    for (int c = 0; c < 4; ++c) {
                        std::snprintf(key, sizeof(key), "W_%d_%d_%d_%d", i, a, b, c);
                        put(key, w(i, a, b, c));
                    }
    }

    /// E table at a chosen Gauss-Legendre order (>= 4 is exact; mb4_scheme.hpp:53-58).
    static std::array<std::array<double, 4>, 3> integrate_e(double alpha1, const std::array<double, 4>& nodes,
                                                            int points) {
        double out[12];
        detail::throw_status(mb4cu_scheme_integrate_e(alpha1, nodes.data(), points, out), mb4cu_create_error());
        std::array<std::array<double, 4>, 3> e{};
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 4; ++j) e[i][j] = out[i * 4 + j];
        return e;
    }

    const mb4cu_scheme& raw() const { return s_; }

private:
    void fill_eig() {
        eig_.t = SmallMat(3, 3);
        eig_.t_inv = SmallMat(3, 3);
        for (int i = 0; i < 3; ++i) {
            eig_.values[i] = s_.lam[i];
            for (int j = 0; j < 3; ++j) {
                eig_.t(i, j) = s_.T[i][j];
                eig_.t_inv(i, j) = s_.Tinv[i][j];
            }
        }
    }
    mb4cu_scheme s_{};
    Eig3 eig_;
};

class GridModel;

enum class MethodId { Rk4, Gauss2, Gauss4, Avf2, Avf4, Mb4 };

/// integrators.cpp:13-43
inline int method_order(MethodId m) { return m == MethodId::Gauss2 || m == MethodId::Avf2 ? 2 : 4; }
inline std::optional<MethodId> parse_method(const std::string& name) {
    std::string u;
    for (char c : name) u.push_back(static_cast<char>(std::toupper(static_cast<unsigned char>(c))));
    static const char* names[] = {"RK4", "GAUSS2", "GAUSS4", "AVF2", "AVF4", "MB4"};
    for (int i = 0; i < 6; ++i)
        if (u == names[i]) return static_cast<MethodId>(i);
    return std::nullopt;
}
inline std::string method_name(MethodId m) {
    static const char* names[] = {"RK4", "GAUSS2", "GAUSS4", "AVF2", "AVF4", "MB4"};
    return names[static_cast<int>(m)];
}

/// RAII device session: one mb4cu context, state resident in HBM; step()/run()
/// advance with `method` (default MB4).
class DeviceSession {
public:
    DeviceSession(const GridModel& model, const Mb4Scheme& scheme, const NewtonConfig& cfg,
                  int neumann_terms = -1, int device = 0, int kernel = 0, MethodId method = MethodId::Mb4);
    ~DeviceSession() { mb4cu_destroy(ctx_); }
    DeviceSession(const DeviceSession&) = delete;
    DeviceSession& operator=(const DeviceSession&) = delete;

    void set_state(const State& u) {
        check(mb4cu_set_state(ctx_, reinterpret_cast<const double*>(u.data())));
    }
    State get_state() const {
        State u(n_);
        check(mb4cu_get_state(ctx_, reinterpret_cast<double*>(u.data())));
        return u;
    }
    void step(double h, StepStats* stats = nullptr) {
        mb4cu_stats st{};
        const int rc = mb4cu_method_step(ctx_, method_, h, &st);
        if (stats) {
            stats->newton_iters += st.newton_iters;
            stats->halvings += st.halvings;
            stats->solve_seconds += st.solve_seconds;
        }
        check(rc, st.last_residual);
    }
    /// nsteps device-resident steps; returns the (nsteps+1) x 7 energy record.
    std::vector<Observables> run(double h, int nsteps, std::vector<int>* iters = nullptr,
                                 StepStats* stats = nullptr) {
        std::vector<Observables> rows(static_cast<size_t>(nsteps) + 1);
        std::vector<int> it(static_cast<size_t>(nsteps));
        mb4cu_stats st{};
        static_assert(sizeof(Observables) == 7 * sizeof(double), "layout");
        const int rc = mb4cu_method_run(ctx_, method_, h, nsteps, reinterpret_cast<double*>(rows.data()), it.data(),
                                        &st);
        if (stats) {
            stats->newton_iters += st.newton_iters;
            stats->halvings += st.halvings;
            stats->solve_seconds += st.solve_seconds;
        }
        check(rc, st.last_residual);
        if (iters) *iters = it;
        return rows;
    }
    Observables observables() const {
        mb4cu_obs o{};
        check(mb4cu_observables(ctx_, &o));
        return {o.u_kinetic, o.u_nonlinear, o.u_external, o.total_energy, o.probability,
                o.participation, o.raw_quartic};
    }
    mb4cu_ctx* handle() const { return ctx_; }

    void check(int rc, double residual = 0.0) const {
        if (rc != MB4CU_OK) detail::throw_status(rc, mb4cu_last_error(ctx_), residual);
    }

private:
    mb4cu_ctx* ctx_ = nullptr;
    int n_ = 0;
    int method_ = MB4CU_METHOD_MB4;
};

class GridModel {
public:
    GridModel(GridSpec grid, double gamma) : GridModel(grid, gamma, std::vector<double>(grid.points(), 0.0)) {}
    GridModel(GridSpec grid, double gamma, std::vector<double> potential)
        : grid_(grid), potential_(std::move(potential)), gamma_(gamma) {
        if (static_cast<int>(potential_.size()) != grid_.points())
            throw std::invalid_argument("GridModel: potential length mismatch");
    }
    const GridSpec& grid() const { return grid_; }
    std::span<const double> potential() const { return potential_; }
    double gamma() const { return gamma_; }
    int points() const { return grid_.points(); }
    double cx() const { return 1.0 / (grid_.hx() * grid_.hx()); }
    double cy() const { return 1.0 / (grid_.hy() * grid_.hy()); }

    /// y = (K + V) u, evaluated on the GPU
    void apply_kv(std::span<const Complex> u, std::span<Complex> y) const {
        DeviceSession s(*this, Mb4Scheme(), NewtonConfig{});
        s.check(mb4cu_apply_kv(s.handle(), reinterpret_cast<const double*>(u.data()),
                               reinterpret_cast<double*>(y.data())));
    }

private:
    GridSpec grid_;
    std::vector<double> potential_;
    double gamma_;
};

inline DeviceSession::DeviceSession(const GridModel& model, const Mb4Scheme& scheme,
                                    const NewtonConfig& cfg, int neumann_terms, int device,
                                    int kernel, MethodId method)
    : method_(static_cast<int>(method)) {
    cfg.validate();
    mb4cu_problem p{};
    p.nx = model.grid().nx;
    p.ny = model.grid().ny;
    p.cx = model.cx();
    p.cy = model.cy();
    p.gamma = model.gamma();
    p.V = model.potential().data();
    p.epsilon = cfg.epsilon;
    p.max_iters = cfg.max_iters;
    p.max_step_halvings = cfg.max_step_halvings;
    p.neumann_terms = neumann_terms;
    p.neumann_first = -1;
    p.ghost = 0;
    p.device = device;
    p.kernel = kernel;
    const int rc = mb4cu_create(&p, &scheme.raw(), &ctx_);
    if (rc != MB4CU_OK) detail::throw_status(rc, mb4cu_create_error());
    n_ = model.points();
}

inline State rhs(const GridModel& model, const State& u) {
    if (static_cast<int>(u.size()) != model.points()) throw std::invalid_argument("rhs: state length mismatch");
    State y(u.size());
    DeviceSession s(model, Mb4Scheme(), NewtonConfig{});
    s.check(mb4cu_rhs(s.handle(), reinterpret_cast<const double*>(u.data()), reinterpret_cast<double*>(y.data())));
    return y;
}

inline Observables observables(const GridModel& model, const State& u) {
    if (static_cast<int>(u.size()) != model.points())
        throw std::invalid_argument("observables: state length mismatch");
    DeviceSession s(model, Mb4Scheme(), NewtonConfig{});
    s.set_state(u);
    return s.observables();
}

inline std::array<State, 3> eval_phi(const GridModel& model, const Mb4Scheme& scheme, const State& u0,
                                     const std::array<State, 3>& stages, double h) {
    std::array<State, 3> phi;
    for (auto& p : phi) p.resize(u0.size());
    DeviceSession s(model, scheme, NewtonConfig{});
    auto d = [](const State& x) { return reinterpret_cast<const double*>(x.data()); };
    auto m = [](State& x) { return reinterpret_cast<double*>(x.data()); };
    s.check(mb4cu_eval_phi(s.handle(), d(u0), d(stages[0]), d(stages[1]), d(stages[2]), h, m(phi[0]),
                           m(phi[1]), m(phi[2])));
    return phi;
}

/// One MB4 step (mb4_integrator.hpp:103-110): host vectors in and out.
inline State mb4_step(const GridModel& model, const Mb4Scheme& scheme, const State& u0, double h,
                      const NewtonConfig& cfg, WorkerPool* = nullptr, StepStats* stats = nullptr,
                      SolverKind = SolverKind::Direct, const std::vector<int>* = nullptr) {
    cfg.validate();
    if (!(h > 0.0)) throw std::invalid_argument("mb4_step: h must be positive");
    DeviceSession s(model, scheme, cfg);
    s.set_state(u0);
    s.step(h, stats);
    return s.get_state();
}

/// The three stage systems (I - h lambda_i J) of one step (mb4_integrator.hpp:76-83).
/// The GPU path forms no matrix: the systems are applied matrix-free and solved by
/// Fourier-preconditioned GMRES inside newton_solve, so the handle only carries h.
/// (The reference's build(jacobian, ...) from a SparseCsr is not offered: no sparse
/// matrix exists on this path.)
struct StageSystem {
    double h = 0.0;
    static StageSystem build(const GridModel&, const Mb4Scheme&, double h, SolverKind = SolverKind::Direct,
                             WorkerPool* = nullptr) {
        if (!(h > 0.0)) throw std::invalid_argument("StageSystem: h must be positive");
        return StageSystem{h};
    }
};

struct NewtonResult {
    std::array<State, 3> stages;
    int iterations = 0;
};

/// Simplified Newton iteration of the stage equations from U = (u0, u0, u0)
/// (mb4_integrator.cpp:194-255): per iteration Phi, T^{-1}, the three decoupled
/// stage solves, T, update, stop when ||r||_inf <= epsilon.  Runs on the GPU through
/// the stage-split entry points (mb4cu_ns_*); the iteration counts are the
/// reference's.  Throws NonConvergenceError as the reference does.
inline NewtonResult newton_solve(const GridModel& model, const Mb4Scheme& scheme, const StageSystem& sys,
                                 const State& u0, double h, const NewtonConfig& cfg, WorkerPool* = nullptr,
                                 double* solve_seconds = nullptr) {
    cfg.validate();
    if (sys.h != h) throw std::invalid_argument("newton_solve: stage system built for another h");
    DeviceSession s(model, scheme, cfg, -1, 0, 3);
    s.set_state(u0);
    mb4cu_ctx* ctx = s.handle();
    s.check(mb4cu_ns_begin(ctx, h));
    NewtonResult res;
    double r = 0.0;
    for (int iter = 1; iter <= cfg.max_iters; ++iter) {
        s.check(mb4cu_ns_phibar(ctx));
        const auto t0 = std::chrono::steady_clock::now();
        for (int k = 0; k < 3; ++k) s.check(mb4cu_ns_solve(ctx, k));
        s.check(mb4cu_ns_update(ctx, &r));
        if (solve_seconds)
            *solve_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        res.iterations = iter;
        if (!std::isfinite(r)) {
            mb4cu_ns_abort(ctx);
            throw NonConvergenceError("newton_solve: iteration diverged (non-finite update)",
                                      std::numeric_limits<double>::infinity());
        }
        if (r <= cfg.epsilon) {
            for (auto& st : res.stages) st.resize(u0.size());
            s.check(mb4cu_ns_get_stages(ctx, reinterpret_cast<double*>(res.stages[0].data()),
                                        reinterpret_cast<double*>(res.stages[1].data()),
                                        reinterpret_cast<double*>(res.stages[2].data())));
            mb4cu_ns_abort(ctx);
            return res;
        }
    }
    mb4cu_ns_abort(ctx);
    throw NonConvergenceError("newton_solve: no convergence after " + std::to_string(cfg.max_iters) + " iterations",
                              r);
}

namespace detail {
inline State plain_method_step(MethodId m, const GridModel& model, const State& u0, double h,
                               const NewtonConfig& cfg, StepStats* stats) {
    cfg.validate();
    if (!(h > 0.0)) throw std::invalid_argument("step: h must be positive");
    // the free functions of integrators.hpp do not halve
    DeviceSession s(model, Mb4Scheme(), NewtonConfig{cfg.epsilon, cfg.max_iters, 0}, -1, 0, 0, m);
    s.set_state(u0);
    s.step(h, stats);
    return s.get_state();
}
}  // namespace detail

/// integrators.hpp:17-43 on the GPU (host vectors in and out)
inline State rk4_step(const GridModel& model, const State& u0, double h) {
    return detail::plain_method_step(MethodId::Rk4, model, u0, h, NewtonConfig{}, nullptr);
}
inline State gauss_step(const GridModel& model, const State& u0, double h, int stages, const NewtonConfig& cfg,
                        StepStats* stats = nullptr, SolverKind = SolverKind::Direct,
                        const std::vector<int>* = nullptr) {
    if (stages != 1 && stages != 2) throw std::invalid_argument("gauss_step: stages must be 1 or 2");
    return detail::plain_method_step(stages == 1 ? MethodId::Gauss2 : MethodId::Gauss4, model, u0, h, cfg, stats);
}
inline State avf2_step(const GridModel& model, const State& u0, double h, const NewtonConfig& cfg,
                       StepStats* stats = nullptr, SolverKind = SolverKind::Direct,
                       const std::vector<int>* = nullptr) {
    return detail::plain_method_step(MethodId::Avf2, model, u0, h, cfg, stats);
}
inline State avf4_step(const GridModel& model, const State& u0, double h, const NewtonConfig& cfg,
                       StepStats* stats = nullptr, SolverKind = SolverKind::Direct,
                       const std::vector<int>* = nullptr) {
    return detail::plain_method_step(MethodId::Avf4, model, u0, h, cfg, stats);
}

/// integrators.hpp:46-66.  Keeps one device session per driver; the halving
/// policy of advance() (integrators.cpp:425-455) runs inside the library.
class StepDriver {
public:
    StepDriver(const GridModel& model, MethodId method, NewtonConfig cfg,
               SolverKind = SolverKind::Direct, WorkerPool* = nullptr)
        : cfg_(cfg) {
        cfg_.validate();
        session_ = std::make_unique<DeviceSession>(model, scheme_, cfg_, -1, 0, 0, method);
    }
    State advance(const State& u0, double h, StepStats* stats = nullptr) {
        if (!(h > 0.0)) throw std::invalid_argument("advance: h must be positive");
        session_->set_state(u0);
        session_->step(h, stats);
        return session_->get_state();
    }
    const Mb4Scheme& scheme() const { return scheme_; }
    DeviceSession& session() { return *session_; }

private:
    NewtonConfig cfg_;
    Mb4Scheme scheme_;
    std::unique_ptr<DeviceSession> session_;
};

}  // namespace nls2d
