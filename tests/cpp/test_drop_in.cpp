// C++ drop-in check: code written against the reference API (proj/include/nls2d)
// compiles unchanged against include/nls2d and runs on the GPU through the C ABI.
// Mirrors reference test cases (test_mb4_integrator.cpp, test_lattice.cpp).
//
// usage: test_drop_in <V.bin> <psi.bin> <nx> <ny> <gamma> <dt> <out_state.bin>
// Steps the given inputs 10 times with StepDriver::advance (host vectors, the
// reference contract) and writes the final state; exit code = number of failures.
#include <cmath>
#include <complex>
#include <cstdio>
#include <fstream>
#include <random>
#include <vector>

#include "nls2d/integrators.hpp"
#include "nls2d/lattice.hpp"
#include "nls2d/mb4_integrator.hpp"
#include "nls2d/mb4_scheme.hpp"

using namespace nls2d;

static int failures = 0;
#define CHECK(cond)                                                          \
    do {                                                                     \
        if (!(cond)) {                                                       \
            std::fprintf(stderr, "CHECK failed at line %d: %s\n", __LINE__, #cond); \
            ++failures;                                                      \
        }                                                                    \
    } while (0)

template <typename T>
static std::vector<T> read_bin(const char* path, size_t n) {
    std::vector<T> v(n);
    std::ifstream f(path, std::ios::binary);
    f.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(n * sizeof(T)));
    return v;
}

static State random_state(int n, unsigned seed) {
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> val(-1.0, 1.0);
    State u(n);
    for (auto& z : u) z = Complex(val(rng), val(rng));
    return u;
}

int main(int argc, char** argv) {
    if (argc != 8) {
        std::fprintf(stderr, "usage: %s V.bin psi.bin nx ny gamma dt out.bin\n", argv[0]);
        return 100;
    }
    const int nx = std::atoi(argv[3]), ny = std::atoi(argv[4]);
    const double gamma = std::atof(argv[5]), dt = std::atof(argv[6]);
    const int n = nx * ny;

    // phi: fixed point at zero step (test_mb4_integrator.cpp:67-76)
    {
        const GridSpec g(4, 4, 2 * M_PI, 2 * M_PI);
        const GridModel model(g, 0.1);
        const Mb4Scheme scheme;
        const State u0 = random_state(g.points(), 9);
        const auto phi = eval_phi(model, scheme, u0, {u0, u0, u0}, 0.0);
        for (const State& p : phi)
            for (const Complex& z : p) CHECK(std::abs(z) == 0.0);
    }
    // scheme validation (mb4_scheme.cpp:84-93)
    {
        bool threw = false;
        try {
            Mb4Scheme bad(-100.0);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    }
    // non-convergence reports the last residual (test_mb4_integrator.cpp:336-345)
    {
        const GridSpec g(6, 6, 2 * M_PI, 2 * M_PI);
        const GridModel model(g, 0.5);
        const Mb4Scheme scheme;
        NewtonConfig cfg;
        cfg.max_iters = 1;
        cfg.max_step_halvings = 0;
        bool threw = false;
        try {
            (void)mb4_step(model, scheme, initial_condition(g), 0.5, cfg);
        } catch (const NonConvergenceError& e) {
            threw = e.last_residual > 0.0;
        }
        CHECK(threw);
    }
    // the other methods through the reference API (test_integrators.cpp:37-42, 64-92)
    {
        const GridModel free_model(GridSpec(6, 6, 2 * M_PI, 2 * M_PI), 0.0);
        const State c0(free_model.points(), Complex(0.7, -0.3));
        const State c1 = rk4_step(free_model, c0, 0.05);
        for (size_t k = 0; k < c0.size(); ++k) CHECK(std::abs(c1[k] - c0[k]) <= 1e-15);
        const GridSpec g(6, 6, 2 * M_PI, 2 * M_PI);
        const GridModel model(g, 0.1);
        const State u0 = initial_condition(g);
        const State f0 = rhs(model, u0);
        for (MethodId m : {MethodId::Gauss2, MethodId::Gauss4, MethodId::Avf2, MethodId::Avf4, MethodId::Mb4}) {
            StepDriver d(model, m, NewtonConfig{});
            const double h = 1e-5;
            const State u1 = d.advance(u0, h);
            double err = 0.0;
            for (int k = 0; k < model.points(); ++k) err = std::max(err, std::abs(u1[k] - u0[k] - h * f0[k]));
            CHECK(err <= 10.0 * h * h);
        }
        const GridModel lin(GridSpec(8, 8, 2 * M_PI, 2 * M_PI), 0.0);
        const State v0 = initial_condition(lin.grid());
        const State a = avf2_step(lin, v0, 0.01, NewtonConfig{});
        const State b = gauss_step(lin, v0, 0.01, 1, NewtonConfig{});
        double num = 0.0, den = 0.0;
        for (size_t k = 0; k < a.size(); ++k) {
            num += std::norm(a[k] - b[k]);
            den += std::norm(b[k]);
        }
        CHECK(std::sqrt(num / den) <= 1e-12);
        CHECK(method_name(MethodId::Avf4) == "AVF4" && method_order(MethodId::Gauss2) == 2);
    }
    // BASELINE inputs: 10 steps through StepDriver::advance (host vectors)
    const std::vector<double> V = read_bin<double>(argv[1], n);
    const State psi = read_bin<Complex>(argv[2], n);
    const GridSpec grid(nx, ny, nx, ny);
    const GridModel model(grid, gamma, V);
    StepDriver driver(model, MethodId::Mb4, NewtonConfig{1e-14, 50, 4});
    const Observables o0 = observables(model, psi);
    State u = psi;
    StepStats stats;
    for (int s = 0; s < 10; ++s) u = driver.advance(u, dt, &stats);
    const Observables o1 = observables(model, u);
    CHECK(std::abs(o1.total_energy - o0.total_energy) <= 1e-13 * std::abs(o0.total_energy));
    CHECK(stats.newton_iters >= 10 && stats.halvings == 0);
    // the device-resident session gives the same trajectory
    DeviceSession sess(model, driver.scheme(), NewtonConfig{1e-14, 50, 4});
    sess.set_state(psi);
    const auto rows = sess.run(dt, 10);
    const State u2 = sess.get_state();
    double d = 0.0, nrm = 0.0;
    for (int k = 0; k < n; ++k) {
        d += std::norm(u2[k] - u[k]);
        nrm += std::norm(u[k]);
    }
    CHECK(std::sqrt(d / nrm) <= 1e-15);
    CHECK(std::abs(rows.back().total_energy - o1.total_energy) <= 1e-14 * std::abs(o1.total_energy));
    std::ofstream out(argv[7], std::ios::binary);
    out.write(reinterpret_cast<const char*>(u.data()), static_cast<std::streamsize>(n * sizeof(Complex)));
    std::printf("test_drop_in: %d failure(s); sweeps=%d\n", failures, stats.newton_iters);
    return failures;
}
