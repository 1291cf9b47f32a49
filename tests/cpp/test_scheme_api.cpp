// Reference-style checks of the scheme / state / Newton surface of the C++ mirror
// (include/nls2d), restating the cases of the reference's test_mb4_scheme.cpp
// (eval_A, lagrange_basis, a_coeff, validation, E / W / eigen tables, dump) and
// lattice.hpp's split_state / join_state against include/nls2d.
//
//   test_scheme_api scheme <exact.txt>        host-only (no GPU): exits 0 when every check passes
//   test_scheme_api newton <u0.bin> <n> <gamma> <h> <out_prefix>
//                                             GPU: newton_solve on the n x n, lx = 2 pi grid;
//                                             writes <out_prefix>{1,2,3}.bin and prints iterations
// exact.txt: "key value" lines written by tests/test_cpp_drop_in.py from
// tests/golden/scheme_exact.json (the reference's exact-rational generator).
#include <cmath>
#include <cstdio>
#include <fstream>
#include <map>
#include <random>
#include <sstream>
#include <string>

#include "nls2d/mb4_integrator.hpp"
#include "nls2d/mb4_scheme.hpp"

using namespace nls2d;

static int failures = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (!(cond)) {                                                           \
            std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                          \
        }                                                                        \
    } while (0)

static bool close_rel(double a, double b, double rel) { return std::abs(a - b) <= rel * std::max(1.0, std::abs(b)); }

template <typename F>
static bool throws_invalid(F&& f) {
    try {
        f();
    } catch (const std::invalid_argument&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static int scheme_checks(const char* exact_path) {
    std::map<std::string, double> ex;
    {
        std::ifstream in(exact_path);
        std::string k;
        double v;
        while (in >> k >> v) ex[k] = v;
    }
    const double kAlpha1 = ex.at("alpha1");

    // eval_A: zero at tau = 0, corner value 1, frozen A(1/2, 1/2)  (test_mb4_scheme.cpp:13-21)
    std::mt19937 rng(1);
    std::uniform_real_distribution<double> unif(0.0, 1.0);
    for (int k = 0; k < 20; ++k) CHECK(eval_A(kAlpha1, 0.0, unif(rng)) == 0.0);
    CHECK(close_rel(eval_A(kAlpha1, 1.0, 0.0), 1.0, 1e-14));
    CHECK(close_rel(eval_A(-500.0, 1.0, 0.0), 1.0, 1e-14));
    CHECK(close_rel(eval_A(kAlpha1, 0.5, 0.5), ex.at("A_half_half"), 1e-14));

    // Lagrange basis: delta property, partition of unity, frozen l_3(1/2)  (:23-39)
    const std::array<double, 4> nodes = {0.0, 1.0 / 3.0, 2.0 / 3.0, 1.0};
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) CHECK(std::abs(lagrange_basis(nodes, i, nodes[j]) - (i == j ? 1.0 : 0.0)) <= 1e-13);
    for (int k = 0; k < 10; ++k) {
        const double z = unif(rng);
        double s = 0.0;
        for (int i = 0; i < 4; ++i) s += lagrange_basis(nodes, i, z);
        CHECK(std::abs(s - 1.0) <= 1e-13);
    }
    CHECK(close_rel(lagrange_basis(nodes, 3, 0.5), ex.at("l3_half"), 1e-15));
    CHECK(throws_invalid([&] { lagrange_basis(nodes, 4, 0.5); }));
    CHECK(throws_invalid([&] { lagrange_basis({0.0, 0.5, 0.5, 1.0}, 1, 0.3); }));

    // eval_A equals the explicit matrix product with a_coeff()  (:41-58)
    const Mb4Scheme scheme;
    const SmallMat m = scheme.a_coeff();
    CHECK(m.rows() == 3 && m.cols() == 3);
    std::mt19937 rng8(8);
    for (int trial = 0; trial < 25; ++trial) {
        const double tau = unif(rng8), zeta = unif(rng8);
        const double tv[3] = {tau, tau * tau / 2.0, tau * tau * tau / 3.0};
        const double zv[3] = {1.0, zeta, zeta * zeta};
        double prod = 0.0;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) prod += tv[i] * m(i, j) * zv[j];
        CHECK(std::abs(scheme.eval_A(tau, zeta) - prod) <= 1e-13 * std::abs(scheme.alpha1()));
        CHECK(scheme.lagrange(2, zeta) == lagrange_basis(scheme.nodes(), 2, zeta));
    }

    // constructor validation  (:60-66)
    CHECK(throws_invalid([] { Mb4Scheme(-200.0); }));
    CHECK(throws_invalid([] { Mb4Scheme(-712.5, {0.5, 0.5, 1.0}); }));
    CHECK(throws_invalid([] { Mb4Scheme(-712.5, {0.3, 0.6, 0.9}); }));

    // E against the exact rationals, row sums, quadrature-order insensitivity  (:68-96)
    for (int i = 1; i <= 3; ++i)
        for (int j = 0; j < 4; ++j) {
            const double e = ex.at("E_" + std::to_string(i) + "_" + std::to_string(j));
            CHECK(std::abs(scheme.e_ext(i, j) - e) <= 1e-14 * std::max(1.0, std::abs(e)));
        }
    const auto e4 = Mb4Scheme::integrate_e(scheme.alpha1(), scheme.nodes(), 4);
    const auto e8 = Mb4Scheme::integrate_e(scheme.alpha1(), scheme.nodes(), 8);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 4; ++j) {
            CHECK(e4[i][j] == scheme.e_ext(i + 1, j));
            CHECK(std::abs(e4[i][j] - e8[i][j]) <= 1e-13 * std::max(1.0, std::abs(e4[i][j])));
        }
    CHECK(throws_invalid([&] { Mb4Scheme::integrate_e(-712.5, scheme.nodes(), 0); }));

    // eigen-decomposition: E_core = T diag(lambda) T^{-1}  (:153-176)
    SmallMat core(3, 3), lam(3, 3);
    for (int i = 0; i < 3; ++i) {
        lam(i, i) = scheme.eigenvalues()[i];
        for (int j = 0; j < 3; ++j) core(i, j) = scheme.e_ext(i + 1, j + 1);
    }
    const SmallMat recon = scheme.t() * lam * scheme.t_inv();
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) CHECK(std::abs(recon(i, j) - core(i, j)) <= 1e-11 * core.inf_norm());
    const SmallMat tt = scheme.t() * scheme.t_inv();
    const SmallMat ti = scheme.t().inverse();
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            CHECK(std::abs(tt(i, j) - (i == j ? 1.0 : 0.0)) <= 1e-12);
            CHECK(std::abs(ti(i, j) - scheme.t_inv()(i, j)) <= 1e-10 * scheme.t_inv().inf_norm());
            CHECK(scheme.t()(i, j) == scheme.t(i, j));
        }
    for (int i = 0; i < 3; ++i) {
        const double l = ex.at("lambda" + std::to_string(i + 1));
        CHECK(std::abs(scheme.eigenvalues()[i] - l) <= 1e-13 * std::abs(l));
    }

    // dump is a parseable key = value table  (:178-204)
    std::ostringstream os;
    scheme.dump(os);
    std::istringstream is(os.str());
    std::string line;
    int count = 0;
    bool saw_alpha = false, saw_w = false;
    while (std::getline(is, line)) {
        const auto eq = line.find(" = ");
        CHECK(eq != std::string::npos);
        if (eq == std::string::npos) break;
        const std::string key = line.substr(0, eq);
        const double value = std::stod(line.substr(eq + 3));
        if (key == "alpha1") {
            saw_alpha = true;
            CHECK(value == -712.5);
        }
        if (key == "W_3_3_3_3") {
            saw_w = true;
            CHECK(close_rel(value, ex.at("W_3_3_3_3"), 1e-15));
        }
        ++count;
    }
    CHECK(saw_alpha && saw_w);
    CHECK(count == 1 + 3 + 12 + 3 + 192);

    // split_state / join_state  (lattice.hpp:17-18)
    State u = {Complex(1.0, -2.0), Complex(3.5, 0.25), Complex(-0.0, 7.0)};
    const std::vector<double> v = split_state(u);
    CHECK(v.size() == 6 && v[0] == 1.0 && v[2] == -0.0 && v[3] == -2.0 && v[5] == 7.0);
    CHECK(join_state(v) == u);
    const std::vector<double> odd(5, 0.0);
    CHECK(throws_invalid([&] { join_state(odd); }));
    return failures;
}

static int newton_run(int argc, char** argv) {
    if (argc < 7) return 2;
    const int n = std::atoi(argv[3]);
    const double gamma = std::atof(argv[4]), h = std::atof(argv[5]);
    State u0(static_cast<size_t>(n) * n);
    {
        std::ifstream in(argv[2], std::ios::binary);
        in.read(reinterpret_cast<char*>(u0.data()), static_cast<std::streamsize>(u0.size() * sizeof(Complex)));
    }
    const GridSpec g(n, n, 2.0 * M_PI, 2.0 * M_PI);
    const GridModel model(g, gamma);
    const Mb4Scheme scheme;
    NewtonConfig cfg;  // epsilon 1e-13, 50 iterations
    const StageSystem sys = StageSystem::build(model, scheme, h);
    double secs = 0.0;
    const NewtonResult r = newton_solve(model, scheme, sys, u0, h, cfg, nullptr, &secs);
    for (int i = 0; i < 3; ++i) {
        std::ofstream out(std::string(argv[6]) + std::to_string(i + 1) + ".bin", std::ios::binary);
        out.write(reinterpret_cast<const char*>(r.stages[i].data()),
                  static_cast<std::streamsize>(r.stages[i].size() * sizeof(Complex)));
    }
    std::printf("iterations %d\n", r.iterations);
    // the non-convergence contract: one iteration cannot meet epsilon = 1e-13
    try {
        NewtonConfig one{1e-13, 1, 0};
        newton_solve(model, scheme, sys, u0, h, one);
        std::printf("no-throw\n");
        return 3;
    } catch (const NonConvergenceError& e) {
        if (!(e.last_residual > 1e-13)) return 4;
    }
    CHECK(throws_invalid([&] { newton_solve(model, scheme, sys, u0, 2 * h, cfg); }));
    return failures;
}

int main(int argc, char** argv) {
    if (argc >= 3 && std::string(argv[1]) == "scheme") {
        const int f = scheme_checks(argv[2]);
        std::printf("%s (%d failures)\n", f ? "FAILED" : "ok", f);
        return f ? 1 : 0;
    }
    if (argc >= 2 && std::string(argv[1]) == "newton") return newton_run(argc, argv);
    std::fprintf(stderr, "usage: test_scheme_api scheme <exact.txt> | newton <u0.bin> <n> <gamma> <h> <prefix>\n");
    return 2;
}
