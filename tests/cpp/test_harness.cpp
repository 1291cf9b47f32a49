// C++ drop-in check for the reference harness API (run_config.hpp, harness.hpp):
// code written against the reference's harness compiles unchanged against
// include/nls2d and runs on the GPU.  usage: test_harness <out_dir>; exit code =
// number of failures.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>

#include "nls2d/harness.hpp"
#include "nls2d/run_config.hpp"

using namespace nls2d;

static int failures = 0;
#define CHECK(cond)                                                                  \
    do {                                                                             \
        if (!(cond)) {                                                               \
            std::fprintf(stderr, "CHECK failed at line %d: %s\n", __LINE__, #cond); \
            ++failures;                                                              \
        }                                                                            \
    } while (0)

int main(int argc, char** argv) {
    if (argc != 2) return 100;
    const std::string dir = argv[1];
    // config file parsing and validation (run_config.cpp)
    {
        std::ofstream f(dir + "/run.cfg");
        f << "# paper-style run\nnx = 16\nny = 16   # trailing comment\nt_end = 0.05\ndt = 0.01\n"
             "method = avf2\nsnapshot_times = 0.0, 0.03\nsolver = gmres\nworkers = 3\n";
    }
    RunConfig cfg = parse_config_file(dir + "/run.cfg");
    CHECK(cfg.nx == 16 && cfg.method == MethodId::Avf2 && cfg.solver == SolverKind::Gmres && cfg.workers == 3);
    CHECK(cfg.snapshot_times.size() == 2 && cfg.snapshot_times[1] == 0.03);
    bool threw = false;
    try {
        apply_key_value(cfg, "no_such_key", "1");
    } catch (const ConfigError&) {
        threw = true;
    }
    CHECK(threw);
    threw = false;
    try {
        RunConfig bad;
        bad.workers = 4;
        bad.validate();
    } catch (const ConfigError&) {
        threw = true;
    }
    CHECK(threw);
    // run() with files: rows, CSV header, snapshots
    cfg.out_dir = dir + "/out";
    const TrajectoryRecord rec = run(cfg);
    CHECK(rec.rows.size() == 6);
    CHECK(rec.max_energy_drift() <= 1e-11);  // AVF2 conserves the energy
    std::ifstream csv(cfg.out_dir + "/trajectory.csv");
    std::string header;
    std::getline(csv, header);
    CHECK(header == "t,UK,UI,UE,H,prob,participation,newton_iters,wall_s");
    CHECK(std::ifstream(cfg.out_dir + "/snapshot_0.03.txt").good());
    // studies
    RunConfig small;
    small.nx = small.ny = 16;
    small.t_end = 0.05;
    const CompareReport cmp = compare_methods(small, {MethodId::Gauss2, MethodId::Mb4, MethodId::Avf4});
    CHECK(cmp.methods.size() == 3 && cmp.methods[1].energy_drift <= 1e-11 && cmp.methods[0].probability_drift <= 1e-12);
    std::ostringstream os;
    cmp.write(os);
    CHECK(os.str().rfind("method  energy_drift", 0) == 0);
    RunConfig conv = small;
    conv.t_end = 0.2;
    const ConvergenceReport cr = convergence_study(conv, {MethodId::Gauss4}, {0.02, 0.01, 0.005});
    CHECK(cr.entries.size() == 1 && std::abs(cr.entries[0].slope - 4.0) < 0.4);
    const BenchReport br = parallel_bench(small);
    CHECK(br.trajectories_identical);
    std::printf("test_harness: %d failure(s)\n", failures);
    return failures;
}
