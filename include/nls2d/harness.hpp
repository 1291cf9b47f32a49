// Reference header name (proj/include/nls2d/harness.hpp): run(), the trajectory
// CSV, snapshots and the method studies, header-only on the GPU path.
//
// Behaviour follows harness.cpp:16-316 (row contents, CSV / snapshot / report
// formats, drift definition, the shorter last step, NonConvergenceError::at_time)
// with one structural difference: the run is stepped device-resident in chunks
// between snapshot times (DeviceSession::run), so the per-step energy rows come
// from the library's energy monitor and wall_s is the chunk's time divided evenly
// over its steps; for MB4 newton_iters counts stage sweeps.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <limits>
#include <ostream>
#include <string>
#include <vector>

#include "nls2d/run_config.hpp"

namespace nls2d {

struct TrajectoryRow {
    double t = 0.0;
    double u_kinetic = 0.0;
    double u_nonlinear = 0.0;
    double u_external = 0.0;
    double total_energy = 0.0;
    double probability = 0.0;
    double participation = 0.0;
    int newton_iters = 0;
    double wall_seconds = 0.0;
};

struct TrajectoryRecord {
    std::vector<TrajectoryRow> rows;
    State final_state;
    double solve_seconds = 0.0;  // device time of the steps
    double wall_seconds = 0.0;   // whole stepping loop

    /// Deviation maxima relative to the t = 0 row (harness.cpp:16-19, 44-58).
    double max_energy_drift() const { return max_drift(&TrajectoryRow::total_energy); }
    double max_probability_drift() const { return max_drift(&TrajectoryRow::probability); }

private:
    double max_drift(double TrajectoryRow::*field) const {
        if (rows.empty()) return 0.0;
        const double base = rows.front().*field;
        double worst = 0.0;
        for (const auto& r : rows) {
            const double v = r.*field;
            const double d = std::isfinite(v) ? std::abs(v - base) / std::max(1.0, std::abs(base))
                                              : std::numeric_limits<double>::infinity();
            worst = std::max(worst, d);
        }
        return worst;
    }
};

namespace detail {
inline std::string fmt(const char* f, double v) {
    char buf[48];
    std::snprintf(buf, sizeof(buf), f, v);
    return buf;
}
inline int steps_to(double t_end, double dt) { return static_cast<int>(std::ceil(t_end / dt - 1e-9)); }

// "# t nx ny", then |u|^2 per site, one grid row per line (harness.cpp:27-40)
inline void snapshot_file(const std::string& path, double t, const GridSpec& g, const State& u) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot open snapshot file: " + path);
    out << "# " << fmt("%.17g", t) << ' ' << g.nx << ' ' << g.ny << '\n';
    for (int j = 0; j < g.ny; ++j)
        for (int i = 0; i < g.nx; ++i)
            out << fmt("%.17g", std::norm(u[g.index(i, j)])) << (i + 1 == g.nx ? '\n' : ' ');
}
}  // namespace detail

inline void write_trajectory_csv(std::ostream& os, const TrajectoryRecord& record) {
    os << "t,UK,UI,UE,H,prob,participation,newton_iters,wall_s\n";
    for (const auto& r : record.rows) {
        const double vals[7] = {r.t, r.u_kinetic, r.u_nonlinear, r.u_external, r.total_energy, r.probability,
                                r.participation};
        for (double v : vals) os << detail::fmt("%.17g", v) << ',';
        os << r.newton_iters << ',' << detail::fmt("%.6g", r.wall_seconds) << '\n';
    }
}

/// Steps the configured problem to t_end on the GPU, one energy row per step;
/// trajectory.csv and snapshot files when cfg.out_dir is set.
inline TrajectoryRecord run(const RunConfig& cfg) {
    cfg.validate();
    const GridModel model = cfg.make_model();
    const NewtonConfig ncfg{cfg.epsilon, cfg.max_iters, cfg.max_halvings};
    DeviceSession session(model, Mb4Scheme(), ncfg, -1, 0, 0, cfg.method);
    session.set_state(cfg.make_initial(model));

    const bool files = !cfg.out_dir.empty();
    if (files) std::filesystem::create_directories(cfg.out_dir);
    std::vector<double> snaps = cfg.snapshot_times;
    std::sort(snaps.begin(), snaps.end());
    std::size_t next_snap = 0;
    auto take_snapshots = [&](double t) {
        while (next_snap < snaps.size() && t + 1e-12 >= snaps[next_snap]) {
            if (files)
                detail::snapshot_file(cfg.out_dir + "/snapshot_" + detail::fmt("%g", snaps[next_snap]) + ".txt", t,
                                      model.grid(), session.get_state());
            ++next_snap;
        }
    };
    TrajectoryRecord rec;
    auto push_row = [&](double t, const Observables& o, int iters, double wall) {
        rec.rows.push_back({t, o.u_kinetic, o.u_nonlinear, o.u_external, o.total_energy, o.probability,
                            cfg.raw_participation ? o.raw_quartic : o.participation, iters, wall});
    };

    const int nsteps = detail::steps_to(cfg.t_end, cfg.dt);
    const double last_h = std::min(nsteps * cfg.dt, cfg.t_end) - (nsteps - 1) * cfg.dt;
    const auto start = std::chrono::steady_clock::now();
    push_row(0.0, session.observables(), 0, 0.0);
    take_snapshots(0.0);
    int done = 0;
    while (done < nsteps) {
        int chunk_end = nsteps;  // up to the next snapshot step
        if (next_snap < snaps.size())
            chunk_end = std::min(nsteps, std::max(done + 1, detail::steps_to(snaps[next_snap], cfg.dt)));
        // uniform steps of dt, then (at the very end) the possibly shorter last step
        const bool short_last = chunk_end == nsteps && std::abs(last_h - cfg.dt) >= 1e-15;
        const int uniform = chunk_end - done - (short_last ? 1 : 0);
        for (int part = 0; part < 2; ++part) {
            const int k = part == 0 ? uniform : (short_last ? 1 : 0);
            if (k <= 0) continue;
            const double h = part == 0 ? cfg.dt : last_h;
            StepStats st;
            std::vector<int> iters;
            const auto t0 = std::chrono::steady_clock::now();
            std::vector<Observables> rows;
            try {
                rows = session.run(h, k, &iters, &st);
            } catch (NonConvergenceError& e) {
                e.at_time = done * cfg.dt;
                throw;
            }
            const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / k;
            rec.solve_seconds += st.solve_seconds;
            for (int q = 0; q < k; ++q) {
                ++done;
                push_row(std::min(done * cfg.dt, cfg.t_end), rows[static_cast<size_t>(q) + 1],
                         iters[static_cast<size_t>(q)], wall);
            }
        }
        take_snapshots(std::min(done * cfg.dt, cfg.t_end));
    }
    rec.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
    rec.final_state = session.get_state();
    if (files) {
        std::ofstream f(cfg.out_dir + "/trajectory.csv");
        if (!f) throw std::runtime_error("cannot open trajectory.csv in " + cfg.out_dir);
        write_trajectory_csv(f, rec);
    }
    return rec;
}

struct MethodReport {
    MethodId method = MethodId::Mb4;
    double energy_drift = 0.0;
    double probability_drift = 0.0;
    double mean_step_seconds = 0.0;
    int total_newton_iters = 0;
};

struct CompareReport {
    std::vector<MethodReport> methods;
    double mb4_over_gauss2 = 0.0;
    double avf4_over_gauss2 = 0.0;

    void write(std::ostream& os) const {  // harness.cpp:180-196
        os << "method  energy_drift  probability_drift  mean_step_seconds  newton_iters\n";
        for (const auto& m : methods) {
            char buf[192];
            std::snprintf(buf, sizeof(buf), "%-7s %.3e     %.3e          %.6f           %d\n",
                          method_name(m.method).c_str(), m.energy_drift, m.probability_drift, m.mean_step_seconds,
                          m.total_newton_iters);
            os << buf;
        }
        os << detail::fmt("time ratio MB4/GAUSS2  = %.3f\n", mb4_over_gauss2);
        os << detail::fmt("time ratio AVF4/GAUSS2 = %.3f\n", avf4_over_gauss2);
    }
};

inline CompareReport compare_methods(const RunConfig& cfg, const std::vector<MethodId>& methods) {
    CompareReport rep;
    double t_gauss2 = 0.0, t_mb4 = 0.0, t_avf4 = 0.0;
    for (MethodId m : methods) {
        RunConfig c = cfg;
        c.method = m;
        c.out_dir.clear();
        const TrajectoryRecord rec = run(c);
        MethodReport mr;
        mr.method = m;
        mr.energy_drift = rec.max_energy_drift();
        mr.probability_drift = rec.max_probability_drift();
        double wall = 0.0;
        for (const auto& r : rec.rows) {
            wall += r.wall_seconds;
            mr.total_newton_iters += r.newton_iters;
        }
        mr.mean_step_seconds = wall / static_cast<double>(std::max<std::size_t>(1, rec.rows.size() - 1));
        if (m == MethodId::Gauss2) t_gauss2 = mr.mean_step_seconds;
        if (m == MethodId::Mb4) t_mb4 = mr.mean_step_seconds;
        if (m == MethodId::Avf4) t_avf4 = mr.mean_step_seconds;
        rep.methods.push_back(mr);
    }
    if (t_gauss2 > 0.0) {
        rep.mb4_over_gauss2 = t_mb4 / t_gauss2;
        rep.avf4_over_gauss2 = t_avf4 / t_gauss2;
    }
    return rep;
}

struct BenchReport {
    double serial_step_seconds = 0.0;
    double parallel_step_seconds = 0.0;
    double speedup = 0.0;
    double solve_fraction = 0.0;
    bool trajectories_identical = false;

    void write(std::ostream& os) const {  // harness.cpp:259-270
        os << detail::fmt("per-step seconds, 1 worker  = %.6f\n", serial_step_seconds);
        os << detail::fmt("per-step seconds, 3 workers = %.6f\n", parallel_step_seconds);
        os << detail::fmt("speedup                     = %.3f\n", speedup);
        os << detail::fmt("solve-phase fraction        = %.3f\n", solve_fraction);
        os << "trajectories bit-identical  = " << (trajectories_identical ? "yes" : "no") << '\n';
    }
};

/// MB4 with workers = 1 and 3 (the GPU path ignores workers: both runs take the same
/// path and must agree bit for bit).
inline BenchReport parallel_bench(const RunConfig& cfg) {
    RunConfig base = cfg;
    base.method = MethodId::Mb4;
    base.out_dir.clear();
    RunConfig one = base, three = base;
    one.workers = 1;
    three.workers = 3;
    const TrajectoryRecord a = run(one), b = run(three);
    const double steps = static_cast<double>(std::max<std::size_t>(1, a.rows.size() - 1));
    BenchReport rep;
    rep.serial_step_seconds = a.wall_seconds / steps;
    rep.parallel_step_seconds = b.wall_seconds / steps;
    rep.speedup = rep.serial_step_seconds / rep.parallel_step_seconds;
    rep.solve_fraction = a.solve_seconds / a.wall_seconds;
    bool same = a.rows.size() == b.rows.size() && a.final_state == b.final_state;
    for (std::size_t i = 0; same && i < a.rows.size(); ++i) {
        const auto &x = a.rows[i], &y = b.rows[i];
        same = x.t == y.t && x.u_kinetic == y.u_kinetic && x.u_nonlinear == y.u_nonlinear &&
               x.u_external == y.u_external && x.total_energy == y.total_energy && x.probability == y.probability &&
               x.participation == y.participation && x.newton_iters == y.newton_iters;
    }
    rep.trajectories_identical = same;
    return rep;
}

struct ConvergenceReport {
    struct Entry {
        MethodId method;
        std::vector<double> h_values;
        std::vector<double> errors;  // relative l2 error at t_end vs the reference run
        double slope = 0.0;          // least-squares log-log fit
    };
    std::vector<Entry> entries;

    void write(std::ostream& os) const {  // harness.cpp:301-313
        for (const auto& e : entries) {
            os << method_name(e.method) << ":\n";
            for (std::size_t i = 0; i < e.h_values.size(); ++i) {
                char buf[96];
                std::snprintf(buf, sizeof(buf), "  h = %-10.6g error = %.6e\n", e.h_values[i], e.errors[i]);
                os << buf;
            }
            os << detail::fmt("  fitted order = %.3f\n", e.slope);
        }
    }
};

/// Errors against a same-method run at h_min / 8 (harness.cpp:272-299).
inline ConvergenceReport convergence_study(const RunConfig& cfg, const std::vector<MethodId>& methods,
                                           const std::vector<double>& h_list) {
    if (h_list.size() < 3) throw ConfigError("convergence_study: need at least 3 h values");
    for (std::size_t i = 1; i < h_list.size(); ++i)
        if (!(h_list[i] < h_list[i - 1])) throw ConfigError("convergence_study: h_list must descend");
    auto norm2 = [](const State& a, const State* b) {
        double s = 0.0;
        for (std::size_t k = 0; k < a.size(); ++k) s += std::norm(b ? a[k] - (*b)[k] : a[k]);
        return std::sqrt(s);
    };
    ConvergenceReport rep;
    for (MethodId m : methods) {
        RunConfig base = cfg;
        base.method = m;
        base.out_dir.clear();
        base.snapshot_times.clear();
        RunConfig fine = base;
        fine.dt = h_list.back() / 8.0;
        const State ref = run(fine).final_state;
        const double ref_norm = norm2(ref, nullptr);
        ConvergenceReport::Entry e{m, {}, {}, 0.0};
        double sx = 0.0, sy = 0.0, sxx = 0.0, sxy = 0.0;
        for (double h : h_list) {
            RunConfig c = base;
            c.dt = h;
            const double err = norm2(run(c).final_state, &ref) / ref_norm;
            e.h_values.push_back(h);
            e.errors.push_back(err);
            const double x = std::log(h), y = std::log(err);
            sx += x;
            sy += y;
            sxx += x * x;
            sxy += x * y;
        }
        const double n = static_cast<double>(h_list.size());
        e.slope = (n * sxy - sx * sy) / (n * sxx - sx * sx);
        rep.entries.push_back(std::move(e));
    }
    return rep;
}

}  // namespace nls2d
