// Reference header name (proj/include/nls2d/run_config.hpp): RunConfig and the
// key = value config files, restated header-only for the GPU path
// (run_config.cpp:9-130).  Same keys, defaults, validation and error texts.
#pragma once

#include <algorithm>
#include <cctype>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "nls2d/mb4cu_api.hpp"

namespace nls2d {

class ConfigError : public std::runtime_error {
public:
    explicit ConfigError(const std::string& what) : std::runtime_error(what) {}
};

enum class InitialKind { Cosine, Uniform };

struct RunConfig {
    double lx = 2.0 * 3.14159265358979323846;
    double ly = 2.0 * 3.14159265358979323846;
    int nx = 70;
    int ny = 70;
    double t_end = 1.0;
    double dt = 0.01;
    double gamma = 0.1;
    double v0 = 0.0;  // depth of the single-point potential; 0 disables
    MethodId method = MethodId::Mb4;
    double epsilon = 1e-13;
    int max_iters = 50;
    int max_halvings = 4;
    int workers = 1;  // 1..3 (accepted; the GPU path has no worker pool)
    InitialKind initial = InitialKind::Cosine;
    bool raw_participation = false;
    SolverKind solver = SolverKind::Direct;  // accepted; no sparse factorization here
    std::vector<double> snapshot_times;
    std::string out_dir;

    void validate() const {
        if (nx < 2 || ny < 2) throw ConfigError("nx and ny must be >= 2");
        if (!(lx > 0.0) || !(ly > 0.0)) throw ConfigError("lx and ly must be positive");
        if (!(dt > 0.0)) throw ConfigError("dt must be positive");
        if (!(t_end >= dt)) throw ConfigError("t_end must be >= dt");
        if (!(epsilon > 0.0)) throw ConfigError("epsilon must be positive");
        if (max_iters < 1) throw ConfigError("max_iters must be >= 1");
        if (max_halvings < 0) throw ConfigError("max_halvings must be >= 0");
        if (workers < 1 || workers > 3) throw ConfigError("workers must be in 1..3");
        for (double t : snapshot_times)
            if (t < 0.0 || t > t_end + 1e-12) throw ConfigError("snapshot time outside [0, t_end]");
    }
    GridModel make_model() const {
        const GridSpec grid(nx, ny, lx, ly);
        if (v0 != 0.0) return GridModel(grid, gamma, build_delta_potential(grid, v0));
        return GridModel(grid, gamma);
    }
    State make_initial(const GridModel& model) const {
        if (initial == InitialKind::Cosine) return initial_condition(model.grid());
        const int n = model.points();
        return State(n, Complex(1.0 / std::sqrt(static_cast<double>(n)), 0.0));
    }
};

namespace detail {
// strict numeric fields: the whole value must parse (run_config.cpp:36-58 semantics)
inline double to_double(const std::string& key, const std::string& v) {
    char* end = nullptr;
    const double x = v.empty() ? 0.0 : std::strtod(v.c_str(), &end);
    if (v.empty() || end != v.c_str() + v.size()) throw ConfigError("invalid numeric value for " + key + ": '" + v + "'");
    return x;
}
inline int to_int(const std::string& key, const std::string& v) {
    char* end = nullptr;
    const long x = v.empty() ? 0 : std::strtol(v.c_str(), &end, 10);
    if (v.empty() || end != v.c_str() + v.size() || x < INT_MIN || x > INT_MAX)
        throw ConfigError("invalid integer value for " + key + ": '" + v + "'");
    return static_cast<int>(x);
}
inline std::string strip(const std::string& s) {
    std::size_t a = 0, b = s.size();
    while (a < b && std::isspace(static_cast<unsigned char>(s[a]))) ++a;
    while (b > a && std::isspace(static_cast<unsigned char>(s[b - 1]))) --b;
    return s.substr(a, b - a);
}
// one of two spellings -> flag, else the reference's error text
inline bool choice(const std::string& v, const char* no, const char* yes, const char* err) {
    if (v == no) return false;
    if (v == yes) return true;
    throw ConfigError(err);
}
}  // namespace detail

/// The reference's keys (run_config.cpp:60-108), table-driven.
inline void apply_key_value(RunConfig& cfg, const std::string& key, const std::string& value) {
    using Setter = void (*)(RunConfig&, const std::string&, const std::string&);
    struct Entry {
        const char* key;
        Setter set;
    };
    static const Entry table[] = {
        {"lx", [](RunConfig& c, const std::string& k, const std::string& v) { c.lx = detail::to_double(k, v); }},
        {"ly", [](RunConfig& c, const std::string& k, const std::string& v) { c.ly = detail::to_double(k, v); }},
        {"nx", [](RunConfig& c, const std::string& k, const std::string& v) { c.nx = detail::to_int(k, v); }},
        {"ny", [](RunConfig& c, const std::string& k, const std::string& v) { c.ny = detail::to_int(k, v); }},
        {"t_end", [](RunConfig& c, const std::string& k, const std::string& v) { c.t_end = detail::to_double(k, v); }},
        {"dt", [](RunConfig& c, const std::string& k, const std::string& v) { c.dt = detail::to_double(k, v); }},
        {"gamma", [](RunConfig& c, const std::string& k, const std::string& v) { c.gamma = detail::to_double(k, v); }},
        {"v0", [](RunConfig& c, const std::string& k, const std::string& v) { c.v0 = detail::to_double(k, v); }},
        {"epsilon",
         [](RunConfig& c, const std::string& k, const std::string& v) { c.epsilon = detail::to_double(k, v); }},
        {"max_iters",
         [](RunConfig& c, const std::string& k, const std::string& v) { c.max_iters = detail::to_int(k, v); }},
        {"max_halvings",
         [](RunConfig& c, const std::string& k, const std::string& v) { c.max_halvings = detail::to_int(k, v); }},
        {"workers", [](RunConfig& c, const std::string& k, const std::string& v) { c.workers = detail::to_int(k, v); }},
        {"method",
         [](RunConfig& c, const std::string&, const std::string& v) {
             const auto m = parse_method(v);
             if (!m) throw ConfigError("unknown method: '" + v + "'");
             c.method = *m;
         }},
        {"initial",
         [](RunConfig& c, const std::string&, const std::string& v) {
             c.initial = detail::choice(v, "cosine", "uniform", "initial must be 'cosine' or 'uniform'")
                             ? InitialKind::Uniform
                             : InitialKind::Cosine;
         }},
        {"participation",
         [](RunConfig& c, const std::string&, const std::string& v) {
             c.raw_participation =
                 detail::choice(v, "normalized", "raw", "participation must be 'normalized' or 'raw'");
         }},
        {"solver",
         [](RunConfig& c, const std::string&, const std::string& v) {
             c.solver = detail::choice(v, "direct", "gmres", "solver must be 'direct' or 'gmres'") ? SolverKind::Gmres
                                                                                                  : SolverKind::Direct;
         }},
        {"snapshot_times",
         [](RunConfig& c, const std::string& k, const std::string& v) {
             c.snapshot_times.clear();
             std::size_t start = 0;
             while (start <= v.size()) {
                 const std::size_t comma = std::min(v.find(',', start), v.size());
                 const std::string item = detail::strip(v.substr(start, comma - start));
                 if (!item.empty()) c.snapshot_times.push_back(detail::to_double(k, item));
                 start = comma + 1;
             }
         }},
        {"out_dir", [](RunConfig& c, const std::string&, const std::string& v) { c.out_dir = v; }},
    };
    for (const Entry& e : table)
        if (key == e.key) return e.set(cfg, key, value);
    throw ConfigError("unknown config key: '" + key + "'");
}

/// Flat key = value file; '#' starts a comment; unknown keys are errors
/// (run_config.cpp:110-128).
inline RunConfig parse_config_file(const std::string& path, RunConfig base = {}) {
    std::ifstream in(path);
    if (!in) throw ConfigError("cannot open config file: " + path);
    int lineno = 0;
    for (std::string raw; std::getline(in, raw);) {
        ++lineno;
        const std::string text = detail::strip(raw.substr(0, raw.find('#')));
        if (text.empty()) continue;
        const auto eq = text.find('=');
        if (eq == std::string::npos)
            throw ConfigError(path + ":" + std::to_string(lineno) + ": expected key = value");
        apply_key_value(base, detail::strip(text.substr(0, eq)), detail::strip(text.substr(eq + 1)));
    }
    return base;
}

}  // namespace nls2d
