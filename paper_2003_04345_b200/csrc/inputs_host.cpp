// BASELINE input generator (host, multithreaded, deterministic).
//
// The reference's RunConfig can only express the single-site delta potential
// and the cosine / uniform initial states (run_config.cpp:22-32), so the
// BASELINE configs (seeded random defects, Gaussian packets) need this new
// layer.  Conventions, fixed here and documented in DESIGN.md:
//  - defects: site with global index k = j*gnx + i is a defect iff
//    u01(splitmix64(seed, k)) < frac; its V is vd_min, or U[vd_min, vd_max)
//    drawn from a second counter stream when vd_max > vd_min;
//  - packets: psi(i,j) = sum_p exp(-(dx^2+dy^2)/(2 sigma^2)) e^{i(kx dx + ky dy + phi_p)}
//    with (dx, dy) the periodic minimum-image offset of (i,j) from the packet
//    centre; the separable 1-D factors are tabulated per packet;
//  - normalisation sum |psi|^2 = 1 is applied by the caller (global sum).
// Counter-based hashing makes every site independent of the decomposition, so
// a rank's sub-block equals the same block of the single-GPU lattice.
#include <algorithm>
#include <cmath>
#include <complex>
#include <thread>
#include <vector>

#include "mb4cu.h"
#include "mb4cu_internal.hpp"

namespace mb4cu {
namespace {

inline uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

inline double u01(uint64_t h) { return static_cast<double>(h >> 11) * (1.0 / 9007199254740992.0); }

inline uint64_t site_hash(uint64_t seed, uint64_t stream, uint64_t k) {
    return splitmix64(splitmix64(seed * 0x2545F4914F6CDD1Dull + stream) ^ k);
}

struct Packet {
    double cx, cy, kx, ky, phase;
};

// minimum-image offset of coordinate i from centre c on a ring of length n
inline double min_image(double i, double c, int n) {
    double d = std::fmod(i - c, static_cast<double>(n));
    if (d < -0.5 * n) d += n;
    if (d >= 0.5 * n) d -= n;
    return d;
}

int resolve_threads(int t) {
    if (t > 0) return t;
    const unsigned hc = std::thread::hardware_concurrency();
    return hc ? static_cast<int>(std::min(hc, 64u)) : 1;
}

template <typename F>
void parallel_rows(int rows, int threads, F&& body) {
    threads = std::max(1, std::min(threads, rows));
    if (threads == 1) {
        body(0, rows);
        return;
    }
    std::vector<std::thread> pool;
    pool.reserve(threads);
    for (int t = 0; t < threads; ++t) {
        const int r0 = static_cast<int>(static_cast<long long>(rows) * t / threads);
        const int r1 = static_cast<int>(static_cast<long long>(rows) * (t + 1) / threads);
        pool.emplace_back([&, r0, r1] { body(r0, r1); });
    }
    for (auto& th : pool) th.join();
}

}  // namespace

int make_inputs(const mb4cu_inputs* sp, int x0, int y0, int lnx, int lny, double* V,
                double* psi, double* psum, std::string& why) {
    if (!sp || sp->gnx < 2 || sp->gny < 2 || lnx < 1 || lny < 1 || x0 < 0 || y0 < 0 ||
        x0 + lnx > sp->gnx || y0 + lny > sp->gny) {
        why = "make_inputs: bad lattice / block";
        return MB4CU_INVALID;
    }
    if (sp->npackets < 0 || (sp->npackets > 0 && !(sp->sigma > 0.0))) {
        why = "make_inputs: bad packet spec";
        return MB4CU_INVALID;
    }
    const int threads = resolve_threads(sp->threads);
    const uint64_t gnx = static_cast<uint64_t>(sp->gnx);

    if (V) {
        parallel_rows(lny, threads, [&](int r0, int r1) {
            for (int jl = r0; jl < r1; ++jl)
                for (int il = 0; il < lnx; ++il) {
                    const uint64_t k = static_cast<uint64_t>(y0 + jl) * gnx + static_cast<uint64_t>(x0 + il);
                    double v = 0.0;
                    if (u01(site_hash(sp->defect_seed, 1, k)) < sp->defect_frac) {
                        v = sp->vd_min;
                        if (sp->vd_max > sp->vd_min)
                            v = sp->vd_min + (sp->vd_max - sp->vd_min) * u01(site_hash(sp->defect_seed, 2, k));
                    }
                    V[static_cast<size_t>(jl) * lnx + il] = v;
                }
        });
    }

    if (psi) {
        std::vector<Packet> pk(static_cast<size_t>(sp->npackets));
        if (sp->random_packets) {
            for (int p = 0; p < sp->npackets; ++p) {
                const uint64_t b = static_cast<uint64_t>(p) * 8;
                pk[p].cx = std::floor(u01(site_hash(sp->packet_seed, 3, b + 0)) * sp->gnx);
                pk[p].cy = std::floor(u01(site_hash(sp->packet_seed, 3, b + 1)) * sp->gny);
                pk[p].kx = sp->k_max * (2.0 * u01(site_hash(sp->packet_seed, 3, b + 2)) - 1.0);
                pk[p].ky = sp->k_max * (2.0 * u01(site_hash(sp->packet_seed, 3, b + 3)) - 1.0);
                pk[p].phase = 2.0 * M_PI * u01(site_hash(sp->packet_seed, 3, b + 4));
            }
        } else {
            for (auto& p : pk) p = Packet{sp->x0, sp->y0, sp->kx, sp->ky, 0.0};
        }
        // separable per-packet factors gx_p(i), gy_p(j)
        const double inv2s2 = sp->npackets ? 1.0 / (2.0 * sp->sigma * sp->sigma) : 0.0;
        std::vector<std::complex<double>> gx(pk.size() * lnx), gy(pk.size() * lny);
        for (size_t p = 0; p < pk.size(); ++p) {
            for (int il = 0; il < lnx; ++il) {
                const double d = min_image(x0 + il, pk[p].cx, sp->gnx);
                gx[p * lnx + il] = std::exp(-d * d * inv2s2) * std::polar(1.0, pk[p].kx * d + pk[p].phase);
            }
            for (int jl = 0; jl < lny; ++jl) {
                const double d = min_image(y0 + jl, pk[p].cy, sp->gny);
                gy[p * lny + jl] = std::exp(-d * d * inv2s2) * std::polar(1.0, pk[p].ky * d);
            }
        }
        std::vector<double> partial(static_cast<size_t>(lny), 0.0);
        parallel_rows(lny, threads, [&](int r0, int r1) {
            for (int jl = r0; jl < r1; ++jl) {
                double rowsum = 0.0;
                for (int il = 0; il < lnx; ++il) {
                    std::complex<double> acc(0.0, 0.0);
                    for (size_t p = 0; p < pk.size(); ++p) acc += gx[p * lnx + il] * gy[p * lny + jl];
                    const size_t k = static_cast<size_t>(jl) * lnx + il;
                    psi[2 * k] = acc.real();
                    psi[2 * k + 1] = acc.imag();
                    rowsum += std::norm(acc);
                }
                partial[jl] = rowsum;
            }
        });
        if (psum) {
            double s = 0.0;  // fixed row order: deterministic for any thread count
            for (double r : partial) s += r;
            *psum = s;
        }
    }
    return MB4CU_OK;
}

int scale_state(double* psi, size_t nsites, double s, int threads) {
    if (!psi) return MB4CU_INVALID;
    const size_t n = 2 * nsites;
    const int rows = static_cast<int>(std::min<size_t>(n / 4096 + 1, 1 << 20));
    parallel_rows(rows, resolve_threads(threads), [&](int r0, int r1) {
        const size_t b = n * static_cast<size_t>(r0) / rows, e = n * static_cast<size_t>(r1) / rows;
        for (size_t i = b; i < e; ++i) psi[i] *= s;
    });
    return MB4CU_OK;
}

}  // namespace mb4cu
