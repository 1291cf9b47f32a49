// Production stage-sweep kernel: one persistent cooperative launch per MB4 step.
//
// Replaces the per-step stage solve of the reference (mb4_single_step +
// newton_solve, mb4_integrator.cpp:194-271): every sweep is the fused
//   Phi (5-point (K+V) stencil + GL-6 cubic)  ->  T^-1  ->  M-term Neumann
//   (I - h lam_k J(u0))^-1  ->  T  ->  U += r  ->  ||r||_inf
// of site_math.cuh, sweeps repeat until ||r||_inf <= eps (same test as :250),
// and a grid-wide barrier separates sweeps.  The energy monitor of u0
// (observables, lattice.cpp:106-137) rides along in the first sweep, which
// already evaluates (K+V) u0.
//
// Layout and schedule:
//  - The lattice is cut into column bands of TX = NT - 2M output columns.  A
//    CTA of NT threads marches down a band row by row; thread t owns column
//    X0 - M + t at level 0.  Work (band-rows) is split evenly over the
//    persistent grid, so every CTA marches ~ (bands*ny)/grid rows.
//  - Stage inputs stream through shared-memory row rings filled by cp.async
//    (LDGSTS) P rows ahead; each level n of the Neumann recursion consumes the
//    previous level's rows from a 4-row ring one iteration later, so a single
//    __syncthreads per row suffices.  Level n at iteration i works on row
//    y0(i) - 2n; the output row trails the load front by 3M+1 rows.
//  - All HBM traffic of a sweep is: u0, V, U_in (read once, plus a thin
//    column halo) and U_out (written once): 120 B/site; the first sweep reads
//    only u0 and V: 72 B/site.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <atomic>

#include "mb4cu_internal.hpp"
#include "site_math.cuh"
#include "async_copy.cuh"

namespace cg = cooperative_groups;

namespace mb4cu {
namespace {

template <int M, int NT>
struct MarchGeom {
    static constexpr int TX = NT - 2 * M;       // output columns per band
    static constexpr int ZW = NT + 2;           // z columns held per row
    static constexpr int P = 2;                 // prefetch depth (rows)
    static constexpr int SU0 = 2 * M + 2 + P;   // u0 / V ring rows
    static constexpr int SU = 3 + P;            // U ring rows
    static constexpr int S0 = (2 * M + 1) > 4 ? (2 * M + 1) : 4;  // level-0 ring (phibar)
    static constexpr int SL = 4;                // level-n ring

    // shared-memory carve-up (bytes, all 16-aligned)
    static constexpr size_t u0_bytes = sizeof(double2) * SU0 * ZW;
    static constexpr size_t v_bytes = ((sizeof(double) * SU0 * ZW + 15) / 16) * 16;
    static constexpr size_t U_bytes = sizeof(double2) * SU * 3 * ZW;
    static constexpr size_t L0_bytes = M >= 1 ? sizeof(double2) * S0 * 3 * NT : 0;
    static constexpr size_t Ln_bytes = M >= 2 ? sizeof(double2) * (M - 1) * SL * 3 * NT : 0;
    static constexpr size_t bytes = u0_bytes + v_bytes + U_bytes + L0_bytes + Ln_bytes;
};

template <int M, int NT, bool FIRST>
struct March {
    using G = MarchGeom<M, NT>;

    double2* u0r;  // [SU0][ZW]
    double* vr;    // [SU0][ZW]
    double2* Ur;   // [SU][3][ZW]
    double2* L0;   // [S0][3][NT]
    double2* Ln;   // [M-1][SL][3][NT]

    __device__ March(unsigned char* smem) {
        u0r = reinterpret_cast<double2*>(smem);
        vr = reinterpret_cast<double*>(smem + G::u0_bytes);
        Ur = reinterpret_cast<double2*>(smem + G::u0_bytes + G::v_bytes);
        L0 = reinterpret_cast<double2*>(smem + G::u0_bytes + G::v_bytes + G::U_bytes);
        Ln = reinterpret_cast<double2*>(smem + G::u0_bytes + G::v_bytes + G::U_bytes + G::L0_bytes);
    }

    __device__ __forceinline__ double2& U_at(int slot, int i, int c) { return Ur[(slot * 3 + i) * G::ZW + c]; }
    __device__ __forceinline__ double2& L0_at(int slot, int k, int t) { return L0[(slot * 3 + k) * NT + t]; }
    __device__ __forceinline__ double2& Ln_at(int n, int slot, int k, int t) {
        return Ln[(((n - 1) * G::SL + slot) * 3 + k) * NT + t];
    }

    // March one band segment: output rows [Y0, Y0 + R) of band `band`.
    __device__ void run(const StepArgs& a, const SweepConsts& c, const double2* const uin[3],
                        double2* const uout[3], int band, int Y0, int R,
                        unsigned long long& rmax, double acc[kObsFields]) {
        const int t = threadIdx.x;
        const int X0 = band * G::TX;
        const int xz0 = X0 - M - 1;
        const int yz0 = Y0 - M - 1;
        const int nzrows = R + 2 * M + 2;
        const int nx = a.nx, ny = a.ny;

        auto issue_row = [&](int j) {
            if (j < nzrows) {
                const size_t rowoff = static_cast<size_t>(wrap_index(yz0 + j, ny)) * nx;
                const int s0 = j % G::SU0, s1 = j % G::SU;
                for (int col = t; col < G::ZW; col += NT) {
                    const size_t g = rowoff + wrap_index(xz0 + col, nx);
                    cp_async16(&u0r[s0 * G::ZW + col], a.u0 + g);
                    cp_async8(&vr[s0 * G::ZW + col], a.V + g);
                    if (!FIRST) {
#pragma unroll
                        for (int q = 0; q < 3; ++q) cp_async16(&U_at(s1, q, col), uin[q] + g);
                    }
                }
            }
            cp_async_commit();
        };

#pragma unroll
        for (int j = 0; j < G::P + 2; ++j) issue_row(j);

        const int niter = R + 3 * M;
        for (int i = 0; i < niter; ++i) {
            cp_async_wait<G::P - 1>();
            __syncthreads();
            issue_row(i + 2 + G::P);

            // final-level U_old reload (L2-resident: read by level 0 ~3M rows ago)
            double2 uold[3];
            const int yout = Y0 + i - 3 * M;
            const int xout = X0 - M + t;
            const bool out_ok = (M == 0 || (i >= 3 * M)) && t >= M && t < NT - M && xout < nx;
            if (M >= 1 && !FIRST && out_ok) {
                const size_t g = static_cast<size_t>(yout) * nx + xout;
#pragma unroll
                for (int q = 0; q < 3; ++q) uold[q] = __ldcg(uin[q] + g);
            }

            // ---- level 0: Phi / phibar at row y0(i) = Y0 - M + i, column t ----
            if (i < R + 2 * M) {
                const int sd = i % G::SU0, sc = (i + 1) % G::SU0, su = (i + 2) % G::SU0;
                const int ud = i % G::SU, uc = (i + 1) % G::SU, uu = (i + 2) % G::SU;
                const int cc = t + 1;
                double2 z[4], w[4];
                const double v = vr[sc * G::ZW + cc];
                z[0] = u0r[sc * G::ZW + cc];
                w[0] = kv_site(c, v, z[0], u0r[sc * G::ZW + cc - 1], u0r[sc * G::ZW + cc + 1],
                               u0r[sd * G::ZW + cc], u0r[su * G::ZW + cc]);
                if (FIRST) {
#pragma unroll
                    for (int q = 1; q < 4; ++q) {
                        z[q] = z[0];
                        w[q] = w[0];
                    }
                } else {
#pragma unroll
                    for (int q = 1; q < 4; ++q) {
                        z[q] = U_at(uc, q - 1, cc);
                        w[q] = kv_site(c, v, z[q], U_at(uc, q - 1, cc - 1), U_at(uc, q - 1, cc + 1),
                                       U_at(ud, q - 1, cc), U_at(uu, q - 1, cc));
                    }
                }
                if (FIRST) {
                    // energy monitor of u0 on owned sites
                    const int x = X0 - M + t;
                    if (t >= M && t < NT - M && x < nx && i >= M && i < M + R) {
                        const double2 u = z[0];
                        const double n2 = fma(u.x, u.x, u.y * u.y);
                        const double vn = v * n2;
                        acc[0] += fma(u.x, w[0].x, u.y * w[0].y) - vn;  // Re conj(u) K u
                        acc[1] += fma(u.x, w[0].y, -u.y * w[0].x);      // Im conj(u) K u
                        acc[2] += n2;
                        acc[3] += n2 * n2;
                        acc[4] += vn;
                    }
                }
                double2 phi[3];
                phi_site(c, z, w, phi);
                if (M == 0) {
                    const int x = X0 + t;
                    if (x < nx) {
                        const size_t g = static_cast<size_t>(Y0 + i) * nx + x;
#pragma unroll
                        for (int q = 0; q < 3; ++q) {
                            const double2 uo = FIRST ? z[0] : z[q + 1];
                            uout[q][g] = make_double2(uo.x - phi[q].x, uo.y - phi[q].y);
                            const unsigned long long bx = abs_bits(phi[q].x), by = abs_bits(phi[q].y);
                            rmax = bx > rmax ? bx : rmax;
                            rmax = by > rmax ? by : rmax;
                        }
                    }
                } else {
                    double2 pb[3];
                    to_eigen(c, phi, pb);
                    const int s = i % G::S0;
#pragma unroll
                    for (int k = 0; k < 3; ++k) L0_at(s, k, t) = pb[k];
                }
            }

            // ---- levels 1..M: b_n = phibar + h lam J b_{n-1} at row y0(i) - 2n ----
#pragma unroll
            for (int n = 1; n <= M; ++n) {
                if (i >= 3 * n && i < R + 2 * M + n && t >= n && t < NT - n) {
                    const int jz = (i - 2 * n + 1) % G::SU0;  // z ring slot of this row
                    const double2 u0c = u0r[jz * G::ZW + t + 1];
                    const double v = vr[jz * G::ZW + t + 1];
                    const JDiag dg = jdiag(u0c);
                    const int sp = (i - 2 * n) % G::S0;  // phibar of this row
                    double2 b[3];
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        double2 tc, tl, tr, td, tu;
                        if (n == 1) {
                            const int r0 = (i - 3) % G::S0, r1 = (i - 2) % G::S0, r2 = (i - 1) % G::S0;
                            tc = L0_at(r1, k, t);
                            tl = L0_at(r1, k, t - 1);
                            tr = L0_at(r1, k, t + 1);
                            td = L0_at(r0, k, t);
                            tu = L0_at(r2, k, t);
                        } else {
                            const int r0 = (i - 3) % G::SL, r1 = (i - 2) % G::SL, r2 = (i - 1) % G::SL;
                            tc = Ln_at(n - 1, r1, k, t);
                            tl = Ln_at(n - 1, r1, k, t - 1);
                            tr = Ln_at(n - 1, r1, k, t + 1);
                            td = Ln_at(n - 1, r0, k, t);
                            tu = Ln_at(n - 1, r2, k, t);
                        }
                        const double2 ak = kv_site(c, v, tc, tl, tr, td, tu);
                        const double2 jt = j_site(c, dg, tc, ak);
                        const double2 pb = L0_at(sp, k, t);
                        b[k] = make_double2(fma(c.hlam[k], jt.x, pb.x), fma(c.hlam[k], jt.y, pb.y));
                    }
                    if (n == M) {
                        if (xout < nx) {
                            double2 rb[3], r[3];
#pragma unroll
                            for (int k = 0; k < 3; ++k) rb[k] = make_double2(-b[k].x, -b[k].y);
                            from_eigen(c, rb, r);
                            const size_t g = static_cast<size_t>(yout) * nx + xout;
#pragma unroll
                            for (int q = 0; q < 3; ++q) {
                                const double2 uo = FIRST ? u0c : uold[q];
                                uout[q][g] = make_double2(uo.x + r[q].x, uo.y + r[q].y);
                                const unsigned long long bx = abs_bits(r[q].x), by = abs_bits(r[q].y);
                                rmax = bx > rmax ? bx : rmax;
                                rmax = by > rmax ? by : rmax;
                            }
                        }
                    } else {
                        const int s = i % G::SL;
#pragma unroll
                        for (int k = 0; k < 3; ++k) Ln_at(n, s, k, t) = b[k];
                    }
                }
            }
        }
        cp_async_wait<0>();
        __syncthreads();
    }
};

// Evenly split the band-rows over the grid and march every segment.
template <int M, int NT, bool FIRST>
__device__ void sweep_all(const StepArgs& a, const SweepConsts& c, unsigned char* smem,
                          const double2* const uin[3], double2* const uout[3],
                          unsigned long long& rmax, double acc[kObsFields]) {
    March<M, NT, FIRST> m(smem);
    const long long G = gridDim.x;
    const long long b0 = a.total * blockIdx.x / G;
    const long long b1 = a.total * (blockIdx.x + 1) / G;
    long long pos = b0;
    while (pos < b1) {
        const int band = static_cast<int>(pos / a.ny);
        const int row = static_cast<int>(pos - static_cast<long long>(band) * a.ny);
        const long long seg_end = static_cast<long long>(band + 1) * a.ny < b1
                                      ? static_cast<long long>(band + 1) * a.ny
                                      : b1;
        const int R = static_cast<int>(seg_end - pos);
        m.run(a, c, uin, uout, band, row, R, rmax, acc);
        pos = seg_end;
    }
}

template <int M, int NT>
__global__ void __launch_bounds__(NT, (M >= 3 ? 1 : 2))
mb4_step_kernel(const StepArgs a, const __grid_constant__ SweepConsts c) {
    extern __shared__ __align__(16) unsigned char smem[];
    cg::grid_group grid = cg::this_grid();
    double acc[kObsFields] = {0.0, 0.0, 0.0, 0.0, 0.0};
    int sweeps = 0, set = 0, converged = 0;
    double rlast = 0.0;
    for (int s = 0; s < a.max_iters; ++s) {
        const int out = s & 1;
        double2* const uout[3] = {a.U[out][0], a.U[out][1], a.U[out][2]};
        unsigned long long rmax = 0ull;
        if (s == 0) {
            const double2* const uin[3] = {a.u0, a.u0, a.u0};
            sweep_all<M, NT, true>(a, c, smem, uin, uout, rmax, acc);
            if (a.want_obs) {
                __shared__ double red[kObsFields][NT / 32];
#pragma unroll
                for (int f = 0; f < kObsFields; ++f) {
                    double v = acc[f];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                    if ((threadIdx.x & 31) == 0) red[f][threadIdx.x >> 5] = v;
                }
                __syncthreads();
                if (threadIdx.x < kObsFields) {
                    double v = 0.0;
                    for (int w = 0; w < NT / 32; ++w) v += red[threadIdx.x][w];
                    a.obs_partial[blockIdx.x * kObsFields + threadIdx.x] = v;
                }
            }
        } else {
            const int in = 1 - out;
            const double2* const uin[3] = {a.U[in][0], a.U[in][1], a.U[in][2]};
            sweep_all<M, NT, false>(a, c, smem, uin, uout, rmax, acc);
        }
        block_max_to(rmax, &a.rmax[s]);
        grid.sync();
        unsigned long long bits = __ldcg(&a.rmax[s]);
        // same widened high-word residual as the production kernel
        if (bits >> 32) bits = (bits & 0xFFFFFFFF00000000ull) | 0xFFFFFFFFull;
        const double rprev = rlast;
        rlast = __longlong_as_double(static_cast<long long>(bits));
        sweeps = s + 1;
        set = out;
        if (!isfinite(rlast)) break;
        if (stage_converged(rlast, rprev, s, a.eps)) {
            converged = 1;
            break;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.status->sweeps = sweeps;
        a.status->set = set;
        a.status->converged = converged;
        a.status->rlast = isfinite(rlast) ? rlast : __longlong_as_double(0x7FF0000000000000ll);  // NaN -> +inf
    }
    if (a.want_obs && blockIdx.x == 0 && threadIdx.x < kObsFields) {
        // fixed-order sum of the block partials written before the first grid.sync
        double v = 0.0;
        for (int b = 0; b < static_cast<int>(gridDim.x); ++b) v += a.obs_partial[b * kObsFields + threadIdx.x];
        a.status->obs[threadIdx.x] = v;
    }
}

template <int M, int NT>
struct Launcher {
    static int grid_size(int device) {
        static std::atomic<int> cached[64];  // per device (0 = not yet computed)
        if (device >= 0 && device < 64 && cached[device].load(std::memory_order_acquire))
            return cached[device].load(std::memory_order_acquire);
        const size_t smem = MarchGeom<M, NT>::bytes;
        cudaFuncSetAttribute(mb4_step_kernel<M, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mb4_step_kernel<M, NT>, NT, smem);
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        const int g = per_sm * sms;
        if (device >= 0 && device < 64) cached[device].store(g, std::memory_order_release);
        return g;
    }

    static cudaError_t launch(StepArgs a, const SweepConsts& c, int device, cudaStream_t s) {
        const int grid = grid_size(device);
        if (grid <= 0) return cudaErrorLaunchOutOfResources;
        a.nbands = (a.nx + MarchGeom<M, NT>::TX - 1) / MarchGeom<M, NT>::TX;
        a.total = static_cast<long long>(a.nbands) * a.ny;
        void* params[] = {&a, const_cast<SweepConsts*>(&c)};
        return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(mb4_step_kernel<M, NT>), dim3(grid),
                                           dim3(NT), params, MarchGeom<M, NT>::bytes, s);
    }
};

}  // namespace

// Host entry: one MB4 (sub)step's stage iteration on the device.
cudaError_t launch_step_march(int m, int nx, int ny, const double2* u0, const double* V,
                              double2* const U[2][3], unsigned long long* rmax,
                              double* obs_partial, void* status, int max_iters, double eps,
                              int want_obs, const SweepConsts& c, int device, cudaStream_t s) {
    StepArgs a{};
    a.nx = nx;
    a.ny = ny;
    a.u0 = u0;
    a.V = V;
    for (int b = 0; b < 2; ++b)
        for (int q = 0; q < 3; ++q) a.U[b][q] = U[b][q];
    a.rmax = rmax;
    a.obs_partial = obs_partial;
    a.status = static_cast<StepStatus*>(status);
    a.max_iters = max_iters;
    a.eps = eps;
    a.want_obs = want_obs;
    switch (m) {
        case 0: return Launcher<0, 128>::launch(a, c, device, s);
        case 1: return Launcher<1, 128>::launch(a, c, device, s);
        case 2: return Launcher<2, 128>::launch(a, c, device, s);
        case 3: return Launcher<3, 64>::launch(a, c, device, s);
    }
    return cudaErrorInvalidValue;
}

int march_grid_size(int m, int device) {
    switch (m) {
        case 0: return Launcher<0, 128>::grid_size(device);
        case 1: return Launcher<1, 128>::grid_size(device);
        case 2: return Launcher<2, 128>::grid_size(device);
        case 3: return Launcher<3, 64>::grid_size(device);
    }
    return 0;
}


}  // namespace mb4cu
