// Production stage-sweep kernel, v2: persistent cooperative launch per MB4 step,
// marching column bands with register windows.
//
// Same algorithm as sweep_march.cu (Phi -> T^-1 -> M-term Neumann
// (I - h lam_k J)^-1 -> T -> update -> ||r||_inf; see site_math.cuh) and the
// same band / work split, but reorganised around the measured bottleneck of
// v1 (shared-memory wavefronts and FP64 latency, profiles/):
//  - Each thread keeps the VERTICAL neighbours of its own column in registers:
//    a 3-row window of z = (u0, U1..U3), and 3-row windows of the Neumann
//    level values (phibar, b1) and of the Jacobian diagonal.  Shared memory
//    carries only the HORIZONTAL neighbours: z rows arrive by cp.async into a
//    row ring; every level publishes its freshly computed row into a
//    double-buffered row that the neighbours read one iteration later.
//  - Level n works on row i - n at iteration i (level n-1 produced row i-n+1
//    this iteration, in registers; the horizontal neighbours of row i-n were
//    published last iteration), so one __syncthreads per row suffices.
//  - The iteration loop is unrolled by 3 so every window slot is static.
//  - The first sweep of a step (U = (u0,u0,u0)) uses the closed form
//    Phi_i = -h c_i f(u0), c_i = sum_j E[i][j].
// HBM traffic per sweep is unchanged: 120 B/site (72 B/site for the first).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "async_copy.cuh"
#include "mb4cu_internal.hpp"
#include "site_math.cuh"

namespace cg = cooperative_groups;

namespace mb4cu {
namespace {

template <int M, int NT>
struct Geom2 {
    static_assert(M >= 0 && M <= 2, "march v2 supports Neumann depth 0..2");
    static constexpr int TX = NT - 2 * M;  // output columns per band
    static constexpr int ZW = NT + 2;      // columns per smem row (1-site pad each side)
    static constexpr int P = 4;            // cp.async prefetch depth (rows)
    static constexpr int S = P + 2;        // z ring rows (6: divisible by the unroll of 3)
    static constexpr size_t zu0_bytes = sizeof(double2) * S * ZW;
    static constexpr size_t zv_bytes = ((sizeof(double) * S * ZW + 15) / 16) * 16;
    static constexpr size_t zU_bytes = sizeof(double2) * S * 3 * ZW;
    static constexpr size_t pub_bytes = sizeof(double2) * 2 * 3 * ZW;  // one level, 2 parities
    static constexpr int NPUB = M;                                      // levels 0..M-1 publish
    static constexpr size_t bytes = zu0_bytes + zv_bytes + zU_bytes + NPUB * pub_bytes;
};

struct JD {  // Jacobian diagonal at a site plus (diag + V)
    double alpha, beta, delta, dv;
};

template <int M, int NT, bool FIRST>
struct March2 {
    using G = Geom2<M, NT>;
    double2* zu0;  // [S][ZW]
    double* zv;    // [S][ZW]
    double2* zU;   // [S][3][ZW]
    double2* pub;  // [NPUB][2][3][ZW]

    // register windows, slot = (level-0 row + 2) mod 3 == (iteration j) mod 3
    double2 zw[3][4];   // own-column z rows (slot of z row k: k mod 3)
    double vw[3];       // own-column V
    double2 pbw[3][3];  // phibar of level-0 rows
    JD jdw[3];
    double2 b1w[3][3];  // level-1 values (M == 2)

    __device__ March2(unsigned char* smem) {
        zu0 = reinterpret_cast<double2*>(smem);
        zv = reinterpret_cast<double*>(smem + G::zu0_bytes);
        zU = reinterpret_cast<double2*>(smem + G::zu0_bytes + G::zv_bytes);
        pub = reinterpret_cast<double2*>(smem + G::zu0_bytes + G::zv_bytes + G::zU_bytes);
    }

    __device__ __forceinline__ double2* pub_row(int level, int parity, int k) {
        return pub + ((level * 2 + parity) * 3 + k) * G::ZW;
    }

    struct Seg {
        int X0, Y0, R;
        int xz0, yz0, nzrows;
    };

    __device__ __forceinline__ void issue_row(const StepArgs& a, const double2* const uin[3],
                                              const Seg& s, int k) {
        if (k < s.nzrows) {
            const size_t rowoff = static_cast<size_t>(wrap_index(s.yz0 + k, a.ny)) * a.nx;
            const int slot = k % G::S;
            for (int col = threadIdx.x; col < G::ZW; col += NT) {
                const size_t g = rowoff + wrap_index(s.xz0 + col, a.nx);
                cp_async16(&zu0[slot * G::ZW + col], a.u0 + g);
                cp_async8(&zv[slot * G::ZW + col], a.V + g);
                if (!FIRST) {
#pragma unroll
                    for (int q = 0; q < 3; ++q) cp_async16(&zU[(slot * 3 + q) * G::ZW + col], uin[q] + g);
                }
            }
        }
        cp_async_commit();
    }

    // One iteration j (level-0 row i = j - 2).  PH = j mod 3 (static); zs = j mod S.
    template <int PH>
    __device__ __forceinline__ void body(const StepArgs& a, const SweepConsts& c,
                                         const double2* const uin[3], double2* const uout[3],
                                         const Seg& s, int j, unsigned long long& rmax,
                                         double acc[kObsFields]) {
        constexpr int S_NEW = PH;            // z row j      (own column, newly loaded)
        constexpr int S_CEN = (PH + 2) % 3;  // z row j - 1  (level-0 centre row)
        constexpr int S_DN = (PH + 1) % 3;   // z row j - 2
        const int t = threadIdx.x;
        const int cc = t + 1;
        const int i = j - 2;                 // level-0 row (relative to Y0 - M)

        cp_async_wait<G::P - 1>();
        __syncthreads();
        issue_row(a, uin, s, j + G::P);

        const int slot_new = j % G::S;
        const int slot_cen = (j + G::S - 1) % G::S;

        // final-level output coordinates (row i - M at level M)
        const int yrel = i - 2 * M;          // output row offset from Y0
        const int xout = s.X0 - M + t;
        const bool out_ok = yrel >= 0 && yrel < s.R && t >= M && t < NT - M && xout < a.nx;
        double2 uold[3];
        if (M == 2 && out_ok) {
            const size_t g = static_cast<size_t>(s.Y0 + yrel) * a.nx + xout;
            if (FIRST) {
                uold[0] = __ldcg(a.u0 + g);
            } else {
#pragma unroll
                for (int q = 0; q < 3; ++q) uold[q] = __ldcg(uin[q] + g);
            }
        }

        // ---- own column: new z row j into the window -------------------------
        zw[S_NEW][0] = zu0[slot_new * G::ZW + cc];
        vw[S_NEW] = zv[slot_new * G::ZW + cc];
        if (!FIRST) {
#pragma unroll
            for (int q = 0; q < 3; ++q) zw[S_NEW][q + 1] = zU[(slot_new * 3 + q) * G::ZW + cc];
        }

        // ---- level 0 at row i: phibar (centre z row j-1) ------------------------
        const double v = vw[S_CEN];
        const double2 u0c = zw[S_CEN][0];
        double2 pb[3];
        {
            const double2 l0 = zu0[slot_cen * G::ZW + cc - 1], r0 = zu0[slot_cen * G::ZW + cc + 1];
            const double2 w0 = kv_site(c, v, u0c, l0, r0, zw[S_DN][0], zw[S_NEW][0]);
            if (FIRST) {
                // f(u0) = -i((K+V)u0 - gamma |u0|^2 u0); phibar_k = first_s[k] * f
                const double n2 = fma(u0c.x, u0c.x, u0c.y * u0c.y);
                const double gx = fma(-c.gamma * n2, u0c.x, w0.x);
                const double gy = fma(-c.gamma * n2, u0c.y, w0.y);
                const double2 f = make_double2(gy, -gx);
#pragma unroll
                for (int k = 0; k < 3; ++k) pb[k] = make_double2(c.first_s[k] * f.x, c.first_s[k] * f.y);
                if (M == 0) {
                    // Picard: U_i = u0 + h c_i f(u0)
                    if (out_ok) {
                        const size_t g = static_cast<size_t>(s.Y0 + yrel) * a.nx + xout;
#pragma unroll
                        for (int q = 0; q < 3; ++q) {
                            const double2 r = make_double2(c.first_c[q] * f.x, c.first_c[q] * f.y);
                            uout[q][g] = make_double2(u0c.x + r.x, u0c.y + r.y);
                            const unsigned long long bx = abs_bits(r.x), by = abs_bits(r.y);
                            rmax = bx > rmax ? bx : rmax;
                            rmax = by > rmax ? by : rmax;
                        }
                    }
                }
                // energy monitor of u0 on owned sites (lattice.cpp:106-137)
                if (i >= M && i < M + s.R && t >= M && t < NT - M && xout < a.nx) {
                    const double vn = v * n2;
                    acc[0] += fma(u0c.x, w0.x, u0c.y * w0.y) - vn;
                    acc[1] += fma(u0c.x, w0.y, -u0c.y * w0.x);
                    acc[2] += n2;
                    acc[3] += n2 * n2;
                    acc[4] += vn;
                }
            } else {
                double2 z[4], w[4];
                z[0] = u0c;
                w[0] = w0;
#pragma unroll
                for (int q = 1; q < 4; ++q) {
                    const double2* row = zU + (slot_cen * 3 + (q - 1)) * G::ZW;
                    z[q] = zw[S_CEN][q];
                    w[q] = kv_site(c, v, z[q], row[cc - 1], row[cc + 1], zw[S_DN][q], zw[S_NEW][q]);
                }
                double2 phi[3];
                phi_site(c, z, w, phi);
                if (M == 0) {
                    if (out_ok) {
                        const size_t g = static_cast<size_t>(s.Y0 + yrel) * a.nx + xout;
#pragma unroll
                        for (int q = 0; q < 3; ++q) {
                            uout[q][g] = make_double2(z[q + 1].x - phi[q].x, z[q + 1].y - phi[q].y);
                            const unsigned long long bx = abs_bits(phi[q].x), by = abs_bits(phi[q].y);
                            rmax = bx > rmax ? bx : rmax;
                            rmax = by > rmax ? by : rmax;
                        }
                    }
                } else {
                    to_eigen(c, phi, pb);
                }
            }
        }
        if (M == 0) return;

        constexpr int R0 = PH;             // slot of level-0 row i   (== S_NEW)
        constexpr int R1 = (PH + 2) % 3;   // row i - 1
        constexpr int R2 = (PH + 1) % 3;   // row i - 2
        const int par = j & 1;             // publish parity of this iteration
        const int ppar = par ^ 1;          // parity published last iteration
        {
            const JD d = {fma(3.0, u0c.x * u0c.x, u0c.y * u0c.y), 2.0 * u0c.x * u0c.y,
                          fma(3.0, u0c.y * u0c.y, u0c.x * u0c.x), c.diag + v};
            jdw[R0] = d;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                pbw[R0][k] = pb[k];
                pub_row(0, par, k)[cc] = pb[k];
            }
        }

        // ---- level 1 at row i - 1 -------------------------------------------
        double2 b1[3];
        {
            const JD d = jdw[R1];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double2* hrow = pub_row(0, ppar, k);
                const double2 tc = pbw[R1][k];
                const double2 tl = hrow[cc - 1], tr = hrow[cc + 1];
                const double2 td = pbw[R2][k], tu = pbw[R0][k];
                double2 ak;
                ak.x = fma(d.dv, tc.x, -(c.cx * (tl.x + tr.x) + c.cy * (td.x + tu.x)));
                ak.y = fma(d.dv, tc.y, -(c.cx * (tl.y + tr.y) + c.cy * (td.y + tu.y)));
                const double nlx = fma(d.alpha, tc.x, d.beta * tc.y);
                const double nly = fma(d.beta, tc.x, d.delta * tc.y);
                const double jx = fma(-c.gamma, nly, ak.y);
                const double jy = fma(c.gamma, nlx, -ak.x);
                b1[k] = make_double2(fma(c.hlam[k], jx, tc.x), fma(c.hlam[k], jy, tc.y));
            }
        }
        if (M == 1) {
            if (out_ok) {
                double2 rb[3], r[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) rb[k] = make_double2(-b1[k].x, -b1[k].y);
                from_eigen(c, rb, r);
                const size_t g = static_cast<size_t>(s.Y0 + yrel) * a.nx + xout;
                // U_old of row i - 1 is z row j - 2 (window slot S_DN)
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const double2 uo = FIRST ? zw[S_DN][0] : zw[S_DN][q + 1];
                    uout[q][g] = make_double2(uo.x + r[q].x, uo.y + r[q].y);
                    const unsigned long long bx = abs_bits(r[q].x), by = abs_bits(r[q].y);
                    rmax = bx > rmax ? bx : rmax;
                    rmax = by > rmax ? by : rmax;
                }
            }
            return;
        }
        // M == 2: publish b1 (row i - 1), keep it in the window
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            b1w[R1][k] = b1[k];
            pub_row(1, par, k)[cc] = b1[k];
        }

        // ---- level 2 at row i - 2 (final) ------------------------------------
        if (out_ok) {
            const JD d = jdw[R2];
            double2 b2[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double2* hrow = pub_row(1, ppar, k);
                // b1 rows: i-3 (slot R0, written 2 iterations ago), i-2 (R2), i-1 (R1)
                const double2 tc = b1w[R2][k];
                const double2 tl = hrow[cc - 1], tr = hrow[cc + 1];
                const double2 td = b1w[R0][k], tu = b1w[R1][k];
                double2 ak;
                ak.x = fma(d.dv, tc.x, -(c.cx * (tl.x + tr.x) + c.cy * (td.x + tu.x)));
                ak.y = fma(d.dv, tc.y, -(c.cx * (tl.y + tr.y) + c.cy * (td.y + tu.y)));
                const double nlx = fma(d.alpha, tc.x, d.beta * tc.y);
                const double nly = fma(d.beta, tc.x, d.delta * tc.y);
                const double jx = fma(-c.gamma, nly, ak.y);
                const double jy = fma(c.gamma, nlx, -ak.x);
                const double2 p0 = pbw[R2][k];
                b2[k] = make_double2(fma(c.hlam[k], jx, p0.x), fma(c.hlam[k], jy, p0.y));
            }
            double2 rb[3], r[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) rb[k] = make_double2(-b2[k].x, -b2[k].y);
            from_eigen(c, rb, r);
            const size_t g = static_cast<size_t>(s.Y0 + yrel) * a.nx + xout;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const double2 uo = FIRST ? uold[0] : uold[q];
                uout[q][g] = make_double2(uo.x + r[q].x, uo.y + r[q].y);
                const unsigned long long bx = abs_bits(r[q].x), by = abs_bits(r[q].y);
                rmax = bx > rmax ? bx : rmax;
                rmax = by > rmax ? by : rmax;
            }
        }
    }

    __device__ void run(const StepArgs& a, const SweepConsts& c, const double2* const uin[3],
                        double2* const uout[3], int band, int Y0, int R, unsigned long long& rmax,
                        double acc[kObsFields]) {
        Seg s;
        s.X0 = band * G::TX;
        s.Y0 = Y0;
        s.R = R;
        s.xz0 = s.X0 - M - 1;
        s.yz0 = Y0 - M - 1;
        s.nzrows = R + 2 * M + 2;
#pragma unroll
        for (int k = 0; k < G::P; ++k) issue_row(a, uin, s, k);
        // iterations j = 0 .. R + 2M + 1 (j = 0, 1 only fill the windows)
        const int jend = R + 2 * M + 2;
        for (int j = 0; j < jend; j += 3) {
            body<0>(a, c, uin, uout, s, j, rmax, acc);
            body<1>(a, c, uin, uout, s, j + 1, rmax, acc);
            body<2>(a, c, uin, uout, s, j + 2, rmax, acc);
        }
        cp_async_wait<0>();
        __syncthreads();
    }
};

template <int M, int NT, bool FIRST>
__device__ void sweep_all2(const StepArgs& a, const SweepConsts& c, unsigned char* smem,
                           const double2* const uin[3], double2* const uout[3],
                           unsigned long long& rmax, double acc[kObsFields]) {
    March2<M, NT, FIRST> m(smem);
    const long long G = gridDim.x;
    const long long b0 = a.total * blockIdx.x / G;
    const long long b1 = a.total * (blockIdx.x + 1) / G;
    long long pos = b0;
    while (pos < b1) {
        const int band = static_cast<int>(pos / a.ny);
        const int row = static_cast<int>(pos - static_cast<long long>(band) * a.ny);
        const long long band_end = static_cast<long long>(band + 1) * a.ny;
        const long long seg_end = band_end < b1 ? band_end : b1;
        m.run(a, c, uin, uout, band, row, static_cast<int>(seg_end - pos), rmax, acc);
        pos = seg_end;
    }
}

template <int M, int NT>
__global__ void __launch_bounds__(NT, 2)
mb4_step2_kernel(const StepArgs a, const __grid_constant__ SweepConsts c) {
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
            sweep_all2<M, NT, true>(a, c, smem, uin, uout, rmax, acc);
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
            sweep_all2<M, NT, false>(a, c, smem, uin, uout, rmax, acc);
        }
        block_max_to(rmax, &a.rmax[s]);
        grid.sync();
        const unsigned long long bits = __ldcg(&a.rmax[s]);
        rlast = __longlong_as_double(static_cast<long long>(bits));
        sweeps = s + 1;
        set = out;
        if (!isfinite(rlast)) break;
        if (rlast <= a.eps) {
            converged = 1;
            break;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.status->sweeps = sweeps;
        a.status->set = set;
        a.status->converged = converged;
        a.status->rlast = rlast;
    }
    if (a.want_obs && blockIdx.x == 0 && threadIdx.x < kObsFields) {
        double v = 0.0;
        for (int b = 0; b < static_cast<int>(gridDim.x); ++b) v += a.obs_partial[b * kObsFields + threadIdx.x];
        a.status->obs[threadIdx.x] = v;
    }
}

template <int M, int NT>
struct Launcher2 {
    static int grid_size(int device) {
        static int cached[64] = {0};
        if (device >= 0 && device < 64 && cached[device]) return cached[device];
        const size_t smem = Geom2<M, NT>::bytes;
        cudaFuncSetAttribute(mb4_step2_kernel<M, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mb4_step2_kernel<M, NT>, NT, smem);
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        const int g = per_sm * sms;
        if (device >= 0 && device < 64) cached[device] = g;
        return g;
    }

    static cudaError_t launch(StepArgs a, const SweepConsts& c, int device, cudaStream_t s) {
        const int grid = grid_size(device);
        if (grid <= 0) return cudaErrorLaunchOutOfResources;
        a.nbands = (a.nx + Geom2<M, NT>::TX - 1) / Geom2<M, NT>::TX;
        a.total = static_cast<long long>(a.nbands) * a.ny;
        void* params[] = {&a, const_cast<SweepConsts*>(&c)};
        return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(mb4_step2_kernel<M, NT>), dim3(grid),
                                           dim3(NT), params, Geom2<M, NT>::bytes, s);
    }
};

}  // namespace

cudaError_t launch_step_march2(int m, int nx, int ny, const double2* u0, const double* V,
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
        case 0: return Launcher2<0, 128>::launch(a, c, device, s);
        case 1: return Launcher2<1, 128>::launch(a, c, device, s);
        case 2: return Launcher2<2, 128>::launch(a, c, device, s);
    }
    return cudaErrorInvalidValue;
}

int march2_grid_size(int m, int device) {
    switch (m) {
        case 0: return Launcher2<0, 128>::grid_size(device);
        case 1: return Launcher2<1, 128>::grid_size(device);
        case 2: return Launcher2<2, 128>::grid_size(device);
    }
    return 0;
}

}  // namespace mb4cu
