// Tiled reference sweep kernel + lattice operator kernels (energy monitor,
// (K+V)u, f(u), Phi).  The tiled sweep is the simple, obviously-correct form
// of one stage iteration; the production path is the persistent marching
// kernel in sweep_march.cu, which is checked against this one.
//
// One stage sweep with Neumann depth M:
//   Phi     = Phi(u0, U)                         (eval_phi, mb4_integrator.cpp:159-192)
//   phibar  = T^-1 Phi                           (:212-219)
//   b_0     = phibar,  b_n = phibar + h lam_k J b_{n-1}   (n = 1..M)
//   rbar    = -b_M    ~= -(I - h lam_k J)^{-1} phibar    (replaces the LU solves :221-229)
//   r = T rbar;  U += r;  ||r||_inf                (:231-250)
// Each level needs its input on a one-site-wider region, so a tile of TX x TY
// outputs stages z on a halo of M+1 sites.
#include <cuda_runtime.h>

#include <atomic>

#include "mb4cu_internal.hpp"
#include "site_math.cuh"

namespace mb4cu {
namespace {

constexpr int kTX = 16, kTY = 16;

template <int M>
struct TiledGeom {
    static constexpr int H = M + 1;
    static constexpr int PX = kTX + 2 * H;
    static constexpr int PY = kTY + 2 * H;
    static constexpr int NP = PX * PY;
    static constexpr int NPE = (NP + 1) & ~1;  // even count keeps double2 alignment
};

template <int M, bool FIRST>
__global__ void __launch_bounds__(kTX * kTY)
sweep_tiled_kernel(const SweepArgs a, const __grid_constant__ SweepConsts c) {
    using G = TiledGeom<M>;
    constexpr int NZ = FIRST ? 1 : 4;
    extern __shared__ double2 smem[];
    double2* zs = smem;                                   // [NZ][NP]
    double* vs = reinterpret_cast<double*>(zs + NZ * G::NP);  // [NPE]
    double2* lev = reinterpret_cast<double2*>(vs + G::NPE);   // [M][3][NP]

    const int tid = threadIdx.x;
    const int nthr = blockDim.x;
    const int gx0 = blockIdx.x * kTX - G::H;
    const int gy0 = blockIdx.y * kTY - G::H;

    for (int idx = tid; idx < G::NP; idx += nthr) {
        const int ly = idx / G::PX, lx = idx - ly * G::PX;
        const size_t g = static_cast<size_t>(wrap_index(gy0 + ly, a.ny)) * a.nx +
                         wrap_index(gx0 + lx, a.nx);
        zs[idx] = a.u0[g];
        if (!FIRST) {
#pragma unroll
            for (int j = 0; j < 3; ++j) zs[(j + 1) * G::NP + idx] = a.uin[j][g];
        }
        vs[idx] = a.V[g];
    }
    __syncthreads();

    auto zat = [&](int j, int idx) -> double2 { return FIRST ? zs[idx] : zs[j * G::NP + idx]; };

    unsigned long long rmax = 0ull;
    auto emit = [&](int lx, int ly, const double2 r[3]) {
        const int gx = gx0 + lx, gy = gy0 + ly;
        if (gx >= a.nx || gy >= a.ny) return;
        const size_t g = static_cast<size_t>(gy) * a.nx + gx;
        const int idx = ly * G::PX + lx;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const double2 u = zat(i + 1, idx);
            a.uout[i][g] = make_double2(u.x + r[i].x, u.y + r[i].y);
            const unsigned long long bx = abs_bits(r[i].x), by = abs_bits(r[i].y);
            rmax = bx > rmax ? bx : rmax;
            rmax = by > rmax ? by : rmax;
        }
    };

    // ---- level 0: Phi (and phibar) on the tile grown by M --------------------
    {
        constexpr int W = G::PX - 2, Hh = G::PY - 2;
        for (int it = tid; it < W * Hh; it += nthr) {
            const int ly = it / W + 1, lx = it % W + 1;
            const int idx = ly * G::PX + lx;
            if (M == 0 && (lx < G::H || lx >= G::H + kTX || ly < G::H || ly >= G::H + kTY)) continue;
            double2 z[4], w[4];
            const double v = vs[idx];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                z[j] = zat(j, idx);
                w[j] = kv_site(c, v, z[j], zat(j, idx - 1), zat(j, idx + 1), zat(j, idx - G::PX),
                               zat(j, idx + G::PX));
            }
            double2 phi[3];
            phi_site(c, z, w, phi);
            if (M == 0) {
                double2 r[3];
#pragma unroll
                for (int i = 0; i < 3; ++i) r[i] = make_double2(-phi[i].x, -phi[i].y);
                emit(lx, ly, r);
            } else {
                double2 pb[3];
                to_eigen(c, phi, pb);
#pragma unroll
                for (int k = 0; k < 3; ++k) lev[k * G::NP + idx] = pb[k];
            }
        }
    }
    // ---- levels 1..M: b_n = phibar + h lam J b_{n-1} --------------------------
#pragma unroll
    for (int n = 1; n <= M; ++n) {
        __syncthreads();
        const double2* prev = lev + (n - 1) * 3 * G::NP;
        double2* cur = lev + n * 3 * G::NP;
        const int lo = n + 1, W = G::PX - 2 * lo, Hh = G::PY - 2 * lo;
        for (int it = tid; it < W * Hh; it += nthr) {
            const int ly = it / W + lo, lx = it % W + lo;
            const int idx = ly * G::PX + lx;
            const double v = vs[idx];
            const JDiag d = jdiag(zs[idx]);
            double2 b[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double2* p = prev + k * G::NP;
                const double2 t = p[idx];
                const double2 ak = kv_site(c, v, t, p[idx - 1], p[idx + 1], p[idx - G::PX], p[idx + G::PX]);
                const double2 jt = j_site(c, d, t, ak);
                const double2 pb = lev[k * G::NP + idx];
                b[k] = make_double2(fma(c.hlam[k], jt.x, pb.x), fma(c.hlam[k], jt.y, pb.y));
            }
            if (n == M) {
                double2 rb[3], r[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) rb[k] = make_double2(-b[k].x, -b[k].y);
                from_eigen(c, rb, r);
                emit(lx, ly, r);
            } else {
#pragma unroll
                for (int k = 0; k < 3; ++k) cur[k * G::NP + idx] = b[k];
            }
        }
    }
    block_max_to(rmax, a.rmax);
}

template <int M, bool FIRST>
size_t tiled_smem() {
    using G = TiledGeom<M>;
    const int nz = FIRST ? 1 : 4;
    const int nlev = M == 0 ? 0 : M;  // lev[0..M-1] (level M goes to global)
    return sizeof(double2) * nz * G::NP + sizeof(double) * G::NPE + sizeof(double2) * 3 * G::NP * nlev;
}

template <int M, bool FIRST>
cudaError_t launch_tiled(const SweepArgs& a, const SweepConsts& c, cudaStream_t s) {
    const size_t smem = tiled_smem<M, FIRST>();
    static std::atomic<bool> configured[64];  // per instantiation and device
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !configured[dev].load(std::memory_order_acquire)) {
        cudaError_t e = cudaFuncSetAttribute(sweep_tiled_kernel<M, FIRST>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        if (dev >= 0 && dev < 64) configured[dev].store(true, std::memory_order_release);
    }
    const dim3 grid((a.nx + kTX - 1) / kTX, (a.ny + kTY - 1) / kTY);
    sweep_tiled_kernel<M, FIRST><<<grid, kTX * kTY, smem, s>>>(a, c);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Energy monitor: observables (lattice.cpp:106-137), deterministic reduction.
// ---------------------------------------------------------------------------
constexpr int kObsThreads = 256;

__global__ void __launch_bounds__(kObsThreads) observables_partial_kernel(const ObsArgs a) {
    double acc[kObsFields] = {0.0, 0.0, 0.0, 0.0, 0.0};
    double car[kObsFields] = {0.0, 0.0, 0.0, 0.0, 0.0};  // compensation (two_sum_add)
    // Tiles of kObsThreads columns x a band of rows; each thread marches down its
    // column with the vertical neighbours in registers (one HBM read of u per site;
    // left/right come from the same row, L1-resident), periodic wrap by
    // compare-and-select.  Fixed work split -> bit-reproducible sums.
    const int ntx = (a.nx + kObsThreads - 1) / kObsThreads;
    const int nby = gridDim.x / ntx;
    const int tx = blockIdx.x % ntx, by = blockIdx.x / ntx;
    const int i = tx * kObsThreads + threadIdx.x;
    if (by < nby && i < a.nx) {
        const int y0 = static_cast<int>(static_cast<long long>(a.ny) * by / nby);
        const int y1 = static_cast<int>(static_cast<long long>(a.ny) * (by + 1) / nby);
        const int il = i == 0 ? a.nx - 1 : i - 1, ir = i == a.nx - 1 ? 0 : i + 1;
        auto at = [&](int j) { return a.u + static_cast<size_t>(j) * a.nx; };
        double2 dn = at(y0 == 0 ? a.ny - 1 : y0 - 1)[i];
        double2 u = at(y0)[i];
        // rows in groups of kObsRows: all their loads issued before the arithmetic (the
        // march is latency-bound with one row's loads in flight per thread)
        constexpr int kObsRows = 4;
        for (int j0 = y0; j0 < y1; j0 += kObsRows) {
            double2 up[kObsRows], l[kObsRows], r[kObsRows];
            double v[kObsRows];
#pragma unroll
            for (int k = 0; k < kObsRows; ++k) {
                const int j = j0 + k;
                if (j < y1) {
                    const double2* row = at(j);
                    up[k] = __ldcs(at(j == a.ny - 1 ? 0 : j + 1) + i);
                    l[k] = row[il];
                    r[k] = row[ir];
                    v[k] = __ldcs(a.V + static_cast<size_t>(j) * a.nx + i);
                }
            }
#pragma unroll
            for (int k = 0; k < kObsRows; ++k) {
                if (j0 + k >= y1) break;
                const double kx = fma(a.diag, u.x, -(a.cx * (l[k].x + r[k].x) + a.cy * (dn.x + up[k].x)));
                const double ky = fma(a.diag, u.y, -(a.cx * (l[k].y + r[k].y) + a.cy * (dn.y + up[k].y)));
                two_sum_add(acc[0], car[0], fma(u.x, kx, u.y * ky));  // Re conj(u) Ku
                acc[1] += fma(u.x, ky, -u.y * kx);                    // Im conj(u) Ku (health check)
                const double n2 = fma(u.x, u.x, u.y * u.y);
                two_sum_add(acc[2], car[2], n2);
                two_sum_add(acc[3], car[3], n2 * n2);
                two_sum_add(acc[4], car[4], v[k] * n2);
                dn = u;
                u = up[k];
            }
        }
    }
    block_csum_store<kObsThreads, kObsFields>(acc, car, a.partial + blockIdx.x * kObsFields);
}

// Fixed-order final sum of the block partials (bit-reproducible).
__global__ void observables_finalize_kernel(const double* partial, int nblocks, double* out) {
    __shared__ double red[kObsFields][256][2];
    double acc[kObsFields] = {0.0, 0.0, 0.0, 0.0, 0.0};
    double car[kObsFields] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x)
#pragma unroll
        for (int f = 0; f < kObsFields; ++f) two_sum_add(acc[f], car[f], partial[b * kObsFields + f]);
#pragma unroll
    for (int f = 0; f < kObsFields; ++f) {
        red[f][threadIdx.x][0] = acc[f];
        red[f][threadIdx.x][1] = car[f];
    }
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s)
#pragma unroll
            for (int f = 0; f < kObsFields; ++f)
                two_sum_merge(red[f][threadIdx.x][0], red[f][threadIdx.x][1], red[f][threadIdx.x + s][0],
                              red[f][threadIdx.x + s][1]);
        __syncthreads();
    }
    if (threadIdx.x < kObsFields) out[threadIdx.x] = red[threadIdx.x][0][0] + red[threadIdx.x][0][1];
}

__global__ void apply_kv_kernel(int nx, int ny, double cx, double cy, const double2* __restrict__ u,
                                const double* __restrict__ V, double gamma, bool rhs,
                                double2* __restrict__ y) {
    const size_t n = static_cast<size_t>(nx) * ny;
    for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(k / nx), i = static_cast<int>(k - static_cast<size_t>(j) * nx);
        const double2 c = u[k];
        const double2 l = u[static_cast<size_t>(j) * nx + wrap_index(i - 1, nx)];
        const double2 r = u[static_cast<size_t>(j) * nx + wrap_index(i + 1, nx)];
        const double2 d = u[static_cast<size_t>(wrap_index(j - 1, ny)) * nx + i];
        const double2 up = u[static_cast<size_t>(wrap_index(j + 1, ny)) * nx + i];
        const double dg = 2.0 * cx + 2.0 * cy;
        double ax = fma(dg, c.x, -(cx * (l.x + r.x) + cy * (d.x + up.x))) + V[k] * c.x;
        double ay = fma(dg, c.y, -(cx * (l.y + r.y) + cy * (d.y + up.y))) + V[k] * c.y;
        if (rhs) {
            const double n2 = fma(c.x, c.x, c.y * c.y);
            ax = fma(-gamma * n2, c.x, ax);
            ay = fma(-gamma * n2, c.y, ay);
            y[k] = make_double2(ay, -ax);  // -i (ax + i ay)
        } else {
            y[k] = make_double2(ax, ay);
        }
    }
}

struct PhiArgs {
    int nx, ny;
    const double2* u0;
    const double* V;
    const double2* st[3];
    double2* phi[3];
};

__global__ void eval_phi_kernel(const PhiArgs a, const __grid_constant__ SweepConsts c) {
    const size_t n = static_cast<size_t>(a.nx) * a.ny;
    for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(k / a.nx), i = static_cast<int>(k - static_cast<size_t>(j) * a.nx);
        const size_t kl = static_cast<size_t>(j) * a.nx + wrap_index(i - 1, a.nx);
        const size_t kr = static_cast<size_t>(j) * a.nx + wrap_index(i + 1, a.nx);
        const size_t kd = static_cast<size_t>(wrap_index(j - 1, a.ny)) * a.nx + i;
        const size_t ku = static_cast<size_t>(wrap_index(j + 1, a.ny)) * a.nx + i;
        const double2* zp[4] = {a.u0, a.st[0], a.st[1], a.st[2]};
        double2 z[4], w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            z[q] = zp[q][k];
            w[q] = kv_site(c, a.V[k], z[q], zp[q][kl], zp[q][kr], zp[q][kd], zp[q][ku]);
        }
        double2 phi[3];
        phi_site(c, z, w, phi);
#pragma unroll
        for (int q = 0; q < 3; ++q) a.phi[q][k] = phi[q];
    }
}

int grid_for(size_t n, int threads) {
    const size_t b = (n + threads - 1) / threads;
    return static_cast<int>(b < 148 * 16 ? (b ? b : 1) : 148 * 16);
}

// max |u|^2 over n sites as the bit pattern of a non-negative double (atomicMax)
// max |u|^2 over the nx x ny owned sites of a (possibly ghost-padded) array
__global__ void amax2_kernel(const double2* __restrict__ u, int nx, size_t n, int pitch,
                             unsigned long long* out) {
    double m = 0.0;
    for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t row = k / static_cast<size_t>(nx), col = k - row * nx;
        const double2 z = __ldcs(u + row * pitch + col);
        m = fmax(m, fma(z.x, z.x, z.y * z.y));
    }
    block_max_to(static_cast<unsigned long long>(__double_as_longlong(m)), out);
}

}  // namespace

size_t tiled_smem_bytes(int m, bool first) {
    switch (m * 2 + (first ? 1 : 0)) {
        case 0: return tiled_smem<0, false>();
        case 1: return tiled_smem<0, true>();
        case 2: return tiled_smem<1, false>();
        case 3: return tiled_smem<1, true>();
        case 4: return tiled_smem<2, false>();
        case 5: return tiled_smem<2, true>();
        case 6: return tiled_smem<3, false>();
        case 7: return tiled_smem<3, true>();
    }
    return 0;
}

cudaError_t launch_sweep_tiled(int m, bool first, const SweepArgs& a, const SweepConsts& c,
                               cudaStream_t s) {
    switch (m * 2 + (first ? 1 : 0)) {
        case 0: return launch_tiled<0, false>(a, c, s);
        case 1: return launch_tiled<0, true>(a, c, s);
        case 2: return launch_tiled<1, false>(a, c, s);
        case 3: return launch_tiled<1, true>(a, c, s);
        case 4: return launch_tiled<2, false>(a, c, s);
        case 5: return launch_tiled<2, true>(a, c, s);
        case 6: return launch_tiled<3, false>(a, c, s);
        case 7: return launch_tiled<3, true>(a, c, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_amax2_2d(const double2* u, int nx, int ny, int pitch, unsigned long long* out, cudaStream_t s) {
    const size_t n = static_cast<size_t>(nx) * ny;
    amax2_kernel<<<grid_for(n, 256), 256, 0, s>>>(u, nx, n, pitch, out);
    return cudaGetLastError();
}

cudaError_t launch_amax2(const double2* u, size_t n, unsigned long long* out, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(*out), s);
    if (e != cudaSuccess) return e;
    amax2_kernel<<<grid_for(n, 256), 256, 0, s>>>(u, static_cast<int>(n), n, static_cast<int>(n), out);
    return cudaGetLastError();
}

int obs_blocks(int nx, int ny) {
    // column tiles x row bands, ~8 blocks per SM, bands of >= 8 rows
    const int ntx = (nx + kObsThreads - 1) / kObsThreads;
    int nby = (148 * 8 + ntx - 1) / ntx;
    if (nby > (ny + 7) / 8) nby = (ny + 7) / 8;
    if (nby < 1) nby = 1;
    return ntx * nby;
}

cudaError_t launch_observables(const ObsArgs& a, double* out5, cudaStream_t s) {
    const int nb = obs_blocks(a.nx, a.ny);
    observables_partial_kernel<<<nb, kObsThreads, 0, s>>>(a);
    observables_finalize_kernel<<<1, 256, 0, s>>>(a.partial, nb, out5);
    return cudaGetLastError();
}

cudaError_t launch_apply_kv(int nx, int ny, double cx, double cy, const double2* u, const double* V,
                            double gamma, bool rhs, double2* y, cudaStream_t s) {
    const size_t n = static_cast<size_t>(nx) * ny;
    apply_kv_kernel<<<grid_for(n, 256), 256, 0, s>>>(nx, ny, cx, cy, u, V, gamma, rhs, y);
    return cudaGetLastError();
}

cudaError_t launch_eval_phi(int nx, int ny, const double2* u0, const double* V,
                            const double2* const st[3], double2* const phi[3],
                            const SweepConsts& c, cudaStream_t s) {
    PhiArgs a;
    a.nx = nx;
    a.ny = ny;
    a.u0 = u0;
    a.V = V;
    for (int q = 0; q < 3; ++q) {
        a.st[q] = st[q];
        a.phi[q] = phi[q];
    }
    const size_t n = static_cast<size_t>(nx) * ny;
    eval_phi_kernel<<<grid_for(n, 128), 128, 0, s>>>(a, c);
    return cudaGetLastError();
}

}  // namespace mb4cu
