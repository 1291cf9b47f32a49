// The reference's other integrators on the GPU, for the
// harness's method comparison / convergence studies: RK4, GAUSS2 (implicit
// midpoint), GAUSS4 (2-stage Gauss), AVF2 and AVF4 (integrators.cpp:45-395).
//
// The implicit methods keep the reference's simplified Newton iteration (the
// Jacobian frozen at u0, ||delta||_inf <= eps over the split reals, the same
// residual forms and final assembly); the linear systems
//     one stage:  (I - h/2 J(u0)) x = b                  (stage_matrix(j, h/2))
//     two stages: (I - h (C (x) J(u0))) x = b, C 2x2    (coupled_matrix2)
// are solved matrix-free by the context's GMRES (mb4cu_api.cu) with the
// matvec kernels below instead of the reference's sparse LU.  Every kernel is
// a site-parallel grid-stride loop; these methods are comparison baselines, not
// the hot path.
#include <cuda_runtime.h>

#include "mb4cu_internal.hpp"
#include "site_math.cuh"

namespace mb4cu {
namespace {

constexpr int kT = 256;

#define MGRID_LOOP(k, n) \
    for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < (n); k += static_cast<size_t>(gridDim.x) * blockDim.x)

struct Nb {
    size_t l, r, d, u;
};

// Every site of the lattice: rows round-robin over the blocks, columns over the
// threads (coalesced); periodic neighbours by compare-and-select, no division.
template <class F>
__device__ __forceinline__ void for_sites(int nx, int ny, const F& f) {
    for (int j = blockIdx.x; j < ny; j += gridDim.x) {
        const size_t row = static_cast<size_t>(j) * nx;
        const size_t dn = static_cast<size_t>(j == 0 ? ny - 1 : j - 1) * nx;
        const size_t up = static_cast<size_t>(j == ny - 1 ? 0 : j + 1) * nx;
        for (int i = threadIdx.x; i < nx; i += blockDim.x) {
            Nb q;
            q.l = row + (i == 0 ? nx - 1 : i - 1);
            q.r = row + (i == nx - 1 ? 0 : i + 1);
            q.d = dn + i;
            q.u = up + i;
            f(row + i, q);
        }
    }
}

__device__ __forceinline__ Nb nbrs(size_t k, int nx, int ny) {
    const int j = static_cast<int>(k / nx), i = static_cast<int>(k - static_cast<size_t>(j) * nx);
    Nb n;
    n.l = static_cast<size_t>(j) * nx + wrap_index(i - 1, nx);
    n.r = static_cast<size_t>(j) * nx + wrap_index(i + 1, nx);
    n.d = static_cast<size_t>(wrap_index(j - 1, ny)) * nx + i;
    n.u = static_cast<size_t>(wrap_index(j + 1, ny)) * nx + i;
    return n;
}

// (K + V) x at a site from the centre and its 4 neighbours, the reference's
// apply_kv (lattice.cpp:86-89) in the same form as the sweep kernels
__device__ __forceinline__ double2 kv5(const MethodConsts& c, double v, double2 xc, double2 xl, double2 xr,
                                       double2 xd, double2 xu) {
    double2 y;
    y.x = fma(c.diag + v, xc.x, -(c.cx * (xl.x + xr.x) + c.cy * (xd.x + xu.x)));
    y.y = fma(c.diag + v, xc.y, -(c.cx * (xl.y + xr.y) + c.cy * (xd.y + xu.y)));
    return y;
}

__device__ __forceinline__ double2 kv_at(const MethodConsts& c, const double2* x, const double* V, size_t k,
                                         const Nb& q) {
    return kv5(c, V[k], x[k], x[q.l], x[q.r], x[q.d], x[q.u]);
}

// f(u) = -i ((K+V) u - gamma |u|^2 u) from a = ((K+V) u)(site) (lattice.cpp:91-104)
__device__ __forceinline__ double2 f_from(const MethodConsts& c, double2 u, double2 a) {
    const double n2 = fma(u.x, u.x, u.y * u.y);
    const double ax = fma(-c.gamma * n2, u.x, a.x);
    const double ay = fma(-c.gamma * n2, u.y, a.y);
    return make_double2(ay, -ax);
}

__device__ __forceinline__ double2 f_at(const MethodConsts& c, const double2* x, const double* V, size_t k,
                                        const Nb& q) {
    return f_from(c, x[k], kv_at(c, x, V, k, q));
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

// -i a + i g b  (the reference's  mi * kv + Complex(0, g) * cubic)
__device__ __forceinline__ double2 vec_field(double2 kv, double g, double2 cub) {
    return make_double2(kv.y - g * cub.y, -kv.x + g * cub.x);
}

// ---- RK4 (integrators.cpp:45-59) -------------------------------------------
// stage 1: k = f(u0); acc = k;        out = u0 + (h/2) k
// stage 2: k = f(x);  acc += 2 k;     out = u0 + (h/2) k
// stage 3: k = f(x);  acc += 2 k;     out = u0 + h k
// stage 4: k = f(x);  out = u0 + (h/6) (acc + k)
__global__ void __launch_bounds__(kT) rk4_stage_kernel(int stage, int nx, int ny, const double2* __restrict__ x,
                                                       const double2* __restrict__ u0, const double* __restrict__ V,
                                                       double2* __restrict__ acc, double2* __restrict__ out,
                                                       const MethodConsts c) {
    const size_t n = static_cast<size_t>(nx) * ny;
    for_sites(nx, ny, [&](size_t k, const Nb& q) {
        const double2 kk = f_at(c, x, V, k, q);
        const double2 u = u0[k];
        if (stage == 1) {
            acc[k] = kk;
            out[k] = cadd(u, cscale(0.5 * c.h, kk));
        } else if (stage < 4) {
            acc[k] = cadd(acc[k], cscale(2.0, kk));
            out[k] = cadd(u, cscale(stage == 2 ? 0.5 * c.h : c.h, kk));
        } else {
            out[k] = cadd(u, cscale(c.h / 6.0, cadd(acc[k], kk)));
        }
        });
}

// ---- residuals b = -G of the implicit methods -------------------------------
// unk holds s contiguous stage fields of n sites.
__global__ void __launch_bounds__(kT) residual_kernel(int method, int nx, int ny, const double2* __restrict__ u0,
                                                      const double* __restrict__ V, const double2* __restrict__ unk,
                                                      double2* __restrict__ b, const MethodConsts c) {
    const size_t n = static_cast<size_t>(nx) * ny;
    for_sites(nx, ny, [&](size_t k, const Nb& q) {
        const double2 z0 = u0[k];
        if (method == kMethodGauss2) {
            // g = u - u0 - (h/2) f(u)   (integrators.cpp:126-128)
            const double2 f = f_at(c, unk, V, k, q);
            const double2 g = csub(csub(unk[k], z0), cscale(0.5 * c.h, f));
            b[k] = make_double2(-g.x, -g.y);
        } else if (method == kMethodGauss4) {
            // g_i = u_i - u0 - h (a_i0 f_0 + a_i1 f_1)   (:178-183)
            const double2 f0 = f_at(c, unk, V, k, q);
            const double2 f1 = f_at(c, unk + n, V, k, q);
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const double2 comb = cadd(cscale(c.a[i][0], f0), cscale(c.a[i][1], f1));
                const double2 g = csub(csub(unk[i * n + k], z0), cscale(c.h, comb));
                b[i * n + k] = make_double2(-g.x, -g.y);
            }
        } else if (method == kMethodAvf2) {
            // mid = (u0 + u1)/2; g = u1 - u0 - h (-i (K+V) mid + i g cubic)   (:239-250)
            const double2* u1 = unk;
            auto mid = [&](size_t s) { return cscale(0.5, cadd(u0[s], u1[s])); };
            const double2 kv = kv5(c, V[k], mid(k), mid(q.l), mid(q.r), mid(q.d), mid(q.u));
            const double2 z[2] = {z0, u1[k]};
            double2 cub = make_double2(0.0, 0.0);
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int bb = 0; bb < 2; ++bb)
#pragma unroll
                    for (int cc = 0; cc < 2; ++cc)
                        cub = cadd(cub, cscale(c.b2[a][bb][cc], cmul(cmul(cconj(z[a]), z[bb]), z[cc])));
            const double2 g = csub(csub(u1[k], z0), cscale(c.h, vec_field(kv, c.gamma, cub)));
            b[k] = make_double2(-g.x, -g.y);
        } else {  // kMethodAvf4
            // combo_i = u0 + mt_i0 z_0 + mt_i1 z_1; g_i = z_i - h (-i (K+V) combo_i + i g cubic_i)   (:352-366)
            const double2* zz0 = unk;
            const double2* zz1 = unk + n;
            const double2 z[3] = {z0, zz0[k], zz1[k]};
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                auto combo = [&](size_t s) {
                    return cadd(cadd(u0[s], cscale(c.a[i][0], zz0[s])), cscale(c.a[i][1], zz1[s]));
                };
                const double2 kv = kv5(c, V[k], combo(k), combo(q.l), combo(q.r), combo(q.d), combo(q.u));
                double2 cub = make_double2(0.0, 0.0);
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int bb = 0; bb < 3; ++bb)
#pragma unroll
                        for (int cc = 0; cc < 3; ++cc)
                            cub = cadd(cub, cscale(c.wt[i][a][bb][cc], cmul(cmul(cconj(z[a]), z[bb]), z[cc])));
                const double2 g = csub(z[1 + i], cscale(c.h, vec_field(kv, c.gamma, cub)));
                b[i * n + k] = make_double2(-g.x, -g.y);
            }
        }
        });
}

// ---- Newton matrix applied matrix-free -------------------------------------
// y_i = x_i - h sum_j C[i][j] J(u0) x_j   (s = 1: C = 1/2)
__global__ void __launch_bounds__(kT) newton_matvec_kernel(int s, int nx, int ny, const double2* __restrict__ x,
                                                           double2* __restrict__ y, const double2* __restrict__ u0,
                                                           const double* __restrict__ V, const MethodConsts c) {
    const size_t n = static_cast<size_t>(nx) * ny;
    for_sites(nx, ny, [&](size_t k, const Nb& q) {
        const double2 z = u0[k];
        const double pp = z.x * z.x, qq = z.y * z.y;
        const double al = fma(3.0, pp, qq), be = 2.0 * z.x * z.y, de = fma(3.0, qq, pp);
        double2 jx[2];
        for (int j = 0; j < s; ++j) {
            const double2* xj = x + j * n;
            const double2 t = xj[k];
            const double2 a = kv_at(c, xj, V, k, q);
            const double nlx = fma(al, t.x, be * t.y);
            const double nly = fma(be, t.x, de * t.y);
            jx[j] = make_double2(fma(-c.gamma, nly, a.y), fma(c.gamma, nlx, -a.x));
        }
        for (int i = 0; i < s; ++i) {
            double2 acc = make_double2(0.0, 0.0);
            for (int j = 0; j < s; ++j) acc = cadd(acc, cscale(c.a[i][j], jx[j]));
            const double2 xi = x[i * n + k];
            y[i * n + k] = make_double2(fma(-c.h, acc.x, xi.x), fma(-c.h, acc.y, xi.y));
        }
        });
}

// unk += x over len complex entries; ||x||_inf over the split reals (bit pattern)
__global__ void __launch_bounds__(kT) newton_add_kernel(double2* __restrict__ unk, const double2* __restrict__ x,
                                                        size_t len, unsigned long long* rmax) {
    unsigned long long m = 0ull;
    MGRID_LOOP(k, len) {
        const double2 d = x[k];
        const double2 u = unk[k];
        unk[k] = make_double2(u.x + d.x, u.y + d.y);
        const unsigned long long bx = abs_bits(d.x), by = abs_bits(d.y);
        m = bx > m ? bx : m;
        m = by > m ? by : m;
    }
    block_max_to(m, rmax);
}

// initial stage increments of AVF4: z_i = h f(u0)   (:342-347)
__global__ void __launch_bounds__(kT) avf4_init_kernel(int nx, int ny, const double2* __restrict__ u0,
                                                       const double* __restrict__ V, double2* __restrict__ unk,
                                                       const MethodConsts c) {
    const size_t n = static_cast<size_t>(nx) * ny;
    for_sites(nx, ny, [&](size_t k, const Nb& q) {
        const double2 z = cscale(c.h, f_at(c, u0, V, k, q));
        unk[k] = z;
        unk[n + k] = z;
        });
}

// final assembly: GAUSS2 u0 + h f(u); GAUSS4 u0 + h (b0 f(u_1) + b1 f(u_2));
// AVF4 u0 + z_0/2 + z_1/2; AVF2 u1 itself
__global__ void __launch_bounds__(kT) final_kernel(int method, int nx, int ny, const double2* __restrict__ u0,
                                                   const double* __restrict__ V, const double2* __restrict__ unk,
                                                   double2* __restrict__ out, const MethodConsts c) {
    const size_t n = static_cast<size_t>(nx) * ny;
    for_sites(nx, ny, [&](size_t k, const Nb& q) {
        const double2 z = u0[k];
        if (method == kMethodGauss2) {
            out[k] = cadd(z, cscale(c.h, f_at(c, unk, V, k, q)));
        } else if (method == kMethodGauss4) {
            const double2 f0 = f_at(c, unk, V, k, q), f1 = f_at(c, unk + n, V, k, q);
            out[k] = cadd(z, cscale(c.h, cadd(cscale(0.5, f0), cscale(0.5, f1))));
        } else if (method == kMethodAvf4) {
            out[k] = cadd(cadd(z, cscale(0.5, unk[k])), cscale(0.5, unk[n + k]));
        } else {
            out[k] = unk[k];
        }
        });
}

int rblocks(int ny) { return ny < 148 * 8 ? ny : 148 * 8; }

int mblocks(size_t n) {
    const size_t b = (n + kT - 1) / kT;
    return static_cast<int>(b < 148 * 16 ? (b ? b : 1) : 148 * 16);
}

}  // namespace

cudaError_t launch_rk4_stage(int stage, int nx, int ny, const double2* x, const double2* u0, const double* V,
                             double2* acc, double2* out, const MethodConsts& c, cudaStream_t s) {
    const size_t n = static_cast<size_t>(nx) * ny;
    rk4_stage_kernel<<<rblocks(ny), kT, 0, s>>>(stage, nx, ny, x, u0, V, acc, out, c);
    return cudaGetLastError();
}

cudaError_t launch_method_residual(int method, int nx, int ny, const double2* u0, const double* V,
                                   const double2* unk, double2* b, const MethodConsts& c, cudaStream_t s) {
    const size_t n = static_cast<size_t>(nx) * ny;
    residual_kernel<<<rblocks(ny), kT, 0, s>>>(method, nx, ny, u0, V, unk, b, c);
    return cudaGetLastError();
}

cudaError_t launch_method_matvec(int stages, int nx, int ny, const double2* x, double2* y, const double2* u0,
                                 const double* V, const MethodConsts& c, cudaStream_t s) {
    const size_t n = static_cast<size_t>(nx) * ny;
    newton_matvec_kernel<<<rblocks(ny), kT, 0, s>>>(stages, nx, ny, x, y, u0, V, c);
    return cudaGetLastError();
}

cudaError_t launch_newton_add(double2* unk, const double2* x, size_t len, unsigned long long* rmax,
                              cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(rmax, 0, sizeof(*rmax), s);
    if (e != cudaSuccess) return e;
    newton_add_kernel<<<mblocks(len), kT, 0, s>>>(unk, x, len, rmax);
    return cudaGetLastError();
}

cudaError_t launch_avf4_init(int nx, int ny, const double2* u0, const double* V, double2* unk,
                             const MethodConsts& c, cudaStream_t s) {
    const size_t n = static_cast<size_t>(nx) * ny;
    avf4_init_kernel<<<rblocks(ny), kT, 0, s>>>(nx, ny, u0, V, unk, c);
    return cudaGetLastError();
}

cudaError_t launch_method_final(int method, int nx, int ny, const double2* u0, const double* V,
                                const double2* unk, double2* out, const MethodConsts& c, cudaStream_t s) {
    const size_t n = static_cast<size_t>(nx) * ny;
    final_kernel<<<rblocks(ny), kT, 0, s>>>(method, nx, ny, u0, V, unk, out, c);
    return cudaGetLastError();
}

}  // namespace mb4cu
