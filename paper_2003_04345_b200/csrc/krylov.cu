// Stiff-regime stage solver (kernel = 3): the reference's simplified Newton
// iteration with matrix-free GMRES stage solves on the GPU.
//
// When h * max|lambda| * rho(J) >~ 1 (the paper's lx = 2 pi setups) the Neumann
// preconditioned sweep of the production kernel cannot converge; this path
// follows the reference algorithm instead (newton_solve, mb4_integrator.cpp:
// 194-255, with the GMRES route of LinearSystem :19-34 / iterative.cpp:68-153,
// here unpreconditioned and matrix-free):
//   b_k = -(T^-1 Phi)_k;  (I - h lam_k J(u0)) x_k = b_k  (GMRES(m), real inner
//   product over the split reals);  r = T x;  U += r;  stop on ||r||_inf.
// Device kernels do every O(N) operation (Phi, J x, the Gram-Schmidt dots and
// AXPYs, norms); the host keeps the (m+1) x m Hessenberg bookkeeping.  Dot
// products are block partials summed on the host in a fixed order, so runs are
// bit-reproducible.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>

#include "mb4cu_internal.hpp"
#include "site_math.cuh"

namespace mb4cu {
namespace {

constexpr int kT = 256;

struct Nbr {
    size_t c, l, r, d, u;
};

// Every site: rows round-robin over the blocks, columns over the threads; periodic
// neighbours by compare-and-select (no integer division in the loop).
template <class F>
__device__ __forceinline__ void for_sites(int nx, int ny, const F& f) {
    for (int j = blockIdx.x; j < ny; j += gridDim.x) {
        const size_t row = static_cast<size_t>(j) * nx;
        const size_t dn = static_cast<size_t>(j == 0 ? ny - 1 : j - 1) * nx;
        const size_t up = static_cast<size_t>(j == ny - 1 ? 0 : j + 1) * nx;
        for (int i = threadIdx.x; i < nx; i += blockDim.x) {
            Nbr q;
            q.c = row + i;
            q.l = row + (i == 0 ? nx - 1 : i - 1);
            q.r = row + (i == nx - 1 ? 0 : i + 1);
            q.d = dn + i;
            q.u = up + i;
            f(q.c, q);
        }
    }
}

int row_blocks(int ny) { return ny < 148 * 8 ? ny : 148 * 8; }

__device__ __forceinline__ Nbr neighbours(size_t k, int nx, int ny) {
    const int j = static_cast<int>(k / nx), i = static_cast<int>(k - static_cast<size_t>(j) * nx);
    Nbr n;
    n.c = k;
    n.l = static_cast<size_t>(j) * nx + wrap_index(i - 1, nx);
    n.r = static_cast<size_t>(j) * nx + wrap_index(i + 1, nx);
    n.d = static_cast<size_t>(wrap_index(j - 1, ny)) * nx + i;
    n.u = static_cast<size_t>(wrap_index(j + 1, ny)) * nx + i;
    return n;
}

#define GRID_LOOP(k, n) \
    for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < (n); k += static_cast<size_t>(gridDim.x) * blockDim.x)

struct PhiIn {
    const double2* u0;
    const double2* st[3];
    const double* V;
    double2* b[3];
    int nx, ny;
};

// b_k = -(T^-1 Phi)_k at every site
__global__ void __launch_bounds__(kT) phibar_kernel(const PhiIn p, const __grid_constant__ SweepConsts c) {
    for_sites(p.nx, p.ny, [&](size_t k, const Nbr& q) {
        const double2* zp[4] = {p.u0, p.st[0], p.st[1], p.st[2]};
        double2 z[4], w[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            z[a] = zp[a][q.c];
            w[a] = kv_site(c, p.V[k], z[a], zp[a][q.l], zp[a][q.r], zp[a][q.d], zp[a][q.u]);
        }
        double2 phi[3], pb[3];
        phi_site(c, z, w, phi);
        to_eigen(c, phi, pb);
#pragma unroll
        for (int s = 0; s < 3; ++s) p.b[s][k] = make_double2(-pb[s].x, -pb[s].y);
    });
}

// y = x - hl * J(u0) x
__global__ void __launch_bounds__(kT) stage_matvec_kernel(const double2* __restrict__ x, double2* __restrict__ y,
                                                          const double2* __restrict__ u0, const double* __restrict__ V,
                                                          int nx, int ny, double hl,
                                                          const __grid_constant__ SweepConsts c) {
    for_sites(nx, ny, [&](size_t k, const Nbr& q) {
        const double2 t = x[q.c];
        const double2 a = kv_site(c, V[k], t, x[q.l], x[q.r], x[q.d], x[q.u]);
        const JDiag d = jdiag(u0[k]);
        const double2 jt = j_site(c, d, t, a);
        y[k] = make_double2(fma(-hl, jt.x, t.x), fma(-hl, jt.y, t.y));
    });
}

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double red[kT / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < kT / 32; ++w) s += red[w];
    __syncthreads();
    return s;
}

struct Basis {
    double2* const* v;  // device array of basis vector pointers
};

// partial[i * gridDim.x + blockIdx.x] = sum over this block's sites of <w, v_i>, i <= j
__global__ void __launch_bounds__(kT) dots_kernel(const double2* __restrict__ w, double2* const* __restrict__ v,
                                                  int nv, size_t n, double* __restrict__ partial) {
    const int i = blockIdx.y;
    if (i >= nv) return;
    const double2* vi = v[i];
    double acc = 0.0;
    GRID_LOOP(k, n) {
        const double2 a = w[k], b = vi[k];
        acc = fma(a.x, b.x, fma(a.y, b.y, acc));
    }
    const double s = block_sum(acc);
    if (threadIdx.x == 0) partial[static_cast<size_t>(i) * gridDim.x + blockIdx.x] = s;
}

// w -= sum_i h_i v_i ; partial[blockIdx.x] = sum |w|^2 (after the update)
__global__ void __launch_bounds__(kT) axpy_norm_kernel(double2* __restrict__ w, double2* const* __restrict__ v,
                                                       const double* __restrict__ h, int nv, size_t n,
                                                       double* __restrict__ partial) {
    double acc = 0.0;
    GRID_LOOP(k, n) {
        double2 a = w[k];
        for (int i = 0; i < nv; ++i) {
            const double2 b = v[i][k];
            a.x = fma(-h[i], b.x, a.x);
            a.y = fma(-h[i], b.y, a.y);
        }
        w[k] = a;
        acc = fma(a.x, a.x, fma(a.y, a.y, acc));
    }
    const double s = block_sum(acc);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// y = alpha * x (+ norm partials)
__global__ void __launch_bounds__(kT) scale_kernel(const double2* __restrict__ x, double2* __restrict__ y, double alpha,
                                                   size_t n) {
    GRID_LOOP(k, n) {
        const double2 a = x[k];
        y[k] = make_double2(alpha * a.x, alpha * a.y);
    }
}

// x += sum_i coef_i v_i
__global__ void __launch_bounds__(kT) combine_kernel(double2* __restrict__ x, double2* const* __restrict__ v,
                                                     const double* __restrict__ coef, int nv, size_t n) {
    GRID_LOOP(k, n) {
        double2 a = x[k];
        for (int i = 0; i < nv; ++i) {
            const double2 b = v[i][k];
            a.x = fma(coef[i], b.x, a.x);
            a.y = fma(coef[i], b.y, a.y);
        }
        x[k] = a;
    }
}

// r = b - y (in place into r) ; partial = |r|^2
__global__ void __launch_bounds__(kT) residual_kernel(const double2* __restrict__ b, const double2* __restrict__ y,
                                                      double2* __restrict__ r, size_t n, double* __restrict__ partial) {
    double acc = 0.0;
    GRID_LOOP(k, n) {
        const double2 a = make_double2(b[k].x - y[k].x, b[k].y - y[k].y);
        r[k] = a;
        acc = fma(a.x, a.x, fma(a.y, a.y, acc));
    }
    const double s = block_sum(acc);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

struct UpdIn {
    double2* st[3];
    const double2* x[3];
};

// r = T x ; U += r ; block max of the split-real |r| (bit patterns)
__global__ void __launch_bounds__(kT) newton_update_kernel(const UpdIn p, size_t n, unsigned long long* rmax,
                                                           const __grid_constant__ SweepConsts c) {
    unsigned long long m = 0ull;
    GRID_LOOP(k, n) {
        double2 xb[3], r[3];
#pragma unroll
        for (int s = 0; s < 3; ++s) xb[s] = p.x[s][k];
        from_eigen(c, xb, r);
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            const double2 u = p.st[s][k];
            p.st[s][k] = make_double2(u.x + r[s].x, u.y + r[s].y);
            const unsigned long long bx = abs_bits(r[s].x), by = abs_bits(r[s].y);
            m = bx > m ? bx : m;
            m = by > m ? by : m;
        }
    }
    block_max_to(m, rmax);
}

int blocks(size_t n) {
    const size_t b = (n + kT - 1) / kT;
    return static_cast<int>(b < 148 * 4 ? (b ? b : 1) : 148 * 4);
}

constexpr int kMaxDots = 32;  // >= the GMRES restart length + 1 (mb4cu_api.cu kKrylovRestart = 30)

// One Arnoldi step after w = A v_j, in ONE cooperative launch (grid barriers
// instead of host round trips): classical Gram-Schmidt twice against v_0..v_j,
// hcol[i] = h_ij (both passes), hcol[j+1] = ||w||, v_{j+1} = w / ||w||.  Dot
// products are block partials summed by block 0 in a fixed order (bit-
// reproducible; the same grid as the other Krylov kernels).
#ifndef MB4_DOT_CHUNK
#define MB4_DOT_CHUNK 8  // 32: all dots in one sweep (118 registers, 2 CTAs per SM; round 1)
#endif
constexpr int kDotChunk = MB4_DOT_CHUNK;

__global__ void __launch_bounds__(kT, MB4_DOT_CHUNK >= 32 ? 1 : 4) arnoldi_kernel(double2* __restrict__ w, double2* const* __restrict__ v, int j_arg,
                                                     size_t n, double* __restrict__ partial,
                                                     double* __restrict__ hbuf, double* __restrict__ hcol,
                                                     int* __restrict__ jdev) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const int G = gridDim.x;
    // jdev != nullptr: the step index lives in device memory and advances here, so one
    // captured graph serves every step of a cycle (kr_gmres_stages)
    const int j = jdev ? *jdev : j_arg;
    for (int pass = 0; pass < 2; ++pass) {
        if (j < kMaxDots) {
            // all j + 1 dot products in one sweep over the sites and ONE block reduction (the
            // per-dot block reductions dominate on small lattices); per-thread, warp and
            // block sums in the same order as the one-dot-at-a-time loop below: bit-identical
            // in chunks of kDotChunk dots (kDotChunk accumulators live: 4 CTAs per SM, so the
            // three stage solves' cooperative launches fit the device together on large
            // lattices); w is re-read once per chunk
            __shared__ double red[kT / 32][kMaxDots];
            for (int c0 = 0; c0 <= j; c0 += kDotChunk) {
                double acc[kDotChunk];
#pragma unroll
                for (int i = 0; i < kDotChunk; ++i) acc[i] = 0.0;
                GRID_LOOP(k, n) {
                    const double2 a = w[k];
#pragma unroll
                    for (int i = 0; i < kDotChunk; ++i)
                        if (c0 + i <= j) {
                            const double2 b = v[c0 + i][k];
                            acc[i] = fma(a.x, b.x, fma(a.y, b.y, acc[i]));
                        }
                }
#pragma unroll
                for (int i = 0; i < kDotChunk; ++i)
                    if (c0 + i <= j) {
                        double t = acc[i];
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
                        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][c0 + i] = t;
                    }
            }
            __syncthreads();
            for (int i = threadIdx.x; i <= j; i += blockDim.x) {
                double t = 0.0;
                for (int q = 0; q < kT / 32; ++q) t += red[q][i];
                partial[static_cast<size_t>(i) * G + blockIdx.x] = t;
            }
        } else {
            for (int i = 0; i <= j; ++i) {
                const double2* vi = v[i];
                double acc = 0.0;
                GRID_LOOP(k, n) {
                    const double2 a = w[k], b = vi[k];
                    acc = fma(a.x, b.x, fma(a.y, b.y, acc));
                }
                const double sblk = block_sum(acc);
                if (threadIdx.x == 0) partial[static_cast<size_t>(i) * G + blockIdx.x] = sblk;
            }
        }
        grid.sync();
        if (blockIdx.x == 0) {
            for (int i = threadIdx.x; i <= j; i += blockDim.x) {
                double t = 0.0;
                for (int b = 0; b < G; ++b) t += partial[static_cast<size_t>(i) * G + b];
                hbuf[i] = t;
                hcol[i] = pass == 0 ? t : hcol[i] + t;
            }
        }
        grid.sync();
        double acc = 0.0;
        GRID_LOOP(k, n) {  // the same sites per thread in every loop: no barrier needed before the next dots
            double2 a = w[k];
            for (int i = 0; i <= j; ++i) {
                const double2 b = v[i][k];
                a.x = fma(-hbuf[i], b.x, a.x);
                a.y = fma(-hbuf[i], b.y, a.y);
            }
            w[k] = a;
            acc = fma(a.x, a.x, fma(a.y, a.y, acc));
        }
        if (pass == 1) {
            const double sblk = block_sum(acc);
            if (threadIdx.x == 0) partial[blockIdx.x] = sblk;
        }
    }
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        double t = 0.0;
        for (int b = 0; b < G; ++b) t += partial[b];
        const double hn = sqrt(t);
        hcol[j + 1] = hn;
        hbuf[0] = hn > 0.0 ? 1.0 / hn : 0.0;
    }
    grid.sync();
    const double inv = hbuf[0];
    double2* vn = v[j + 1];
    if (inv > 0.0) {
        GRID_LOOP(k, n) {
            const double2 a = w[k];
            vn[k] = make_double2(inv * a.x, inv * a.y);
        }
    }
    if (jdev && blockIdx.x == 0 && threadIdx.x == 0) *jdev = j + 1;  // every block read *jdev before the syncs
}

// y = v[*jdev] (the basis vector of the current Arnoldi step, index in device memory)
__global__ void gather_basis_kernel(double2* __restrict__ y, double2* const* __restrict__ v, const int* __restrict__ jdev,
                                    size_t n) {
    const double2* src = v[*jdev];
    GRID_LOOP(k, n) y[k] = src[k];
}

}  // namespace

// co-resident Arnoldi blocks on the current device (the three batched stage solves'
// concurrent cooperative launches must fit together)
int arnoldi_capacity() {
    static std::atomic<int> cap[64];  // co-resident blocks per device (0 = unknown)
    int dev = 0;
    cudaGetDevice(&dev);
    int c = dev >= 0 && dev < 64 ? cap[dev].load(std::memory_order_acquire) : 0;
    if (!c) {
        int per_sm = 0, sms = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, arnoldi_kernel, kT, 0);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        c = per_sm * sms;
        if (dev >= 0 && dev < 64) cap[dev].store(c, std::memory_order_release);
    }
    return c;
}

// Grid of one Arnoldi launch: at most 2 blocks per SM even where 4 fit -- block 0 sums
// the per-block partials of every dot in sequence, which a wider grid only lengthens
// (measured: 400^2 Newton-Krylov step 16.4 ms at 296 blocks, 19.2 ms at 592)
int arnoldi_grid(size_t n) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int c = std::min(arnoldi_capacity(), 2 * sms);
    const int b = blocks(n);
    return b < c ? b : c;
}

cudaError_t kr_arnoldi(double2* w, double2* const* v_dev, int j, size_t n, double* partial, double* hbuf,
                       double* hcol, cudaStream_t s, int* jdev) {
    const int g = arnoldi_grid(n);
    void* args[] = {&w, const_cast<double2***>(&v_dev), &j, &n, &partial, &hbuf, &hcol, &jdev};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(arnoldi_kernel), dim3(g), dim3(kT), args, 0, s);
}

cudaError_t kr_gather_basis(double2* y, double2* const* v_dev, const int* jdev, size_t n, cudaStream_t s) {
    gather_basis_kernel<<<blocks(n), kT, 0, s>>>(y, v_dev, jdev, n);
    return cudaGetLastError();
}

int krylov_blocks(size_t n) { return blocks(n); }

cudaError_t kr_phibar(int nx, int ny, const double2* u0, const double2* const st[3], const double* V,
                      double2* const b[3], const SweepConsts& c, cudaStream_t s) {
    PhiIn p;
    p.u0 = u0;
    p.V = V;
    p.nx = nx;
    p.ny = ny;
    for (int i = 0; i < 3; ++i) {
        p.st[i] = st[i];
        p.b[i] = b[i];
    }
    phibar_kernel<<<row_blocks(ny), kT, 0, s>>>(p, c);
    return cudaGetLastError();
}

cudaError_t kr_matvec(const double2* x, double2* y, const double2* u0, const double* V, int nx, int ny, double hl,
                      const SweepConsts& c, cudaStream_t s) {
    stage_matvec_kernel<<<row_blocks(ny), kT, 0, s>>>(x, y, u0, V, nx, ny, hl, c);
    return cudaGetLastError();
}

cudaError_t kr_dots(const double2* w, double2* const* v_dev, int nv, size_t n, double* partial, cudaStream_t s) {
    dots_kernel<<<dim3(blocks(n), nv), kT, 0, s>>>(w, v_dev, nv, n, partial);
    return cudaGetLastError();
}

cudaError_t kr_axpy_norm(double2* w, double2* const* v_dev, const double* h_dev, int nv, size_t n, double* partial,
                         cudaStream_t s) {
    axpy_norm_kernel<<<blocks(n), kT, 0, s>>>(w, v_dev, h_dev, nv, n, partial);
    return cudaGetLastError();
}

cudaError_t kr_scale(const double2* x, double2* y, double alpha, size_t n, cudaStream_t s) {
    scale_kernel<<<blocks(n), kT, 0, s>>>(x, y, alpha, n);
    return cudaGetLastError();
}

cudaError_t kr_combine(double2* x, double2* const* v_dev, const double* coef_dev, int nv, size_t n, cudaStream_t s) {
    combine_kernel<<<blocks(n), kT, 0, s>>>(x, v_dev, coef_dev, nv, n);
    return cudaGetLastError();
}

cudaError_t kr_residual(const double2* b, const double2* y, double2* r, size_t n, double* partial, cudaStream_t s) {
    residual_kernel<<<blocks(n), kT, 0, s>>>(b, y, r, n, partial);
    return cudaGetLastError();
}

cudaError_t kr_update(double2* const st[3], const double2* const x[3], size_t n, unsigned long long* rmax,
                      const SweepConsts& c, cudaStream_t s) {
    UpdIn p;
    for (int i = 0; i < 3; ++i) {
        p.st[i] = st[i];
        p.x[i] = x[i];
    }
    newton_update_kernel<<<blocks(n), kT, 0, s>>>(p, n, rmax, c);
    return cudaGetLastError();
}

}  // namespace mb4cu
