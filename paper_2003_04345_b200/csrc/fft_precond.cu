// Fourier preconditioner for the matrix-free Krylov solves (stiff MB4 steps and
// the implicit comparison methods).
//
// The Newton matrices are  I - sigma J(u0)  (one stage, sigma = h lambda_k or
// h/2) or  I - h (C (x) J(u0))  (coupled 2-stage methods), with
//     J t = -i (K + V) t + i gamma (2|u0|^2 t + u0^2 conj(t)).
// Their stiff part is the periodic 5-point K, which the 2-D DFT diagonalises:
// K e_k = mu_k e_k with mu_k = 2cx (1 - cos(2 pi kx/nx)) + 2cy (1 - cos(2 pi ky/ny)).
// The preconditioner keeps K plus the mean of the C-linear diagonal,
//     s = mean(V) - 2 gamma mean(|u0|^2),
//     P = I + i sigma (K + s)            (one stage)
//     P = I + i h C (x) (K + s)          (two stages: a 2x2 system per mode),
// and applies P^-1 as FFT -> per-mode scaling -> inverse FFT (cuFFT).  Only the
// preconditioner is approximate (the defect, the delta potential and the
// conj(t) term stay in the operator), so the Krylov solution is unchanged; the
// iteration count drops from O(sqrt(sigma rho(K))) to a handful (the reference
// solves these systems by sparse LU instead, mb4_integrator.cpp:141-157).
#include <cuda_runtime.h>
#include <cufft.h>

#include "mb4cu_internal.hpp"

namespace mb4cu {
namespace {

constexpr int kT = 256;

__device__ __forceinline__ double mode_mu(int kx, int ky, int nx, int ny, double cx, double cy) {
    const double two_pi = 6.283185307179586476925286766559;
    return 2.0 * cx * (1.0 - cos(two_pi * kx / nx)) + 2.0 * cy * (1.0 - cos(two_pi * ky / ny));
}

// one stage: y_k *= 1 / ((1 + i sigma (mu_k + s)) N)
__global__ void __launch_bounds__(kT) scale1_kernel(double2* __restrict__ y, int nx, int ny, double cx, double cy,
                                                    double shift_arg, double sigma, const double* __restrict__ shift_dev) {
    const double shift = shift_dev ? *shift_dev : shift_arg;  // device copy: graph-invariant
    const size_t n = static_cast<size_t>(nx) * ny;
    const double inv_n = 1.0 / static_cast<double>(n);
    for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int ky = static_cast<int>(k / nx), kx = static_cast<int>(k - static_cast<size_t>(ky) * nx);
        const double b = sigma * (mode_mu(kx, ky, nx, ny, cx, cy) + shift);  // d = 1 + i b
        const double den = inv_n / fma(b, b, 1.0);
        const double2 v = y[k];
        // v / (1 + i b) = v (1 - i b) / (1 + b^2)
        y[k] = make_double2(fma(b, v.y, v.x) * den, fma(-b, v.x, v.y) * den);
    }
}

// two stages: [y0; y1] <- M^-1 [y0; y1] / N with M = I + i h (mu_k + s) C
__global__ void __launch_bounds__(kT) scale2_kernel(double2* __restrict__ y0, double2* __restrict__ y1, int nx,
                                                    int ny, double cx, double cy, double shift, double h,
                                                    double c00, double c01, double c10, double c11) {
    const size_t n = static_cast<size_t>(nx) * ny;
    const double inv_n = 1.0 / static_cast<double>(n);
    for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int ky = static_cast<int>(k / nx), kx = static_cast<int>(k - static_cast<size_t>(ky) * nx);
        const double t = h * (mode_mu(kx, ky, nx, ny, cx, cy) + shift);
        // M = [[1 + i t c00, i t c01], [i t c10, 1 + i t c11]] (complex entries)
        const double2 m00 = make_double2(1.0, t * c00), m01 = make_double2(0.0, t * c01);
        const double2 m10 = make_double2(0.0, t * c10), m11 = make_double2(1.0, t * c11);
        // det = m00 m11 - m01 m10
        const double2 det = make_double2(m00.x * m11.x - m00.y * m11.y - (m01.x * m10.x - m01.y * m10.y),
                                         m00.x * m11.y + m00.y * m11.x - (m01.x * m10.y + m01.y * m10.x));
        const double dd = inv_n / fma(det.x, det.x, det.y * det.y);
        const double2 idet = make_double2(det.x * dd, -det.y * dd);  // 1 / (det N)
        const double2 a = y0[k], b = y1[k];
        // M^-1 = adj(M) / det, adj = [[m11, -m01], [-m10, m00]]
        const double2 r0 = make_double2(m11.x * a.x - m11.y * a.y - (m01.x * b.x - m01.y * b.y),
                                        m11.x * a.y + m11.y * a.x - (m01.x * b.y + m01.y * b.x));
        const double2 r1 = make_double2(m00.x * b.x - m00.y * b.y - (m10.x * a.x - m10.y * a.y),
                                        m00.x * b.y + m00.y * b.x - (m10.x * a.y + m10.y * a.x));
        y0[k] = make_double2(r0.x * idet.x - r0.y * idet.y, r0.x * idet.y + r0.y * idet.x);
        y1[k] = make_double2(r1.x * idet.x - r1.y * idet.y, r1.x * idet.y + r1.y * idet.x);
    }
}

// s = mean(V) - 2 gamma mean(|u0|^2): block partial sums (fixed order)
__global__ void __launch_bounds__(kT) shift_partial_kernel(const double2* __restrict__ u0,
                                                           const double* __restrict__ V, size_t n,
                                                           double* __restrict__ partial) {
    double sv = 0.0, su = 0.0;
    for (size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const double2 z = u0[k];
        sv += V[k];
        su += fma(z.x, z.x, z.y * z.y);
    }
    __shared__ double red[2][kT / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sv += __shfl_xor_sync(0xffffffffu, sv, o);
        su += __shfl_xor_sync(0xffffffffu, su, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = sv;
        red[1][threadIdx.x >> 5] = su;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        double v = 0.0;
        for (int w = 0; w < kT / 32; ++w) v += red[threadIdx.x][w];
        partial[2 * blockIdx.x + threadIdx.x] = v;
    }
}

int pblocks(size_t n) {
    const size_t b = (n + kT - 1) / kT;
    return static_cast<int>(b < 148 * 8 ? (b ? b : 1) : 148 * 8);
}

}  // namespace

int fft_shift_blocks(size_t n) { return pblocks(n); }

cudaError_t launch_fft_shift_partials(const double2* u0, const double* V, size_t n, double* partial,
                                      cudaStream_t s) {
    shift_partial_kernel<<<pblocks(n), kT, 0, s>>>(u0, V, n, partial);
    return cudaGetLastError();
}

cudaError_t launch_fft_scale1(double2* y, int nx, int ny, double cx, double cy, double shift, double sigma,
                              cudaStream_t s, const double* shift_dev) {
    scale1_kernel<<<pblocks(static_cast<size_t>(nx) * ny), kT, 0, s>>>(y, nx, ny, cx, cy, shift, sigma, shift_dev);
    return cudaGetLastError();
}

cudaError_t launch_fft_scale2(double2* y0, double2* y1, int nx, int ny, double cx, double cy, double shift,
                              double h, const double C[2][2], cudaStream_t s) {
    scale2_kernel<<<pblocks(static_cast<size_t>(nx) * ny), kT, 0, s>>>(y0, y1, nx, ny, cx, cy, shift, h, C[0][0],
                                                                       C[0][1], C[1][0], C[1][1]);
    return cudaGetLastError();
}

}  // namespace mb4cu
