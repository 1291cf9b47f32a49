// Per-site FP64 math of the MB4 stage sweep, shared by every sweep kernel.
//
// Notation: z = (u0, U1, U2, U3) at a site,
//   c_i     = sum_j E[i][j] z_j                      (mb4_integrator.cpp:168-171)
//   U_q     = sum_a L[q][a] z_a   (q = 1..6, GL-6 nodes of the collocation polynomial)
//   Phi_i   = U_i - u0 - h [ -i (K+V) c_i + i gamma sum_q WA[i][q] |U_q|^2 U_q ]
// which equals the reference's W-tensor form (mb4_integrator.cpp:172-188)
// because W[i][a][b][c] = sum_q WA[i][q] L[q][a] L[q][b] L[q][c] exactly
// (degree-11 integrand, 6-point Gauss rule).
//   J t     = -i (K+V) t + i gamma (2|u0|^2 t + u0^2 conj(t))
// is the real-split Jacobian of mb4_integrator.hpp:52-55 in complex form.
#pragma once

#include <cuda_runtime.h>

#include "mb4cu_internal.hpp"

namespace mb4cu {

__device__ __forceinline__ int wrap_index(int x, int n) {
    x %= n;
    return x < 0 ? x + n : x;
}

// (K + V) x at a site from the centre value and its 4 neighbours.
__device__ __forceinline__ double2 kv_site(const SweepConsts& c, double v, double2 x, double2 xl,
                                           double2 xr, double2 xd, double2 xu) {
    double2 y;
    y.x = fma(c.diag + v, x.x, -(c.cx * (xl.x + xr.x) + c.cy * (xd.x + xu.x)));
    y.y = fma(c.diag + v, x.y, -(c.cx * (xl.y + xr.y) + c.cy * (xd.y + xu.y)));
    return y;
}

// Stage residuals Phi_i at one site from z (centre) and w_j = ((K+V) z_j)(site).
__device__ __forceinline__ void phi_site(const SweepConsts& c, const double2 z[4],
                                         const double2 w[4], double2 phi[3]) {
    double2 cub[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) cub[i] = make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        double ur = c.L[q][0] * z[0].x, ui = c.L[q][0] * z[0].y;
#pragma unroll
        for (int a = 1; a < 4; ++a) {
            ur = fma(c.L[q][a], z[a].x, ur);
            ui = fma(c.L[q][a], z[a].y, ui);
        }
        const double n2 = fma(ur, ur, ui * ui);
        const double gr = n2 * ur, gi = n2 * ui;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            cub[i].x = fma(c.WA[i][q], gr, cub[i].x);
            cub[i].y = fma(c.WA[i][q], gi, cub[i].y);
        }
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        double kr = c.E[i][0] * w[0].x, ki = c.E[i][0] * w[0].y;
#pragma unroll
        for (int j = 1; j < 4; ++j) {
            kr = fma(c.E[i][j], w[j].x, kr);
            ki = fma(c.E[i][j], w[j].y, ki);
        }
        // R = -i (K+V)c + i gamma cub
        const double rr = fma(-c.gamma, cub[i].y, ki);
        const double ri = fma(c.gamma, cub[i].x, -kr);
        phi[i].x = fma(-c.h, rr, z[i + 1].x - z[0].x);
        phi[i].y = fma(-c.h, ri, z[i + 1].y - z[0].y);
    }
}

// phibar = T^{-1} phi (per site, 3x3 real times complex)
__device__ __forceinline__ void to_eigen(const SweepConsts& c, const double2 phi[3], double2 out[3]) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        out[k].x = fma(c.Tinv[k][0], phi[0].x, fma(c.Tinv[k][1], phi[1].x, c.Tinv[k][2] * phi[2].x));
        out[k].y = fma(c.Tinv[k][0], phi[0].y, fma(c.Tinv[k][1], phi[1].y, c.Tinv[k][2] * phi[2].y));
    }
}

// r = T rbar
__device__ __forceinline__ void from_eigen(const SweepConsts& c, const double2 rb[3], double2 out[3]) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        out[i].x = fma(c.T[i][0], rb[0].x, fma(c.T[i][1], rb[1].x, c.T[i][2] * rb[2].x));
        out[i].y = fma(c.T[i][0], rb[0].y, fma(c.T[i][1], rb[1].y, c.T[i][2] * rb[2].y));
    }
}

// Diagonal (nonlinear) part of J at u0: alpha = 3p^2+q^2, beta = 2pq, delta = p^2+3q^2.
struct JDiag {
    double alpha, beta, delta;
};

__device__ __forceinline__ JDiag jdiag(double2 u0) {
    const double pp = u0.x * u0.x, qq = u0.y * u0.y;
    JDiag d;
    d.alpha = fma(3.0, pp, qq);
    d.beta = 2.0 * u0.x * u0.y;
    d.delta = fma(3.0, qq, pp);
    return d;
}

// J t at a site given a = ((K+V) t)(site).
__device__ __forceinline__ double2 j_site(const SweepConsts& c, const JDiag& d, double2 t,
                                          double2 a) {
    const double nlx = fma(d.alpha, t.x, d.beta * t.y);
    const double nly = fma(d.beta, t.x, d.delta * t.y);
    return make_double2(fma(-c.gamma, nly, a.y), fma(c.gamma, nlx, -a.x));
}

__device__ __forceinline__ unsigned long long abs_bits(double x) {
    return static_cast<unsigned long long>(__double_as_longlong(x)) & 0x7FFFFFFFFFFFFFFFull;
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}

// Block-wide max of a per-thread bit pattern, folded into *dst with atomicMax.
// NaN bit patterns (with the sign cleared) compare above +inf, so a non-finite
// update always surfaces as a non-finite residual.
__device__ __forceinline__ void block_max_to(unsigned long long v, unsigned long long* dst) {
    __shared__ unsigned long long red[32];
    v = warp_max_u64(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nthreads = blockDim.x * blockDim.y;
    const int tid = threadIdx.x + threadIdx.y * blockDim.x;
    (void)lane;
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    if (tid < 32) {
        v = tid < (nthreads + 31) / 32 ? red[tid] : 0ull;
        v = warp_max_u64(v);
        if (tid == 0 && v) atomicMax(dst, v);
    }
    (void)warp;
}

}  // namespace mb4cu
