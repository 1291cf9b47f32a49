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

// Compensated summation (Knuth TwoSum, branch-free): s + c carries the running sum with
// the rounding error of every addition kept in c, so the energy monitor's relative error
// does not grow with the number of sites a thread, block or grid adds up.
__device__ __forceinline__ void two_sum_add(double& s, double& c, double x) {
    const double t = s + x;
    const double z = t - s;
    c += (s - (t - z)) + (x - z);
    s = t;
}
// (s, c) += (s2, c2)
__device__ __forceinline__ void two_sum_merge(double& s, double& c, double s2, double c2) {
    two_sum_add(s, c, s2);
    c += c2;
}

// Compensated block reduction of NF per-thread (sum, carry) pairs, fixed order; thread f < NF
// of the block writes field f's block total (one rounding) to out[f].
template <int NT, int NF>
__device__ __forceinline__ void block_csum_store(const double* acc, const double* car, double* out) {
    __shared__ double red[NF][NT / 32][2];
#pragma unroll
    for (int f = 0; f < NF; ++f) {
        double v = acc[f], c = car[f];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double v2 = __shfl_xor_sync(0xffffffffu, v, o), c2 = __shfl_xor_sync(0xffffffffu, c, o);
            two_sum_merge(v, c, v2, c2);
        }
        if ((threadIdx.x & 31) == 0) {
            red[f][threadIdx.x >> 5][0] = v;
            red[f][threadIdx.x >> 5][1] = c;
        }
    }
    __syncthreads();
    if (threadIdx.x < NF) {
        double v = 0.0, c = 0.0;
        for (int w = 0; w < NT / 32; ++w) two_sum_merge(v, c, red[threadIdx.x][w][0], red[threadIdx.x][w][1]);
        out[threadIdx.x] = v + c;
    }
}

// Energy monitor accumulators of a first-sweep thread: plain sums of the current block of
// rows (fields 0..4), max|u0|^2, and the compensated totals (sum, carry) into which
// monitor_flush folds the block sums every kMonitorRows rows -- the per-site cost of
// plain accumulation with the accuracy of compensated summation (a block sum of <= 16
// terms is the only uncompensated step).
constexpr int kAccMax = kObsFields;            // max |u0|^2
constexpr int kAccTot = kObsFields + 1;        // compensated totals of fields 0..4
constexpr int kAccCarry = kAccTot + kObsFields;  // their carries
constexpr int kAccSize = kAccCarry + kObsFields;
constexpr int kMonitorRows = 16;
#ifndef MB4_MONITOR_COMP
#define MB4_MONITOR_COMP 1  // 0: plain block folding (experiment knob)
#endif
#ifndef MB4_MONITOR_AMAX
#define MB4_MONITOR_AMAX 1  // 0: no max|u0|^2 in the monitor (experiment knob)
#endif

__device__ __forceinline__ void monitor_add(double* acc, double kin, double kin_im, double n2, double vn) {
    acc[0] += kin;
    acc[1] += kin_im;
    acc[2] += n2;
    acc[3] += n2 * n2;
    acc[4] += vn;
    if (MB4_MONITOR_AMAX) acc[kAccMax] = fmax(acc[kAccMax], n2);  // max |u0|^2 (spectral bound)
}

__device__ __forceinline__ void monitor_flush(double* acc) {
#pragma unroll
    for (int f = 0; f < kObsFields; ++f) {
        if (f == 1 || !MB4_MONITOR_COMP) {
            acc[kAccTot + f] += acc[f];  // imaginary kinetic part: a health check, plain
        } else {
            two_sum_add(acc[kAccTot + f], acc[kAccCarry + f], acc[f]);
        }
        acc[f] = 0.0;
    }
}

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
