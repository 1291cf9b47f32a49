// Sub-domain (multi-GPU) support kernels: halo pack / unpack between padded
// local arrays and contiguous exchange buffers, and the energy monitor on a
// padded sub-domain.  The exchange itself (NCCL send/recv between the 4 torus
// neighbours, x phase then y phase so corners propagate) is driven by the host
// (paper_2003_04345_b200/dist.py); see DESIGN.md section 8.
#include <cuda_runtime.h>

#include "mb4cu_internal.hpp"
#include "site_math.cuh"

namespace mb4cu {
namespace {

template <typename T>
__global__ void halo_copy_kernel(T* const* arrays, int narr, int pitch, int ghost, int x0, int y0, int w,
                                 int h, T* buf, bool pack) {
    const size_t per = static_cast<size_t>(w) * h;
    const size_t total = per * narr;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int a = static_cast<int>(e / per);
        const size_t r = e - static_cast<size_t>(a) * per;
        const int y = static_cast<int>(r / w), x = static_cast<int>(r - static_cast<size_t>(y) * w);
        const size_t g = static_cast<size_t>(y0 + y + ghost) * pitch + (x0 + x + ghost);
        if (pack)
            buf[e] = arrays[a][g];
        else
            arrays[a][g] = buf[e];
    }
}

struct Ptrs2 {
    double2* p[3];
};

__global__ void halo_copy2_kernel(Ptrs2 arrays, int narr, int pitch, int ghost, int x0, int y0, int w, int h,
                                  double2* buf, bool pack) {
    const size_t per = static_cast<size_t>(w) * h;
    const size_t total = per * narr;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int a = static_cast<int>(e / per);
        const size_t r = e - static_cast<size_t>(a) * per;
        const int y = static_cast<int>(r / w), x = static_cast<int>(r - static_cast<size_t>(y) * w);
        const size_t g = static_cast<size_t>(y0 + y + ghost) * pitch + (x0 + x + ghost);
        if (pack)
            buf[e] = arrays.p[a][g];
        else
            arrays.p[a][g] = buf[e];
    }
}

// Periodic wrap of a sub-domain onto itself (a process-grid dimension of extent 1): the
// owned strips go straight into the opposite ghost strips, one launch per phase instead
// of a pack and an unpack per side.  phase 0: columns (owned rows); phase 1: rows (the
// full padded width, after phase 0, so the corners follow).  narr double2 arrays, or one
// double array (V) when d1 != nullptr.
__global__ void halo_wrap_kernel(Ptrs2 arrays, double* d1, int narr, int pitch, int ghost, int nx, int ny, int g,
                                 int phase) {
    const int w = phase == 0 ? g : nx + 2 * g, h = phase == 0 ? ny : g;
    const size_t per = static_cast<size_t>(w) * h;  // sites of one ghost strip
    const size_t total = 2 * per * narr;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int a = static_cast<int>(e / (2 * per));
        size_t r = e - static_cast<size_t>(a) * 2 * per;
        const int hi = r >= per ? 1 : 0;
        r -= hi * per;
        const int y = static_cast<int>(r / w), x = static_cast<int>(r - static_cast<size_t>(y) * w);
        int dx, dy, sx, sy;  // ghost (destination) and owned (source) coordinates
        if (phase == 0) {
            dy = sy = y;
            dx = hi ? nx + x : x - g;
            sx = hi ? x : nx - g + x;
        } else {
            dx = sx = x - g;
            dy = hi ? ny + y : y - g;
            sy = hi ? y : ny - g + y;
        }
        const size_t gd = static_cast<size_t>(dy + ghost) * pitch + (dx + ghost);
        const size_t gs = static_cast<size_t>(sy + ghost) * pitch + (sx + ghost);
        if (d1)
            d1[gd] = d1[gs];
        else
            arrays.p[a][gd] = arrays.p[a][gs];
    }
}

__global__ void halo_copy1_kernel(double* array, int pitch, int ghost, int x0, int y0, int w, int h,
                                  double* buf, bool pack) {
    const size_t total = static_cast<size_t>(w) * h;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int y = static_cast<int>(e / w), x = static_cast<int>(e - static_cast<size_t>(y) * w);
        const size_t g = static_cast<size_t>(y0 + y + ghost) * pitch + (x0 + x + ghost);
        if (pack)
            buf[e] = array[g];
        else
            array[g] = buf[e];
    }
}

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads)
observables_ghost_kernel(const ObsArgs a, int ghost, int pitch) {
    double acc[kObsFields] = {0.0, 0.0, 0.0, 0.0, 0.0};
    double car[kObsFields] = {0.0, 0.0, 0.0, 0.0, 0.0};  // compensation (two_sum_add)
    // rows round-robin over the blocks, columns over the threads (no division)
    for (int j = blockIdx.x; j < a.ny; j += gridDim.x) {
        const size_t g0 = static_cast<size_t>(j + ghost) * pitch + ghost;
        for (int i = threadIdx.x; i < a.nx; i += blockDim.x) {
            const size_t g = g0 + i;
            const double2 u = a.u[g], l = a.u[g - 1], r = a.u[g + 1], d = a.u[g - pitch], up = a.u[g + pitch];
            const double kx = fma(a.diag, u.x, -(a.cx * (l.x + r.x) + a.cy * (d.x + up.x)));
            const double ky = fma(a.diag, u.y, -(a.cx * (l.y + r.y) + a.cy * (d.y + up.y)));
            two_sum_add(acc[0], car[0], fma(u.x, kx, u.y * ky));
            acc[1] += fma(u.x, ky, -u.y * kx);
            const double n2 = fma(u.x, u.x, u.y * u.y);
            two_sum_add(acc[2], car[2], n2);
            two_sum_add(acc[3], car[3], n2 * n2);
            two_sum_add(acc[4], car[4], a.V[g] * n2);
        }
    }
    block_csum_store<kThreads, kObsFields>(acc, car, a.partial + blockIdx.x * kObsFields);
}

__global__ void observables_ghost_finalize(const double* partial, int nblocks, double* out) {
    if (threadIdx.x < kObsFields) {
        double v = 0.0, c = 0.0;
        for (int b = 0; b < nblocks; ++b) two_sum_add(v, c, partial[b * kObsFields + threadIdx.x]);
        out[threadIdx.x] = v + c;
    }
}

int blocks_for(size_t n) {
    const size_t b = (n + kThreads - 1) / kThreads;
    return static_cast<int>(b < 148 * 8 ? (b ? b : 1) : 148 * 8);
}

}  // namespace

cudaError_t launch_halo_copy2(double2* const* arrays, int narr, int pitch, int ghost, int x0, int y0,
                              int w, int h, double2* buf, bool pack, cudaStream_t s) {
    Ptrs2 p{};
    for (int i = 0; i < narr && i < 3; ++i) p.p[i] = arrays[i];
    halo_copy2_kernel<<<blocks_for(static_cast<size_t>(w) * h * narr), kThreads, 0, s>>>(
        p, narr, pitch, ghost, x0, y0, w, h, buf, pack);
    return cudaGetLastError();
}

cudaError_t launch_halo_wrap(double2* const* arrays, double* d1, int narr, int pitch, int ghost, int nx, int ny,
                             int g, int phase, cudaStream_t s) {
    Ptrs2 p{};
    for (int i = 0; i < narr && i < 3; ++i) p.p[i] = arrays ? arrays[i] : nullptr;
    const size_t sites = 2 * static_cast<size_t>(phase == 0 ? g * ny : g * (nx + 2 * g)) * (d1 ? 1 : narr);
    halo_wrap_kernel<<<blocks_for(sites), kThreads, 0, s>>>(p, d1, d1 ? 1 : narr, pitch, ghost, nx, ny, g, phase);
    return cudaGetLastError();
}

cudaError_t launch_halo_copy1(double* array, int pitch, int ghost, int x0, int y0, int w, int h,
                              double* buf, bool pack, cudaStream_t s) {
    halo_copy1_kernel<<<blocks_for(static_cast<size_t>(w) * h), kThreads, 0, s>>>(array, pitch, ghost, x0, y0,
                                                                                  w, h, buf, pack);
    return cudaGetLastError();
}

namespace {
// Convergence test of sweep s of a decomposed (sub)step on the device, after the all-reduce
// of its residual: out[s * stride] = the global ||r||_inf (non-finite reported as +inf).
// state[0] = done (converged or diverged: the later sweeps enqueued ahead become no-ops),
// state[1] = sweeps of the converged iterate, state[2] = diverged.
__global__ void dist_converge_kernel(const double* out, int stride, int s, double eps, int* state) {
    if (state[0]) return;  // an earlier sweep ended the sub-step (this one was skipped)
    const double r = out[static_cast<size_t>(s) * stride];
    const double rp = s > 0 ? out[static_cast<size_t>(s - 1) * stride] : 0.0;
    if (!isfinite(r)) {
        state[2] = 1;
        state[0] = 1;
        state[1] = s + 1;
    } else if (stage_converged(r, rp, s, eps)) {
        state[0] = 1;
        state[1] = s + 1;
    }
}
}  // namespace

cudaError_t launch_dist_converge(const double* out, int stride, int s, double eps, int* state, cudaStream_t st) {
    dist_converge_kernel<<<1, 1, 0, st>>>(out, stride, s, eps, state);
    return cudaGetLastError();
}

cudaError_t launch_observables_ghost(const ObsArgs& a, int ghost, int pitch, double* out5, cudaStream_t s) {
    // a.partial must hold obs_blocks(nx, ny) * kObsFields doubles
    const int nb = obs_blocks(a.nx, a.ny);
    observables_ghost_kernel<<<nb, kThreads, 0, s>>>(a, ghost, pitch);
    observables_ghost_finalize<<<1, 32, 0, s>>>(a.partial, nb, out5);
    return cudaGetLastError();
}

}  // namespace mb4cu
