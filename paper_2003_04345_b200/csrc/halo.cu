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

cudaError_t launch_halo_copy1(double* array, int pitch, int ghost, int x0, int y0, int w, int h,
                              double* buf, bool pack, cudaStream_t s) {
    halo_copy1_kernel<<<blocks_for(static_cast<size_t>(w) * h), kThreads, 0, s>>>(array, pitch, ghost, x0, y0,
                                                                                  w, h, buf, pack);
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
