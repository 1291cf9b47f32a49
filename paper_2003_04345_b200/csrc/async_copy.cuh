// cp.async (LDGSTS) helpers shared by the marching sweep kernels.
#pragma once

#include <cuda_runtime.h>

namespace mb4cu {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

}  // namespace mb4cu

// ---- bulk (TMA engine) row copies completing on an mbarrier -----------------------
// One thread copies a whole row segment global -> shared with cp.async.bulk; the bytes
// bypass the LSU data pipe (a warp's 16-byte cp.async of a row segment that is not
// 128-byte aligned costs ~9.5 shared wavefronts instead of 4: profiles/r02_*).
namespace mb4cu {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// make initialised mbarriers visible to the async proxy (then a CTA barrier)
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// Wait for the phase of `parity`; a phase that never completes (a bug: bytes never
// issued) traps after ~4 s instead of hanging the device.
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    if (mbar_try_wait(bar, parity)) return;
    const long long t0 = clock64();
    while (!mbar_try_wait(bar, parity))
        if (clock64() - t0 > (8ll << 30)) __trap();
}

// bytes: multiple of 16; src / dst 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// NCOL consecutive double2 of a lattice row into shared memory, starting at (wrapped)
// column c0: periodic rows wrap at width w (any number of times on small lattices);
// ghost-padded rows stop at the padded width w instead (the clamped columns only feed
// masked outputs).  Returns the bytes copied.
template <bool WRAP>
__device__ __forceinline__ unsigned bulk_row(double2* sdst, const double2* grow, int c0, int ncol, int w,
                                             unsigned long long* bar) {
    if (!WRAP) {
        const int len = ncol < w - c0 ? ncol : w - c0;
        bulk_g2s(sdst, grow + c0, 16u * len, bar);
        return 16u * len;
    }
    int done = 0, c = c0;
    while (done < ncol) {
        const int len = ncol - done < w - c ? ncol - done : w - c;
        bulk_g2s(sdst + done, grow + c, 16u * len, bar);
        done += len;
        c = 0;
    }
    return 16u * ncol;
}

// bytes bulk_row<WRAP> will copy (for the mbarrier's expected transaction count)
template <bool WRAP>
__device__ __forceinline__ unsigned bulk_row_bytes(int c0, int ncol, int w) {
    if (!WRAP) return 16u * (ncol < w - c0 ? ncol : w - c0);
    return 16u * ncol;
}

}  // namespace mb4cu
