// Microbenchmark: FP64 pipe throughput on one SM as a function of resident warps per
// SM sub-partition and independent DFMA chains per thread (ILP), plain and with one
// integer / one shared-memory load interleaved per DFMA.  Prints the fraction of the
// 16 lanes/clk/sub-partition peak.  nvcc -arch=sm_100a -O3 fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP, int MIX>
__global__ void chains(double* out, int iters, long long* cyc) {
    __shared__ double sm[1024];
    sm[threadIdx.x] = threadIdx.x * 1e-9;
    __syncthreads();
    double a[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) a[k] = threadIdx.x * 1e-3 + k;
    const double b = 0.999999, c = 1e-7;
    int iacc = threadIdx.x;
    double sacc = 0.0;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
            for (int k = 0; k < ILP; ++k) {
                a[k] = fma(a[k], b, c);
                if (MIX == 1) iacc = iacc * 3 + r;  // one integer op per DFMA
                if (MIX == 2) sacc += sm[(iacc + k + r * ILP) & 1023];  // (adds a DADD too)
            }
        }
        if (MIX == 2) iacc += 7;
    }
    const long long t1 = clock64();
    double s = sacc + iacc;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int ILP, int MIX>
void run(double* out, long long* cyc, int warps_per_smsp) {
    const int iters = 2000;
    const int threads = 32 * 4 * warps_per_smsp;  // one CTA on one SM
    if (threads > 1024) return;
    chains<ILP, MIX><<<1, threads>>>(out, iters, cyc);
    chains<ILP, MIX><<<1, threads>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    // FP64 instructions per sub-partition: warps * iters * 8 * ILP (MIX 2: twice), 2 clk each
    const double inst = (double)warps_per_smsp * iters * 8 * ILP * (MIX == 2 ? 2 : 1);
    printf("mix %d  warps/smsp %d  ilp %d : %.3f of peak (%.1f clk per dependent DFMA)\n", MIX, warps_per_smsp, ILP,
           2.0 * inst / h, (double)h / (iters * 8.0));
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1024 * sizeof(double));
    cudaMalloc(&cyc, sizeof(long long));
    const int ws[] = {1, 2, 3, 4, 6, 8};
    for (int w : ws) {
        run<1, 0>(out, cyc, w);
        run<2, 0>(out, cyc, w);
        run<3, 0>(out, cyc, w);
        run<4, 0>(out, cyc, w);
        run<6, 0>(out, cyc, w);
        run<8, 0>(out, cyc, w);
    }
    for (int w : ws) {
        run<2, 1>(out, cyc, w);
        run<4, 1>(out, cyc, w);
        run<2, 2>(out, cyc, w);
        run<4, 2>(out, cyc, w);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
