// Probe: do warp shuffles share the L1/shared data pipe with LDS?  Times a loop of
// (a) 2 LDS.128 per iteration, (b) 8 SHFL.32 per iteration, (c) both, at 8 warps/SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, int iters) {
  __shared__ double2 buf[2][256];
  const int t = threadIdx.x;
  buf[0][t] = make_double2(t, t + 1); buf[1][t] = make_double2(t * 2, t);
  __syncthreads();
  double2 a = make_double2(t, 0), b = a;
  int off = 0;
  for (int i = 0; i < iters; ++i) {
    if (MODE & 1) {
      const double2 l = buf[i & 1][(t + 255 + off) & 255], r = buf[(i + 1) & 1][(t + 1 + off) & 255];
      a.x += l.x * l.y; a.y += r.x * r.y;
    }
    if (MODE & 2) {
      b.x += __shfl_up_sync(0xffffffffu, b.y, 1); b.y += __shfl_down_sync(0xffffffffu, b.x, 1);
      a.x += __shfl_up_sync(0xffffffffu, a.y, 1); a.y += __shfl_down_sync(0xffffffffu, a.x, 1);
    }
    off += (int)a.x & 1;
  }
  out[blockIdx.x * blockDim.x + t] = a.x + a.y + b.x + b.y;
}
template <int MODE> float run(double* out, int iters) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE><<<148 * 4, 256>>>(out, iters);
  cudaEventRecord(e0);
  k<MODE><<<148 * 4, 256>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); return ms;
}
int main() {
  double* out; cudaMalloc(&out, 148 * 4 * 256 * 8);
  const int it = 20000;
  printf("LDS (2x LDS.128/iter): %.3f ms\n", run<1>(out, it));
  printf("SHFL (8x SHFL.32 as 4x 64-bit/iter): %.3f ms\n", run<2>(out, it));
  printf("both: %.3f ms\n", run<3>(out, it));
  return 0;
}
