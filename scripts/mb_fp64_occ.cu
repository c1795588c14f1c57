// FP64 modular-product throughput vs resident warps per SM and independent chains per thread
// (nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/mb_fp64_occ.cu -o /tmp/mb && /tmp/mb)
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double fmulmod(double a, double w, double q, double qi) {
    const double h = a * w; const double l = fma(a, w, -h); const double e = rint(h * qi); return fma(-e, q, h) + l;
}
__device__ __forceinline__ double fmulmod_m(double a, double w, double q, double qi) {  // magic rounding
    const double h = a * w; const double l = fma(a, w, -h);
    const double e = fma(h, qi, 6755399441055744.0) - 6755399441055744.0; return fma(-e, q, h) + l;
}
template <int CH, bool MAGIC>
__global__ void k(double *sink, int iters, double q, double w) {
    const double qi = 1.0 / q; double x[CH];
    for (int k = 0; k < CH; k++) x[k] = (double)(threadIdx.x * 8 + k + blockIdx.x);
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int k = 0; k < CH; k++) x[k] = MAGIC ? fmulmod_m(x[k], w, q, qi) : fmulmod(x[k], w, q, qi);
    double s = 0; for (int k = 0; k < CH; k++) s += x[k];
    if (s == 12345.0) sink[0] = s;
}
template <int CH, bool MAGIC> void run(int warps_per_sm) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *sink; cudaMalloc(&sink, 64);
    const int threads = 32 * warps_per_sm, iters = 2048;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms = 0;
    for (int r = 0; r < 2; r++) {
        cudaEventRecord(e0); k<CH, MAGIC><<<sms, threads>>>(sink, iters, 1099511480321.0, 123456789.0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    const double per = (double)sms * threads * iters * CH / (ms * 1e-3);
    printf("warps/SM %2d chains %d magic %d: %.2e fmulmod/s = %.1f per SM-cycle (at 1.9 GHz)\n", warps_per_sm, CH, MAGIC,
           per, per / sms / 1.9e9);
    cudaFree(sink);
}
int main() {
    for (int w : {4, 8, 16, 32}) { run<4, false>(w); run<8, false>(w); run<8, true>(w); }
    return 0;
}
