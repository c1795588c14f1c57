// Microbenchmark: FP64 pipe rates on one B200 -- raw DFMA, FRND.F64, and the
// exact modular product (fmulmod) with rint vs magic-number rounding.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_fp64 mb_fp64.cu && ./mb_fp64
#include <cstdint>
#include <cstdio>

__global__ void k_dfma(double *out, int iters, double a, double b) {
    double x[8];
    for (int i = 0; i < 8; i++) x[i] = threadIdx.x + i;
    for (int it = 0; it < iters; it++)
#pragma unroll
        for (int i = 0; i < 8; i++) x[i] = fma(x[i], a, b);
    double s = 0;
    for (int i = 0; i < 8; i++) s += x[i];
    if (s == 12345.0) out[0] = s;
}
__global__ void k_frnd(double *out, int iters, double a) {
    double x[8];
    for (int i = 0; i < 8; i++) x[i] = threadIdx.x + i + 0.25;
    for (int it = 0; it < iters; it++)
#pragma unroll
        for (int i = 0; i < 8; i++) x[i] = rint(x[i]) + a;
    double s = 0;
    for (int i = 0; i < 8; i++) s += x[i];
    if (s == 12345.0) out[0] = s;
}
__device__ __forceinline__ double fm_rint(double a, double w, double q, double qi) {
    const double h = a * w, l = fma(a, w, -h), e = rint(h * qi);
    return fma(-e, q, h) + l;
}
__device__ __forceinline__ double fm_magic(double a, double w, double q, double qi) {
    const double M = 6755399441055744.0;  // 1.5 * 2^52
    const double h = a * w, l = fma(a, w, -h), e = fma(h, qi, M) - M;
    return fma(-e, q, h) + l;
}
template <int V>
__global__ void k_fm(double *out, int iters, double q, double w) {
    const double qi = 1.0 / q;
    double x[8];
    for (int i = 0; i < 8; i++) x[i] = (double)(threadIdx.x * 8 + i + blockIdx.x);
    for (int it = 0; it < iters; it++)
#pragma unroll
        for (int i = 0; i < 8; i++) x[i] = V == 0 ? fm_rint(x[i], w, q, qi) : fm_magic(x[i], w, q, qi);
    double s = 0;
    for (int i = 0; i < 8; i++) s += x[i];
    if (s == 12345.0) out[0] = s;
}

template <typename F>
double run(F f, double n) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms = 0;
    for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        f();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    return n / (ms * 1e-3);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *sink;
    cudaMalloc(&sink, 64);
    const double q = 1099511480321.0, w = 123456789012.0;
    const int blocks = sms * 8, threads = 256, iters = 4096;
    const double n = (double)blocks * threads * iters * 8;
    printf("DFMA            : %.3e /s\n", run([&] { k_dfma<<<blocks, threads>>>(sink, iters, 0.999, 1e-3); }, n));
    printf("FRND.F64 + DADD : %.3e /s\n", run([&] { k_frnd<<<blocks, threads>>>(sink, iters, 0.25); }, n));
    printf("fmulmod (rint)  : %.3e /s\n", run([&] { k_fm<0><<<blocks, threads>>>(sink, iters, q, w); }, n));
    printf("fmulmod (magic) : %.3e /s\n", run([&] { k_fm<1><<<blocks, threads>>>(sink, iters, q, w); }, n));
    return 0;
}
