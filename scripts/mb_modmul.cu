// Microbenchmark: modular multiplication throughput on one B200, integer
// Shoup (64-bit IMAD emulation) vs an FP64 Barrett variant for q < 2^50.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_modmul mb_modmul.cu && ./mb_modmul
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t shoup_lazy(uint64_t a, uint64_t w, uint64_t wp, uint64_t q) {
    return a * w - __umul64hi(a, wp) * q;
}

// 8 independent chains per thread, ITER rounds
__global__ void k_int(uint64_t *out, int iters, uint64_t q, uint64_t w, uint64_t wp) {
    uint64_t x[8];
    for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 8 + i + blockIdx.x;
    for (int it = 0; it < iters; it++)
#pragma unroll
        for (int i = 0; i < 8; i++) x[i] = shoup_lazy(x[i], w, wp, q);
    uint64_t s = 0;
    for (int i = 0; i < 8; i++) s ^= x[i];
    if (s == 12345) out[0] = s;
}

// FP64: a, w exact integers < 2^52 (q < 2^50); r = a*w mod q in (-q, 2q) without conversions
__device__ __forceinline__ double fmod_mul(double a, double w, double q, double qinv) {
    const double h = a * w;
    const double l = fma(a, w, -h);
    const double qe = rint(h * qinv);
    double r = fma(-qe, q, h) + l;
    return r;
}
__global__ void k_fp(double *out, int iters, double q, double w, double qinv) {
    double x[8];
    for (int i = 0; i < 8; i++) x[i] = (double)(threadIdx.x * 8 + i + blockIdx.x);
    for (int it = 0; it < iters; it++)
#pragma unroll
        for (int i = 0; i < 8; i++) {
            double r = fmod_mul(x[i], w, q, qinv);
            x[i] = r < 0 ? r + q : r;
        }
    double s = 0;
    for (int i = 0; i < 8; i++) s += x[i];
    if (s == 12345.0) out[0] = s;
}
// FP64 with u64 <-> f64 conversions around every product (worst case)
__global__ void k_fpc(uint64_t *out, int iters, double q, double w, double qinv) {
    uint64_t x[8];
    for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 8 + i + blockIdx.x;
    for (int it = 0; it < iters; it++)
#pragma unroll
        for (int i = 0; i < 8; i++) {
            double r = fmod_mul((double)x[i], w, q, qinv);
            r = r < 0 ? r + q : r;
            x[i] = (uint64_t)r;
        }
    uint64_t s = 0;
    for (int i = 0; i < 8; i++) s ^= x[i];
    if (s == 12345) out[0] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    void *sink;
    cudaMalloc(&sink, 64);
    const uint64_t q = 1099511480321ull;  // a 40-bit prime
    const uint64_t w = 123456789012ull % q;
    const uint64_t wp = (uint64_t)(((unsigned __int128)w << 64) / q);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    const double n = (double)blocks * threads * iters * 8;
    for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(e0);
        k_int<<<blocks, threads>>>((uint64_t *)sink, iters, q, w, wp);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("integer Shoup lazy : %.3e modmul/s\n", n / (ms * 1e-3));
    for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(e0);
        k_fp<<<blocks, threads>>>((double *)sink, iters, (double)q, (double)w, 1.0 / (double)q);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FP64 Barrett       : %.3e modmul/s\n", n / (ms * 1e-3));
    for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(e0);
        k_fpc<<<blocks, threads>>>((uint64_t *)sink, iters, (double)q, (double)w, 1.0 / (double)q);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FP64 + conversions : %.3e modmul/s\n", n / (ms * 1e-3));
    return 0;
}
