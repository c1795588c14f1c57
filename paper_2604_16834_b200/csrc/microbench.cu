// microbench.cu -- integer-pipe peak measurement for the roofline denominators.
//
// MEASURED_PEAKS.json carries only HBM and bf16 tensor peaks; the NTT, key
// switching and CUDA-core linear combination are integer-pipe bound, so the
// engine measures the pipe it runs on: independent 32-bit IMAD chains
// (8 per thread, full grid) and the 64x64->128 multiply-accumulate the
// kernels use (mad.lo.cc.u64 + madc.hi.u64).
#include "ntt_core.cuh"  // fmulmod: the FP64 modular product of the < 2^42 prime path

namespace {

__global__ void k_imad32(uint32_t *sink, int iters, uint32_t seed) {
    uint32_t a[8];
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = seed + threadIdx.x * 8 + k;
    const uint32_t m = seed | 1u;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 8; k++) a[k] = a[k] * m + (uint32_t)k;
    }
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) s ^= a[k];
    if (s == 0x12345678u) sink[0] = s;
}

__global__ void k_mac128(uint64_t *sink, int iters, uint64_t seed) {
    u128 acc[4] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
    uint64_t x = seed + threadIdx.x, w = seed * 3 + 1;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 4; k++) mac128(acc[k], x + k, w);
        x += acc[0].lo & 1;
    }
    uint64_t s = acc[0].hi ^ acc[1].hi ^ acc[2].hi ^ acc[3].lo;
    if (s == 0x123456789ull) sink[0] = s;
}

// FP64 modular products (fmulmod, the key-switch / NTT datapath for primes
// below 2^42): 8 independent chains per thread on a 40-bit prime
__global__ void k_fmulmod(double *sink, int iters, double q, double w) {
    const double qi = 1.0 / q;
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = (double)(threadIdx.x * 8 + k + blockIdx.x);
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = fmulmod(x[k], w, q, qi);  // lazy: |x| < 3q stays exact
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) s += x[k];
    if (s == 12345.0) sink[0] = s;
}

// mma.sync.m16n8k32 u8 x s8 -> s32 (the fused conv's tensor-core instruction):
// 8 independent accumulators per warp, full grid
__global__ void k_imma(int *sink, int iters, uint32_t seed) {
    int c[8][4];
#pragma unroll
    for (int k = 0; k < 8; k++) c[k][0] = c[k][1] = c[k][2] = c[k][3] = 0;
    uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7;
    const uint32_t b0 = seed * 11, b1 = seed * 13;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 8; k++)
            asm volatile(
                "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+r"(c[k][0]), "+r"(c[k][1]), "+r"(c[k][2]), "+r"(c[k][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
        a0 += 1;
    }
    int s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) s ^= c[k][0] ^ c[k][3];
    if (s == 0x12345678) sink[0] = s;
}

}  // namespace

// int8 multiply-accumulates per second through mma.sync m16n8k32 (u8 x s8),
// the instruction of the fused conv kernels (convsq_kernel.cuh)
extern "C" int he_microbench_imma(int device, double *mac_per_s) {
    HE_CHECK_CUDA(cudaSetDevice(device));
    int sms = 0;
    HE_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    void *sink;
    HE_CHECK_CUDA(cudaMalloc(&sink, 64));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 4, threads = 256, iters = 2048;
    float ms = 0;
    for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(e0);
        k_imma<<<blocks, threads>>>((int *)sink, iters, 12345u);
        cudaEventRecord(e1);
        HE_CHECK_CUDA(cudaEventSynchronize(e1));
    }
    cudaEventElapsedTime(&ms, e0, e1);
    *mac_per_s = (double)blocks * (threads / 32) * iters * 8 * (16.0 * 8 * 32) / (ms * 1e-3);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// FP64 modular products per second (fmulmod on a 40-bit prime, full grid)
extern "C" int he_microbench_fp64(int device, double *modmul_per_s) {
    HE_CHECK_CUDA(cudaSetDevice(device));
    int sms = 0;
    HE_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    void *sink;
    HE_CHECK_CUDA(cudaMalloc(&sink, 64));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    float ms = 0;
    for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(e0);
        k_fmulmod<<<blocks, threads>>>((double *)sink, iters, 1099511480321.0, 123456789012.0);
        cudaEventRecord(e1);
        HE_CHECK_CUDA(cudaEventSynchronize(e1));
    }
    cudaEventElapsedTime(&ms, e0, e1);
    *modmul_per_s = (double)blocks * threads * iters * 8 / (ms * 1e-3);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// ops_per_s[0] = 32-bit IMAD/s, ops_per_s[1] = 64x64->128 MAC/s (blocking)
extern "C" int he_microbench_intpipe(int device, double *ops_per_s) {
    HE_CHECK_CUDA(cudaSetDevice(device));
    int sms = 0;
    HE_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    void *sink;
    HE_CHECK_CUDA(cudaMalloc(&sink, 64));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    float ms = 0;
    for (int rep = 0; rep < 2; rep++) {  // first run warms clocks
        cudaEventRecord(e0);
        k_imad32<<<blocks, threads>>>((uint32_t *)sink, iters, 12345u);
        cudaEventRecord(e1);
        HE_CHECK_CUDA(cudaEventSynchronize(e1));
    }
    cudaEventElapsedTime(&ms, e0, e1);
    ops_per_s[0] = (double)blocks * threads * iters * 8 / (ms * 1e-3);
    for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(e0);
        k_mac128<<<blocks, threads>>>((uint64_t *)sink, iters, 12345u);
        cudaEventRecord(e1);
        HE_CHECK_CUDA(cudaEventSynchronize(e1));
    }
    cudaEventElapsedTime(&ms, e0, e1);
    ops_per_s[1] = (double)blocks * threads * iters * 4 / (ms * 1e-3);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    HE_CHECK_LAUNCH();
    return HE_OK;
}
