// Does a running tcgen05.mma (kind::i8) stream slow the FP64 pipe of the same SM?
// 16 warps run fmulmod / DFMA chains (ILP 4) while one extra warp issues back-to-back
// M=128 N=32 K=32 int8 MMAs (mode 1) or idles (mode 0).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2604_16834_b200/csrc -o mb_fp64_vs_mma mb_fp64_vs_mma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc5.cuh"

constexpr int BK = 256;

template <int KIND>  // 0: fmulmod chains, 1: dfma chains, 2: integer IMAD chains
__global__ void __launch_bounds__(17 * 32, 1) k(int N, int mma_on, int iters, unsigned long long *cyc, double *sink, double q,
                                                double w) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t taddr_s;
    __shared__ volatile int stop;
    const int abytes = 128 * BK;
    for (int i = threadIdx.x; i < abytes + N * BK; i += blockDim.x) sm[i] = (uint8_t)(i * 2654435761u >> 24);
    tc5::fence_async_smem();
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tc5::tmem_alloc<256>(&taddr_s);
    if (threadIdx.x == 0) {
        tc5::mbar_init(&bar, 1);
        tc5::mbar_fence_init();
        stop = 0;
    }
    tc5::tc_fence_before();
    __syncthreads();
    tc5::tc_fence_after();
    const uint32_t taddr = taddr_s;
    if (warp == 16) {
        if (threadIdx.x == 16 * 32 && mma_on) {
            const uint32_t idesc = tc5::idesc_u8s8(128, N);
            const uint32_t sa = tc5::smem_u32(sm), sb = tc5::smem_u32(sm + abytes);
            const uint32_t a_lbo = 2048, a_sbo = 128, b_lbo = (uint32_t)N * 16;
            unsigned long long n = 0;
            const unsigned long long t0 = clock64();
            while (!stop) {
#pragma unroll
                for (int t = 0; t < BK / 32; t++)
                    tc5::mma_i8(taddr + (uint32_t)((t % 4) * N), tc5::sdesc(sa + 2 * t * a_lbo, a_lbo, a_sbo),
                                tc5::sdesc(sb + 2 * t * b_lbo, b_lbo, 128), idesc, n != 0);
                n += BK / 32;
                if ((n & 63) == 0) {  // bound the in-flight queue
                    tc5::tc_commit(&bar);
                    tc5::mbar_wait(&bar, (uint32_t)((n / 64 - 1) & 1));
                }
            }
            if (blockIdx.x == 0) {
                cyc[1] = n;
                cyc[2] = clock64() - t0;
            }
        }
    } else {
        const double qi = 1.0 / q;
        double x[4];
        uint32_t u[4];
#pragma unroll
        for (int k2 = 0; k2 < 4; k2++) {
            x[k2] = (double)(threadIdx.x * 8 + k2 + blockIdx.x);
            u[k2] = threadIdx.x * 8 + k2;
        }
        asm volatile("bar.sync 1, 512;");
        const unsigned long long t0 = clock64();
        for (int i = 0; i < iters; i++)
#pragma unroll
            for (int k2 = 0; k2 < 4; k2++) {
                if (KIND == 0) {
                    const double h = x[k2] * w, l = fma(x[k2], w, -h), e = rint(h * qi);
                    x[k2] = fma(-e, q, h) + l;
                } else if (KIND == 1) {
                    x[k2] = fma(x[k2], 1.0000001, q);
                } else {
                    u[k2] = u[k2] * 2654435761u + 12345u;
                }
            }
        asm volatile("bar.sync 1, 512;");
        if (threadIdx.x == 0) {
            if (blockIdx.x == 0) cyc[0] = clock64() - t0;
            stop = 1;
        }
        double s = 0;
#pragma unroll
        for (int k2 = 0; k2 < 4; k2++) s += x[k2] + u[k2];
        if (s == 12345.0) sink[0] = s;
    }
    tc5::tc_fence_before();
    __syncthreads();
    if (warp == 0) tc5::tmem_free<256>(taddr);
}

int main() {
    unsigned long long *cyc, h[3];
    double *sink;
    cudaMalloc(&cyc, 24);
    cudaMalloc(&sink, 8);
    const int iters = 1 << 15, N = 32;
    const int smem = 128 * BK + N * BK;
    auto run = [&](auto kern, const char *name, int per_step) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int mma = 0; mma < 2; mma++) {
            cudaMemset(cyc, 0, 24);
            kern<<<148, 17 * 32, smem>>>(N, mma, iters, cyc, sink, 1099511480321.0, 123456789012.0);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(h, cyc, 24, cudaMemcpyDeviceToHost);
            printf("%s mma %d: %s, %.1f cycles per chain step per SMSP (4 warps, ILP 4), FP64 lanes/clk/SM %.1f; MMAs %llu in %llu cycles (%.1f cycles each)\n",
                   name, mma, cudaGetErrorString(e), (double)h[0] / (iters * 4.0 * 4.0),
                   16.0 * 32 * iters * 4 * per_step / (double)h[0], h[1], h[2], h[1] ? (double)h[2] / h[1] : 0.0);
        }
    };
    run(k<0>, "fmulmod", 5);
    run(k<1>, "dfma   ", 1);
    run(k<2>, "imad   ", 1);
    return 0;
}
