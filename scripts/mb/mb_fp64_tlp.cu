// FP64 pipe throughput on sm_100a as a function of resident warps per SM and independent
// chains per thread (ILP): DFMA chains and fmulmod (DMUL/DFMA/FRND) chains.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_fp64_tlp mb_fp64_tlp.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP, bool MODMUL>
__global__ void k(double *sink, int iters, double q, double w) {
    const double qi = 1.0 / q;
    double x[ILP];
#pragma unroll
    for (int k = 0; k < ILP; k++) x[k] = (double)(threadIdx.x * 8 + k + blockIdx.x);
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int k = 0; k < ILP; k++) {
            if (MODMUL) {
                const double h = x[k] * w, l = fma(x[k], w, -h), e = rint(h * qi);
                x[k] = fma(-e, q, h) + l;
            } else {
                x[k] = fma(x[k], w, q);
            }
        }
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; k++) s += x[k];
    if (s == 12345.0) sink[0] = s;
}

template <int ILP, bool MODMUL>
void run(int warps_per_sm, int sms, double *sink, double mhz) {
    const int threads = warps_per_sm >= 32 ? 1024 : warps_per_sm * 32;
    const int blocks = sms * (warps_per_sm >= 32 ? warps_per_sm / 32 : 1);
    const int iters = 1 << 14;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms = 0;
    for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(e0);
        k<ILP, MODMUL><<<blocks, threads>>>(sink, iters, 1099511480321.0, MODMUL ? 123456789012.0 : 1.0000001);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * threads * iters * ILP;  // chain steps
    const double fp64_per_step = MODMUL ? 5 : 1;
    const double cyc = ms * 1e-3 * mhz * 1e6;
    printf("%s warps/SM %2d ILP %d: %.3e steps/s, FP64-pipe lanes/clk/SM %.1f, cycles per warp-step %.1f\n",
           MODMUL ? "fmulmod" : "dfma   ", warps_per_sm, ILP, ops / (ms * 1e-3), ops * fp64_per_step / cyc / sms,
           cyc / ((double)iters * ILP));
}

int main() {
    int sms = 0, khz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double mhz = khz / 1e3;
    double *sink;
    cudaMalloc(&sink, 64);
    printf("SMs %d, %0.f MHz\n", sms, mhz);
    for (int w : {4, 8, 16, 32, 64}) {
        run<1, false>(w, sms, sink, mhz);
        run<4, false>(w, sms, sink, mhz);
        run<8, false>(w, sms, sink, mhz);
        run<1, true>(w, sms, sink, mhz);
        run<4, true>(w, sms, sink, mhz);
        run<8, true>(w, sms, sink, mhz);
    }
    return 0;
}
