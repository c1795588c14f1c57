// tc5probe.cu -- tcgen05.mma kind::i8 self-test and throughput probe.
//
// he_tc5_selftest: one CTA multiplies a deterministic u8 A (128 x 64) by a
// deterministic s8 B (N x 64), both K-major in the no-swizzle core-matrix
// layout, accumulating in TMEM, and returns D (128 x N int32) so the host can
// check the descriptor encodings (tests/test_gpu_tc5.py).  Two operand
// layouts are exercised: layout 0 puts the two 16-byte K chunks of a K step
// 2 KB apart and 8-row groups 128 B apart; layout 1 interleaves them (chunk
// stride 128 B, group stride 512 B).
//
// he_microbench_tc5: int8 MAC/s of a long back-to-back MMA chain (M = 128,
// the given N, K = 32 per instruction, both operands read from shared memory)
// on every SM: the tcgen05 roofline denominator of the conv kernels.
#include "common.cuh"
#include "tc5.cuh"

namespace {

__host__ __device__ inline uint32_t probe_hash(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

constexpr int PK = 64;  // self-test K (two MMAs)

// byte offset of (row r, K byte k) in a K-major no-swizzle operand
__device__ __forceinline__ uint32_t koff(int r, int k, uint32_t lbo, uint32_t sbo) {
    return (uint32_t)(r >> 3) * sbo + (uint32_t)(k >> 4) * lbo + (uint32_t)(r & 7) * 16 + (uint32_t)(k & 15);
}

__global__ void __launch_bounds__(128, 1) k_tc5_selftest(int N, int layout, int32_t *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t taddr_s;
    // A: 128 rows; B: N rows; K = 64 bytes = 4 chunks
    const uint32_t a_lbo = layout ? 128 : 2048, a_sbo = layout ? 512 : 128;  // layout 1: [group][chunk][8x16]
    const uint32_t b_lbo = layout ? 128 : (uint32_t)N * 16, b_sbo = layout ? 512 : 128;
    uint8_t *A = sm, *B = sm + 128 * PK;
    for (int i = threadIdx.x; i < 128 * PK; i += blockDim.x) {
        const int r = i / PK, k = i % PK;
        A[koff(r, k, a_lbo, a_sbo)] = (uint8_t)(probe_hash((uint32_t)i) & 0xFF);
    }
    for (int i = threadIdx.x; i < N * PK; i += blockDim.x) {
        const int r = i / PK, k = i % PK;
        B[koff(r, k, b_lbo, b_sbo)] = (uint8_t)(probe_hash(0x9E3779B9u + (uint32_t)i) & 0xFF);
    }
    tc5::fence_async_smem();
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tc5::tmem_alloc<256>(&taddr_s);
    if (threadIdx.x == 0) {
        tc5::mbar_init(&bar, 1);
        tc5::mbar_fence_init();
    }
    tc5::tc_fence_before();
    __syncthreads();
    tc5::tc_fence_after();
    const uint32_t taddr = taddr_s;
    if (threadIdx.x == 0) {
        const uint32_t idesc = tc5::idesc_u8s8(128, N);
        const uint32_t sa = tc5::smem_u32(A), sb = tc5::smem_u32(B);
        for (int t = 0; t < PK / 32; t++)  // K step t: chunks 2t, 2t+1
            tc5::mma_i8(taddr, tc5::sdesc(sa + 2 * t * a_lbo, a_lbo, a_sbo), tc5::sdesc(sb + 2 * t * b_lbo, b_lbo, b_sbo),
                        idesc, t > 0);
        tc5::tc_commit(&bar);
    }
    __syncwarp();
    tc5::mbar_wait(&bar, 0);
    tc5::tc_fence_after();
    const int row = warp * 32 + (threadIdx.x & 31);
    for (int c = 0; c < N; c += 8) {
        uint32_t v[8];
        tc5::tld8(taddr + ((uint32_t)(warp * 32) << 16) + (uint32_t)c, v);
        tc5::tld_wait();
        for (int j = 0; j < 8; j++) out[(size_t)row * N + c + j] = (int32_t)v[j];
    }
    tc5::tc_fence_before();
    __syncthreads();
    if (warp == 0) tc5::tmem_free<256>(taddr);
}

constexpr int BK = 256;  // throughput probe: K bytes resident (8 K steps)

__global__ void __launch_bounds__(128, 1) k_tc5_rate(int N, int iters, unsigned long long *cyc, uint32_t a_sbo,
                                                     uint32_t a_lbo, int abytes, int ndst) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t taddr_s;
    uint8_t *A = sm, *B = sm + abytes;
    for (int i = threadIdx.x; i < abytes + N * BK; i += blockDim.x) sm[i] = (uint8_t)probe_hash((uint32_t)i);
    tc5::fence_async_smem();
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tc5::tmem_alloc<256>(&taddr_s);
    if (threadIdx.x == 0) {
        tc5::mbar_init(&bar, 1);
        tc5::mbar_fence_init();
    }
    tc5::tc_fence_before();
    __syncthreads();
    tc5::tc_fence_after();
    const uint32_t taddr = taddr_s;
    if (threadIdx.x == 0) {
        const uint32_t idesc = tc5::idesc_u8s8(128, N);
        const uint32_t sa = tc5::smem_u32(A), sb = tc5::smem_u32(B);
        const uint32_t b_lbo = (uint32_t)N * 16;
        const unsigned long long t0 = clock64();
        for (int it = 0; it < iters; it++)
#pragma unroll
            for (int t = 0; t < BK / 32; t++)
                tc5::mma_i8(taddr + (uint32_t)((t % ndst) * N), tc5::sdesc(sa + 2 * t * a_lbo, a_lbo, a_sbo),
                            tc5::sdesc(sb + 2 * t * b_lbo, b_lbo, 128), idesc, it != 0);
        tc5::tc_commit(&bar);
        tc5::mbar_wait(&bar, 0);
        if (blockIdx.x == 0) *cyc = clock64() - t0;
    }
    __syncwarp();
    tc5::mbar_wait(&bar, 0);
    tc5::tc_fence_before();
    __syncthreads();
    if (warp == 0) tc5::tmem_free<256>(taddr);
}

// TMEM -> register read throughput: `warps` warps each load `cols` consecutive columns of
// their lane quarter (32x32b.x{cols}) per iteration, waiting after every `batch` loads
template <int COLS>
__global__ void k_tmem_ld_rate(int iters, int batch, unsigned long long *cyc, uint32_t *sink) {
    __shared__ uint32_t taddr_s;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tc5::tmem_alloc<512>(&taddr_s);
    tc5::tc_fence_before();
    __syncthreads();
    tc5::tc_fence_after();
    const uint32_t t0 = taddr_s + ((uint32_t)((warp & 3) * 32) << 16);
    uint32_t acc = 0;
    __syncthreads();
    const unsigned long long c0 = clock64();
    for (int it = 0; it < iters; it++) {
        uint32_t r[COLS];
        for (int b = 0; b < batch; b++) {
            const uint32_t a = t0 + (uint32_t)(((it * batch + b) * COLS + (warp >> 2) * 8) & 511 & ~(COLS - 1));
            if constexpr (COLS == 4) {
                uint32_t (&rr)[4] = *reinterpret_cast<uint32_t(*)[4]>(r);
                tc5::tld4(a, rr);
            } else if constexpr (COLS == 8) {
                uint32_t (&rr)[8] = *reinterpret_cast<uint32_t(*)[8]>(r);
                tc5::tld8(a, rr);
            } else {
                uint32_t (&rr)[16] = *reinterpret_cast<uint32_t(*)[16]>(r);
                tc5::tld16(a, rr);
            }
            tc5::tld_wait();
#pragma unroll
            for (int k = 0; k < COLS; k++) acc += r[k];
        }
    }
    __syncthreads();
    const unsigned long long c1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = c1 - c0;
    if (acc == 0x12345678u) *sink = acc;
    tc5::tc_fence_before();
    __syncthreads();
    if (warp == 0) tc5::tmem_free<512>(taddr_s);
}

}  // namespace

// rates[0] = bytes / cycle / SM read from TMEM by `warps` warps (32x32b.x{cols}), rates[1] = cycles
extern "C" int he_microbench_tmem_ld(int device, int warps, int cols, double *rates) {
    if (!rates || warps < 4 || warps > 32 || warps % 4 || (cols != 4 && cols != 8 && cols != 16)) {
        he_set_error("he_microbench_tmem_ld: warps in {4..32} (multiple of 4), cols in {4, 8, 16}");
        return HE_EINVAL;
    }
    HE_CHECK_CUDA(cudaSetDevice(device));
    unsigned long long *cyc;
    uint32_t *sink;
    HE_CHECK_CUDA(cudaMalloc(&cyc, 8));
    HE_CHECK_CUDA(cudaMalloc(&sink, 4));
    const int iters = 2048, batch = 4;
    for (int rep = 0; rep < 2; rep++) {
        if (cols == 4) k_tmem_ld_rate<4><<<1, warps * 32>>>(iters, batch, cyc, sink);
        else if (cols == 8) k_tmem_ld_rate<8><<<1, warps * 32>>>(iters, batch, cyc, sink);
        else k_tmem_ld_rate<16><<<1, warps * 32>>>(iters, batch, cyc, sink);
        HE_CHECK_CUDA(cudaDeviceSynchronize());
    }
    unsigned long long c = 0;
    HE_CHECK_CUDA(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    rates[0] = (double)warps * 32 * 4 * cols * iters * batch / (double)c;
    rates[1] = (double)c;
    cudaFree(cyc);
    cudaFree(sink);
    return HE_OK;
}

extern "C" int he_tc5_selftest(int device, int n, int layout, int32_t *d_out) {
    if (n < 16 || n > 256 || n % 16 || (layout != 0 && layout != 1) || !d_out) {
        he_set_error("he_tc5_selftest: N must be a multiple of 16 in [16, 256], layout 0 or 1");
        return HE_EINVAL;
    }
    HE_CHECK_CUDA(cudaSetDevice(device));
    const size_t smem = (size_t)(128 + n) * PK;
    HE_CHECK_CUDA(cudaFuncSetAttribute(k_tc5_selftest, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_tc5_selftest<<<1, 128, smem>>>(n, layout, d_out);
    HE_CHECK_LAUNCH();
    HE_CHECK_CUDA(cudaDeviceSynchronize());
    return HE_OK;
}

// rates[0] = int8 MAC/s over all SMs, rates[1] = cycles per MMA (M=128, N=n, K=32) on one SM.
// a_sbo = 0: A contiguous (8-row groups 128 B apart); else the A operand's 8-row groups sit
// a_sbo bytes apart and its K chunks a_lbo bytes apart (the conv kernels' pixel-strided rings).
// ndst: the MMAs rotate over ndst disjoint accumulators (ndst = 1: one dependent chain)
static int tc5_rate(int device, int n, uint32_t a_sbo, uint32_t a_lbo, double *rates, int ndst = 1);
extern "C" int he_microbench_tc5(int device, int n, double *rates) { return tc5_rate(device, n, 0, 0, rates); }
extern "C" int he_microbench_tc5_strided(int device, int n, int a_sbo, int a_lbo, double *rates) {
    return tc5_rate(device, n, (uint32_t)a_sbo, (uint32_t)a_lbo, rates);
}
extern "C" int he_microbench_tc5_indep(int device, int n, int ndst, double *rates) {
    return tc5_rate(device, n, 0, 0, rates, ndst);
}
static int tc5_rate(int device, int n, uint32_t a_sbo, uint32_t a_lbo, double *rates, int ndst) {
    if (n < 16 || n > 256 || n % 16 || !rates || ndst < 1 || ndst > BK / 32 || ndst * n > 256) {
        he_set_error("he_microbench_tc5: N must be a multiple of 16 in [16, 256], ndst * N <= 256, ndst <= 8");
        return HE_EINVAL;
    }
    HE_CHECK_CUDA(cudaSetDevice(device));
    int sms = 0;
    HE_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    if (a_sbo == 0) {
        a_sbo = 128;
        a_lbo = 128 * 16;
    }
    // A spans 16 row groups and 2 * (BK / 32) K chunks
    const int abytes = (int)(((15 * a_sbo + (2 * (BK / 32) - 1) * a_lbo + 128) + 1023) & ~1023u);
    const size_t smem = (size_t)abytes + (size_t)n * BK;
    if (smem > 227 * 1024) {
        he_set_error("he_microbench_tc5: operand layout needs %zu bytes", smem);
        return HE_EINVAL;
    }
    HE_CHECK_CUDA(cudaFuncSetAttribute(k_tc5_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    unsigned long long *cyc;
    HE_CHECK_CUDA(cudaMalloc(&cyc, 8));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    float ms = 0;
    for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(e0);
        k_tc5_rate<<<sms, 128, smem>>>(n, iters, cyc, a_sbo, a_lbo, abytes, ndst);
        cudaEventRecord(e1);
        HE_CHECK_CUDA(cudaEventSynchronize(e1));
    }
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long c = 0;
    HE_CHECK_CUDA(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    const double mmas = (double)iters * (BK / 32);
    rates[0] = (double)sms * mmas * 128.0 * n * 32 / (ms * 1e-3);
    rates[1] = (double)c / mmas;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(cyc);
    HE_CHECK_LAUNCH();
    return HE_OK;
}
