// convsq.cu -- fused feature-major 3x3 conv -> degree-2 activation (square,
// no relinearisation) -> 2x2 pool / global sum, on the tensor cores.
//
// Replaces the chain  conv_mma -> tensor_batch -> add_const -> lincomb_int
// (featuremajor.run_cnn, lazy + deferred plan) with one kernel that never
// materialises the conv output: for config 3's conv1 that map is 16384
// ciphertexts (240 GB at 14 limbs) written and read back once each.
//
// Per CTA: one limb l and one chunk of 8 coefficients, ALL windows of the
// launch.  For every output pixel the conv is an exact int8 GEMM
//     C_d[(comp, j)][(e, m)] = sum_k  byte_d(x_{k, comp, j}) * W_e[m][k]
// (rows: 2 components x 8 coefficients, so the lane holding row j of
// component 0 also holds component 1 -- the square needs both), one
// mma.sync m16n8k32 u8 x s8 per (digit plane d, 32-tap block, weight digit e).
// Digit planes beyond the limb's byte length (5 for 40-bit primes) are
// skipped.  The lane recombines its values exactly (int64 partial sums at
// 2^0 / 2^32 / 2^64, one signed 128-bit total), reduces with ONE Montgomery
// step (y R^-1), squares in the Montgomery domain and accumulates the window
// sums; the window result is scaled back with R^4 and stored as three
// components.  Bit-identical to conv -> tensor -> add_const -> sum, because
// every step is exact arithmetic mod q.
//
// Data path: taps are gathered from global memory one pixel ahead into
// registers (software pipeline), byte-transposed with PRMT and stored
// digit-planar ([d][tap word][row], 24-word rows: conflict-free STS and LDS);
// the weight digits live in registers for the whole kernel.
#include <algorithm>

#include "common.cuh"

namespace {

constexpr int CT = 128;  // 4 warps: MG channel groups x PS pixel streams
constexpr int RS = 24;   // words per tap-word row of a digit plane (16 rows + 8 pad)

struct SqArgs {
    const uint64_t *ptab;       // [npix][Tpad] input ciphertext address of every tap slot (0 = zero tap)
    const int32_t *sched;       // [steps][PS] launch pixel of every (step, stream), -1 = idle
    uint64_t *const *out;       // 3-component outputs, ell limbs
    const uint32_t *bfrag;      // [MG][KB][E][32] uint2 B fragments
    const uint64_t *bias;       // [M][ell] bias * R^-1 mod q (component 0), or nullptr
    const uint64_t *cst;        // [ell] constant added to component 0 of every output, or nullptr
    const uint64_t *r4;         // [ell] R^4 mod q
    const ModConst *mc;
    int M, ell, logN, pool, nwin, steps;
};

// acc += a * b (signed 32 x 32 -> 64, one IMAD.WIDE)
__device__ __forceinline__ void madw(int64_t &acc, int a, int b) {
    asm("mad.wide.s32 %0, %1, %2, %0;" : "+l"(acc) : "r"(a), "r"(b));
}

__device__ __forceinline__ void mma_u8s8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         const uint2 b) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b.x), "r"(b.y));
}

// 4x4 byte transpose: o[d] = byte d of w0..w3 (w0 in the low byte)
__device__ __forceinline__ void tr4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t (&o)[4]) {
    const uint32_t t0 = __byte_perm(w0, w1, 0x5140), t1 = __byte_perm(w2, w3, 0x5140);
    const uint32_t t2 = __byte_perm(w0, w1, 0x7362), t3 = __byte_perm(w2, w3, 0x7362);
    o[0] = __byte_perm(t0, t1, 0x5410);
    o[1] = __byte_perm(t0, t1, 0x7632);
    o[2] = __byte_perm(t2, t3, 0x5410);
    o[3] = __byte_perm(t2, t3, 0x7632);
}

// Montgomery product a b R^-1 (a, b canonical)
__device__ __forceinline__ uint64_t mont(uint64_t a, uint64_t b, const ModConst &c) {
    return redc(mulhi(a, b), a * b, c.q, c.qinv);
}

template <int KB, int MG>
struct Gather {
    static constexpr int PS = 4 / MG;
    static constexpr int KW = KB * 8;
    static constexpr int TASKS = PS * KB;  // per thread: PS streams x 2 comps x KW/4 quads x 32 lanes / CT
    uint64_t v[TASKS][4];

    // task t = tid + CT * i -> (stream, comp, quad of tap words, kw sub, coefficient j)
    __device__ __forceinline__ static void decode(int t, int &ps, int &comp, int &kw, int &j) {
        const int ln = t & 31, rest = t >> 5;
        j = ln & 7;
        const int kq = rest % (KW / 4), r2 = rest / (KW / 4);
        kw = kq * 4 + (ln >> 3);
        comp = r2 & 1;
        ps = r2 >> 1;
    }

    __device__ __forceinline__ void load(const SqArgs &a, int s, int l, size_t coff) {
        const size_t N = (size_t)1 << a.logN;
#pragma unroll
        for (int i = 0; i < TASKS; i++) {
            int ps, comp, kw, j;
            decode(threadIdx.x + CT * i, ps, comp, kw, j);
            const int pix = __ldg(a.sched + s * PS + ps);
            v[i][0] = v[i][1] = v[i][2] = v[i][3] = 0;
            if (pix >= 0) {
                const ulonglong2 *pp = (const ulonglong2 *)(a.ptab + ((size_t)pix * KW + kw) * 4);
                const ulonglong2 p01 = __ldg(pp), p23 = __ldg(pp + 1);
                const size_t off = ((size_t)comp * a.ell + l) * N + coff + j;
                if (p01.x) v[i][0] = __ldg((const uint64_t *)p01.x + off);
                if (p01.y) v[i][1] = __ldg((const uint64_t *)p01.y + off);
                if (p23.x) v[i][2] = __ldg((const uint64_t *)p23.x + off);
                if (p23.y) v[i][3] = __ldg((const uint64_t *)p23.y + off);
            }
        }
    }

    // digit-planar store: word (d, kw, row = comp*8 + j) of the stream's buffer
    __device__ __forceinline__ void store(uint32_t *buf, int nb) const {
        constexpr int PLANE = KW * RS;
#pragma unroll
        for (int i = 0; i < TASKS; i++) {
            int ps, comp, kw, j;
            decode(threadIdx.x + CT * i, ps, comp, kw, j);
            uint32_t lo[4], hi[4];
            tr4((uint32_t)v[i][0], (uint32_t)v[i][1], (uint32_t)v[i][2], (uint32_t)v[i][3], lo);
            tr4((uint32_t)(v[i][0] >> 32), (uint32_t)(v[i][1] >> 32), (uint32_t)(v[i][2] >> 32),
                (uint32_t)(v[i][3] >> 32), hi);
            uint32_t *dst = buf + (size_t)ps * 8 * PLANE + kw * RS + comp * 8 + j;
#pragma unroll
            for (int d = 0; d < 4; d++) dst[d * PLANE] = lo[d];
#pragma unroll
            for (int d = 0; d < 4; d++)
                if (d + 4 < nb) dst[(d + 4) * PLANE] = hi[d];
        }
    }
};

template <int KB, int E, int MG>
__global__ void __launch_bounds__(CT) k_conv_sqsum(const SqArgs a) {
    constexpr int PS = 4 / MG, KW = KB * 8, PLANE = KW * RS, BUF = PS * 8 * PLANE;
    extern __shared__ __align__(16) uint32_t xs[];  // [2][BUF] digit-planar staging
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const int cg = warp % MG, ps = warp / MG;
    const int l = blockIdx.y;
    const size_t N = (size_t)1 << a.logN, coff = (size_t)blockIdx.x * 8;
    const ModConst c = a.mc[l];
    const int nb = c.q < (1ull << 40) ? 5 : (c.q < (1ull << 48) ? 6 : (c.q < (1ull << 56) ? 7 : 8));

    uint2 bw[KB][E];
#pragma unroll
    for (int kb = 0; kb < KB; kb++)
#pragma unroll
        for (int e = 0; e < E; e++) bw[kb][e] = ((const uint2 *)a.bfrag)[((cg * KB + kb) * E + e) * 32 + lane];
    const int m0 = cg * 8 + 2 * tig;  // this lane's channels m0, m0 + 1
    uint64_t bias[2] = {0, 0};
    if (a.bias) {
        if (m0 < a.M) bias[0] = a.bias[(size_t)m0 * a.ell + l];
        if (m0 + 1 < a.M) bias[1] = a.bias[(size_t)(m0 + 1) * a.ell + l];
    }

    Gather<KB, MG> g;
    g.load(a, 0, l, coff);
    g.store(xs, nb);
    __syncthreads();

    // window sums of the products (y R^-1)(y' R^-1), exact 128-bit (hi kept < 2q)
    u128 acc[3][2];
#pragma unroll
    for (int k = 0; k < 3; k++) acc[k][0] = acc[k][1] = u128{0, 0};
    for (int s = 0; s < a.steps; s++) {
        if (s + 1 < a.steps) g.load(a, s + 1, l, coff);
        if (__ldg(a.sched + s * PS + ps) >= 0) {
            const uint32_t *X = xs + (s & 1) * BUF + ps * 8 * PLANE + tig * RS + gid;
            int64_t P[3][4];  // partial sums at 2^0, 2^32, 2^64 for the 4 fragment values
#pragma unroll
            for (int h = 0; h < 3; h++) P[h][0] = P[h][1] = P[h][2] = P[h][3] = 0;
#pragma unroll
            for (int d = 0; d < 8; d++) {
                if (d < nb) {
                    int C[E][4];
#pragma unroll
                    for (int e = 0; e < E; e++) C[e][0] = C[e][1] = C[e][2] = C[e][3] = 0;
#pragma unroll
                    for (int kb = 0; kb < KB; kb++) {
                        const uint32_t *Pd = X + d * PLANE + kb * 8 * RS;
                        const uint32_t a0 = Pd[0], a1 = Pd[8], a2 = Pd[4 * RS], a3 = Pd[4 * RS + 8];
#pragma unroll
                        for (int e = 0; e < E; e++) mma_u8s8(C[e], a0, a1, a2, a3, bw[kb][e]);
                    }
#pragma unroll
                    for (int e = 0; e < E; e++) {
                        const int sh = d + e;
#pragma unroll
                        for (int q = 0; q < 4; q++) madw(P[sh >> 2][q], C[e][q], 1 << (8 * (sh & 3)));
                    }
                }
            }
            // fragment values: q=0,1 -> component 0, channels m0, m0+1; q=2,3 -> component 1
            uint64_t yv[4];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const uint64_t lo = (uint64_t)P[0][q] + ((uint64_t)P[1][q] << 32);
                const uint64_t cy = lo < (uint64_t)P[0][q] ? 1 : 0;
                const int64_t hi = (P[0][q] >> 63) + (P[1][q] >> 32) + (int64_t)cy + P[2][q];
                const uint64_t hic = hi < 0 ? (uint64_t)(hi + (int64_t)c.q) : (uint64_t)hi;  // |hi| < q
                yv[q] = redc(hic, lo, c.q, c.qinv);  // conv * R^-1
            }
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const uint64_t y0 = add_mod(yv[h], bias[h], c.q), y1 = yv[2 + h];
                mac128(acc[0][h], y0, y0);
                mac128(acc[1][h], y0, y1);
                mac128(acc[2][h], y1, y1);
            }
            if ((s & 7) == 7) {  // each product adds < q/16 to hi: fold every 8 pixels
#pragma unroll
                for (int k = 0; k < 3; k++)
#pragma unroll
                    for (int h = 0; h < 2; h++)
                        if (acc[k][h].hi >= c.q) acc[k][h].hi -= c.q;
            }
            if (a.pool && (s & 3) == 3) {  // window complete
                const uint64_t r4 = a.r4[l], cst = a.cst ? a.cst[l] : 0;
                const int win = (s >> 2) * PS + ps;
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int m = m0 + h;
                    if (m < a.M) {
                        uint64_t *o = a.out[(size_t)m * a.nwin + win] + coff + gid;
#pragma unroll
                        for (int k = 0; k < 3; k++) {
                            const uint64_t hi = acc[k][h].hi >= c.q ? acc[k][h].hi - c.q : acc[k][h].hi;
                            uint64_t r = redc(hi, acc[k][h].lo, c.q, c.qinv);  // sum R^-3
                            if (k == 1) r = add_mod(r, r, c.q);
                            uint64_t v = mont(r, r4, c);
                            if (k == 0) v = add_mod(v, cst, c.q);
                            o[((size_t)k * a.ell + l) * N] = v;
                        }
                    }
#pragma unroll
                    for (int k = 0; k < 3; k++) acc[k][h] = u128{0, 0};
                }
            }
        }
        if (s + 1 < a.steps) g.store(xs + ((s + 1) & 1) * BUF, nb);
        __syncthreads();
    }
    if (!a.pool) {  // global sum: reduce, combine the pixel streams, then store
        uint64_t r[3][2];
#pragma unroll
        for (int k = 0; k < 3; k++)
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const uint64_t hi = acc[k][h].hi >= c.q ? acc[k][h].hi - c.q : acc[k][h].hi;
                r[k][h] = redc(hi, acc[k][h].lo, c.q, c.qinv);
            }
        uint64_t *red = (uint64_t *)xs;
        if (PS > 1) {
#pragma unroll
            for (int k = 0; k < 3; k++)
#pragma unroll
                for (int h = 0; h < 2; h++) red[((ps * MG + cg) * 32 + lane) * 6 + k * 2 + h] = r[k][h];
            __syncthreads();
            if (ps == 0)
                for (int o = 1; o < PS; o++)
#pragma unroll
                    for (int k = 0; k < 3; k++)
#pragma unroll
                        for (int h = 0; h < 2; h++)
                            r[k][h] = add_mod(r[k][h], red[((o * MG + cg) * 32 + lane) * 6 + k * 2 + h], c.q);
        }
        if (ps == 0) {
            const uint64_t r4 = a.r4[l], cst = a.cst ? a.cst[l] : 0;
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int m = m0 + h;
                if (m >= a.M) continue;
                uint64_t *o = a.out[m] + coff + gid;
#pragma unroll
                for (int k = 0; k < 3; k++) {
                    const uint64_t rr = k == 1 ? add_mod(r[k][h], r[k][h], c.q) : r[k][h];
                    uint64_t v = mont(rr, r4, c);
                    if (k == 0) v = add_mod(v, cst, c.q);
                    o[((size_t)k * a.ell + l) * N] = v;
                }
            }
        }
    }
}

template <int KB, int E, int MG>
int launch_sq(dim3 grid, size_t smem, cudaStream_t s, const SqArgs &a) {
    if (smem > 48 * 1024)
        HE_CHECK_CUDA(cudaFuncSetAttribute(k_conv_sqsum<KB, E, MG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
    k_conv_sqsum<KB, E, MG><<<grid, CT, smem, s>>>(a);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

template <int KB, int E>
int dispatch_mg(int MG, dim3 grid, size_t smem, cudaStream_t s, const SqArgs &a) {
    if (MG == 1) return launch_sq<KB, E, 1>(grid, smem, s, a);
    if (MG == 2) return launch_sq<KB, E, 2>(grid, smem, s, a);
    return launch_sq<KB, E, 4>(grid, smem, s, a);
}

template <int KB>
int dispatch_e(int E, int MG, dim3 grid, size_t smem, cudaStream_t s, const SqArgs &a) {
    if (E == 1) return dispatch_mg<KB, 1>(MG, grid, smem, s, a);
    if (E == 2) return dispatch_mg<KB, 2>(MG, grid, smem, s, a);
    return dispatch_mg<KB, 3>(MG, grid, smem, s, a);
}

int dispatch_sq(int KB, int E, int MG, dim3 grid, size_t smem, cudaStream_t s, const SqArgs &a) {
    switch (KB) {
        case 1: return dispatch_e<1>(E, MG, grid, smem, s, a);
        case 2: return dispatch_e<2>(E, MG, grid, smem, s, a);
        case 3: return dispatch_e<3>(E, MG, grid, smem, s, a);
        case 4: return dispatch_e<4>(E, MG, grid, smem, s, a);
        case 5: return dispatch_e<5>(E, MG, grid, smem, s, a);
    }
    he_set_error("he_conv_square_sum: no kernel for KB=%d", KB);
    return HE_EINVAL;
}

// balanced signed base-256 digit e of w
inline int digit_s8(int64_t w, int e) {
    for (int i = 0; i < e; i++) {
        int64_t d = (int8_t)(uint8_t)(w & 0xFF);
        w = (w - d) >> 8;
    }
    return (int8_t)(uint8_t)(w & 0xFF);
}

}  // namespace

// Fused 3x3/pad-1 conv (p -> M channels over an H x W map, conv output rows
// [y0, y1)) + square (tensor product, no relinearisation) + window sum:
//   pool = 1: out[m * nwin + (y/2 - y0/2) * (W/2) + x/2] = sum over the 2x2 window
//   pool = 0: out[m] = sum over every pixel of rows [y0, y1)
// of (y0^2, 2 y0 y1, y1^2), y = sum_k weights[m][k] in[tap k] (+ bias[m] on
// component 0), then + cst on component 0.  Inputs in[i*H*W + y*W + x] are 2
// components x ell limbs; outputs 3 components x ell limbs.  Tap order
// k = i*9 + (dy+1)*3 + (dx+1).  Returns HE_EINVAL when a tensor-core bound
// does not hold (9p > 160, M > 32, |w| >= 2^23 or a prime below 2^36).
extern "C" int he_conv_square_sum(he_ctx *c, const uint64_t *const *in, int p, int H, int W, uint64_t *const *out,
                                  int M, int pool, int y0, int y1, const int64_t *weights, const uint64_t *bias,
                                  const uint64_t *cst, int ell, void *stream) {
    if (!c || !in || !out || !weights || p < 1 || H < 1 || W < 1 || M < 1 || ell < 1 || ell > c->L || y0 < 0 ||
        y1 > H || y0 >= y1) {
        he_set_error("he_conv_square_sum: bad arguments");
        return HE_EINVAL;
    }
    if (pool && ((y0 | y1 | H | W) & 1)) {
        he_set_error("he_conv_square_sum: 2x2 pooling needs even H, W and row range");
        return HE_EINVAL;
    }
    const int T = 9 * p, KB = (T + 31) / 32, MG = (M + 7) / 8;
    if (KB > 5 || M > 32 || c->N % 8 || c->N < 8) {
        he_set_error("he_conv_square_sum: 9p=%d taps / M=%d channels beyond the fused kernel", T, M);
        return HE_EINVAL;
    }
    for (int l = 0; l < ell; l++)
        if (c->mod[l] < (1ull << 36)) {
            he_set_error("he_conv_square_sum: prime %d below 2^36", l);
            return HE_EINVAL;
        }
    int64_t wmax = 0;
    for (int i = 0; i < M * T; i++) wmax = std::max<int64_t>(wmax, weights[i] < 0 ? -weights[i] : weights[i]);
    int E = 1;
    int64_t cap = 127;
    while (wmax > cap && E < 3) {
        E++;
        cap = cap * 256 + 127;
    }
    if (wmax > cap) {
        he_set_error("he_conv_square_sum: weights need more than 3 signed byte digits");
        return HE_EINVAL;
    }
    const int MGk = MG == 3 ? 4 : MG;  // kernels exist for 1, 2, 4 channel groups
    // B fragments [MGk][KB][E][lane][2]: b.x = taps kb*32 + tig*4 + 0..3, b.y = +16; column gid -> channel
    std::vector<uint32_t> bf((size_t)MGk * KB * E * 32 * 2, 0);
    for (int cg = 0; cg < MGk; cg++)
        for (int kb = 0; kb < KB; kb++)
            for (int e = 0; e < E; e++)
                for (int lane = 0; lane < 32; lane++) {
                    const int gid = lane >> 2, tig = lane & 3, m = cg * 8 + gid;
                    for (int r = 0; r < 2; r++) {
                        uint32_t reg = 0;
                        for (int i = 0; i < 4; i++) {
                            const int k = kb * 32 + r * 16 + tig * 4 + i;
                            const int dg = (m < M && k < T) ? digit_s8(weights[(size_t)m * T + k], e) : 0;
                            reg |= (uint32_t)(uint8_t)(int8_t)dg << (8 * i);
                        }
                        bf[((((size_t)cg * KB + kb) * E + e) * 32 + lane) * 2 + r] = reg;
                    }
                }
    // per-limb constants: R^4, bias * R^-1
    std::vector<uint64_t> r4(ell), bres(bias ? (size_t)M * ell : 0);
    for (int l = 0; l < ell; l++) {
        const uint64_t q = c->mod[l], R = (uint64_t)(((unsigned __int128)1 << 64) % q);
        const uint64_t R2 = he_h_mulmod(R, R, q);
        r4[l] = he_h_mulmod(R2, R2, q);
        if (cst && cst[l] >= q) {
            he_set_error("he_conv_square_sum: residue not canonical");
            return HE_EINVAL;
        }
        if (bias) {
            const uint64_t Rinv = he_h_inv(R, q);
            for (int m = 0; m < M; m++) {
                if (bias[(size_t)m * ell + l] >= q) {
                    he_set_error("he_conv_square_sum: residue not canonical");
                    return HE_EINVAL;
                }
                bres[(size_t)m * ell + l] = he_h_mulmod(bias[(size_t)m * ell + l], Rinv, q);
            }
        }
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int nwin = pool ? ((y1 - y0) / 2) * (W / 2) : 1;
    const int n_out = pool ? M * nwin : M, npix = (y1 - y0) * W, Tpad = KB * 32, PS = 4 / MGk;
    const int steps = pool ? ((nwin + PS - 1) / PS) * 4 : (npix + PS - 1) / PS;
    // tap address table [launch pixel][tap slot] and the (step, stream) -> pixel schedule
    std::vector<uint64_t> ptab((size_t)npix * Tpad, 0);
    for (int y = y0; y < y1; y++)
        for (int x = 0; x < W; x++)
            for (int k = 0; k < T; k++) {
                const int i = k / 9, t = k % 9, yy = y + t / 3 - 1, xx = x + t % 3 - 1;
                if (yy >= 0 && yy < H && xx >= 0 && xx < W)
                    ptab[((size_t)(y - y0) * W + x) * Tpad + k] = (uint64_t)in[(size_t)i * H * W + yy * W + xx];
            }
    std::vector<int32_t> sched((size_t)steps * PS, -1);
    for (int st = 0; st < steps; st++)
        for (int q = 0; q < PS; q++) {
            if (pool) {
                const int w = (st >> 2) * PS + q, k = st & 3, Wo = W / 2;
                if (w < nwin) sched[(size_t)st * PS + q] = (2 * (w / Wo) + (k >> 1)) * W + 2 * (w % Wo) + (k & 1);
            } else if (st * PS + q < npix) {
                sched[(size_t)st * PS + q] = st * PS + q;
            }
        }
    void **dout = nullptr;
    HE_TRY(he_upload_ptrs((const void *const *)out, n_out, &dout, s));
    const size_t b_bf = bf.size() * 4, b_pt = ptab.size() * 8, b_sc = sched.size() * 4, b_r4 = (size_t)ell * 8,
                 b_b = bres.size() * 8, b_c = cst ? (size_t)ell * 8 : 0;
    char *meta = nullptr;
    HE_TRY(he_scratch_alloc((void **)&meta, b_bf + b_pt + b_sc + b_r4 + b_b + b_c + 128, s));
    size_t off = 0;
    auto carve = [&](size_t bytes) {
        char *p = meta + off;
        off = (off + bytes + 15) & ~(size_t)15;
        return p;
    };
    uint32_t *dbf = (uint32_t *)carve(b_bf);
    uint64_t *dpt = (uint64_t *)carve(b_pt);
    int32_t *dsc = (int32_t *)carve(b_sc);
    uint64_t *dr4 = (uint64_t *)carve(b_r4);
    uint64_t *db = bias ? (uint64_t *)carve(b_b) : nullptr;
    uint64_t *dc = cst ? (uint64_t *)carve(b_c) : nullptr;
    HE_CHECK_CUDA(cudaMemcpyAsync(dbf, bf.data(), b_bf, cudaMemcpyHostToDevice, s));
    HE_CHECK_CUDA(cudaMemcpyAsync(dpt, ptab.data(), b_pt, cudaMemcpyHostToDevice, s));
    HE_CHECK_CUDA(cudaMemcpyAsync(dsc, sched.data(), b_sc, cudaMemcpyHostToDevice, s));
    HE_CHECK_CUDA(cudaMemcpyAsync(dr4, r4.data(), b_r4, cudaMemcpyHostToDevice, s));
    if (db) HE_CHECK_CUDA(cudaMemcpyAsync(db, bres.data(), b_b, cudaMemcpyHostToDevice, s));
    if (dc) HE_CHECK_CUDA(cudaMemcpyAsync(dc, cst, b_c, cudaMemcpyHostToDevice, s));
    SqArgs a;
    a.ptab = dpt;
    a.sched = dsc;
    a.out = (uint64_t *const *)dout;
    a.bfrag = dbf;
    a.bias = db;
    a.cst = dc;
    a.r4 = dr4;
    a.mc = c->d_mc;
    a.M = M;
    a.ell = ell;
    a.logN = c->logN;
    a.pool = pool;
    a.nwin = nwin;
    a.steps = steps;
    const size_t smem = (size_t)2 * PS * 8 * (KB * 8 * RS) * 4;
    dim3 grid((unsigned)(c->N / 8), (unsigned)ell);
    int rc = dispatch_sq(KB, E, MGk, grid, smem, s, a);
    he_scratch_free(meta, s);
    he_scratch_free(dout, s);
    return rc;
}
