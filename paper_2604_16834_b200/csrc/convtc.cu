// convtc.cu -- the fused conv3x3 -> square -> 2x2 pool / global sum of
// featuremajor.run_cnn on the 5th-generation tensor cores (tcgen05).
//
// Same arithmetic contract as convsq_kernel.cuh (exact int8 digit GEMMs, exact
// recombination, FP64 modular products of the window/GAP squares; results
// are canonical residues identical to the conv -> tensor -> add_const -> sum
// chain), restructured for Blackwell:
//
//   * The MMA is tcgen05.mma.cta_group::1.kind::i8 (u8 x s8 -> s32), issued by
//     one thread, accumulators in TMEM.  M = 128 rows = 16 output pixels of one
//     image row x 8 coefficients of one limb; the CTA owns one (limb,
//     8-coefficient chunk) work item at a time (persistent grid).
//   * Inputs are byte-transposed ONCE per input row into a shared-memory ring
//     laid out as UMMA core matrices (8 coefficients x 16 bytes), so every tap
//     is a plain shared-memory descriptor: the 8-row groups of the A operand are
//     consecutive pixels (SBO = pixel stride) and the two 16-byte K chunks of a
//     K step are two taps (LBO = tap distance) -- an implicit GEMM with no
//     im2col copy.  Taps pair as (dy,0)+(dy,1) for dy = 0,1,2, then (0,2)+(1,2)
//     (ring-order dependent: a swapped B variant covers the wrap), then (2,2)
//     with a zero-weight partner: 5 K steps for 9 taps.
//   * Packing P1 (p <= 3 input channels, conv1): one 16-byte K chunk holds all
//     five byte planes of the three channels (byte 5 i + d), and the byte shift
//     goes into N: B[(i,d)][(s,m)] = digit_{s-d}(w[m][i][tap]), so one MMA
//     (N = NSH x 16) produces every shift sum C[s] of all 16 output channels.
//   * Warp roles: warps 0-15 epilogue (four per TMEM lane quarter, 4 channels
//     each: tcgen05.ld -> exact recombination on the integer pipe -> FP64
//     window products -> window sums -> stores), warps 16-18 producers (128-bit
//     global loads -> PRMT byte packing -> shared ring), warp 19 TMEM allocator
//     + MMA issuer.  After the role split the epilogue warpgroups raise their
//     register limit and the producer / MMA warpgroup lowers its own
//     (setmaxnreg, RegSplit).  On B200 the FP64 pipe and the tensor core share
//     one issue resource (scripts/mb/mb_fp64_vs_mma.cu), so what bounds these
//     kernels is MMA cycles + FP64 cycles: FP64 work is kept to the window
//     products (recombine_fold does the rest in integers).  mbarriers
//     connect them: ring row full (producers -> MMA), ring row empty
//     (tcgen05.commit -> producers), TMEM slot full (commit -> epilogue), TMEM
//     slot empty (epilogue -> MMA).  Four TMEM slots of 128 columns (one per
//     (row step, component)) let the MMAs of the next components run while
//     the epilogue does its FP64 work.
#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "ntt_core.cuh"  // u2d / d2u / fmulmod / fcanon
#include "tc5.cuh"

namespace convtc {

constexpr int P1_NCOL = 128;     // P1 MMA N: 4 channel groups x 32 columns (NSH x 4 used)
constexpr int NB = 5;            // byte planes of a 40-bit residue
constexpr int EPI_WARPS = 16;    // warps 0-15: four per TMEM lane quarter, CPT channels each
constexpr int CPT = 4;           // output channels per epilogue thread
constexpr int PROD_WARPS = 3;    // warps 16-18
constexpr int MMA_WARP = 19;
constexpr int THREADS = 32 * 20;  // 5 warps per SM sub-partition: 96 registers per thread
// setmaxnreg: the four epilogue warpgroups grow to EPI registers per thread, the producer / MMA
// warpgroup shrinks to AUX; 512 * EPI + 128 * AUX <= 640 * 96 (the launch allocation), or the
// epilogue's request never completes
template <int EPI, int AUX>
struct RegSplit {
    static_assert(512 * EPI + 128 * AUX <= 640 * 96 && EPI % 8 == 0 && AUX % 8 == 0 && AUX >= 24, "register pool");
    static __device__ __forceinline__ void epilogue() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(EPI)); }
    static __device__ __forceinline__ void aux() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(AUX)); }
};
#ifndef P1_EPI_REGS
#define P1_EPI_REGS 104
#define P1_AUX_REGS 64
#endif
#ifndef P16_EPI_REGS
#define P16_EPI_REGS 112  // planar carry: the producers only issue bulk copies
#define P16_AUX_REGS 32
#endif
using P1Regs = RegSplit<P1_EPI_REGS, P1_AUX_REGS>;
using P16Regs = RegSplit<104, 64>;  // pointer-list inputs: the producers transpose in registers
using P16RegsPlanar = RegSplit<P16_EPI_REGS, P16_AUX_REGS>;
constexpr int NSLOT = 4;         // TMEM accumulator slots (128 columns each)
constexpr int MC = 16;           // output channels per CTA

struct TcArgs {
    const uint64_t *const *in;   // [p*H*W] input ciphertexts (NCI components x ell limbs)
    const uint64_t *ibase;       // input i = ibase + ioff[i] * 32 words (256-byte units; staged in shared memory)
    const uint32_t *ioff;
    uint64_t *const *out;        // pool: [M][nwin] (3 components); GAP: [M]
    uint64_t *obase;             // != nullptr: out[k] = obase + k * ostride (one batch allocation)
    long long ostride;           // elements
    const uint8_t *btiles;       // B tiles (global), copied to shared memory once per CTA
    const double *biasd;         // [MC][ell] plain-domain bias (component 0), canonical
    const uint64_t *cst;         // [ell] constant added to component 0 of every output (or nullptr)
    const ModConst *mc;
    const int32_t *limbs;        // [nlimbs] limb of limb-index
    int nlimbs, ell, logN, p, H, W, M, y0, y1, nwin, nitems;
    int btile_bytes, nshift;     // bytes per B tile, shift sums (N = nshift * 16)
    unsigned long long *prof;    // != nullptr: per-role cycle counters (he_convtc_profile)
    int exp;                     // diagnostics (CONVTC_EXP): 1 = epilogue skips the products
    // planar carry (conv1 -> conv2 of the config-3 plan): layout [limb][N/8 coefficient chunks]
    // [y][x][component][byte plane][8 coefficients x 16 channels] -- conv2's ring row layout, so
    // one input row of one (limb, chunk) is a contiguous (W x 1920)-byte block
    uint8_t *pl_out;             // P1: pooled outputs written planar (16 channels, H/2 x W/2)
    const uint8_t *pl_in;        // P16: inputs read planar (p = 16 channels, H x W)
};

// role timing (he_convtc_profile): [0] producer wait-empty, [1] producer total, [2] MMA wait-full,
// [3] MMA wait-dempty, [4] MMA total, [5] epilogue wait-dfull, [6] epilogue total (one sampled
// thread per role, summed over CTAs)
#define PWAIT(slot, call)                                       \
    do {                                                        \
        const long long _t0 = prof_on ? clock64() : 0;          \
        call;                                                   \
        if (prof_on) pc[slot] += clock64() - _t0;               \
    } while (0)

// diagnostic build (-DCONVTC_PHASES, scripts/gpu): only the sampled epilogue thread reports, and
// counters [0], [2], [3] hold its TMEM-load, recombination and window-product cycles
#ifdef CONVTC_PHASES
#define PH_ONLY_EPI (threadIdx.x == 0)
#define PH_START() long long tph = clock64()
#define PH(i)                                  \
    if (prof_on) {                             \
        const long long _n = clock64();        \
        pc[i] += _n - tph;                     \
        tph = _n;                              \
    }
#define PH_RESET() \
    if (prof_on) tph = clock64()
#else
#define PH_ONLY_EPI true
#define PH_START()
#define PH(i)
#define PH_RESET()
#endif

// ---------------------------------------------------------------- shared layout
// ring row: (W + 3) pixel slots (halo, W pixels, halo, pad) x NCI components x
// 128 bytes (8 coefficients x 16-byte chunk); RR rows
template <int NCI>
struct P1Layout {
    static constexpr int PS = NCI * 128;  // pixel stride (bytes) = A operand SBO
    static constexpr int RR = 6;          // ring rows (4 in use for a pool step + 2 prefetched)
};

__device__ __forceinline__ int64_t madw(int64_t acc, int a, int b) {
    asm("mad.wide.s32 %0, %1, %2, %0;" : "+l"(acc) : "r"(a), "r"(b));
    return acc;
}

// K independent FP64 modular products issued stage by stage (the K dependency chains
// interleave in program order instead of running one after the other); each lane of the
// batch computes exactly fmulmod(a, b)
template <int K>
__device__ __forceinline__ void fmulmod_v(const double (&a)[K], const double (&b)[K], double (&r)[K], double q,
                                          double qi) {
    double h[K], e[K];
#pragma unroll
    for (int k = 0; k < K; k++) h[k] = a[k] * b[k];
#pragma unroll
    for (int k = 0; k < K; k++) e[k] = rint(h[k] * qi);
#pragma unroll
    for (int k = 0; k < K; k++) r[k] = fma(a[k], b[k], -h[k]);
#pragma unroll
    for (int k = 0; k < K; k++) h[k] = fma(-e[k], q, h[k]);
#pragma unroll
    for (int k = 0; k < K; k++) r[k] = h[k] + r[k];
}
// Recombination on the INTEGER pipe.  On B200 the FP64 pipe and the tensor core share one
// issue resource (scripts/mb/mb_fp64_vs_mma.cu: a running tcgen05.mma stream cuts FP64
// throughput 3x and is itself slowed), so every FP64 instruction the epilogue does not issue is
// tensor time.  With kq = 2^40 - q < 2^25 (the 40-bit NTT primes are 2^40 - j 2N + 1, j small):
//   S = sum_{s<6} C[s] 2^(8s) (int64, |S| < 2^62.2) = S_hi 2^40 + S_lo, 0 <= S_lo < 2^40
//   y = S_lo + (S_hi + 2^8 C[6]) kq  == S + C[6] 2^48 (mod q)
// and, with a seventh shift sum, one more fold; the result is an exact integer |y| < 2^47,
// congruent to recombine<NSH>() (which differs from it by a multiple of q).
template <int NSH>
__device__ __forceinline__ double recombine_fold(const int (&C)[NSH], int kq) {
    static_assert(NSH >= 5 && NSH <= 7, "40-bit limbs: 5 byte planes, 1-3 weight digits");
    constexpr int64_t M40 = (1ll << 40) - 1;
    const int q0 = C[0] + C[1] * 256, q1 = C[2] + C[3] * 256;
    const int q2 = NSH > 5 ? C[4] + C[NSH > 5 ? 5 : 4] * 256 : C[4];
    const int64_t S = (int64_t)q0 + ((int64_t)q1 << 16) + ((int64_t)q2 << 32);
    int hi = (int)(S >> 40);  // |hi| < 2^22.2
    if (NSH > 6) hi += C[NSH > 6 ? 6 : 4] * 256;  // |hi| < 2^30.2
    int64_t y = madw(S & M40, hi, kq);
    if (NSH > 6) y = madw(y & M40, (int)(y >> 40), kq);  // |y >> 40| < 2^15
    return __longlong_as_double(0x4338000000000000ll + y) - 6755399441055744.0;
}
// recombination of K channels at once
template <int NSH, int K>
__device__ __forceinline__ void recombine_v(const int (&C)[K][NSH], int kq, double (&y)[K]) {
#pragma unroll
    for (int k = 0; k < K; k++) y[k] = recombine_fold<NSH>(C[k], kq);
}

// exact integer-valued double |x| < 2^50 -> canonical residue (magic-constant
// rounding: |x / q| < 2^14, so x q^-1 + 1.5 2^52 rounds to the nearest integer)
__device__ __forceinline__ uint64_t canon_fast(double x, double q, double qi) {
    const double e = fma(x, qi, 6755399441055744.0) - 6755399441055744.0;
    double r = fma(-e, q, x);  // exact, in (-q, q)
    r = r < 0.0 ? r + q : r;
    return (uint64_t)(__double_as_longlong(r + 4503599627370496.0) - 0x4330000000000000ll);
}

__device__ __forceinline__ void ldg128(const uint64_t *p, uint64_t &a, uint64_t &b) {
    asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d));
}

// P1 chunk of one coefficient: byte 5 i + d = byte d of channel i (i < 3, d < 5), byte 15 = 0
__device__ __forceinline__ void pack_p1(uint64_t v0, uint64_t v1, uint64_t v2, uint32_t (&w)[4]) {
    const uint32_t l0 = (uint32_t)v0, h0 = (uint32_t)(v0 >> 32);
    const uint32_t l1 = (uint32_t)v1, h1 = (uint32_t)(v1 >> 32);
    const uint32_t l2 = (uint32_t)v2, h2 = (uint32_t)(v2 >> 32);
    w[0] = l0;
    w[1] = __byte_perm(h0, l1, 0x6540);                        // h0.b0, l1.b0, l1.b1, l1.b2
    w[2] = __byte_perm(__byte_perm(l1, h1, 0x0043), l2, 0x5410);  // l1.b3, h1.b0 | l2.b0, l2.b1
    w[3] = __byte_perm(l2, h2, 0x0432) & 0x00FFFFFFu;          // l2.b2, l2.b3, h2.b0, 0
}

// ---------------------------------------------------------------- the P1 kernel (conv1 shape)
// NCI = 2 input components, p <= 3 channels, MC = 16 output channels, 2x2 pool, W % 16 == 0.
template <int NSH>
__global__ void __launch_bounds__(THREADS, 1) k_convtc_p1_pool(const TcArgs a) {
    constexpr int NCI = 2;
    using LY = P1Layout<NCI>;
    constexpr int PS = LY::PS, RR = LY::RR;
    // MMA N = 128: column block cg*32 + s*4 + mm holds shift sum s of channel 4 cg + mm, so
    // an epilogue thread's NSH x 4 sums are contiguous (one x16 + one x8/x4 TMEM load)
    constexpr int NCOL = P1_NCOL;
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar_full[RR], bar_empty[RR], bar_dfull[NSLOT], bar_dempty[NSLOT], bar_b;
    __shared__ uint32_t taddr_s;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int W = a.W, H = a.H, XB = W / 16;
    const int RS = (W + 3) * PS;  // ring row stride
    uint8_t *ring = smem;
    uint8_t *bsm = smem + (size_t)RR * RS;
    // input address table (32-bit offsets), staged once: every work item reads the same ciphertexts
    uint32_t *ptab = (uint32_t *)(bsm + 6 * (size_t)a.btile_bytes);
    for (int i = threadIdx.x; i < a.p * a.H * a.W; i += THREADS) ptab[i] = a.ioff[i];
    const size_t N = (size_t)1 << a.logN;
    const int nchunk = (int)(N / 8);
    const int rows_in = a.y1 - a.y0 + 2;
    const int npairs = (a.y1 - a.y0) / 2;

    if (threadIdx.x == 0) {
        for (int i = 0; i < RR; i++) {
            tc5::mbar_init(&bar_full[i], PROD_WARPS * 32);
            tc5::mbar_init(&bar_empty[i], 1);
        }
        for (int i = 0; i < NSLOT; i++) {
            tc5::mbar_init(&bar_dfull[i], 1);
            tc5::mbar_init(&bar_dempty[i], EPI_WARPS * 32);
        }
        tc5::mbar_init(&bar_b, 1);
        tc5::mbar_fence_init();
    }
    // zero the whole ring once: halo pixel slots are never written again
    for (int i = threadIdx.x * 16; i < RR * RS; i += THREADS * 16) *(uint4 *)(ring + i) = make_uint4(0, 0, 0, 0);
    // B tiles: one bulk copy per CTA (TMA engine, completes on bar_b)
    if (threadIdx.x == 0) {
        tc5::mbar_arrive_expect_tx(&bar_b, (uint32_t)(6 * a.btile_bytes));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         tc5::smem_u32(bsm)),
                     "l"(a.btiles), "r"((uint32_t)(6 * a.btile_bytes)), "r"(tc5::smem_u32(&bar_b))
                     : "memory");
    }
    if (warp == MMA_WARP) tc5::tmem_alloc<512>(&taddr_s);
    tc5::fence_async_smem();
    tc5::tc_fence_before();
    __syncthreads();
    tc5::tc_fence_after();
    const uint32_t tmem = taddr_s;
    const bool prof_on = a.prof && PH_ONLY_EPI && (threadIdx.x == 0 || threadIdx.x == EPI_WARPS * 32 || threadIdx.x == MMA_WARP * 32);
    long long pc[7] = {0, 0, 0, 0, 0, 0, 0};
    const long long t_start = clock64();

    if (warp >= EPI_WARPS && warp < EPI_WARPS + PROD_WARPS) {
        // ======================= producers: input rows -> packed ring rows
        P1Regs::aux();
        const int pt = threadIdx.x - EPI_WARPS * 32;  // 0..95
        constexpr int PT = PROD_WARPS * 32;
        const uint32_t ring_s = tc5::smem_u32(ring);
        const int ntask = W * NCI * 4;  // (pixel, component, coefficient pair); <= 3 per thread for W <= 32
        constexpr int TPT = 3;
        int k = 0;
        for (int item = blockIdx.x; item < a.nitems; item += gridDim.x, k++) {
            const int l = a.limbs[item / nchunk];
            const size_t coff = (size_t)(item % nchunk) * 8;
            for (int rr = 0; rr < rows_in; rr++) {
                const int G = k * rows_in + rr, slot = G % RR, use = G / RR;
                if (use > 0) {  // one warp polls the slot barrier, the others park on a named barrier
                    if (warp == EPI_WARPS) PWAIT(0, tc5::mbar_wait(&bar_empty[slot], (use - 1) & 1));
                    asm volatile("bar.sync 1, %0;" ::"n"(PROD_WARPS * 32) : "memory");
                }
                const int y = a.y0 - 1 + rr;
                const bool inside = y >= 0 && y < H;
                const uint32_t rbase = ring_s + slot * RS;
                for (int t0 = pt; t0 < ntask; t0 += TPT * PT) {
                    // every load of the batch is in flight before the first pack
                    uint64_t v[TPT][3][2];
#pragma unroll
                    for (int u = 0; u < TPT; u++) {
                        const int t = t0 + u * PT;
                        const int jp = t & 3, c = (t >> 2) % NCI, x = (t >> 2) / NCI;
#pragma unroll
                        for (int i = 0; i < 3; i++) {
                            v[u][i][0] = v[u][i][1] = 0;
                            if (t < ntask && inside && i < a.p) {
                                const uint64_t *src = a.ibase + (size_t)ptab[i * H * W + y * W + x] * 32;
                                ldg128(src + ((size_t)c * a.ell + l) * N + coff + 2 * jp, v[u][i][0], v[u][i][1]);
                            }
                        }
                    }
#pragma unroll
                    for (int u = 0; u < TPT; u++) {
                        const int t = t0 + u * PT;
                        if (t >= ntask) break;
                        const int jp = t & 3, c = (t >> 2) % NCI, x = (t >> 2) / NCI;
                        const uint32_t dst = rbase + (x + 1) * PS + c * 128 + jp * 32;
#pragma unroll
                        for (int h = 0; h < 2; h++) {
                            uint32_t w[4];
                            pack_p1(v[u][0][h], v[u][1][h], v[u][2][h], w);
                            sts128(dst + h * 16, w[0], w[1], w[2], w[3]);
                        }
                    }
                }
                tc5::fence_async_smem();
                tc5::mbar_arrive(&bar_full[slot]);
            }
        }
    } else if (warp == MMA_WARP) {
        P1Regs::aux();
        // ======================= MMA issuer
        if (lane == 0) {
            tc5::mbar_wait(&bar_b, 0);
            const uint32_t ring_s = tc5::smem_u32(ring), b_s = tc5::smem_u32(bsm);
            const uint32_t idesc = tc5::idesc_u8s8(128, NCOL);
            const uint32_t blbo = NCOL * 16;  // B: chunk 0 rows then chunk 1 rows
            const uint32_t ahi = tc5::sdesc_hi(PS), lps = tc5::sdesc_lbo(PS);
            uint64_t bd[6];
            for (int t = 0; t < 6; t++) bd[t] = tc5::sdesc(b_s + t * a.btile_bytes, blbo, 128);
            int k = 0, S = 0;
            for (int item = blockIdx.x; item < a.nitems; item += gridDim.x, k++) {
                const int Gb = k * rows_in;  // ring index of input row y0 - 1
                auto slot_of = [&](int y) { return (Gb + (y - (a.y0 - 1))) % RR; };
                for (int pr = 0; pr < npairs; pr++) {
                    const int yp = a.y0 + 2 * pr;
                    // rows yp-1 .. yp+2 must be resident
                    for (int y = yp - 1; y <= yp + 2; y++) {
                        const int G = Gb + (y - (a.y0 - 1));
                        PWAIT(2, tc5::mbar_wait(&bar_full[G % RR], (G / RR) & 1));
                    }
                    tc5::tc_fence_after();
                    for (int xb = 0; xb < XB; xb++)
                        for (int dyb = 0; dyb < 2; dyb++) {
                            const int y = yp + dyb;
                            // descriptor low words: (address >> 4) | LBO field
                            const uint32_t r0 = (ring_s + slot_of(y - 1) * RS) >> 4,
                                           r1 = (ring_s + slot_of(y) * RS) >> 4,
                                           r2 = (ring_s + slot_of(y + 1) * RS) >> 4;
                            const uint32_t xo = (uint32_t)(xb * 16) * (PS >> 4);
                            const uint32_t lv = r1 > r0 ? tc5::sdesc_lbo((r1 - r0) << 4) : tc5::sdesc_lbo((r0 - r1) << 4);
                            const uint32_t a3 = (r1 > r0 ? r0 : r1) + 2 * (PS >> 4) + lv;
                            const uint64_t b3 = r1 > r0 ? bd[3] : bd[5];
                            for (int c = 0; c < NCI; c++, S++) {
                                const int ds = S % NSLOT;
                                if (S >= NSLOT) PWAIT(3, tc5::mbar_wait(&bar_dempty[ds], ((S / NSLOT) - 1) & 1));
                                tc5::tc_fence_after();
                                const uint32_t d = tmem + (uint32_t)ds * 128;
                                const uint32_t co = xo + c * (128 >> 4);
                                // K steps: (dy,0)+(dy,1) for dy = 0..2; (0,2)+(1,2); (2,2)+pad
                                tc5::mma_i8_set(d, tc5::sdesc_hl(ahi, r0 + co + lps), bd[0], idesc);
                                tc5::mma_i8_acc(d, tc5::sdesc_hl(ahi, r1 + co + lps), bd[1], idesc);
                                tc5::mma_i8_acc(d, tc5::sdesc_hl(ahi, r2 + co + lps), bd[2], idesc);
                                tc5::mma_i8_acc(d, tc5::sdesc_hl(ahi, a3 + co), b3, idesc);
                                tc5::mma_i8_acc(d, tc5::sdesc_hl(ahi, r2 + co + 2 * (PS >> 4) + lps), bd[4], idesc);
                                tc5::tc_commit(&bar_dfull[ds]);
                            }
                        }
                    // rows yp-1, yp are not read by later pairs
                    tc5::tc_commit(&bar_empty[slot_of(yp - 1)]);
                    tc5::tc_commit(&bar_empty[slot_of(yp)]);
                }
                tc5::tc_commit(&bar_empty[slot_of(a.y1 - 1)]);
                tc5::tc_commit(&bar_empty[slot_of(a.y1)]);
            }
        }
        __syncwarp();
    } else if (warp < EPI_WARPS) {
        // ======================= epilogue
        P1Regs::epilogue();
        const int qd = warp & 3, cg = warp >> 2;  // TMEM lane quarter, channel group (CPT channels)
        const int row = qd * 32 + lane, xl = row >> 3, j = row & 7;
        const uint32_t tq = tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(cg * 32);
        const int par = xl & 1;  // window partners (x, x+1) split the stores: par 0 -> comps 0, 2; par 1 -> comp 1
        int k = 0, S = 0;
        for (int item = blockIdx.x; item < a.nitems; item += gridDim.x, k++) {
            const int li = item / nchunk, l = a.limbs[li];
            const size_t coff = (size_t)(item % nchunk) * 8;
            const ModConst c = a.mc[l];
            const int kq = (int)(1099511627776.0 - c.qd);  // 2^40 - q < 2^25 (checked by the launcher)
            const double cstd = a.cst ? (double)a.cst[l] : 0.0;  // canonical, < 2^40
            double biasd[CPT];
#pragma unroll
            for (int m = 0; m < CPT; m++) biasd[m] = a.biasd[(size_t)(cg * CPT + m) * a.ell + l];
            const size_t lo = (size_t)l * N + coff + j;  // limb / coefficient offset inside an output
            const size_t cs = (size_t)a.ell * N;         // component stride
            uint64_t *obm[CPT];                          // strided outputs: window 0 of channel cg CPT + m
#pragma unroll
            for (int m = 0; m < CPT; m++)
                obm[m] = a.obase ? a.obase + (size_t)(cg * CPT + m) * a.nwin * a.ostride + lo : nullptr;
            PH_START();
            for (int pr = 0; pr < npairs; pr++) {
                for (int xb = 0; xb < XB; xb++) {
                    double acc[CPT][3];
#pragma unroll
                    for (int m = 0; m < CPT; m++) acc[m][0] = acc[m][1] = acc[m][2] = 0.0;
                    for (int dyb = 0; dyb < 2; dyb++) {
                        double yv[2][CPT];
#pragma unroll
                        for (int cc = 0; cc < NCI; cc++, S++) {
                            const int ds = S % NSLOT;
                            PWAIT(5, tc5::mbar_wait(&bar_dfull[ds], (S / NSLOT) & 1));
                            PH_RESET();
                            tc5::tc_fence_after();
                            int C[CPT][NSH];
                            const uint32_t ta = tq + (uint32_t)ds * 128;
                            uint32_t r0[16], r1[8], r2[4];
                            tc5::tld16(ta, r0);
                            if constexpr (NSH >= 6) tc5::tld8(ta + 16, r1);
                            if constexpr (NSH == 5) tc5::tld4(ta + 16, r2);
                            if constexpr (NSH == 7) tc5::tld4(ta + 24, r2);
                            tc5::tld_wait();
#pragma unroll
                            for (int s2 = 0; s2 < NSH; s2++)
#pragma unroll
                                for (int m = 0; m < CPT; m++)
                                    C[m][s2] = (int)(s2 < 4 ? r0[s2 * 4 + m]
                                                     : NSH == 5 ? r2[m]
                                                     : s2 < 6 ? r1[(s2 - 4) * 4 + m] : r2[m]);
                            tc5::tc_fence_before();
                            tc5::mbar_arrive(&bar_dempty[ds]);
                            PH(0);
                            recombine_v<NSH, CPT>(C, kq, yv[cc]);
                            PH(2);
                        }
                        {
                            double d0[CPT], t[CPT];
#pragma unroll
                            for (int m = 0; m < CPT; m++) d0[m] = yv[0][m] + biasd[m];
                            fmulmod_v<CPT>(d0, d0, t, c.qd, c.qid);
#pragma unroll
                            for (int m = 0; m < CPT; m++) acc[m][0] += t[m];
                            fmulmod_v<CPT>(d0, yv[1], t, c.qd, c.qid);
#pragma unroll
                            for (int m = 0; m < CPT; m++) acc[m][1] += t[m];
                            fmulmod_v<CPT>(yv[1], yv[1], t, c.qd, c.qid);
#pragma unroll
                            for (int m = 0; m < CPT; m++) acc[m][2] += t[m];
                        }
                        PH(3);
                    }
                    // window = this pixel + its x-neighbour (lane ^ 8), rows yp, yp+1.  Reduce-scatter
                    // over the pair: lane par keeps channels 2 par, 2 par + 1 of its window (no
                    // divergent finalisation).  The constant (added once per window) and the factor 2
                    // of the cross term are folded into the exact FP64 sums (|sum| < 2^50).
                    const int x = xb * 16 + xl;
                    const int win = pr * (W / 2) + x / 2;
                    if (a.pl_out) {  // planar carry: 5 byte planes, channels (2 par + h) as 16-bit pairs
                        uint64_t v[2][3];
#pragma unroll
                        for (int h = 0; h < 2; h++)
#pragma unroll
                            for (int s2 = 0; s2 < 3; s2++) {
                                const double mine = par ? acc[2 + h][s2] : acc[h][s2];
                                const double give = par ? acc[h][s2] : acc[2 + h][s2];
                                const double keep = mine + __shfl_xor_sync(0xffffffffu, give, 8);
                                v[h][s2] = canon_fast(s2 == 0 ? keep + cstd : s2 == 1 ? 2.0 * keep : keep, c.qd, c.qid);
                            }
                        PH(1);
                        const int H2 = a.H >> 1, W2 = W >> 1, y2 = (a.y0 >> 1) + pr, x2 = x >> 1;
                        uint8_t *pb = a.pl_out +
                                      ((((size_t)l * nchunk + (size_t)(item % nchunk)) * H2 + y2) * W2 + x2) * (3 * 5 * 128) +
                                      j * 16 + cg * CPT + 2 * par;
#pragma unroll
                        for (int s2 = 0; s2 < 3; s2++) {
                            // byte d of both channels -> one 16-bit store per byte plane (one PRMT each)
                            const uint32_t al = (uint32_t)v[0][s2], ah = (uint32_t)(v[0][s2] >> 32);
                            const uint32_t bl = (uint32_t)v[1][s2], bh = (uint32_t)(v[1][s2] >> 32);
#pragma unroll
                            for (int d = 0; d < 5; d++) {
                                const uint32_t u = d < 4 ? __byte_perm(al, bl, 0x0040 + 0x0011 * d)
                                                         : __byte_perm(ah, bh, 0x0040);
                                *(unsigned short *)(pb + (s2 * 5 + d) * 128) = (unsigned short)u;
                            }
                        }
                        PH(4);
                    } else
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        double keep[3];
#pragma unroll
                        for (int s2 = 0; s2 < 3; s2++) {
                            const double mine = par ? acc[2 + h][s2] : acc[h][s2];
                            const double give = par ? acc[h][s2] : acc[2 + h][s2];
                            keep[s2] = mine + __shfl_xor_sync(0xffffffffu, give, 8);
                        }
                        const int mo = cg * CPT + 2 * par + h;
                        if (mo < a.M) {
                            uint64_t *o = a.obase ? (par ? obm[2 + h] : obm[h]) + (size_t)win * a.ostride
                                                  : a.out[(size_t)mo * a.nwin + win] + lo;
                            o[0] = canon_fast(keep[0] + cstd, c.qd, c.qid);
                            o[cs] = canon_fast(2.0 * keep[1], c.qd, c.qid);
                            o[2 * cs] = canon_fast(keep[2], c.qd, c.qid);
                        }
                    }
                }
            }
        }
    }
    if (prof_on) {
        const int tot = threadIdx.x == 0 ? 6 : threadIdx.x == EPI_WARPS * 32 ? 1 : 4;
        pc[tot] = clock64() - t_start;
        for (int i = 0; i < 7; i++)
            if (pc[i]) atomicAdd(a.prof + i, (unsigned long long)pc[i]);
    }
    tc5::tc_fence_before();
    __syncthreads();
    if (warp == MMA_WARP) tc5::tmem_free<512>(tmem);
}

// ---------------------------------------------------------------- the P16 kernel (conv2 shape)
// NCI = 3 input components (carried, unrelinearised squares), p = 16 input channels,
// MC = 16 output channels per CTA (blockIdx parity selects the channel half), W = 16,
// global sum over rows [y0, y1) -> 5-component outputs.
//
// Packing P16: one 16-byte K chunk = byte plane d of the 16 input channels at one
// pixel (core matrix = 8 coefficients x 16 channels).  Planes are multiplied
// separately; the byte shift lives in the accumulator's TMEM COLUMN offset: plane
// d's MMA (N = 32 = 2 weight digits x 16 channels) writes columns d*16 .. d*16+31,
// i.e. shift blocks d and d+1, so the shift sums accumulate in place.  The first
// MMA of a (row step, component) uses an N = 96 B tile whose blocks 2..5 are zero,
// which initialises all six shift blocks (no TMEM clearing pass).
struct P16Layout {
    static constexpr int NCI = 3, PLANES = 5;
    static constexpr int PS = NCI * PLANES * 128;  // pixel stride (bytes)
    static constexpr int RR = 4;                   // ring rows (3 in use + 1; plus 2 half rows staged)
    static constexpr int STG = 2 * 8 * NCI * 16 * 64;  // cp.async staging: 2 half rows
    static constexpr int TB = 32 * 32;             // B tile (N = 32 rows x 32 bytes)
    static constexpr int TB0 = 96 * 32;            // zero-extended K step 0 (N = 96)
    static constexpr int TBP = 48 * 32;            // tap 8 of planes d and d + 1 in one K step (N = 48)
    static constexpr int BBYTES = 6 * TB + TB0 + TBP;
};

__device__ __forceinline__ void tr4b(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t (&o)[4]) {
    const uint32_t t0 = __byte_perm(w0, w1, 0x5140), t1 = __byte_perm(w2, w3, 0x5140);
    const uint32_t t2 = __byte_perm(w0, w1, 0x7362), t3 = __byte_perm(w2, w3, 0x7362);
    o[0] = __byte_perm(t0, t1, 0x5410);
    o[1] = __byte_perm(t0, t1, 0x7632);
    o[2] = __byte_perm(t2, t3, 0x5410);
    o[3] = __byte_perm(t2, t3, 0x7632);
}

template <bool PLANAR>
__global__ void __launch_bounds__(THREADS, 1) k_convtc_p16_gap(const TcArgs a) {
    using Regs = std::conditional_t<PLANAR, P16RegsPlanar, P16Regs>;
    using LY = P16Layout;
    constexpr int NCI = 3, PS = LY::PS, RR = LY::RR, NSH = 6;
    constexpr int NSL = 5, SLC = 96;  // TMEM slots: 5 x 96 columns (one per (row step, component))
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar_full[RR], bar_empty[RR], bar_dfull[NSL], bar_dempty[NSL], bar_b;
    __shared__ uint32_t taddr_s;
    __shared__ unsigned int fin_cnt[4];  // planar: arrivals of a channel group's four lane quarters

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int W = a.W, H = a.H;
    const int RS = (W + 3) * PS;
    uint8_t *ring = smem;
    uint8_t *bsm = smem + (size_t)RR * RS;
    double *red = (double *)(bsm + LY::BBYTES);        // [4 cg][4 m][5 s][8 j] cross-quarter GAP sums
    uint32_t *ptab = (uint32_t *)(red + (PLANAR ? 16 : 4) * CPT * 5 * 8);  // input offsets (256-byte units)
    uint8_t *stg = (uint8_t *)(((uintptr_t)(ptab + a.p * a.H * a.W) + 127) & ~(uintptr_t)127);  // 2 x 24 KB staging
    if (!PLANAR)
        for (int i = threadIdx.x; i < a.p * a.H * a.W; i += THREADS) ptab[i] = a.ioff[i];
    const size_t N = (size_t)1 << a.logN;
    const int nchunk = (int)(N / 8);
    const int rows_in = a.y1 - a.y0 + 2;
    const int nrows = a.y1 - a.y0;
    const int half = blockIdx.x & 1;  // grid is even: a CTA always owns the same channel half

    if (threadIdx.x == 0) {
        for (int i = 0; i < RR; i++) {
            tc5::mbar_init(&bar_full[i], PLANAR ? 1 : PROD_WARPS * 32);
            tc5::mbar_init(&bar_empty[i], 1);
        }
        for (int i = 0; i < NSL; i++) {
            tc5::mbar_init(&bar_dfull[i], 1);
            tc5::mbar_init(&bar_dempty[i], EPI_WARPS * 32);
        }
        tc5::mbar_init(&bar_b, 1);
        tc5::mbar_fence_init();
        fin_cnt[0] = fin_cnt[1] = fin_cnt[2] = fin_cnt[3] = 0;
    }
    for (int i = threadIdx.x * 16; i < RR * RS; i += THREADS * 16) *(uint4 *)(ring + i) = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        tc5::mbar_arrive_expect_tx(&bar_b, (uint32_t)LY::BBYTES);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         tc5::smem_u32(bsm)),
                     "l"(a.btiles + (size_t)half * LY::BBYTES), "r"((uint32_t)LY::BBYTES), "r"(tc5::smem_u32(&bar_b))
                     : "memory");
    }
    if (warp == MMA_WARP) tc5::tmem_alloc<512>(&taddr_s);
    tc5::fence_async_smem();
    tc5::tc_fence_before();
    __syncthreads();
    tc5::tc_fence_after();
    const uint32_t tmem = taddr_s;
    const bool prof_on = a.prof && PH_ONLY_EPI && (threadIdx.x == 0 || threadIdx.x == EPI_WARPS * 32 || threadIdx.x == MMA_WARP * 32);
    long long pc[7] = {0, 0, 0, 0, 0, 0, 0};
    const long long t_start = clock64();

    if (warp >= EPI_WARPS && warp < EPI_WARPS + PROD_WARPS) {
        // ======================= producers: input rows -> plane-separated ring rows
        Regs::aux();
        // Half rows (8 pixels x 3 components x 16 channels x 8 coefficients = 24 KB) are
        // copied raw into two shared staging buffers with cp.async (no registers held, a half
        // row in flight while the other is transposed), then byte-transposed into the ring.
        // Staging layout [pixel, component][channel i ^ ((i >> 2) & 1)][4 x 16 bytes]: the
        // swizzle spreads a transposition load over all 32 banks.
        const int pt = threadIdx.x - EPI_WARPS * 32;
        constexpr int PT = PROD_WARPS * 32;
        const uint32_t ring_s = tc5::smem_u32(ring), stg_s = tc5::smem_u32(stg);
        constexpr int HX = 8;                         // pixels per staging unit (half row)
        constexpr int NU = 2;                         // staging units per row = buffers
        constexpr int NSEG = HX * NCI * 16 * 4;       // 16-byte copies per half row
        constexpr int NTASK = HX * NCI * 16;          // (pixel, component, coefficient pair, channel group)
        int k = 0;
        int issued = 0;  // staging units whose copies were issued (global counter, NU buffers)
        // issue the copies of unit hr (row hr / NU of item kk) into buffer issued % NU
        auto issue = [&](int kk, int item_i, int hr) {
            const int it = item_i >> 1;
            const int l = a.limbs[it / nchunk];
            const size_t coff = (size_t)(it % nchunk) * 8;
            const int y = a.y0 - 1 + hr / NU, xh = (hr % NU) * HX;
            const uint32_t dst0 = stg_s + (uint32_t)(issued % NU) * (NSEG * 16);
            if (y >= 0 && y < H)
                for (int sgi = pt; sgi < NSEG; sgi += PT) {
                    // segment = (pixel, component, channel, quarter of the 64-byte coefficient chunk)
                    const int q4 = sgi & 3, is = (sgi >> 2) & 15, i = is ^ ((is >> 2) & 1), cx = sgi >> 6,
                              c = cx % NCI, x = xh + cx / NCI;
                    const uint64_t *src = a.ibase + (size_t)ptab[i * H * W + y * W + x] * 32 +
                                          ((size_t)c * a.ell + l) * N + coff + 2 * q4;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst0 + sgi * 16), "l"(src)
                                 : "memory");
                }
            asm volatile("cp.async.commit_group;" ::: "memory");
            issued++;
            (void)kk;
        };
        if constexpr (PLANAR) {
            // planar carry: one bulk copy (TMA engine) per input row into pixel slots 1..W
            const uint32_t rowb = (uint32_t)W * PS;
            for (int item = blockIdx.x; item < a.nitems; item += gridDim.x, k++) {
                const int it = item >> 1;
                const int l = a.limbs[it / nchunk];
                const size_t chunk = (size_t)(it % nchunk);
                for (int rr = 0; rr < rows_in; rr++) {
                    const int G = k * rows_in + rr, slot = G % RR, use = G / RR;
                    const int y = a.y0 - 1 + rr;
                    const bool inside = y >= 0 && y < H;
                    if (use > 0) {
                        if (warp == EPI_WARPS) PWAIT(0, tc5::mbar_wait(&bar_empty[slot], (use - 1) & 1));
                        asm volatile("bar.sync 1, %0;" ::"n"(PT) : "memory");
                    }
                    if (inside) {
                        if (pt == 0) {
                            tc5::mbar_arrive_expect_tx(&bar_full[slot], rowb);
                            const uint8_t *src = a.pl_in + (((size_t)l * nchunk + chunk) * H + y) * rowb;
                            asm volatile(
                                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                    ring_s + slot * RS + PS),
                                "l"(src), "r"(rowb), "r"(tc5::smem_u32(&bar_full[slot]))
                                : "memory");
                        }
                    } else {  // zero padding row
                        for (uint32_t o = (uint32_t)pt * 16; o < rowb; o += PT * 16)
                            asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(ring_s + slot * RS + PS + o),
                                         "r"(0u));
                        tc5::fence_async_smem();
                        asm volatile("bar.sync 1, %0;" ::"n"(PT) : "memory");
                        if (pt == 0) tc5::mbar_arrive(&bar_full[slot]);
                    }
                }
            }
        } else {
        int nk = 0, nitem = blockIdx.x, nhr = 0;  // next half row to issue
        auto issue_next = [&]() {
            if (nitem >= a.nitems) {
                asm volatile("cp.async.commit_group;" ::: "memory");  // keep the group count uniform
                issued++;
                return;
            }
            issue(nk, nitem, nhr);
            if (++nhr == NU * rows_in) {
                nhr = 0;
                nitem += gridDim.x;
                nk++;
            }
        };
        for (int u = 0; u < NU - 1; u++) issue_next();
        for (int item = blockIdx.x; item < a.nitems; item += gridDim.x, k++) {
            for (int rr = 0; rr < rows_in; rr++) {
                const int G = k * rows_in + rr, slot = G % RR, use = G / RR;
                const int y = a.y0 - 1 + rr;
                const bool inside = y >= 0 && y < H;
                const uint32_t rbase = ring_s + slot * RS;
                if (use > 0) {
                    if (warp == EPI_WARPS) PWAIT(0, tc5::mbar_wait(&bar_empty[slot], (use - 1) & 1));
                    asm volatile("bar.sync 1, %0;" ::"n"(PT) : "memory");
                }
                for (int h = 0; h < NU; h++) {
                    const int cur = (issued - (NU - 1)) % NU;  // buffer of the unit now landing
                    issue_next();                               // later units stream in meanwhile
                    asm volatile("cp.async.wait_group %0;" ::"n"(NU - 1) : "memory");
                    asm volatile("bar.sync 1, %0;" ::"n"(PT) : "memory");  // every thread's copies landed
                    const uint32_t sb = stg_s + (uint32_t)cur * (NSEG * 16);
                    for (int t = pt; t < NTASK; t += PT) {
                        const int g = t & 3, jp = (t >> 2) & 3, cx = t >> 4, c = cx % NCI, x = h * HX + cx / NCI;
                        const uint32_t base = rbase + (x + 1) * PS + c * (5 * 128) + g * 4;
                        uint64_t v[4][2];
#pragma unroll
                        for (int ch = 0; ch < 4; ch++) {
                            if (inside) {
                                const int is = (4 * g + ch) ^ (g & 1);
                                const uint32_t sa = sb + (uint32_t)(((cx * 16 + is) * 4 + jp) * 16);
                                asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(v[ch][0]), "=l"(v[ch][1]) : "r"(sa));
                            } else {
                                v[ch][0] = v[ch][1] = 0;
                            }
                        }
#pragma unroll
                        for (int kc = 0; kc < 2; kc++) {
                            uint32_t lo[4], hi[4];
                            const uint64_t a0 = v[0][kc], a1 = v[1][kc], a2 = v[2][kc], a3 = v[3][kc];
                            tr4b((uint32_t)a0, (uint32_t)a1, (uint32_t)a2, (uint32_t)a3, lo);
                            tr4b((uint32_t)(a0 >> 32), (uint32_t)(a1 >> 32), (uint32_t)(a2 >> 32), (uint32_t)(a3 >> 32),
                                 hi);
                            const uint32_t dst = base + (2 * jp + kc) * 16;
#pragma unroll
                            for (int d = 0; d < 4; d++)
                                asm volatile("st.shared.u32 [%0], %1;" ::"r"(dst + d * 128), "r"(lo[d]));
                            asm volatile("st.shared.u32 [%0], %1;" ::"r"(dst + 4 * 128), "r"(hi[0]));
                        }
                    }
                    asm volatile("bar.sync 1, %0;" ::"n"(PT) : "memory");  // staging buffer cur is free again
                }
                tc5::fence_async_smem();
                tc5::mbar_arrive(&bar_full[slot]);
            }
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
    } else if (warp == MMA_WARP) {
        Regs::aux();
        // ======================= MMA issuer (warp-uniform loop, one elected lane issues)
        {
            tc5::mbar_wait(&bar_b, 0);
            const uint32_t ring_s = tc5::smem_u32(ring), b_s = tc5::smem_u32(bsm);
            const uint32_t idesc32 = tc5::idesc_u8s8(128, 32), idesc96 = tc5::idesc_u8s8(128, 96),
                           idesc48 = tc5::idesc_u8s8(128, 48);
            const uint32_t blbo = 32 * 16, blbo0 = 96 * 16;
            const uint32_t ahi = tc5::sdesc_hi(PS), lps = tc5::sdesc_lbo(PS), lpl = tc5::sdesc_lbo(128);
            uint64_t bd[7];
            for (int t = 0; t < 6; t++) bd[t] = tc5::sdesc(b_s + t * LY::TB, blbo, 128);
            bd[6] = tc5::sdesc(b_s + 6 * LY::TB, blbo0, 128);
            const uint64_t bdp = tc5::sdesc(b_s + 6 * LY::TB + LY::TB0, 48 * 16, 128);
            int k = 0, S = 0;
            for (int item = blockIdx.x; item < a.nitems; item += gridDim.x, k++) {
                const int Gb = k * rows_in;
                auto slot_of = [&](int y) { return (Gb + (y - (a.y0 - 1))) % RR; };
                for (int y = a.y0; y < a.y1; y++) {
                    for (int yy = y - 1; yy <= y + 1; yy++) {
                        const int G = Gb + (yy - (a.y0 - 1));
                        PWAIT(2, tc5::mbar_wait(&bar_full[G % RR], (G / RR) & 1));
                    }
                    tc5::tc_fence_after();
                    const uint32_t r0 = (ring_s + slot_of(y - 1) * RS) >> 4, r1 = (ring_s + slot_of(y) * RS) >> 4,
                                   r2 = (ring_s + slot_of(y + 1) * RS) >> 4;
                    const uint32_t lv = r1 > r0 ? tc5::sdesc_lbo((r1 - r0) << 4) : tc5::sdesc_lbo((r0 - r1) << 4);
                    const uint32_t a3 = (r1 > r0 ? r0 : r1) + 2 * (PS >> 4) + lv;
                    const uint64_t b3 = r1 > r0 ? bd[3] : bd[5];
                    // one component at a time, each committed as soon as its 25 MMAs are issued,
                    // so the epilogue starts on component 0 while components 1 and 2 multiply
                    // (dependent accumulations cost no MMA throughput: tests/test_gpu_tc5.py)
#pragma unroll
                    for (int c = 0; c < NCI; c++) {
                        const int Sc = S + c, ds = Sc % NSL;
                        if (Sc >= NSL) PWAIT(3, tc5::mbar_wait(&bar_dempty[ds], ((Sc / NSL) - 1) & 1));
                        tc5::tc_fence_after();
                        const uint32_t dslc = tmem + (uint32_t)ds * SLC;
#pragma unroll
                        for (int d = 0; d < 5; d++) {
                            const uint32_t dcol = dslc + d * 16;
                            const uint32_t co = (uint32_t)(c * 5 + d) * (128 >> 4);
                            if (d == 0)
                                tc5::mma_i8_w(dcol, tc5::sdesc_hl(ahi, r0 + co + lps), bd[6], idesc96, false);
                            else
                                tc5::mma_i8_w(dcol, tc5::sdesc_hl(ahi, r0 + co + lps), bd[0], idesc32, true);
                            tc5::mma_i8_w(dcol, tc5::sdesc_hl(ahi, r1 + co + lps), bd[1], idesc32, true);
                            tc5::mma_i8_w(dcol, tc5::sdesc_hl(ahi, r2 + co + lps), bd[2], idesc32, true);
                            tc5::mma_i8_w(dcol, tc5::sdesc_hl(ahi, a3 + co), b3, idesc32, true);
                            // tap 8: planes (0, 1) and (2, 3) share one K step (the two K chunks are
                            // the two planes, 128 bytes apart; N = 48 covers shift blocks d .. d + 2)
                            if (d == 0 || d == 2)
                                tc5::mma_i8_w(dcol, tc5::sdesc_hl(ahi, r2 + co + 2 * (PS >> 4) + lpl), bdp, idesc48, true);
                            else if (d == 4)
                                tc5::mma_i8_w(dcol, tc5::sdesc_hl(ahi, r2 + co + 2 * (PS >> 4) + lps), bd[4], idesc32, true);
                        }
                        tc5::tc_commit_w(&bar_dfull[Sc % NSL]);
                    }
                    S += NCI;
                    tc5::tc_commit_w(&bar_empty[slot_of(y - 1)]);  // row y-1 is not read again
                }
                tc5::tc_commit_w(&bar_empty[slot_of(a.y1 - 1)]);
                tc5::tc_commit_w(&bar_empty[slot_of(a.y1)]);
            }
        }
    } else if (warp < EPI_WARPS) {
        // ======================= epilogue
        Regs::epilogue();
        const int qd = warp & 3, cg = warp >> 2;
        const int row = qd * 32 + lane, j = row & 7;
        const bool exp1 = a.exp == 1, hasb = a.biasd != nullptr;  // no bias: no per-row loads
        const uint32_t tq = tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(cg * CPT);
        int k = 0, S = 0;
        int li_cur = -1, l = 0, kq = 0;
        ModConst c;
        for (int item = blockIdx.x; item < a.nitems; item += gridDim.x, k++) {
            const int it = item >> 1;
            const size_t coff = (size_t)(it % nchunk) * 8;
            if (it / nchunk != li_cur) {  // a CTA's consecutive items mostly share the limb: reload on change only
                li_cur = it / nchunk;
                l = a.limbs[li_cur];
                c = a.mc[l];
                kq = (int)(1099511627776.0 - c.qd);  // 2^40 - q < 2^25 (checked by the launcher)
            }
            const int m0 = half * MC + cg * CPT;  // this thread's first output channel
            double gs[CPT][5];  // (y0 y0, y0 y1, 2 y0 y2 + y1 y1, y1 y2, y2 y2) over the thread's pixel column
#pragma unroll
            for (int m = 0; m < CPT; m++)
#pragma unroll
                for (int s2 = 0; s2 < 5; s2++) gs[m][s2] = 0.0;
            PH_START();
            for (int yr = 0; yr < nrows; yr++) {
                double yv[NCI][CPT];
#pragma unroll
                for (int cc = 0; cc < NCI; cc++, S++) {
                    const int ds = S % NSL;
                    PWAIT(5, tc5::mbar_wait(&bar_dfull[ds], (S / NSL) & 1));
                    PH_RESET();
                    tc5::tc_fence_after();
                    int C[CPT][NSH];
                    const uint32_t ta = tq + (uint32_t)ds * SLC;
#pragma unroll
                    for (int s2 = 0; s2 < NSH; s2++) {
                        uint32_t r[4];
                        tc5::tld4(ta + s2 * 16, r);
#pragma unroll
                        for (int m = 0; m < CPT; m++) C[m][s2] = (int)r[m];
                    }
                    tc5::tld_wait();
                    tc5::tc_fence_before();
                    tc5::mbar_arrive(&bar_dempty[ds]);
                    PH(0);
                    recombine_v<NSH, CPT>(C, kq, yv[cc]);
                    PH(2);
                }
                if (exp1) {
#pragma unroll
                    for (int m = 0; m < CPT; m++) gs[m][0] += yv[0][m] + yv[1][m] + yv[2][m];
                } else {
                    double t[CPT], d00[CPT];
                    if (hasb)
#pragma unroll
                        for (int m = 0; m < CPT; m++) yv[0][m] += a.biasd[(size_t)(m0 + m) * a.ell + l];
                    fmulmod_v<CPT>(yv[0], yv[0], t, c.qd, c.qid);
#pragma unroll
                    for (int m = 0; m < CPT; m++) gs[m][0] += t[m];
                    fmulmod_v<CPT>(yv[0], yv[1], t, c.qd, c.qid);
#pragma unroll
                    for (int m = 0; m < CPT; m++) gs[m][1] += t[m];
#pragma unroll
                    for (int m = 0; m < CPT; m++) d00[m] = yv[0][m] + yv[0][m];
                    fmulmod_v<CPT>(d00, yv[2], t, c.qd, c.qid);
                    fmulmod_v<CPT>(yv[1], yv[1], d00, c.qd, c.qid);
#pragma unroll
                    for (int m = 0; m < CPT; m++) gs[m][2] += t[m] + d00[m];
                    fmulmod_v<CPT>(yv[1], yv[2], t, c.qd, c.qid);
#pragma unroll
                    for (int m = 0; m < CPT; m++) gs[m][3] += t[m];
                    fmulmod_v<CPT>(yv[2], yv[2], t, c.qd, c.qid);
#pragma unroll
                    for (int m = 0; m < CPT; m++) gs[m][4] += t[m];
                }
                PH(3);
                if ((yr & 15) == 15 && yr + 1 < nrows)  // keep the exact sums below 2^53: centre every 16 rows
#pragma unroll
                    for (int m = 0; m < CPT; m++)
#pragma unroll
                        for (int s2 = 0; s2 < 5; s2++) {
                            const double e = fma(gs[m][s2], c.qid, 6755399441055744.0) - 6755399441055744.0;
                            gs[m][s2] = fma(-e, c.qd, gs[m][s2]);
                        }
            }
            // centre, then sum the 16 pixels of the row: 4 per warp (lanes ^ 8, ^ 16), 4 quarters via shared memory
#pragma unroll
            for (int m = 0; m < CPT; m++)
#pragma unroll
                for (int s2 = 0; s2 < 5; s2++) {
                    double v = gs[m][s2];
                    const double e = fma(v, c.qid, 6755399441055744.0) - 6755399441055744.0;
                    v = fma(-e, c.qd, v);  // |v| <= q/2 + 1
                    v += __shfl_xor_sync(0xffffffffu, v, 8);
                    v += __shfl_xor_sync(0xffffffffu, v, 16);
                    gs[m][s2] = v;
                }
            PH(1);
            if constexpr (PLANAR) {
                // no warp waits for another: each quarter leaves its partial sums in its own
                // shared-memory block and counts in; the LAST of the channel group's four warps
                // to arrive adds the four blocks and writes the outputs.  (A warp cannot reach the
                // end of the next item before every warp has finished this one: the TMEM slots
                // of the next item's rows are released by all sixteen warps.)
                double *blk = red + (size_t)(cg * 4 + qd) * (CPT * 5 * 8);
                if (lane < 8)
#pragma unroll
                    for (int m = 0; m < CPT; m++)
#pragma unroll
                        for (int s2 = 0; s2 < 5; s2++) blk[(m * 5 + s2) * 8 + lane] = gs[m][s2];
                __syncwarp();
                unsigned int old = 0;
                if (lane == 0) {
                    __threadfence_block();
                    old = atomicAdd(&fin_cnt[cg], 1u);
                }
                old = __shfl_sync(0xffffffffu, old, 0);
                PH(4);
                if ((old & 3u) == 3u) {
                    __threadfence_block();
                    const double *b0 = red + (size_t)(cg * 4) * (CPT * 5 * 8);
                    const size_t cs = (size_t)a.ell * N;
                    const double cstd = a.cst ? (double)a.cst[l] : 0.0;
#pragma unroll
                    for (int i = 0; i < CPT * 5 * 8 / 32; i++) {
                        const int idx = lane + 32 * i, jj = idx & 7, s2 = (idx >> 3) % 5, m = idx / 40;
                        const volatile double *p = b0 + idx;
                        double v = p[0] + p[CPT * 5 * 8] + p[2 * CPT * 5 * 8] + p[3 * CPT * 5 * 8];
                        v = s2 == 0 ? v + cstd : (s2 & 1) ? 2.0 * v : v;
                        const int mo = m0 + m;
                        if (mo < a.M) {
                            uint64_t *o = (a.obase ? a.obase + (size_t)mo * a.ostride : a.out[mo]) + (size_t)l * N + coff;
                            o[(size_t)s2 * cs + jj] = canon_fast(v, c.qd, c.qid);
                        }
                    }
                }
                __syncwarp();
            } else {
            // quarters 0..3 add into red[cg] in turn (named barrier over the epilogue warps)
            double *rr2 = red + (size_t)cg * (CPT * 5 * 8);
            for (int q2 = 0; q2 < 4; q2++) {
                if (qd == q2 && lane < 8)
#pragma unroll
                    for (int m = 0; m < CPT; m++)
#pragma unroll
                        for (int s2 = 0; s2 < 5; s2++) {
                            double *p = rr2 + (m * 5 + s2) * 8 + lane;
                            const double v = q2 ? *p + gs[m][s2] : gs[m][s2];
                            if (q2 < 3)
                                *p = v;
                            else
                                gs[m][s2] = v;
                        }
                // only the four warps of this channel group (one per lane quarter) meet here
                switch (cg) {
                    case 0: asm volatile("bar.sync 2, 128;" ::: "memory"); break;
                    case 1: asm volatile("bar.sync 3, 128;" ::: "memory"); break;
                    case 2: asm volatile("bar.sync 4, 128;" ::: "memory"); break;
                    default: asm volatile("bar.sync 5, 128;" ::: "memory"); break;
                }
            }
            PH(4);
            if (qd == 3 && lane < 8) {
                const size_t lo = (size_t)l * N + coff + j;
                const size_t cs = (size_t)a.ell * N;
                const double cstd = a.cst ? (double)a.cst[l] : 0.0;
#pragma unroll
                for (int m = 0; m < CPT; m++) {
                    const int mo = m0 + m;
                    if (mo >= a.M) break;
                    uint64_t *o = (a.obase ? a.obase + (size_t)mo * a.ostride : a.out[mo]) + lo;
                    o[0] = canon_fast(gs[m][0] + cstd, c.qd, c.qid);
                    o[cs] = canon_fast(2.0 * gs[m][1], c.qd, c.qid);
                    o[2 * cs] = canon_fast(gs[m][2], c.qd, c.qid);
                    o[3 * cs] = canon_fast(2.0 * gs[m][3], c.qd, c.qid);
                    o[4 * cs] = canon_fast(gs[m][4], c.qd, c.qid);
                }
            }
            }
        }
    }
    if (prof_on) {
        const int tot = threadIdx.x == 0 ? 6 : threadIdx.x == EPI_WARPS * 32 ? 1 : 4;
        pc[tot] = clock64() - t_start;
        for (int i = 0; i < 7; i++)
            if (pc[i]) atomicAdd(a.prof + i, (unsigned long long)pc[i]);
    }
    tc5::tc_fence_before();
    __syncthreads();
    if (warp == MMA_WARP) tc5::tmem_free<512>(tmem);
}

// balanced signed base-256 digit e of w
inline int digit_s8(int64_t w, int e) {
    for (int i = 0; i < e; i++) {
        int64_t d = (int8_t)(uint8_t)(w & 0xFF);
        w = (w - d) >> 8;
    }
    return (int8_t)(uint8_t)(w & 0xFF);
}

}  // namespace convtc

using namespace convtc;

// B tiles of the P1 packing: tile t (0..5) = K step t; tile 5 = K step 3 with its two taps swapped.
// Tile layout (K-major, no swizzle): [chunk k][row group n/8][8 rows x 16 bytes], row n = (m / 4) * 32 + s * 4 + m % 4 (P1_NCOL columns, s < NSH).
static void build_btiles_p1(const int64_t *weights, int M, int p, int E, int NSH, std::vector<uint8_t> &bt) {
    const int NCOL = P1_NCOL, TB = NCOL * 32;
    // taps (dy, dx) of the two chunks of each K step; (-1,-1) = zero chunk
    const int ks[6][2][2] = {{{0, 0}, {0, 1}}, {{1, 0}, {1, 1}}, {{2, 0}, {2, 1}},
                             {{0, 2}, {1, 2}}, {{2, 2}, {-1, -1}}, {{1, 2}, {0, 2}}};
    bt.assign((size_t)6 * TB, 0);
    for (int t = 0; t < 6; t++)
        for (int k = 0; k < 2; k++) {
            const int dy = ks[t][k][0], dx = ks[t][k][1];
            if (dy < 0) continue;
            const int tap = dy * 3 + dx;
            for (int n = 0; n < NCOL; n++) {
                // column block cg*32 + s*4 + mm: shift s of channel m = 4 cg + mm (s >= NSH: zero)
                const int s = (n % 32) / 4, m = (n / 32) * 4 + n % 4;
                if (m >= M || s >= NSH) continue;
                for (int kb = 0; kb < 15; kb++) {
                    const int i = kb / 5, d = kb % 5, e = s - d;
                    if (i >= p || e < 0 || e >= E) continue;
                    const int dg = digit_s8(weights[(size_t)m * p * 9 + i * 9 + tap], e);
                    bt[(size_t)t * TB + (size_t)k * NCOL * 16 + (size_t)(n / 8) * 128 + (n % 8) * 16 + kb] =
                        (uint8_t)(int8_t)dg;
                }
            }
        }
}

// B tiles of the P16 packing for channel half h (rows n = e * 16 + m, m = output channel 16 h + m):
// tiles 0..5 as P1 (N = 32), tile 6 = K step 0 zero-extended to N = 96 (initialises all six shift blocks).
static void build_btiles_p16(const int64_t *weights, int M, int p, std::vector<uint8_t> &bt) {
    const int ks[6][2][2] = {{{0, 0}, {0, 1}}, {{1, 0}, {1, 1}}, {{2, 0}, {2, 1}},
                             {{0, 2}, {1, 2}}, {{2, 2}, {-1, -1}}, {{1, 2}, {0, 2}}};
    const int BB = P16Layout::BBYTES;
    bt.assign((size_t)2 * BB, 0);
    for (int h = 0; h < 2; h++)
        for (int t = 0; t < 7; t++) {
            const int kt = t == 6 ? 0 : t, NR = t == 6 ? 96 : 32;
            uint8_t *tile = bt.data() + (size_t)h * BB + (size_t)t * P16Layout::TB;
            for (int k = 0; k < 2; k++) {
                const int dy = ks[kt][k][0], dx = ks[kt][k][1];
                if (dy < 0) continue;
                const int tap = dy * 3 + dx;
                for (int n = 0; n < 32; n++) {
                    const int e = n / 16, m = h * 16 + n % 16;
                    if (m >= M) continue;
                    for (int i = 0; i < p && i < 16; i++)
                        tile[(size_t)k * NR * 16 + (size_t)(n / 8) * 128 + (n % 8) * 16 + i] =
                            (uint8_t)(int8_t)digit_s8(weights[(size_t)m * p * 9 + i * 9 + tap], e);
                }
            }
        }
    // pair tile: K chunk k = tap 8 of byte plane d + k; row n = b * 16 + m is shift block d + b,
    // so chunk k holds digit b - k of the weight (zero outside 0..1)
    for (int h = 0; h < 2; h++) {
        uint8_t *tile = bt.data() + (size_t)h * BB + (size_t)6 * P16Layout::TB + P16Layout::TB0;
        for (int k = 0; k < 2; k++)
            for (int n = 0; n < 48; n++) {
                const int e = n / 16 - k, m = h * 16 + n % 16;
                if (m >= M || e < 0 || e > 1) continue;
                for (int i = 0; i < p && i < 16; i++)
                    tile[(size_t)k * 48 * 16 + (size_t)(n / 8) * 128 + (n % 8) * 16 + i] =
                        (uint8_t)(int8_t)digit_s8(weights[(size_t)m * p * 9 + i * 9 + 8], e);
            }
    }
}

static int g_conv_tc = 1;  // he_set_conv_tc: 0 forces the mma.sync kernels (A/B tests)
static unsigned long long *g_prof = nullptr;

// role timing of the tcgen05 conv kernels (diagnostics): on != 0 enables and zeroes the
// counters, on == 0 copies the 7 summed counters (see PWAIT) to out and disables
extern "C" int he_convtc_profile(int on, double *out) {
    if (on) {
        if (!g_prof) HE_CHECK_CUDA(cudaMalloc(&g_prof, 64));
        HE_CHECK_CUDA(cudaMemset(g_prof, 0, 64));
        return HE_OK;
    }
    if (!g_prof) return HE_EINVAL;
    unsigned long long h[7];
    HE_CHECK_CUDA(cudaDeviceSynchronize());
    HE_CHECK_CUDA(cudaMemcpy(h, g_prof, 56, cudaMemcpyDeviceToHost));
    for (int i = 0; i < 7; i++) out[i] = (double)h[i];
    cudaFree(g_prof);
    g_prof = nullptr;
    return HE_OK;
}

extern "C" int he_set_conv_tc(int on) {
    const int old = g_conv_tc;
    g_conv_tc = on;
    return old;
}

// Eligibility + launch of the tcgen05 path; HE_EINVAL (no work enqueued) when the shape is not covered.
// pl_in / pl_out: planar carry input (P16) / output (P1) instead of ciphertext pointer lists.
static int convtc_launch(he_ctx *c, const uint64_t *const *in, int nci, int p, int H, int W, uint64_t *const *out,
                         int M, int pool, int y0, int y1, const int64_t *weights, const uint64_t *bias,
                         const uint64_t *cst, int ell, const uint8_t *pl_in, uint8_t *pl_out, void *stream) {
    if (!c || (!in && !pl_in) || (!out && !pl_out) || !weights || ell < 1 || ell > c->L || y0 < 0 || y1 > H ||
        y0 >= y1) {
        he_set_error("he_conv_square_sum_tc: bad arguments");
        return HE_EINVAL;
    }
    const bool p1 = nci == 2 && p <= 3 && pool && M <= MC && W % 16 == 0 && W <= 64 && !((y0 | y1 | H) & 1);
    const bool p16 = nci == 3 && p == 16 && !pool && M <= 2 * MC && W == 16;
    if ((pl_in && !p16) || (pl_out && !(p1 && M == MC))) {
        he_set_error("he_conv_square_sum_pl: planar carry needs the conv2 shape (input) / 16 pooled channels (output)");
        return HE_EINVAL;
    }
    if (!p1 && !p16) {
        he_set_error("he_conv_square_sum_tc: shape (nci=%d p=%d M=%d W=%d pool=%d) not covered", nci, p, M, W, pool);
        return HE_EINVAL;
    }
    for (int l = 0; l < ell; l++)
        if (c->mod[l] <= (1ull << 40) - (1ull << 25) || c->mod[l] >= (1ull << 40)) {  // recombine_fold: 2^40 - q < 2^25
            he_set_error("he_conv_square_sum_tc: prime %d outside (2^40 - 2^25, 2^40)", l);
            return HE_EINVAL;
        }
    int64_t wmax = 0;
    for (int i = 0; i < M * p * 9; i++) wmax = std::max<int64_t>(wmax, weights[i] < 0 ? -weights[i] : weights[i]);
    int E = 1;
    int64_t cap = 127;
    while (wmax > cap && E < 3) {
        E++;
        cap = cap * 256 + 127;
    }
    if (wmax > cap || (p16 && E > 2)) {
        he_set_error("he_conv_square_sum_tc: weights need more than %d signed byte digits", p16 ? 2 : 3);
        return HE_EINVAL;
    }
    // worst-case shift sums: |C[s]| <= 255 * sum over the digits and the K = 9 p weights of one
    // output channel of |digit|.  The epilogue combines C[s] + 2^8 C[s+1] in 32 bits and
    // (C[4] + 2^8 C[5]) 2^32 in 64 (recombine_fold), which is exact below 2^22.5.
    for (int m = 0; m < M; m++) {
        int64_t dsum = 0;
        for (int i = 0; i < p * 9; i++)
            for (int e = 0; e < E; e++) dsum += std::abs(digit_s8(weights[(size_t)m * p * 9 + i], e));
        if (255 * dsum >= 5931641) {  // 2^22.5
            he_set_error("he_conv_square_sum_tc: weights of channel %d too heavy for the 32-bit shift sums", m);
            return HE_EINVAL;
        }
    }
    const int NSH = p16 ? 6 : NB + E - 1;
    std::vector<uint8_t> bt;
    if (p16)
        build_btiles_p16(weights, M, p, bt);
    else
        build_btiles_p1(weights, M, p, E, NSH, bt);
    const int TB = p16 ? P16Layout::TB : P1_NCOL * 32;
    std::vector<double> biasd((size_t)2 * MC * ell, 0.0);
    for (int l = 0; l < ell; l++) {
        const uint64_t q = c->mod[l];
        if (cst && cst[l] >= q) {
            he_set_error("he_conv_square_sum_tc: residue not canonical");
            return HE_EINVAL;
        }
        if (bias)
            for (int m = 0; m < M; m++) {
                if (bias[(size_t)m * ell + l] >= q) {
                    he_set_error("he_conv_square_sum_tc: residue not canonical");
                    return HE_EINVAL;
                }
                biasd[(size_t)m * ell + l] = (double)bias[(size_t)m * ell + l];
            }
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int nwin = pool ? ((y1 - y0) / 2) * (W / 2) : 1;
    const int n_in = p * H * W, n_out = M * nwin;
    const size_t smem = p16 ? (size_t)P16Layout::RR * (W + 3) * P16Layout::PS + P16Layout::BBYTES +
                                  (pl_in ? 0 : (size_t)n_in * 4 + 128 + P16Layout::STG) + (size_t)(pl_in ? 16 : 4) * CPT * 5 * 8 * 8
                            : (size_t)P1Layout<2>::RR * (W + 3) * P1Layout<2>::PS + 6 * (size_t)TB + (size_t)n_in * 4;
    // inputs as 32-bit offsets from the lowest address in 256-byte units (every ciphertext of a
    // batch allocation is 256-byte aligned); anything else takes the mma.sync kernels
    uintptr_t ib = UINTPTR_MAX;
    for (int i = 0; i < n_in && in; i++) ib = std::min(ib, (uintptr_t)in[i]);
    std::vector<uint32_t> ioff(in ? n_in : 0);
    for (int i = 0; i < n_in && in; i++) {
        const uintptr_t d = (uintptr_t)in[i] - ib;
        if ((d & 255) || (d >> 8) > 0xFFFFFFFFull) {
            he_set_error("he_conv_square_sum_tc: inputs not addressable by 32-bit 256-byte offsets");
            return HE_EINVAL;
        }
        ioff[i] = (uint32_t)(d >> 8);
    }
    if (smem > 227 * 1024) {
        he_set_error("he_conv_square_sum_tc: %zu bytes of shared memory (input table of %d)", smem, n_in);
        return HE_EINVAL;
    }
    void **din = nullptr, **dout = nullptr;
    if (in) HE_TRY(he_upload_ptrs((const void *const *)in, n_in, &din, s));
    if (out) HE_TRY(he_upload_ptrs((const void *const *)out, n_out, &dout, s));
    std::vector<int32_t> lorder(ell);
    for (int l = 0; l < ell; l++) lorder[l] = l;
    const size_t b_bt = bt.size(), b_bias = biasd.size() * 8, b_lo = (size_t)ell * 4,
                 b_c = cst ? (size_t)ell * 8 : 0, b_io = in ? (size_t)n_in * 4 : 16;
    char *meta = nullptr;
    HE_TRY(he_scratch_alloc((void **)&meta, b_bt + b_bias + b_lo + b_c + b_io + 1024, s));
    size_t off = 0;
    auto carve = [&](size_t bytes) {
        char *q = meta + off;
        off = (off + bytes + 127) & ~(size_t)127;
        return q;
    };
    uint8_t *dbt = (uint8_t *)carve(b_bt);
    double *dbias = (double *)carve(b_bias);
    int32_t *dlo = (int32_t *)carve(b_lo);
    uint64_t *dc = cst ? (uint64_t *)carve(b_c) : nullptr;
    uint32_t *dio = (uint32_t *)carve(b_io);
    if (in) HE_CHECK_CUDA(he_h2d(dio, ioff.data(), b_io, s));
    HE_CHECK_CUDA(he_h2d(dbt, bt.data(), b_bt, s));
    HE_CHECK_CUDA(he_h2d(dbias, biasd.data(), b_bias, s));
    HE_CHECK_CUDA(he_h2d(dlo, lorder.data(), b_lo, s));
    if (dc) HE_CHECK_CUDA(he_h2d(dc, cst, b_c, s));
    TcArgs a;
    a.in = (const uint64_t *const *)din;
    a.ibase = (const uint64_t *)ib;
    a.ioff = dio;
    a.out = (uint64_t *const *)dout;
    a.obase = nullptr;
    a.ostride = 0;
    a.pl_in = pl_in;
    a.pl_out = pl_out;
    if (out && n_out > 1) {  // outputs of one batch allocation: strided addressing, no pointer loads
        const long long st = (long long)(out[1] - out[0]);
        bool uni = st > 0;
        for (int i = 2; i < n_out && uni; i++) uni = (out[i] - out[i - 1]) == st;
        if (uni) {
            a.obase = out[0];
            a.ostride = st;
        }
    }
    a.btiles = dbt;
    // P16 reads the bias per row only when there is one (config 3's biases are zero)
    a.biasd = (p16 && std::all_of(biasd.begin(), biasd.end(), [](double v) { return v == 0.0; })) ? nullptr : dbias;
    a.cst = dc;
    a.mc = c->d_mc;
    a.limbs = dlo;
    a.nlimbs = ell;
    a.ell = ell;
    a.logN = c->logN;
    a.p = p;
    a.H = H;
    a.W = W;
    a.M = M;
    a.y0 = y0;
    a.y1 = y1;
    a.nwin = nwin;
    a.nitems = ell * (c->N / 8) * (p16 ? 2 : 1);
    a.btile_bytes = TB;
    a.prof = g_prof;
    a.exp = getenv("CONVTC_EXP") ? atoi(getenv("CONVTC_EXP")) : 0;
    a.nshift = NSH;
    int sms = 0;
    HE_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    const dim3 grid((unsigned)(p16 ? std::min(sms, a.nitems) & ~1 : std::min(sms, a.nitems)));  // P16: even
    int rc = HE_OK;
    auto launch = [&](auto kern) -> int {
        HE_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<grid, THREADS, smem, s>>>(a);
        HE_CHECK_LAUNCH();
        return HE_OK;
    };
    if (p16 && pl_in) rc = launch(k_convtc_p16_gap<true>);
    else if (p16) rc = launch(k_convtc_p16_gap<false>);
    else if (NSH == 5) rc = launch(k_convtc_p1_pool<5>);
    else if (NSH == 6) rc = launch(k_convtc_p1_pool<6>);
    else rc = launch(k_convtc_p1_pool<7>);
    he_scratch_free(meta, s);
    if (din) he_scratch_free(din, s);
    if (dout) he_scratch_free(dout, s);
    return rc;
}

extern "C" int he_conv_square_sum_tc(he_ctx *c, const uint64_t *const *in, int nci, int p, int H, int W,
                                     uint64_t *const *out, int M, int pool, int y0, int y1, const int64_t *weights,
                                     const uint64_t *bias, const uint64_t *cst, int ell, void *stream) {
    if (!in || !out) {
        he_set_error("he_conv_square_sum_tc: bad arguments");
        return HE_EINVAL;
    }
    return convtc_launch(c, in, nci, p, H, W, out, M, pool, y0, y1, weights, bias, cst, ell, nullptr, nullptr, stream);
}

extern "C" int he_conv_square_sum_pl(he_ctx *c, const uint64_t *const *in, int nci, int p, int H, int W,
                                     uint64_t *const *out, int M, int pool, int y0, int y1, const int64_t *weights,
                                     const uint64_t *bias, const uint64_t *cst, int ell, const void *pl_in,
                                     void *pl_out, void *stream) {
    return convtc_launch(c, pl_in ? nullptr : in, nci, p, H, W, pl_out ? nullptr : out, M, pool, y0, y1, weights,
                         bias, cst, ell, (const uint8_t *)pl_in, (uint8_t *)pl_out, stream);
}

// ---------------------------------------------------------------- planar carry <-> ciphertexts
// planar byte offset of (limb l, coefficient k, y, x, component cp, plane d, channel m), C = 16 channels
__device__ __forceinline__ size_t pl_off(int l, size_t k, int y, int x, int cp, int d, int m, int H, int W,
                                        size_t nchunk) {
    return ((((size_t)l * nchunk + (k >> 3)) * H + y) * W + x) * (3 * 5 * 128) + (size_t)(cp * 5 + d) * 128 +
           (k & 7) * 16 + m;
}
// one thread per (channel group of 4, coefficient, pixel, component, limb)
__global__ void k_planar_pack(const uint64_t *const *in, int C, int H, int W, int ell, int logN, uint8_t *pl) {
    const size_t N = (size_t)1 << logN, nchunk = N >> 3;
    const size_t tot = (size_t)ell * 3 * H * W * N * 4;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < tot; t += (size_t)gridDim.x * blockDim.x) {
        const int g = (int)(t & 3);
        size_t r = t >> 2;
        const size_t k = r % N;
        r /= N;
        const int px = (int)(r % ((size_t)H * W));
        r /= (size_t)H * W;
        const int cp = (int)(r % 3), l = (int)(r / 3);
        uint64_t v[4];
        for (int u = 0; u < 4; u++) {
            const int ch = 4 * g + u;
            v[u] = ch < C ? in[(size_t)ch * H * W + px][((size_t)cp * ell + l) * N + k] : 0;
        }
        const size_t o = pl_off(l, k, px / W, px % W, cp, 0, 4 * g, H, W, nchunk);
        for (int d = 0; d < 5; d++) {
            uint32_t w = 0;
            for (int u = 0; u < 4; u++) w |= (uint32_t)((v[u] >> (8 * d)) & 0xFF) << (8 * u);
            *(uint32_t *)(pl + o + (size_t)d * 128) = w;
        }
    }
}
__global__ void k_planar_unpack(const uint8_t *pl, int C, int H, int W, int ell, int logN, uint64_t *const *out) {
    const size_t N = (size_t)1 << logN, nchunk = N >> 3;
    const size_t tot = (size_t)ell * 3 * H * W * N * C;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < tot; t += (size_t)gridDim.x * blockDim.x) {
        size_t r = t;
        const size_t k = r % N;
        r /= N;
        const int px = (int)(r % ((size_t)H * W));
        r /= (size_t)H * W;
        const int ch = (int)(r % C);
        r /= C;
        const int cp = (int)(r % 3), l = (int)(r / 3);
        const size_t o = pl_off(l, k, px / W, px % W, cp, 0, ch, H, W, nchunk);
        uint64_t v = 0;
        for (int d = 0; d < 5; d++) v |= (uint64_t)pl[o + (size_t)d * 128] << (8 * d);
        out[(size_t)ch * H * W + px][((size_t)cp * ell + l) * N + k] = v;
    }
}

// ciphertexts (C <= 16 channels x H x W, 3 components, residues < 2^40 on ell limbs) -> planar carry
extern "C" int he_planar_pack(he_ctx *c, const uint64_t *const *in, int C, int H, int W, int ell, void *pl,
                              void *stream) {
    if (!c || !in || !pl || C < 1 || C > 16 || H < 1 || W < 1 || ell < 1 || ell > c->L) {
        he_set_error("he_planar_pack: bad arguments");
        return HE_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    void **din = nullptr;
    HE_TRY(he_upload_ptrs((const void *const *)in, C * H * W, &din, s));
    HE_CHECK_CUDA(cudaMemsetAsync(pl, 0, (size_t)ell * (c->N / 8) * H * W * 1920, s));
    k_planar_pack<<<148 * 16, 256, 0, s>>>((const uint64_t *const *)din, C, H, W, ell, c->logN, (uint8_t *)pl);
    HE_CHECK_LAUNCH();
    he_scratch_free(din, s);
    return HE_OK;
}
extern "C" int he_planar_unpack(he_ctx *c, const void *pl, int C, int H, int W, int ell, uint64_t *const *out,
                                void *stream) {
    if (!c || !out || !pl || C < 1 || C > 16 || H < 1 || W < 1 || ell < 1 || ell > c->L) {
        he_set_error("he_planar_unpack: bad arguments");
        return HE_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    void **dout = nullptr;
    HE_TRY(he_upload_ptrs((const void *const *)out, C * H * W, &dout, s));
    k_planar_unpack<<<148 * 16, 256, 0, s>>>((const uint8_t *)pl, C, H, W, ell, c->logN, (uint64_t *const *)dout);
    HE_CHECK_LAUNCH();
    he_scratch_free(dout, s);
    return HE_OK;
}


int he_conv_tc_enabled() { return g_conv_tc; }
