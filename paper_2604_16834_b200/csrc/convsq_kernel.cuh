// convsq_kernel.cuh -- the fused conv + square + pool/GAP kernel of convsq.cu,
// templated on the input component count NCI (2: fresh / relinearised
// ciphertexts -> 3-component window sums; 3: unrelinearised squares from the
// previous block -> 5-component sums).  convsq.cu instantiates NCI = 2 and the
// host entry points, convsq3.cu instantiates NCI = 3 (parallel compilation).
//
// Per CTA: one limb l and one chunk of 8 coefficients, ALL windows of the
// launch.  For every output pixel the conv is an exact int8 GEMM
//     C_d[(comp, j)][(e, m)] = sum_k  byte_d(x_{k, comp, j}) * W_e[m][k]
// one mma.sync m16n8k32 u8 x s8 per (input byte plane d, 32-byte K block,
// weight digit e).  Tile T0 has rows (component 0, coefficient j) and
// (component 1, j), so the lane holding row j of component 0 also holds
// component 1 -- the square needs both.  With NCI = 3, tile T1 holds component
// 2 of coefficient j at two horizontally adjacent pixels (x, x+1), so pixels are
// processed in pairs and component 2 costs half a tile per pixel (1.5 tiles per
// pixel in all, the ideal 3/2 of the 2-component kernel).  Byte planes beyond
// the limb's length (5 for 40-bit primes) are skipped.  The lane recombines
// its values exactly (int32 sums per byte shift, IMAD.WIDE into int64 partial
// sums at 2^0 / 2^32 / 2^64); 40-bit primes finish with one FP64 modular
// product (plain domain), wider primes with one Montgomery step (y R^-1).  The
// window's products (y0^2, y0 y1, y1^2; with NCI = 3 also y0 y2, y1 y2, y2^2)
// accumulate exactly and are reduced once; outputs are the square's components
//   NCI = 2: (s00, 2 s01, s11)
//   NCI = 3: (s00, 2 s01, 2 s02 + s11, 2 s12, s22).
// Bit-identical to conv -> tensor square -> add_const -> sum: every step is
// exact arithmetic mod q.
//
// Data path: the K dimension is ordered (tap, group of 4 input channels), so
// one 32-bit A-operand word is "byte d of 4 channels at one input pixel".
// Input rows are loaded ONCE per CTA into a shared-memory ring (R rows x
// (W+2) pixels incl. a zero halo), byte-transposed with PRMT into that
// digit-planar, channel-interleaved layout (8 NCI rows per channel group and
// plane); every output pixel then reads its 9 taps straight from the ring.
// Strides are chosen so the A-fragment loads are bank-conflict free.  Weight
// digits stay in registers for the whole kernel.
#pragma once
#include <algorithm>

#include "ntt_core.cuh"  // u2d / d2u / fmulmod / fcanon (FP64 modular products)

namespace convsq {

#ifndef CONV2_CTAS
#define CONV2_CTAS 3  // resident CTAs/SM of the 3-component, 4-group kernel (2 column tiles; 4 tiles at 4 CTAs measured slower)
#endif

constexpr int CT = 128;  // 4 warps: MG channel groups x PS pixel streams

struct SqArgs {
    const uint64_t *const *in;  // [p*H*W] NCI-component input ciphertexts (device array of addresses)
    uint64_t *const *out;       // (2 NCI - 1)-component outputs, ell limbs
    const uint32_t *bfrag;      // [MG][KB][E][32] uint2 B fragments
    const uint32_t *bfrag8;     // tap-8 packing (one channel group, 40-bit primes): [MG][4 + E][32] uint2
    const uint64_t *bias;       // [M][ell] bias * R^-1 mod q (component 0), or nullptr
    const uint64_t *cst;        // [ell] constant added to component 0 of every output, or nullptr
    const uint64_t *r4;         // [ell] R^4 mod q
    const double *yc;           // [ell][2] R mod q and 2^32 mod q as doubles (FP64 recombination)
    const ModConst *mc;
    const int32_t *limbs;       // [gridDim.y] limb handled by blockIdx.y (one byte-plane count per launch)
    int p, H, W, M, ell, logN, pool, y0, y1, nwin;
    int x0, Wt;                 // column tile of blockIdx.z: output columns [x0 + z Wt, x0 + (z+1) Wt) (GAP)
    int ncg, nb, R;             // channel groups of 4, byte planes stored, ring rows
    int pstr, rstr;             // ring strides in 32-bit words: pixel, ring row
    int mul[4];                 // 1, 2^8, 2^16, 2^24
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

// Row r (= component * 8 + coefficient) of channel group cg inside a pixel's
// plane.  NCI = 2: 16 rows per group, groups 2, 3 swap their halves so the
// four groups read by one A-fragment load hit 32 distinct banks.  NCI = 3: 24
// rows per group (group strides 24 words already spread the banks).
// LS (ldmatrix layout, NCI = 3 with 4 channel groups): the 4 groups of a row
// are one contiguous 16-byte ldmatrix row, rows follow at 16 bytes.
template <int NCI, bool LS = false>
__device__ __forceinline__ int rowpos(int cg, int r) {
    if constexpr (LS) return r * 4 + cg;
    if constexpr (NCI == 2) return cg * 16 + (r ^ (8 * ((cg >> 1) & 1)));
    return cg * 24 + r;
}

// Input row yy -> ring slot: word (x' + 1) * pstr + d * (8 NCI ncg) + rowpos(cg, comp*8 + j)
// holds byte d of channels 4cg .. 4cg+3 at pixel (yy, x'), coefficient j of component comp.
template <int NCI, bool LS, int NCG, int NB>
__device__ __forceinline__ void load_row(const SqArgs &a, uint32_t *slot, const uint64_t **prow, int yy, int l,
                                         size_t coff) {
    constexpr int RW = 8 * NCI;    // rows per channel group
    constexpr int RC = RW * NCG;   // tasks per pixel: (row, channel group)
    constexpr int DSTR = RC;       // words per byte plane of a pixel
    const size_t N = (size_t)1 << a.logN, compstr = (size_t)a.ell * N, base = (size_t)l * N + coff;
    // ring slots [s_lo, s_lo + ns) <-> image columns xb - 1 + slot: the whole row
    // (slots 1..W; the halo slots stay zero) or a column tile with its halo
    const bool tiled = a.Wt < a.W;
    const int xb = a.x0 + (int)blockIdx.z * a.Wt, s_lo = tiled ? 0 : 1, ns = tiled ? a.Wt + 2 : a.W;
    const int ntask = ns * RC;
    const bool inside = yy >= 0 && yy < a.H;
    // the row's input addresses (p x ns) are staged in shared memory once, so no
    // task waits on a dependent address-table load
    __syncthreads();  // the previous row's table is no longer read
    if (inside)
        for (int k = threadIdx.x; k < a.p * ns; k += CT) {
            const int x = xb - 1 + s_lo + k % ns;
            prow[k] = (x >= 0 && x < a.W) ? a.in[(size_t)(k / ns) * a.H * a.W + yy * a.W + x] : nullptr;
        }
    __syncthreads();
    // LU tasks per thread per batch: their data loads are all in flight before
    // the first transpose (one memory latency per batch)
    constexpr int LU = 4;
    for (int t0 = threadIdx.x; t0 < ntask; t0 += LU * CT) {
        const uint64_t *src[LU][4];
#pragma unroll
        for (int j = 0; j < LU; j++) {
            const int t = t0 + j * CT, rc = t % RC, x = t / RC;  // compile-time divisors
            // LS: channel group fastest, so a warp's stores are contiguous words
            const int r = LS ? rc / 4 : rc % RW, cg = LS ? rc % 4 : rc / RW;
            const size_t off = (size_t)(r >> 3) * compstr + base + (r & 7);
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int i = cg * 4 + u;
                const uint64_t *pr = (inside && t < ntask && i < a.p) ? prow[i * ns + x] : nullptr;
                src[j][u] = pr ? pr + off : nullptr;
            }
        }
        uint64_t v[LU][4];
#pragma unroll
        for (int j = 0; j < LU; j++)
#pragma unroll
            for (int u = 0; u < 4; u++) v[j][u] = src[j][u] ? __ldg(src[j][u]) : 0;
#pragma unroll
        for (int j = 0; j < LU; j++) {
            const int t = t0 + j * CT, rc = t % RC, x = t / RC;
            if (t >= ntask) break;
            const int r = LS ? rc / 4 : rc % RW, cg = LS ? rc % 4 : rc / RW;
            uint32_t lo[4], hi[4];
            tr4((uint32_t)v[j][0], (uint32_t)v[j][1], (uint32_t)v[j][2], (uint32_t)v[j][3], lo);
            tr4((uint32_t)(v[j][0] >> 32), (uint32_t)(v[j][1] >> 32), (uint32_t)(v[j][2] >> 32),
                (uint32_t)(v[j][3] >> 32), hi);
            uint32_t *dst = slot + (x + s_lo) * a.pstr + rowpos<NCI, LS>(cg, r);
#pragma unroll
            for (int d = 0; d < 4; d++) dst[d * DSTR] = lo[d];
#pragma unroll
            for (int d = 0; d < 4; d++)
                if (d + 4 < NB) dst[(d + 4) * DSTR] = hi[d];
        }
    }
}

// One input byte plane D on the tensor cores.  Products with the same byte
// shift s = D + e accumulate in ONE int32 fragment C[s] (the mma's own
// accumulator), so the exact recombination sees NB + E - 1 shift sums instead
// of NB * E digit products: |C[s]| <= 3 * 144 * 255 * 128 < 2^24 for the
// accepted shapes (p <= 16, |w| < 2^23), no overflow.
template <int D, int KB, int E, int NB, int DSTR, int NSH>
__device__ __forceinline__ void digit_plane(const uint32_t *X, const int (&o0)[KB][2], const int (&o1)[KB][2],
                                            const uint2 (&bw)[KB][E], int (&C)[NSH][4]) {
    if (D >= NB) return;
    const uint32_t *Xd = X + D * DSTR;  // compile-time plane offset: an LDS immediate
#pragma unroll
    for (int kb = 0; kb < KB; kb++) {
        const uint32_t a0 = Xd[o0[kb][0]], a1 = Xd[o1[kb][0]], a2 = Xd[o0[kb][1]], a3 = Xd[o1[kb][1]];
#pragma unroll
        for (int e = 0; e < E; e++) mma_u8s8(C[D + e], a0, a1, a2, a3, bw[kb][e]);
    }
}

// The tile's four fragment values: exact conv over all byte planes (tile rows
// from o0 / o1), recombined from the shift sums: P0 = sum_{s<4} C[s] 2^(8s),
// P1 = sum_{4<=s<8} C[s] 2^(8(s-4)), P2 = the rest.  FP (40-bit primes):
// T = P0 + P1 2^32 with |P0| < 2^48.1, |P1| < 2^40; y = P0 + [P1 2^32 mod q]
// (one FP64 modular product) is returned as an integer-valued double,
// NOT reduced: |y| < 2^48.2 (the square accumulator takes unreduced
// operands).  Integer path: canonical y R^-1 (one Montgomery step) in yv.
// Tap-8 packing (one channel group: 9 taps = 9 K words, the second K block
// would hold 1 real word): per plane only block 0 (taps 0..7) is multiplied;
// tap 8 of ALL planes shares one block -- word k = tap 8 of plane k -- and is
// multiplied once per byte shift s with B8[s] (word k = weight digit s - k),
// which lands every product in its shift sum C[s].  NB * KB * E mma become
// NB * E + NSH (conv1: 30 -> 22).  o0[1][0] / o1[1][0] carry this lane's tap-8
// row offsets (plane 0); the block's words sit DSTR apart.
template <int KB, int E, int NB, int DSTR, bool TP8 = false>
__device__ __forceinline__ void tile_values(const uint32_t *X, const int (&o0)[KB][2], const int (&o1)[KB][2],
                                            const uint2 (&bw)[KB][E], const int (&mul)[4], const ModConst &c,
                                            double yc1, double (&yd)[4], uint64_t (&yv)[4],
                                            const uint2 *bw8 = nullptr) {
    constexpr int NSH = NB + E - 1;  // byte shifts 0 .. NB + E - 2
    constexpr int KBM = TP8 ? 1 : KB;  // K blocks multiplied per plane
    int C[NSH][4];
#pragma unroll
    for (int s = 0; s < NSH; s++) C[s][0] = C[s][1] = C[s][2] = C[s][3] = 0;
    digit_plane<0, KBM, E, NB, DSTR, NSH>(X, (const int(&)[KBM][2])o0, (const int(&)[KBM][2])o1,
                                          (const uint2(&)[KBM][E])bw, C);
    digit_plane<1, KBM, E, NB, DSTR, NSH>(X, (const int(&)[KBM][2])o0, (const int(&)[KBM][2])o1,
                                          (const uint2(&)[KBM][E])bw, C);
    digit_plane<2, KBM, E, NB, DSTR, NSH>(X, (const int(&)[KBM][2])o0, (const int(&)[KBM][2])o1,
                                          (const uint2(&)[KBM][E])bw, C);
    digit_plane<3, KBM, E, NB, DSTR, NSH>(X, (const int(&)[KBM][2])o0, (const int(&)[KBM][2])o1,
                                          (const uint2(&)[KBM][E])bw, C);
    digit_plane<4, KBM, E, NB, DSTR, NSH>(X, (const int(&)[KBM][2])o0, (const int(&)[KBM][2])o1,
                                          (const uint2(&)[KBM][E])bw, C);
    digit_plane<5, KBM, E, NB, DSTR, NSH>(X, (const int(&)[KBM][2])o0, (const int(&)[KBM][2])o1,
                                          (const uint2(&)[KBM][E])bw, C);
    digit_plane<6, KBM, E, NB, DSTR, NSH>(X, (const int(&)[KBM][2])o0, (const int(&)[KBM][2])o1,
                                          (const uint2(&)[KBM][E])bw, C);
    digit_plane<7, KBM, E, NB, DSTR, NSH>(X, (const int(&)[KBM][2])o0, (const int(&)[KBM][2])o1,
                                          (const uint2(&)[KBM][E])bw, C);
    if constexpr (TP8) {
        static_assert(NB <= 5, "tap-8 block holds one word per plane: planes 0..4 in words 0..4");
        const int tig = threadIdx.x & 3;
        const uint32_t *X0 = X + o0[1][0], *X1 = X + o1[1][0];
        const uint32_t a0 = X0[tig * DSTR], a1 = X1[tig * DSTR];  // words tig: plane tig
        const uint32_t a2 = tig == 0 ? X0[4 * DSTR] : 0u, a3 = tig == 0 ? X1[4 * DSTR] : 0u;  // word 4: plane 4
#pragma unroll
        for (int s = 0; s < NSH; s++) mma_u8s8(C[s], a0, a1, a2, a3, __ldg(bw8 + s * 32));
    }
    int64_t P[3][4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
        P[0][q] = C[0][q];
        P[1][q] = NSH > 4 ? C[NSH > 4 ? 4 : 0][q] : 0;
        P[2][q] = NSH > 8 ? C[NSH > 8 ? 8 : 0][q] : 0;
#pragma unroll
        for (int s = 1; s < NSH; s++)
            if (s & 3) madw(P[s >> 2][q], C[s][q], mul[s & 3]);
    }
    if constexpr (NB == 5) {
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const double p0 = __longlong_as_double(0x4338000000000000ll + P[0][q]) - 6755399441055744.0;
            const double p1 = __longlong_as_double(0x4338000000000000ll + P[1][q]) - 6755399441055744.0;
            yd[q] = p0 + fmulmod(p1, yc1, c.qd, c.qid);  // T = P0 + P1 2^32 (mod q), |T'| < 2^48.2
        }
    } else {
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const uint64_t lo = (uint64_t)P[0][q] + ((uint64_t)P[1][q] << 32);
            const uint64_t cy = lo < (uint64_t)P[0][q] ? 1 : 0;
            const int64_t hi = (P[0][q] >> 63) + (P[1][q] >> 32) + (int64_t)cy + P[2][q];
            const uint64_t hic = hi < 0 ? (uint64_t)(hi + (int64_t)c.q) : (uint64_t)hi;  // |hi| < q
            yv[q] = redc(hic, lo, c.q, c.qinv);  // conv * R^-1
        }
    }
}

__device__ __forceinline__ void ldsm4(uint32_t addr, uint32_t &a0, uint32_t &a1, uint32_t &a2, uint32_t &a3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                 : "r"(addr));
}

// shift sums -> value (as tile_values): FP path only (40-bit primes)
template <int NSH>
__device__ __forceinline__ void recombine_fp(const int (&C)[NSH][4], const int (&mul)[4], const ModConst &c,
                                             double yc1, double (&yd)[4]) {
#pragma unroll
    for (int q = 0; q < 4; q++) {
        int64_t p0 = C[0][q], p1 = NSH > 4 ? C[NSH > 4 ? 4 : 0][q] : 0;
#pragma unroll
        for (int s = 1; s < NSH && s < 4; s++) madw(p0, C[s][q], mul[s]);
#pragma unroll
        for (int s = 5; s < NSH; s++) madw(p1, C[s][q], mul[s - 4]);
        const double d0 = __longlong_as_double(0x4338000000000000ll + p0) - 6755399441055744.0;
        const double d1 = __longlong_as_double(0x4338000000000000ll + p1) - 6755399441055744.0;
        yd[q] = d0 + fmulmod(d1, yc1, c.qd, c.qid);
    }
}

// ldmatrix.x4 at addr + OFF (OFF: compile-time byte offset, folded into the instruction)
template <int OFF>
__device__ __forceinline__ void ldsm4i(uint32_t addr, uint32_t &a0, uint32_t &a1, uint32_t &a2, uint32_t &a3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4+%5];"
                 : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                 : "r"(addr), "n"(OFF));
}

// LS layout (NCI = 3, 4 channel groups, 40-bit primes): the A fragment of a
// (plane, K block) is ONE ldmatrix.x4 -- this lane supplies the row address
// (bytes, plane 0) of matrix lane/8, row lane%8.  Three independent tiles are
// interleaved so their mma chains overlap: y[0] = T1 at ad[0][kb], y[1] = T0 of
// pixel x at ad[1][kb], y[2] = T0 of pixel x + 1 at ad[1][kb] + PSTRB.
template <int D, int KB, int E, int DSTRB, int PSTRB, int NSH, int KBM = KB>
__device__ __forceinline__ void plane_ls(const uint32_t (&ad)[2][KB], const uint2 (&bw)[KB][E], int (&C)[3][NSH][4]) {
#pragma unroll
    for (int kb = 0; kb < KBM; kb++) {  // K blocks 0 .. KBM-1 of the plane
        uint32_t a[3][4];
        ldsm4i<D * DSTRB>(ad[0][kb], a[0][0], a[0][1], a[0][2], a[0][3]);
        ldsm4i<D * DSTRB>(ad[1][kb], a[1][0], a[1][1], a[1][2], a[1][3]);
        ldsm4i<D * DSTRB + PSTRB>(ad[1][kb], a[2][0], a[2][1], a[2][2], a[2][3]);
#pragma unroll
        for (int t = 0; t < 3; t++)
#pragma unroll
            for (int e = 0; e < E; e++) mma_u8s8(C[t][D + e], a[t][0], a[t][1], a[t][2], a[t][3], bw[kb][e]);
    }
}

// LS8 (E = 2): the last K block (tap 8 + 4 zero words) is not multiplied per
// plane; instead one block per byte shift s holds [tap 8 of plane s | tap 8 of
// plane s - 1] against [W0 | W1] (halves outside 0..4 read a valid plane with
// zero weights): 5 x 2 mma per tile become 6.  ad[*][KB-1] addresses tap 8 of
// plane 0 for every lane; lanes of matrices 2, 3 (h1) read plane s - 1.
template <int T, int S, int DSTRB, int PSTRB>
__device__ __forceinline__ void tap8_ls(uint32_t base, uint32_t baseh, int (&C)[3][6][4], uint2 b) {
    uint32_t a0, a1, a2, a3;
    constexpr int OFF = (T == 2 ? PSTRB : 0);
    if (S == 0)
        ldsm4i<OFF>(base, a0, a1, a2, a3);
    else if (S == 5)
        ldsm4i<4 * DSTRB + OFF>(base, a0, a1, a2, a3);
    else
        ldsm4i<S * DSTRB + OFF>(baseh, a0, a1, a2, a3);
    mma_u8s8(C[T][S], a0, a1, a2, a3, b);
}

template <int KB, int E, int DSTRB, int PSTRB, bool LS8 = false>
__device__ __forceinline__ void tile_values_ls(const uint32_t (&ad)[2][KB], const uint2 (&bw)[KB][E],
                                               const int (&mul)[4], const ModConst &c, double yc1,
                                               double (&yd)[3][4], const uint2 (&b8)[3] = {}, int h1 = 0) {
    constexpr int NB = 5, NSH = NB + E - 1;
    constexpr int KBM = LS8 ? KB - 1 : KB;
    int C[3][NSH][4];
#pragma unroll
    for (int t = 0; t < 3; t++)
#pragma unroll
        for (int s = 0; s < NSH; s++) C[t][s][0] = C[t][s][1] = C[t][s][2] = C[t][s][3] = 0;
    plane_ls<0, KB, E, DSTRB, PSTRB, NSH, KBM>(ad, bw, C);
    plane_ls<1, KB, E, DSTRB, PSTRB, NSH, KBM>(ad, bw, C);
    plane_ls<2, KB, E, DSTRB, PSTRB, NSH, KBM>(ad, bw, C);
    plane_ls<3, KB, E, DSTRB, PSTRB, NSH, KBM>(ad, bw, C);
    plane_ls<4, KB, E, DSTRB, PSTRB, NSH, KBM>(ad, bw, C);
    if constexpr (LS8) {
        static_assert(E == 2, "two planes per tap-8 block");
        const uint32_t dh = h1 ? (uint32_t)DSTRB : 0u;  // h1 lanes: plane s - 1
        const uint32_t b1 = ad[1][KB - 1], b0 = ad[0][KB - 1];
        // (tile T and shift S are template constants: unrolled by hand)
        tap8_ls<0, 0, DSTRB, PSTRB>(b0, b0 - dh, (int(&)[3][6][4])C, b8[0]);
        tap8_ls<1, 0, DSTRB, PSTRB>(b1, b1 - dh, (int(&)[3][6][4])C, b8[0]);
        tap8_ls<2, 0, DSTRB, PSTRB>(b1, b1 - dh, (int(&)[3][6][4])C, b8[0]);
        tap8_ls<0, 1, DSTRB, PSTRB>(b0, b0 - dh, (int(&)[3][6][4])C, b8[1]);
        tap8_ls<1, 1, DSTRB, PSTRB>(b1, b1 - dh, (int(&)[3][6][4])C, b8[1]);
        tap8_ls<2, 1, DSTRB, PSTRB>(b1, b1 - dh, (int(&)[3][6][4])C, b8[1]);
        tap8_ls<0, 2, DSTRB, PSTRB>(b0, b0 - dh, (int(&)[3][6][4])C, b8[1]);
        tap8_ls<1, 2, DSTRB, PSTRB>(b1, b1 - dh, (int(&)[3][6][4])C, b8[1]);
        tap8_ls<2, 2, DSTRB, PSTRB>(b1, b1 - dh, (int(&)[3][6][4])C, b8[1]);
        tap8_ls<0, 3, DSTRB, PSTRB>(b0, b0 - dh, (int(&)[3][6][4])C, b8[1]);
        tap8_ls<1, 3, DSTRB, PSTRB>(b1, b1 - dh, (int(&)[3][6][4])C, b8[1]);
        tap8_ls<2, 3, DSTRB, PSTRB>(b1, b1 - dh, (int(&)[3][6][4])C, b8[1]);
        tap8_ls<0, 4, DSTRB, PSTRB>(b0, b0 - dh, (int(&)[3][6][4])C, b8[1]);
        tap8_ls<1, 4, DSTRB, PSTRB>(b1, b1 - dh, (int(&)[3][6][4])C, b8[1]);
        tap8_ls<2, 4, DSTRB, PSTRB>(b1, b1 - dh, (int(&)[3][6][4])C, b8[1]);
        tap8_ls<0, 5, DSTRB, PSTRB>(b0, b0 - dh, (int(&)[3][6][4])C, b8[2]);
        tap8_ls<1, 5, DSTRB, PSTRB>(b1, b1 - dh, (int(&)[3][6][4])C, b8[2]);
        tap8_ls<2, 5, DSTRB, PSTRB>(b1, b1 - dh, (int(&)[3][6][4])C, b8[2]);
    }
#pragma unroll
    for (int t = 0; t < 3; t++) recombine_fp<NSH>(C[t], mul, c, yc1, yd[t]);
}

// Window sums of the products of y = conv (plain domain, FP path) or
// y = conv * R^-1 (integer path).  NS = 3: (y0 y0, y0 y1, y1 y1);
// NS = 6: (y0 y0, y0 y1, y0 y2, y1 y1, y1 y2, y2 y2).
// 40-bit primes: exact FP64 modular products of the unreduced conv values
// accumulated as doubles (folded every 32) on the FP64 pipe; wider primes:
// exact 128-bit sums.  value(k) returns the canonical plain-domain sum.
template <bool FP, int NS>
struct SqAcc;
template <int NS>
struct SqAcc<true, NS> {
    double a[NS];
    int n;
    __device__ __forceinline__ SqAcc() { reset(); }
    // operands are unreduced integer-valued doubles, |y| < 2^49: each modular
    // product is then below q/2 + 2^98-52 < 2^46.1 in magnitude, so 32 of them
    // plus a centred residue stay exact (< 2^53); fold every 32
    __device__ __forceinline__ void fold(const ModConst &c) {
        if (++n == 32) {
            n = 0;
#pragma unroll
            for (int k = 0; k < NS; k++) a[k] = fma(-rint(a[k] * c.qid), c.qd, a[k]);  // |a| <= q/2 + 1
        }
    }
    __device__ __forceinline__ void addd(double d0, double d1, const ModConst &c) {  // |d| < 2^49
        a[0] += fmulmod(d0, d0, c.qd, c.qid);
        a[1] += fmulmod(d0, d1, c.qd, c.qid);
        a[NS == 3 ? 2 : 3] += fmulmod(d1, d1, c.qd, c.qid);
        fold(c);
    }
    __device__ __forceinline__ void addd3(double d0, double d1, double d2, const ModConst &c) {
        a[0] += fmulmod(d0, d0, c.qd, c.qid);
        a[1] += fmulmod(d0, d1, c.qd, c.qid);
        a[2] += fmulmod(d0, d2, c.qd, c.qid);
        a[3] += fmulmod(d1, d1, c.qd, c.qid);
        a[4] += fmulmod(d1, d2, c.qd, c.qid);
        a[5] += fmulmod(d2, d2, c.qd, c.qid);
        fold(c);
    }
    __device__ __forceinline__ uint64_t value(int k, const ModConst &c, uint64_t) const {
        return fcanon(a[k], c.qd, c.qid);
    }
    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int k = 0; k < NS; k++) a[k] = 0.0;
        n = 0;
    }
};
template <int NS>
struct SqAcc<false, NS> {
    u128 a[NS];
    int n;
    __device__ __forceinline__ SqAcc() { reset(); }
    __device__ __forceinline__ void fold(const ModConst &c) {
        if (++n == 8) {  // each product adds < q/16 to hi: fold every 8
            n = 0;
#pragma unroll
            for (int k = 0; k < NS; k++)
                if (a[k].hi >= c.q) a[k].hi -= c.q;
        }
    }
    __device__ __forceinline__ void add(uint64_t y0, uint64_t y1, const ModConst &c) {
        mac128(a[0], y0, y0);
        mac128(a[1], y0, y1);
        mac128(a[NS == 3 ? 2 : 3], y1, y1);
        fold(c);
    }
    __device__ __forceinline__ void add3(uint64_t y0, uint64_t y1, uint64_t y2, const ModConst &c) {
        mac128(a[0], y0, y0);
        mac128(a[1], y0, y1);
        mac128(a[2], y0, y2);
        mac128(a[3], y1, y1);
        mac128(a[4], y1, y2);
        mac128(a[5], y2, y2);
        fold(c);
    }
    __device__ __forceinline__ uint64_t value(int k, const ModConst &c, uint64_t r4) const {
        const uint64_t hi = a[k].hi >= c.q ? a[k].hi - c.q : a[k].hi;
        return mont(redc(hi, a[k].lo, c.q, c.qinv), r4, c);  // sum R^-3 -> plain
    }
    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int k = 0; k < NS; k++) a[k] = u128{0, 0};
        n = 0;
    }
};

// output component k of the square from the product sums (NCI = 2 or 3)
template <int NCI, class Acc>
__device__ __forceinline__ uint64_t square_comp(const Acc &acc, int k, const ModConst &c, uint64_t r4) {
    if constexpr (NCI == 2) {
        const uint64_t v = acc.value(k, c, r4);
        return k == 1 ? add_mod(v, v, c.q) : v;
    } else {
        if (k == 0) return acc.value(0, c, r4);
        if (k == 4) return acc.value(5, c, r4);
        if (k == 1) {
            const uint64_t v = acc.value(1, c, r4);
            return add_mod(v, v, c.q);
        }
        if (k == 3) {
            const uint64_t v = acc.value(4, c, r4);
            return add_mod(v, v, c.q);
        }
        const uint64_t v = acc.value(2, c, r4);
        return add_mod(add_mod(v, v, c.q), acc.value(3, c, r4), c.q);
    }
}

template <int KB, int E, int MG, int NB, int NCI>
__global__ void __launch_bounds__(CT, NCI == 3 ? (KB == 5 ? CONV2_CTAS : 2) : (KB <= 2 ? 4 : 3)) k_conv_sqsum(const SqArgs a) {
    constexpr int PS = 4 / MG;
    constexpr int NO = 2 * NCI - 1;  // output components
    extern __shared__ __align__(16) uint32_t xs[];  // ring [R][rstr]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const int cg = warp % MG, ps = warp / MG;
    const int l = a.limbs[blockIdx.y];
    const size_t N = (size_t)1 << a.logN, coff = (size_t)blockIdx.x * 8;
    const ModConst c = a.mc[l];
    constexpr int NCG = KB == 2 ? 1 : KB - 1;  // channel groups of 4 implied by the K blocks
    constexpr int DSTR = 8 * NCI * NCG;
    constexpr bool LS = NCI == 3 && KB == 5 && NB == 5;  // ldmatrix layout (4 channel groups)
    constexpr bool TP8 = KB == 2 && NB == 5;               // tap-8 packing (one channel group)
    constexpr bool LS8 = LS && E == 2;                     // tap-8 packing on the ldmatrix path

    uint2 bw[KB][E];
#pragma unroll
    for (int kb = 0; kb < KB; kb++)
#pragma unroll
        for (int e = 0; e < E; e++) bw[kb][e] = ((const uint2 *)a.bfrag)[((cg * KB + kb) * E + e) * 32 + lane];
    const uint2 *bw8 = TP8 ? (const uint2 *)a.bfrag8 + (size_t)cg * (4 + E) * 32 + lane : nullptr;
    // LS tap-8 block fragments: [W0 | 0] (shift 0), [W0 | W1] (shifts 1..4), [0 | W1] (shift 5)
    uint2 bw8ls[3] = {};
    if (LS8)
#pragma unroll
        for (int k = 0; k < 3; k++) bw8ls[k] = ((const uint2 *)a.bfrag8)[((size_t)cg * 3 + k) * 32 + lane];
    const int mul[4] = {a.mul[0], a.mul[1], a.mul[2], a.mul[3]};
    const int m0 = cg * 8 + 2 * tig;  // this lane's channels m0, m0 + 1
    uint64_t bias[2] = {0, 0};
    if (a.bias) {
        if (m0 < a.M) bias[0] = a.bias[(size_t)m0 * a.ell + l];
        if (m0 + 1 < a.M) bias[1] = a.bias[(size_t)(m0 + 1) * a.ell + l];
    }
    // FP path: plain-domain bias (bias R^-1 * R) and 2^32 mod q
    const double yc0 = a.yc[2 * l], yc1 = a.yc[2 * l + 1];
    const double biasd[2] = {fcanond(fmulmod(u2d(bias[0]), yc0, c.qd, c.qid), c.qd, c.qid),
                             fcanond(fmulmod(u2d(bias[1]), yc0, c.qd, c.qid), c.qd, c.qid)};
    // this lane's A words: word w = kb*8 + h*4 + tig -> (tap t, channel group g);
    // words past the 9 taps carry zero weights and read tap 0
    // packed per word: offset inside the ring row (dx * pstr + row position of
    // component 0) in bits 3.., tap row dy in bits 0..1, bit 2 = component 1 sits 8 words lower
    int wd[KB][2];
#pragma unroll
    for (int kb = 0; kb < KB; kb++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int w = kb * 8 + h * 4 + tig;
            int t = w / a.ncg, g = w % a.ncg;
            if (t >= 9) t %= 9;  // zero-weight word: any in-bounds tap, spread over the banks
            if (TP8 && kb == 1 && h == 0) t = 8, g = 0;  // tap-8 block base (every lane)
            const int r0 = rowpos<NCI>(g, gid), r1 = rowpos<NCI>(g, gid + 8);
            wd[kb][h] = (((t % 3) * a.pstr + r0) << 3) | (r1 < r0 ? 4 : 0) | (t / 3);
        }

    const uint64_t **prow = (const uint64_t **)(xs + a.R * a.rstr);  // [p * W] input addresses of one row
    for (int i = tid; i < a.R * a.rstr; i += CT) xs[i] = 0;  // zero halo pixels stay zero
    __syncthreads();
    const int R = a.R, nrow0 = a.pool ? 4 : 3;
    for (int k = 0; k < nrow0; k++) {
        const int yy = a.y0 - 1 + k;
        load_row<NCI, LS, NCG, NB>(a, xs + ((yy + R) % R) * a.rstr, prow, yy, l, coff);
    }
    __syncthreads();

    SqAcc<NB == 5, NCI == 2 ? 3 : 6> acc[2];  // window sums for this lane's two channels
    const int rows_per_blk = a.pool ? 2 : 1;
    for (int yb = a.y0; yb < a.y1; yb += rows_per_blk) {
        // ring-row bases of the input rows yb - 1 .. yb + 2
        int sb[4];
#pragma unroll
        for (int k = 0; k < 4; k++) sb[k] = ((yb - 1 + k + R) % R) * a.rstr;
        // A-word offsets at x = 0 for the block's two rows (dyb = 0, 1)
        int bo[2][KB][2];
#pragma unroll
        for (int dyb = 0; dyb < 2; dyb++)
#pragma unroll
            for (int kb = 0; kb < KB; kb++)
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int v = wd[kb][h], r = (v & 3) + dyb;
                    bo[dyb][kb][h] = (r == 0 ? sb[0] : r == 1 ? sb[1] : r == 2 ? sb[2] : sb[3]) + (v >> 3);
                }
        int o0[KB][2], o1[KB][2];
        if constexpr (NCI == 2) {
            // per-pixel work list: pool -> windows wx = ps, ps+PS, ... (4 pixels each); GAP -> x = ps, ps+PS, ...
            const int nitems = a.pool ? (a.W / 2) : a.W, npx = a.pool ? 4 : 1;
            for (int it = ps; it < nitems; it += PS) {
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    if (k >= npx) break;
                    const int xo = (npx == 4 ? 2 * it + (k & 1) : it) * a.pstr;
#pragma unroll
                    for (int kb = 0; kb < KB; kb++)
#pragma unroll
                        for (int h = 0; h < 2; h++) {
                            o0[kb][h] = bo[k >> 1][kb][h] + xo;
                            o1[kb][h] = o0[kb][h] + ((wd[kb][h] & 4) ? -8 : 8);
                        }
                    // fragment values: q=0,1 -> component 0, channels m0, m0+1; q=2,3 -> component 1
                    double yd[4];
                    uint64_t yv[4];
                    tile_values<KB, E, NB, DSTR, TP8>(xs, o0, o1, bw, mul, c, yc1, yd, yv, bw8);
                    if constexpr (NB == 5) {
#pragma unroll
                        for (int h = 0; h < 2; h++)
                            acc[h].addd(yd[h] + biasd[h], yd[2 + h], c);
                    } else {
#pragma unroll
                        for (int h = 0; h < 2; h++) acc[h].add(add_mod(yv[h], bias[h], c.q), yv[2 + h], c);
                    }
                }
                if (a.pool) {  // window complete
                    const uint64_t r4 = a.r4[l], cst = a.cst ? a.cst[l] : 0;
                    const int win = ((yb - a.y0) >> 1) * (a.W >> 1) + it;
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        const int m = m0 + h;
                        if (m < a.M) {
                            uint64_t *o = a.out[(size_t)m * a.nwin + win] + coff + gid;
#pragma unroll
                            for (int k = 0; k < NO; k++) {
                                uint64_t v = square_comp<NCI>(acc[h], k, c, r4);
                                if (k == 0) v = add_mod(v, cst, c.q);
                                o[((size_t)k * a.ell + l) * N] = v;
                            }
                        }
                        acc[h].reset();
                    }
                }
            }
        } else if constexpr (LS) {
            // pixel pairs as below; A fragments by ldmatrix, the pair's two T0
            // tiles interleaved.  Lane = (matrix mi, row rr): tap 2 kb + (mi >> 1),
            // tile rows 8 (mi & 1) + rr.
            const int mi = lane >> 3, rr = lane & 7;
            constexpr int PSTR = NB * NCG * 8 * NCI;  // pixel stride (words) of the LS ring (host: ncg % 4 == 0)
            const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(xs);
            const int nitems = a.W / 2, npair = a.pool ? 2 : 1;
            // per K block: this lane's T0 row address at pixel 0 of the block's rows
            // (pr = 0, 1), bytes; T1 sits dT1 bytes further, T0(x + 1) PSTR words
            uint32_t rbase[2][KB];
#pragma unroll
            for (int kb = 0; kb < KB; kb++) {
                int t = 2 * kb + (mi >> 1);
                if (t >= 9) t -= 9;  // zero-weight half of the last K block
                if (LS8 && kb == KB - 1) t = 8;  // tap-8 block: every lane addresses tap 8
#pragma unroll
                for (int pr = 0; pr < 2; pr++) {
                    const int dy = t / 3 + pr;
                    rbase[pr][kb] = sbase + 4 * ((dy == 0 ? sb[0] : dy == 1 ? sb[1] : dy == 2 ? sb[2] : sb[3]) +
                                                 (t % 3) * PSTR + 4 * rr + (mi & 1) * 32);
                }
            }
            const uint32_t dT1 = 4 * ((mi & 1) * (PSTR - 32) + 64);  // component 2, pixel x + (mi & 1)
            const int nit = a.Wt / 2;  // pixel pairs of this CTA's column tile
            for (int it = ps; it < nit; it += PS) {
                for (int pr = 0; pr < npair; pr++) {
                    uint32_t ad[2][KB];  // tile 0: T1 (component 2 of the pair), tile 1: T0 of x (x + 1 by offset)
                    const uint32_t xoff = 4 * 2 * it * PSTR;
#pragma unroll
                    for (int kb = 0; kb < KB; kb++) {
                        ad[1][kb] = rbase[pr][kb] + xoff;
                        ad[0][kb] = ad[1][kb] + dT1;
                    }
                    double y[3][4];
                    tile_values_ls<KB, E, 4 * DSTR, 4 * PSTR, LS8>(ad, bw, mul, c, yc1, y, bw8ls, mi >> 1);
#pragma unroll
                    for (int k = 0; k < 2; k++)
#pragma unroll
                        for (int h = 0; h < 2; h++)
                            acc[h].addd3(y[1 + k][h] + biasd[h], y[1 + k][2 + h], y[0][2 * k + h], c);
                }
                if (a.pool) {  // window complete
                    const uint64_t r4 = a.r4[l], cst = a.cst ? a.cst[l] : 0;
                    const int win = ((yb - a.y0) >> 1) * (a.W >> 1) + it;
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        const int m = m0 + h;
                        if (m < a.M) {
                            uint64_t *o = a.out[(size_t)m * a.nwin + win] + coff + gid;
#pragma unroll
                            for (int k = 0; k < NO; k++) {
                                uint64_t v = square_comp<NCI>(acc[h], k, c, r4);
                                if (k == 0) v = add_mod(v, cst, c.q);
                                o[((size_t)k * a.ell + l) * N] = v;
                            }
                        }
                        acc[h].reset();
                    }
                }
            }
        } else {
            // pixel pairs (x, x+1), x even: pool -> the window's two rows (dyb = 0, 1);
            // GAP -> pairs it = ps, ps+PS, ... of the row
            const int nitems = a.W / 2, npair = a.pool ? 2 : 1;
            for (int it = ps; it < nitems; it += PS) {
                for (int pr = 0; pr < npair; pr++) {
                    const int xo = 2 * it * a.pstr;
                    // T1: component 2 (rows 16..23 of the group) at pixels x (tile rows 0..7)
                    // and x+1 (tile rows 8..15)
#pragma unroll
                    for (int kb = 0; kb < KB; kb++)
#pragma unroll
                        for (int h = 0; h < 2; h++) {
                            o0[kb][h] = bo[pr][kb][h] + xo + 16;
                            o1[kb][h] = o0[kb][h] + a.pstr;
                        }
                    double y2d[4];
                    uint64_t y2v[4];
                    tile_values<KB, E, NB, DSTR, TP8>(xs, o0, o1, bw, mul, c, yc1, y2d, y2v, bw8);
#pragma unroll
                    for (int k = 0; k < 2; k++) {  // T0 of pixel x + k
#pragma unroll
                        for (int kb = 0; kb < KB; kb++)
#pragma unroll
                            for (int h = 0; h < 2; h++) {
                                o0[kb][h] = bo[pr][kb][h] + xo + k * a.pstr;
                                o1[kb][h] = o0[kb][h] + 8;
                            }
                        double yd[4];
                        uint64_t yv[4];
                        tile_values<KB, E, NB, DSTR, TP8>(xs, o0, o1, bw, mul, c, yc1, yd, yv, bw8);
                        if constexpr (NB == 5) {
#pragma unroll
                            for (int h = 0; h < 2; h++)
                                acc[h].addd3(yd[h] + biasd[h], yd[2 + h], y2d[2 * k + h], c);
                        } else {
#pragma unroll
                            for (int h = 0; h < 2; h++)
                                acc[h].add3(add_mod(yv[h], bias[h], c.q), yv[2 + h], y2v[2 * k + h], c);
                        }
                    }
                }
                if (a.pool) {  // window complete
                    const uint64_t r4 = a.r4[l], cst = a.cst ? a.cst[l] : 0;
                    const int win = ((yb - a.y0) >> 1) * (a.W >> 1) + it;
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        const int m = m0 + h;
                        if (m < a.M) {
                            uint64_t *o = a.out[(size_t)m * a.nwin + win] + coff + gid;
#pragma unroll
                            for (int k = 0; k < NO; k++) {
                                uint64_t v = square_comp<NCI>(acc[h], k, c, r4);
                                if (k == 0) v = add_mod(v, cst, c.q);
                                o[((size_t)k * a.ell + l) * N] = v;
                            }
                        }
                        acc[h].reset();
                    }
                }
            }
        }
        // slide the ring: the rows of this block's top are no longer needed
        const int ynext = yb + rows_per_blk;
        if (ynext < a.y1) {
            __syncthreads();
            for (int k = 0; k < rows_per_blk; k++) {
                const int yy = ynext + 1 + k;  // pool: rows ynext+1, ynext+2; GAP: row ynext+1
                load_row<NCI, LS, NCG, NB>(a, xs + ((yy + R) % R) * a.rstr, prow, yy, l, coff);
            }
            __syncthreads();
        }
    }
    if (!a.pool) {  // global sum: reduce, combine the pixel streams, then store
        uint64_t r[NO][2];
        const uint64_t r4v = a.r4[l];
#pragma unroll
        for (int k = 0; k < NO; k++)
#pragma unroll
            for (int h = 0; h < 2; h++) r[k][h] = square_comp<NCI>(acc[h], k, c, r4v);
        uint64_t *red = (uint64_t *)xs;
        if (PS > 1) {
            __syncthreads();
#pragma unroll
            for (int k = 0; k < NO; k++)
#pragma unroll
                for (int h = 0; h < 2; h++) red[((ps * MG + cg) * 32 + lane) * 2 * NO + k * 2 + h] = r[k][h];
            __syncthreads();
            if (ps == 0)
                for (int o = 1; o < PS; o++)
#pragma unroll
                    for (int k = 0; k < NO; k++)
#pragma unroll
                        for (int h = 0; h < 2; h++)
                            r[k][h] = add_mod(r[k][h], red[((o * MG + cg) * 32 + lane) * 2 * NO + k * 2 + h], c.q);
        }
        if (ps == 0) {
            const uint64_t cst = a.cst && blockIdx.z == 0 ? a.cst[l] : 0;  // the GAP constant once, not per tile
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int m = m0 + h;
                if (m >= a.M) continue;
                uint64_t *o = a.out[m + blockIdx.z * a.M] + coff + gid;  // tile z's partial sums
#pragma unroll
                for (int k = 0; k < NO; k++) {
                    uint64_t v = r[k][h];
                    if (k == 0) v = add_mod(v, cst, c.q);
                    o[((size_t)k * a.ell + l) * N] = v;
                }
            }
        }
    }
}

template <int KB, int E, int MG, int NB, int NCI>
int launch_sq(dim3 grid, size_t smem, cudaStream_t s, const SqArgs &a) {
    if (smem > 48 * 1024)
        HE_CHECK_CUDA(cudaFuncSetAttribute(k_conv_sqsum<KB, E, MG, NB, NCI>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_conv_sqsum<KB, E, MG, NB, NCI><<<grid, CT, smem, s>>>(a);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

template <int KB, int E, int MG, int NCI>
int dispatch_nb(dim3 grid, size_t smem, cudaStream_t s, const SqArgs &a) {
    return a.nb == 5 ? launch_sq<KB, E, MG, 5, NCI>(grid, smem, s, a) : launch_sq<KB, E, MG, 8, NCI>(grid, smem, s, a);
}

template <int KB, int E, int NCI>
int dispatch_mg(int MG, dim3 grid, size_t smem, cudaStream_t s, const SqArgs &a) {
    if (MG == 1) return dispatch_nb<KB, E, 1, NCI>(grid, smem, s, a);
    if (MG == 2) return dispatch_nb<KB, E, 2, NCI>(grid, smem, s, a);
    return dispatch_nb<KB, E, 4, NCI>(grid, smem, s, a);
}

template <int KB, int NCI>
int dispatch_e(int E, int MG, dim3 grid, size_t smem, cudaStream_t s, const SqArgs &a) {
    if (E == 1) return dispatch_mg<KB, 1, NCI>(MG, grid, smem, s, a);
    if (E == 2) return dispatch_mg<KB, 2, NCI>(MG, grid, smem, s, a);
    return dispatch_mg<KB, 3, NCI>(MG, grid, smem, s, a);
}

template <int NCI>
int dispatch_sq(int KB, int E, int MG, dim3 grid, size_t smem, cudaStream_t s, const SqArgs &a) {
    switch (KB) {
        case 2: return dispatch_e<2, NCI>(E, MG, grid, smem, s, a);
        case 3: return dispatch_e<3, NCI>(E, MG, grid, smem, s, a);
        case 4: return dispatch_e<4, NCI>(E, MG, grid, smem, s, a);
        case 5: return dispatch_e<5, NCI>(E, MG, grid, smem, s, a);
    }
    he_set_error("he_conv_square_sum: no kernel for KB=%d", KB);
    return HE_EINVAL;
}

// instantiated in convsq.cu (NCI = 2) and convsq3.cu (NCI = 3)
int dispatch_sq2(int KB, int E, int MG, dim3 grid, size_t smem, cudaStream_t s, const SqArgs &a);
int dispatch_sq3(int KB, int E, int MG, dim3 grid, size_t smem, cudaStream_t s, const SqArgs &a);

}  // namespace convsq
