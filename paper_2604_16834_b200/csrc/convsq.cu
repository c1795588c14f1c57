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
// mma.sync m16n8k32 u8 x s8 per (input byte plane d, 32-byte K block, weight
// digit e).  Byte planes beyond the limb's length (5 for 40-bit primes) are
// skipped.  The lane recombines its values exactly (int32 sums per byte
// shift, IMAD.WIDE into int64 partial sums at 2^0 / 2^32 / 2^64, one signed
// 128-bit total), reduces with ONE Montgomery step (y R^-1), accumulates the
// window's squares as exact 128-bit sums and reduces them once; the window
// result is scaled back with R^4 and stored as three components.
// Bit-identical to conv -> tensor -> add_const -> sum: every step is exact
// arithmetic mod q.
//
// Data path: the K dimension is ordered (tap, group of 4 input channels), so
// one 32-bit A-operand word is "byte d of 4 channels at one input pixel".
// Input rows are loaded ONCE per CTA into a shared-memory ring (R rows x
// (W+2) pixels incl. a zero halo), byte-transposed with PRMT into that
// digit-planar, channel-interleaved layout; every output pixel then reads its
// 9 taps straight from the ring (no per-tap gather).  Strides are chosen so
// the A-fragment loads are bank-conflict free.  Weight digits stay in
// registers for the whole kernel.
#include <algorithm>

#include "ntt_core.cuh"  // u2d / d2u / fmulmod / fcanon (FP64 modular products)

namespace {

constexpr int CT = 128;  // 4 warps: MG channel groups x PS pixel streams

struct SqArgs {
    const uint64_t *const *in;  // [p*H*W] 2-component input ciphertexts (device array of addresses)
    uint64_t *const *out;       // 3-component outputs, ell limbs
    const uint32_t *bfrag;      // [MG][KB][E][32] uint2 B fragments
    const uint64_t *bias;       // [M][ell] bias * R^-1 mod q (component 0), or nullptr
    const uint64_t *cst;        // [ell] constant added to component 0 of every output, or nullptr
    const uint64_t *r4;         // [ell] R^4 mod q
    const double *yc;           // [ell][2] R mod q and 2^32 mod q as doubles (FP64 recombination)
    const ModConst *mc;
    const int32_t *limbs;       // [gridDim.y] limb handled by blockIdx.y (one byte-plane count per launch)
    int p, H, W, M, ell, logN, pool, y0, y1, nwin;
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

// row r of channel group cg inside a pixel: groups 2, 3 swap their halves so
// the four groups read by one A-fragment load hit 32 distinct banks
__device__ __forceinline__ int rowpos(int cg, int r) { return cg * 16 + (r ^ (8 * ((cg >> 1) & 1))); }

// Input row yy -> ring slot: word (x' + 1) * pstr + d * (16 ncg) + rowpos(cg, comp*8 + j)
// holds byte d of channels 4cg .. 4cg+3 at pixel (yy, x'), coefficient j of component comp.
__device__ __forceinline__ void load_row(const SqArgs &a, uint32_t *slot, int yy, int l, size_t coff) {
    const size_t N = (size_t)1 << a.logN;
    const int dstr = 16 * a.ncg, ntask = a.W * a.ncg * 16;
    const bool inside = yy >= 0 && yy < a.H;
    for (int t = threadIdx.x; t < ntask; t += CT) {
        const int r = t & 15, rest = t >> 4, cg = rest % a.ncg, x = rest / a.ncg;
        uint64_t v[4] = {0, 0, 0, 0};
        if (inside) {
            const size_t off = ((size_t)(r >> 3) * a.ell + l) * N + coff + (r & 7);
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int i = cg * 4 + u;
                if (i < a.p) v[u] = __ldg(a.in[(size_t)i * a.H * a.W + yy * a.W + x] + off);
            }
        }
        uint32_t lo[4], hi[4];
        tr4((uint32_t)v[0], (uint32_t)v[1], (uint32_t)v[2], (uint32_t)v[3], lo);
        tr4((uint32_t)(v[0] >> 32), (uint32_t)(v[1] >> 32), (uint32_t)(v[2] >> 32), (uint32_t)(v[3] >> 32), hi);
        uint32_t *dst = slot + (x + 1) * a.pstr + rowpos(cg, r);
#pragma unroll
        for (int d = 0; d < 4; d++) dst[d * dstr] = lo[d];
#pragma unroll
        for (int d = 0; d < 4; d++)
            if (d + 4 < a.nb) dst[(d + 4) * dstr] = hi[d];
    }
}

// One input byte plane D: C[e] = sum_k byte_D(x_k) W_e[k] on the tensor cores,
// then the exact recombination.  W[j][q] is the int32 sum of the products with
// byte shift D + j still open (|C| < 2^23, <= E terms: no overflow); a
// completed shift s is folded into P[s/4] with one IMAD.WIDE by 2^(8 (s%4))
// (multipliers held in registers so ptxas keeps IMAD.WIDE).
template <int D, int KB, int E, int NB, int DSTR>
__device__ __forceinline__ void digit_plane(const uint32_t *X, const int (&o0)[KB][2], const int (&o1)[KB][2],
                                            const uint2 (&bw)[KB][E], int (&W)[E][4], int64_t (&P)[3][4],
                                            const int (&mul)[4]) {
    if (D >= NB) return;
    const uint32_t *Xd = X + D * DSTR;  // compile-time plane offset: an LDS immediate
    int C[E][4];
#pragma unroll
    for (int e = 0; e < E; e++) C[e][0] = C[e][1] = C[e][2] = C[e][3] = 0;
#pragma unroll
    for (int kb = 0; kb < KB; kb++) {
        const uint32_t a0 = Xd[o0[kb][0]], a1 = Xd[o1[kb][0]], a2 = Xd[o0[kb][1]], a3 = Xd[o1[kb][1]];
#pragma unroll
        for (int e = 0; e < E; e++) mma_u8s8(C[e], a0, a1, a2, a3, bw[kb][e]);
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
#pragma unroll
        for (int e = 0; e < E; e++) W[e][q] += C[e][q];
        madw(P[D >> 2][q], W[0][q], mul[D & 3]);  // shift D is complete
#pragma unroll
        for (int j = 0; j + 1 < E; j++) W[j][q] = W[j + 1][q];
        W[E - 1][q] = 0;
    }
    if (D == NB - 1) {  // last byte plane: flush shifts NB .. NB + E - 2
#pragma unroll
        for (int j = 0; j + 1 < E; j++)
#pragma unroll
            for (int q = 0; q < 4; q++) madw(P[(D + 1 + j) >> 2][q], W[j][q], mul[(D + 1 + j) & 3]);
    }
}

// Window sums of the squares (y0^2, y0 y1, y1^2) of y = conv * R^-1.
// 40-bit primes (NB = 5): exact FP64 modular products accumulated as doubles
// (|sum| < 2q per product, folded every 64), which moves the squares to the FP64
// pipe while the integer pipe recombines; wider primes: exact 128-bit sums.
// value(k) returns the canonical sum in the plain domain (times R^2, or R^4
// after the 128-bit path's extra Montgomery step).
template <bool FP>
struct SqAcc;
template <>
struct SqAcc<true> {
    double a[3] = {0.0, 0.0, 0.0};
    int n = 0;
    __device__ __forceinline__ void add(uint64_t y0, uint64_t y1, const ModConst &c) { addd(u2d(y0), u2d(y1), c); }
    __device__ __forceinline__ void addd(double d0, double d1, const ModConst &c) {  // canonical doubles
        a[0] += fmulmod(d0, d0, c.qd, c.qid);
        a[1] += fmulmod(d0, d1, c.qd, c.qid);
        a[2] += fmulmod(d1, d1, c.qd, c.qid);
        if (++n == 64) {
            n = 0;
#pragma unroll
            for (int k = 0; k < 3; k++) a[k] = u2d(fcanon(a[k], c.qd, c.qid));
        }
    }
    __device__ __forceinline__ uint64_t value(int k, const ModConst &c, uint64_t) const {
        return fcanon(a[k], c.qd, c.qid);  // the FP path squares the plain conv value
    }
    __device__ __forceinline__ void reset() { a[0] = a[1] = a[2] = 0.0; n = 0; }
};
template <>
struct SqAcc<false> {
    u128 a[3] = {{0, 0}, {0, 0}, {0, 0}};
    int n = 0;
    __device__ __forceinline__ void add(uint64_t y0, uint64_t y1, const ModConst &c) {
        mac128(a[0], y0, y0);
        mac128(a[1], y0, y1);
        mac128(a[2], y1, y1);
        if (++n == 8) {  // each product adds < q/16 to hi: fold every 8
            n = 0;
#pragma unroll
            for (int k = 0; k < 3; k++)
                if (a[k].hi >= c.q) a[k].hi -= c.q;
        }
    }
    __device__ __forceinline__ uint64_t value(int k, const ModConst &c, uint64_t r4) const {
        const uint64_t hi = a[k].hi >= c.q ? a[k].hi - c.q : a[k].hi;
        return mont(redc(hi, a[k].lo, c.q, c.qinv), r4, c);  // sum R^-3 -> plain
    }
    __device__ __forceinline__ void reset() {
        a[0] = a[1] = a[2] = u128{0, 0};
        n = 0;
    }
};

template <int KB, int E, int MG, int NB>
__global__ void __launch_bounds__(CT, KB <= 2 ? 4 : 3) k_conv_sqsum(const SqArgs a) {
    constexpr int PS = 4 / MG;
    extern __shared__ __align__(16) uint32_t xs[];  // ring [R][rstr]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const int cg = warp % MG, ps = warp / MG;
    const int l = a.limbs[blockIdx.y];
    const size_t N = (size_t)1 << a.logN, coff = (size_t)blockIdx.x * 8;
    const ModConst c = a.mc[l];
    constexpr int NCG = KB == 2 ? 1 : KB - 1;  // channel groups of 4 implied by the K blocks
    constexpr int DSTR = 16 * NCG;

    uint2 bw[KB][E];
#pragma unroll
    for (int kb = 0; kb < KB; kb++)
#pragma unroll
        for (int e = 0; e < E; e++) bw[kb][e] = ((const uint2 *)a.bfrag)[((cg * KB + kb) * E + e) * 32 + lane];
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
            const int r0 = rowpos(g, gid), r1 = rowpos(g, gid + 8);
            wd[kb][h] = (((t % 3) * a.pstr + r0) << 3) | (r1 < r0 ? 4 : 0) | (t / 3);
        }

    for (int i = tid; i < a.R * a.rstr; i += CT) xs[i] = 0;  // zero halo pixels stay zero
    __syncthreads();
    const int R = a.R, nrow0 = a.pool ? 4 : 3;
    for (int k = 0; k < nrow0; k++) {
        const int yy = a.y0 - 1 + k;
        load_row(a, xs + ((yy + R) % R) * a.rstr, yy, l, coff);
    }
    __syncthreads();

    SqAcc<NB == 5> acc[2];  // window sums for this lane's two channels
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
                int64_t P[3][4];  // partial sums at 2^0, 2^32, 2^64 for the 4 fragment values
#pragma unroll
                for (int hh = 0; hh < 3; hh++) P[hh][0] = P[hh][1] = P[hh][2] = P[hh][3] = 0;
                int W[E][4];
#pragma unroll
                for (int j = 0; j < E; j++) W[j][0] = W[j][1] = W[j][2] = W[j][3] = 0;
                digit_plane<0, KB, E, NB, DSTR>(xs, o0, o1, bw, W, P, mul);
                digit_plane<1, KB, E, NB, DSTR>(xs, o0, o1, bw, W, P, mul);
                digit_plane<2, KB, E, NB, DSTR>(xs, o0, o1, bw, W, P, mul);
                digit_plane<3, KB, E, NB, DSTR>(xs, o0, o1, bw, W, P, mul);
                digit_plane<4, KB, E, NB, DSTR>(xs, o0, o1, bw, W, P, mul);
                digit_plane<5, KB, E, NB, DSTR>(xs, o0, o1, bw, W, P, mul);
                digit_plane<6, KB, E, NB, DSTR>(xs, o0, o1, bw, W, P, mul);
                digit_plane<7, KB, E, NB, DSTR>(xs, o0, o1, bw, W, P, mul);
                // fragment values: q=0,1 -> component 0, channels m0, m0+1; q=2,3 -> component 1
                if constexpr (NB == 5) {
                    // 40-bit primes: shifts stop at 6, so T = P0 + P1 2^32 with |P0|, |P1| < 2^50;
                    // y = T mod q with one FP64 modular product (exact, see fmulmod); the
                    // squares are taken of the plain value (no Montgomery factor on this path)
                    double yd[4];
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const double p0 = __longlong_as_double(0x4338000000000000ll + P[0][q]) - 6755399441055744.0;
                        const double p1 = __longlong_as_double(0x4338000000000000ll + P[1][q]) - 6755399441055744.0;
                        yd[q] = p0 + fmulmod(p1, yc1, c.qd, c.qid);  // T = P0 + P1 2^32 (mod q), |T'| < 2^51
                    }
#pragma unroll
                    for (int h = 0; h < 2; h++)
                        acc[h].addd(fcanond(yd[h] + biasd[h], c.qd, c.qid), fcanond(yd[2 + h], c.qd, c.qid), c);
                } else {
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
                        for (int k = 0; k < 3; k++) {
                            uint64_t v = acc[h].value(k, c, r4);
                            if (k == 1) v = add_mod(v, v, c.q);
                            if (k == 0) v = add_mod(v, cst, c.q);
                            o[((size_t)k * a.ell + l) * N] = v;
                        }
                    }
                    acc[h].reset();
                }
            }
        }
        // slide the ring: the rows of this block's top are no longer needed
        const int ynext = yb + rows_per_blk;
        if (ynext < a.y1) {
            __syncthreads();
            for (int k = 0; k < rows_per_blk; k++) {
                const int yy = ynext + 1 + k;  // pool: rows ynext+1, ynext+2; GAP: row ynext+1
                load_row(a, xs + ((yy + R) % R) * a.rstr, yy, l, coff);
            }
            __syncthreads();
        }
    }
    if (!a.pool) {  // global sum: reduce, combine the pixel streams, then store
        uint64_t r[3][2];
        const uint64_t r4v = a.r4[l];
#pragma unroll
        for (int k = 0; k < 3; k++)
#pragma unroll
            for (int h = 0; h < 2; h++) r[k][h] = acc[h].value(k, c, r4v);
        uint64_t *red = (uint64_t *)xs;
        if (PS > 1) {
            __syncthreads();
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
            const uint64_t cst = a.cst ? a.cst[l] : 0;
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int m = m0 + h;
                if (m >= a.M) continue;
                uint64_t *o = a.out[m] + coff + gid;
#pragma unroll
                for (int k = 0; k < 3; k++) {
                    uint64_t v = k == 1 ? add_mod(r[k][h], r[k][h], c.q) : r[k][h];
                    if (k == 0) v = add_mod(v, cst, c.q);
                    o[((size_t)k * a.ell + l) * N] = v;
                }
            }
        }
    }
}

template <int KB, int E, int MG, int NB>
int launch_sq(dim3 grid, size_t smem, cudaStream_t s, const SqArgs &a) {
    if (smem > 48 * 1024)
        HE_CHECK_CUDA(cudaFuncSetAttribute(k_conv_sqsum<KB, E, MG, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
    k_conv_sqsum<KB, E, MG, NB><<<grid, CT, smem, s>>>(a);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

template <int KB, int E, int MG>
int dispatch_nb(dim3 grid, size_t smem, cudaStream_t s, const SqArgs &a) {
    return a.nb == 5 ? launch_sq<KB, E, MG, 5>(grid, smem, s, a) : launch_sq<KB, E, MG, 8>(grid, smem, s, a);
}

template <int KB, int E>
int dispatch_mg(int MG, dim3 grid, size_t smem, cudaStream_t s, const SqArgs &a) {
    if (MG == 1) return dispatch_nb<KB, E, 1>(grid, smem, s, a);
    if (MG == 2) return dispatch_nb<KB, E, 2>(grid, smem, s, a);
    return dispatch_nb<KB, E, 4>(grid, smem, s, a);
}

template <int KB>
int dispatch_e(int E, int MG, dim3 grid, size_t smem, cudaStream_t s, const SqArgs &a) {
    if (E == 1) return dispatch_mg<KB, 1>(MG, grid, smem, s, a);
    if (E == 2) return dispatch_mg<KB, 2>(MG, grid, smem, s, a);
    return dispatch_mg<KB, 3>(MG, grid, smem, s, a);
}

int dispatch_sq(int KB, int E, int MG, dim3 grid, size_t smem, cudaStream_t s, const SqArgs &a) {
    switch (KB) {
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

int round_up_mod(int v, int mod, int rem) {  // smallest v' >= v with v' = rem (mod mod)
    while (((v % mod) + mod) % mod != rem) v++;
    return v;
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
// does not hold (p > 16, M > 32, |w| >= 2^23 or a prime below 2^36).
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
    const int T = 9 * p, ncg = (p + 3) / 4, KB = std::max(2, (9 * ncg + 7) / 8), MG = (M + 7) / 8;
    if (p > 16 || M > 32 || c->N % 8 || c->N < 8) {
        he_set_error("he_conv_square_sum: p=%d input / M=%d output channels beyond the fused kernel", p, M);
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
    // B fragments [MGk][KB][E][lane][2]: b.x = K word kb*8 + tig, b.y = word kb*8 + 4 + tig;
    // word w = (tap t = w / ncg, channel group g = w % ncg), byte u -> channel 4g + u; column gid -> channel m
    std::vector<uint32_t> bf((size_t)MGk * KB * E * 32 * 2, 0);
    for (int cg = 0; cg < MGk; cg++)
        for (int kb = 0; kb < KB; kb++)
            for (int e = 0; e < E; e++)
                for (int lane = 0; lane < 32; lane++) {
                    const int gid = lane >> 2, tig = lane & 3, m = cg * 8 + gid;
                    for (int r = 0; r < 2; r++) {
                        const int w = kb * 8 + r * 4 + tig, t = w / ncg, g = w % ncg;
                        uint32_t reg = 0;
                        for (int u = 0; u < 4; u++) {
                            const int i = 4 * g + u;
                            const int dg = (m < M && t < 9 && i < p) ? digit_s8(weights[(size_t)m * T + i * 9 + t], e) : 0;
                            reg |= (uint32_t)(uint8_t)(int8_t)dg << (8 * u);
                        }
                        bf[((((size_t)cg * KB + kb) * E + e) * 32 + lane) * 2 + r] = reg;
                    }
                }
    // per-limb constants: R^4, bias * R^-1, and R^-1, 2^32 R^-1 as doubles
    std::vector<uint64_t> r4(ell), bres(bias ? (size_t)M * ell : 0);
    std::vector<double> yc(2 * (size_t)ell);
    for (int l = 0; l < ell; l++) {
        const uint64_t q = c->mod[l], Rm = (uint64_t)(((unsigned __int128)1 << 64) % q);
        const uint64_t R2 = he_h_mulmod(Rm, Rm, q);
        r4[l] = he_h_mulmod(R2, R2, q);
        const uint64_t Ri = he_h_inv(Rm, q);
        yc[2 * l] = (double)Rm;                          // R mod q: bias R^-1 -> plain
        yc[2 * l + 1] = (double)(((uint64_t)1 << 32) % q);  // 2^32 mod q
        (void)Ri;
        if (cst && cst[l] >= q) {
            he_set_error("he_conv_square_sum: residue not canonical");
            return HE_EINVAL;
        }
        if (bias) {
            const uint64_t Rinv = he_h_inv(Rm, q);
            for (int m = 0; m < M; m++) {
                if (bias[(size_t)m * ell + l] >= q) {
                    he_set_error("he_conv_square_sum: residue not canonical");
                    return HE_EINVAL;
                }
                bres[(size_t)m * ell + l] = he_h_mulmod(bias[(size_t)m * ell + l], Rinv, q);
            }
        }
    }
    // limbs grouped by byte length (one launch, one ring layout per group)
    std::vector<int32_t> lorder;
    std::vector<std::pair<int, int>> groups;  // (nb, count)
    for (int nb = 5; nb <= 8; nb += 3) {  // 40-bit primes: 5 byte planes; anything longer: all 8
        int n = 0;
        for (int l = 0; l < ell; l++) {
            const int b = c->mod[l] < (1ull << 40) ? 5 : 8;
            if (b == nb) {
                lorder.push_back(l);
                n++;
            }
        }
        if (n) groups.push_back({nb, n});
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int nwin = pool ? ((y1 - y0) / 2) * (W / 2) : 1;
    const int n_in = p * H * W, n_out = pool ? M * nwin : M;
    void **din = nullptr, **dout = nullptr;
    HE_TRY(he_upload_ptrs((const void *const *)in, n_in, &din, s));
    HE_TRY(he_upload_ptrs((const void *const *)out, n_out, &dout, s));
    const size_t b_bf = bf.size() * 4, b_lo = lorder.size() * 4, b_r4 = (size_t)ell * 8, b_b = bres.size() * 8,
                 b_c = cst ? (size_t)ell * 8 : 0, b_yc = yc.size() * 8;
    char *meta = nullptr;
    HE_TRY(he_scratch_alloc((void **)&meta, b_bf + b_lo + b_r4 + b_b + b_c + b_yc + 160, s));
    size_t off = 0;
    auto carve = [&](size_t bytes) {
        char *p = meta + off;
        off = (off + bytes + 15) & ~(size_t)15;
        return p;
    };
    uint32_t *dbf = (uint32_t *)carve(b_bf);
    int32_t *dlo = (int32_t *)carve(b_lo);
    uint64_t *dr4 = (uint64_t *)carve(b_r4);
    uint64_t *db = bias ? (uint64_t *)carve(b_b) : nullptr;
    uint64_t *dc = cst ? (uint64_t *)carve(b_c) : nullptr;
    double *dyc = (double *)carve(b_yc);
    HE_CHECK_CUDA(he_h2d(dyc, yc.data(), b_yc, s));
    HE_CHECK_CUDA(he_h2d(dbf, bf.data(), b_bf, s));
    HE_CHECK_CUDA(he_h2d(dlo, lorder.data(), b_lo, s));
    HE_CHECK_CUDA(he_h2d(dr4, r4.data(), b_r4, s));
    if (db) HE_CHECK_CUDA(he_h2d(db, bres.data(), b_b, s));
    if (dc) HE_CHECK_CUDA(he_h2d(dc, cst, b_c, s));
    SqArgs a;
    a.in = (const uint64_t *const *)din;
    a.out = (uint64_t *const *)dout;
    a.bfrag = dbf;
    a.bias = db;
    a.cst = dc;
    a.r4 = dr4;
    a.yc = dyc;
    a.mc = c->d_mc;
    a.p = p;
    a.H = H;
    a.W = W;
    a.M = M;
    a.ell = ell;
    a.logN = c->logN;
    a.pool = pool;
    a.y0 = y0;
    a.y1 = y1;
    a.nwin = nwin;
    a.ncg = ncg;
    for (int k = 0; k < 4; k++) a.mul[k] = 1 << (8 * k);
    int rc = HE_OK, first = 0;
    for (auto &g : groups) {
        a.nb = g.first;
        a.limbs = dlo + first;
        // bank-conflict-free A loads: with 4 channel groups per tap the 4 groups
        // fill the 32 banks by themselves; otherwise consecutive taps must sit
        // 8 banks apart (pixel stride = 24, ring-row stride = 8 mod 32, 4 rows)
        if (ncg % 4 == 0) {
            a.pstr = a.nb * ncg * 16;
            a.rstr = (W + 2) * a.pstr;
            a.R = pool ? 4 : 3;
        } else {
            a.pstr = round_up_mod(a.nb * ncg * 16, 32, 24);
            a.rstr = round_up_mod((W + 2) * a.pstr, 32, 8);
            a.R = 4;
        }
        const size_t smem = (size_t)a.R * a.rstr * 4;
        if (smem > 227 * 1024) {
            he_set_error("he_conv_square_sum: row ring needs %zu bytes of shared memory (W=%d too wide)", smem, W);
            rc = HE_EINVAL;
            break;
        }
        dim3 grid((unsigned)(c->N / 8), (unsigned)g.second);
        rc = dispatch_sq(KB, E, MGk, grid, smem, s, a);
        if (rc != HE_OK) break;
        first += g.second;
    }
    he_scratch_free(meta, s);
    he_scratch_free(din, s);
    he_scratch_free(dout, s);
    return rc;
}
