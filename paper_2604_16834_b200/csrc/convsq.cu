// convsq.cu -- fused feature-major 3x3 conv -> degree-2 activation (square,
// no relinearisation) -> 2x2 pool / global sum, on the tensor cores.
//
// Replaces the chain  conv_mma -> tensor_batch -> add_const -> lincomb_int
// (featuremajor.run_cnn, lazy + deferred plan) with one kernel that never
// materialises the conv output: for config 3's conv1 that map is 16384
// ciphertexts (240 GB at 14 limbs) written and read back once each.
//
// The kernel (tile layout, exact recombination, shared-memory ring) is in
// convsq_kernel.cuh; this file holds the NCI = 2 instantiations and the host
// entry points (B fragments, per-limb constants, limb groups, ring strides).
#include "convsq_kernel.cuh"

using namespace convsq;

int convsq::dispatch_sq2(int KB, int E, int MG, dim3 grid, size_t smem, cudaStream_t s, const SqArgs &a) {
    return dispatch_sq<2>(KB, E, MG, grid, smem, s, a);
}

namespace {

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
// of the square of y = sum_k weights[m][k] in[tap k] (+ bias[m] on component
// 0), then + cst on component 0.  Inputs in[i*H*W + y*W + x] are nci = 2 or 3
// components x ell limbs; outputs 2 nci - 1 components x ell limbs:
// (y0^2, 2 y0 y1, y1^2) or (y0^2, 2 y0 y1, 2 y0 y2 + y1^2, 2 y1 y2, y2^2) summed.  Tap order
// k = i*9 + (dy+1)*3 + (dx+1).  Returns HE_EINVAL when a tensor-core bound
// does not hold (p > 16, M > 32, |w| >= 2^23 or a prime below 2^36).
// out[m] (canonical, [NO][ell][N]) += part[m] (mod q of the limb)
__global__ void k_add_parts(uint64_t *const *out, const uint64_t *part, int M, int polys, int ell, int logN,
                            const ModConst *mc) {
    const size_t N = (size_t)1 << logN, per = (size_t)polys * N, tot = (size_t)M * per;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
        const size_t m = i / per, r = i % per;
        const uint64_t q = mc[(r >> logN) % ell].q;
        uint64_t *o = out[m] + r;
        *o = add_mod(*o, part[i], q);
    }
}

int he_conv_tc_enabled();  // convtc.cu

extern "C" int he_conv_square_sum_n(he_ctx *c, const uint64_t *const *in, int nci, int p, int H, int W,
                                    uint64_t *const *out, int M, int pool, int y0, int y1, const int64_t *weights,
                                    const uint64_t *bias, const uint64_t *cst, int ell, void *stream) {
    // the tcgen05 kernels (convtc.cu) take every shape they cover; the mma.sync
    // kernels below handle the rest (and serve as the A/B reference in tests)
    if (he_conv_tc_enabled() && he_conv_square_sum_tc(c, in, nci, p, H, W, out, M, pool, y0, y1, weights, bias, cst,
                                                       ell, stream) == HE_OK)
        return HE_OK;
    if (!c || !in || !out || !weights || p < 1 || H < 1 || W < 1 || M < 1 || ell < 1 || ell > c->L || y0 < 0 ||
        y1 > H || y0 >= y1 || (nci != 2 && nci != 3)) {
        he_set_error("he_conv_square_sum: bad arguments");
        return HE_EINVAL;
    }
    if (nci == 3 && (W & 1)) {
        he_set_error("he_conv_square_sum: 3-component inputs are processed in pixel pairs (even W)");
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
    // tap-8 packing (one channel group, 40-bit limbs): [MGk][4 + E][lane][2], entry s = byte
    // shift s; K word k (< 5) of the block is tap 8 of input byte plane k, so it carries
    // weight digit s - k (zero outside 0 .. E-1); words 5..7 are zero
    const int NSH8 = 4 + E;
    const bool ls8 = ncg == 4 && nci == 3 && E == 2;  // ldmatrix path: [W0 | 0], [W0 | W1], [0 | W1] of tap 8
    std::vector<uint32_t> bf8(ncg == 1 ? (size_t)MGk * NSH8 * 32 * 2 : ls8 ? (size_t)MGk * 3 * 32 * 2 : 0, 0);
    if (ls8)
        for (int cg = 0; cg < MGk; cg++)
            for (int k = 0; k < 3; k++)
                for (int lane = 0; lane < 32; lane++) {
                    const int gid = lane >> 2, tig = lane & 3, m = cg * 8 + gid;
                    for (int r = 0; r < 2; r++) {  // r = K half: 0 -> digit 0 (not for k = 2), 1 -> digit 1 (not k = 0)
                        uint32_t reg = 0;
                        const bool on = r == 0 ? k != 2 : k != 0;
                        if (on && m < M)
                            for (int u = 0; u < 4; u++) {
                                const int i = 4 * tig + u;  // channel group tig of tap 8
                                if (i < p) {
                                    const int dg = digit_s8(weights[(size_t)m * T + i * 9 + 8], r);
                                    reg |= (uint32_t)(uint8_t)(int8_t)dg << (8 * u);
                                }
                            }
                        bf8[(((size_t)cg * 3 + k) * 32 + lane) * 2 + r] = reg;
                    }
                }
    if (ncg == 1)
        for (int cg = 0; cg < MGk; cg++)
            for (int sh = 0; sh < NSH8; sh++)
                for (int lane = 0; lane < 32; lane++) {
                    const int gid = lane >> 2, tig = lane & 3, m = cg * 8 + gid;
                    for (int r = 0; r < 2; r++) {
                        const int k = r * 4 + tig, e = sh - k;  // plane k, weight digit e
                        uint32_t reg = 0;
                        if (k < 5 && e >= 0 && e < E && m < M)
                            for (int u = 0; u < 4; u++)
                                if (u < p) {
                                    const int dg = digit_s8(weights[(size_t)m * T + u * 9 + 8], e);
                                    reg |= (uint32_t)(uint8_t)(int8_t)dg << (8 * u);
                                }
                        bf8[(((size_t)cg * NSH8 + sh) * 32 + lane) * 2 + r] = reg;
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
    // column tiles (3-component GAP on the ldmatrix path, 40-bit limbs): two CTAs per
    // (limb, coefficient chunk) each own half the columns, so the ring (and shared
    // memory per CTA) halves and three CTAs fit an SM; tile 1 writes partial sums to
    // scratch, added into out afterwards
    const int tiles = (nci == 3 && !pool && ncg % 4 == 0 && W % 4 == 0 && W >= 16) ? 2 : 1;
    const int NO = 2 * nci - 1;
    uint64_t *part = nullptr;
    std::vector<const uint64_t *> outs((const uint64_t *const *)out, (const uint64_t *const *)out + n_out);
    if (tiles > 1) {  // tiles 1 .. T-1 write partial sums to scratch [T-1][M][NO][ell][N]
        const size_t per = (size_t)NO * ell * c->N, bytes = (size_t)(tiles - 1) * M * per * 8;
        HE_TRY(he_scratch_alloc((void **)&part, bytes, s));
        HE_CHECK_CUDA(cudaMemsetAsync(part, 0, bytes, s));
        for (int z = 1; z < tiles; z++)
            for (int m = 0; m < M; m++) outs.push_back(part + ((size_t)(z - 1) * M + m) * per);
    }
    HE_TRY(he_upload_ptrs((const void *const *)outs.data(), (int)outs.size(), &dout, s));
    const size_t b_bf8 = bf8.size() * 4;
    const size_t b_bf = bf.size() * 4, b_lo = lorder.size() * 4, b_r4 = (size_t)ell * 8, b_b = bres.size() * 8,
                 b_c = cst ? (size_t)ell * 8 : 0, b_yc = yc.size() * 8;
    char *meta = nullptr;
    HE_TRY(he_scratch_alloc((void **)&meta, b_bf + b_bf8 + b_lo + b_r4 + b_b + b_c + b_yc + 192, s));
    size_t off = 0;
    auto carve = [&](size_t bytes) {
        char *p = meta + off;
        off = (off + bytes + 15) & ~(size_t)15;
        return p;
    };
    uint32_t *dbf = (uint32_t *)carve(b_bf);
    uint32_t *dbf8 = b_bf8 ? (uint32_t *)carve(b_bf8) : nullptr;
    int32_t *dlo = (int32_t *)carve(b_lo);
    uint64_t *dr4 = (uint64_t *)carve(b_r4);
    uint64_t *db = bias ? (uint64_t *)carve(b_b) : nullptr;
    uint64_t *dc = cst ? (uint64_t *)carve(b_c) : nullptr;
    double *dyc = (double *)carve(b_yc);
    HE_CHECK_CUDA(he_h2d(dyc, yc.data(), b_yc, s));
    HE_CHECK_CUDA(he_h2d(dbf, bf.data(), b_bf, s));
    if (dbf8) HE_CHECK_CUDA(he_h2d(dbf8, bf8.data(), b_bf8, s));
    HE_CHECK_CUDA(he_h2d(dlo, lorder.data(), b_lo, s));
    HE_CHECK_CUDA(he_h2d(dr4, r4.data(), b_r4, s));
    if (db) HE_CHECK_CUDA(he_h2d(db, bres.data(), b_b, s));
    if (dc) HE_CHECK_CUDA(he_h2d(dc, cst, b_c, s));
    SqArgs a;
    a.in = (const uint64_t *const *)din;
    a.out = (uint64_t *const *)dout;
    a.bfrag = dbf;
    a.bfrag8 = dbf8;
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
        const bool tile_g = tiles > 1 && a.nb == 5;  // the ldmatrix kernel of this group takes tiles
        a.x0 = 0;
        a.Wt = tile_g ? W / tiles : W;
        if (ncg % 4 == 0) {
            a.pstr = a.nb * ncg * 8 * nci;
            a.rstr = (a.Wt + 2) * a.pstr;
            a.R = pool ? 4 : 3;
        } else {
            a.pstr = round_up_mod(a.nb * ncg * 8 * nci, 32, 24);
            a.rstr = round_up_mod((W + 2) * a.pstr, 32, 8);
            a.R = 4;
        }
        // ring + one row's input-address table (8-byte aligned: rstr is even)
        const size_t smem = (size_t)a.R * a.rstr * 4 + (size_t)p * (a.Wt + 2) * 8;
        if (smem > 227 * 1024) {
            he_set_error("he_conv_square_sum: row ring needs %zu bytes of shared memory (W=%d too wide)", smem, W);
            rc = HE_EINVAL;
            break;
        }
        dim3 grid((unsigned)(c->N / 8), (unsigned)g.second, tile_g ? (unsigned)tiles : 1u);
        rc = nci == 2 ? dispatch_sq2(KB, E, MGk, grid, smem, s, a) : dispatch_sq3(KB, E, MGk, grid, smem, s, a);
        if (rc != HE_OK) break;
        first += g.second;
    }
    if (rc == HE_OK && part) {  // out += tile-1 partial sums (zero for untiled limb groups)
        for (int z = 1; z < tiles && rc == HE_OK; z++) {
            k_add_parts<<<(unsigned)std::min<size_t>(((size_t)M * NO * ell * c->N + 255) / 256, (size_t)148 * 64), 256,
                          0, s>>>((uint64_t *const *)dout, part + (size_t)(z - 1) * M * NO * ell * c->N, M, NO * ell,
                                  ell, c->logN, c->d_mc);
            he_count_launch(1);
            if (cudaGetLastError() != cudaSuccess) rc = HE_ECUDA;
        }
    }
    if (part) he_scratch_free(part, s);
    he_scratch_free(meta, s);
    he_scratch_free(din, s);
    he_scratch_free(dout, s);
    return rc;
}

extern "C" int he_conv_square_sum(he_ctx *c, const uint64_t *const *in, int p, int H, int W, uint64_t *const *out,
                                  int M, int pool, int y0, int y1, const int64_t *weights, const uint64_t *bias,
                                  const uint64_t *cst, int ell, void *stream) {
    return he_conv_square_sum_n(c, in, 2, p, H, W, out, M, pool, y0, y1, weights, bias, cst, ell, stream);
}
