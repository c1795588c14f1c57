// mma.cu -- exact modular feature-major convolution on the tensor cores
// (int8 digit decomposition, mma.sync m16n8k32 u8 x s8 -> s32).
//
// For one output pixel g the conv is a tiny dense product
//     out[m] = sum_k W[m][k] * x_k          (k = the 9p taps, x_k residues < q)
// with W small signed integers (deferred-rescale weights, |W| < 2^31).  Split
//     x_k = sum_d x_{k,d} 256^d   (unsigned bytes: the uint64 residue's own
//                                   little-endian bytes, d < 8)
//     W   = sum_e W_e 256^e       (balanced signed bytes, e < E <= 4)
// then  sum_k W x = sum_{d,e} 256^(d+e) C[(j,d)][(e,m)],
//     C[(j,d)][(e,m)] = sum_k x_{k,j,d} W_e[m][k]      (exact int32)
// is an int8 GEMM: rows (coefficient j, digit d), columns (weight digit e,
// channel m), the taps as the reduction.  The recombination is exact in
// 128 bits, then one Montgomery pair reduces mod q_l, so the result is
// bit-identical to the CUDA-core he_lincomb_grouped.
//
// Data path per CTA (4 warps) = a group of pixels x a run of 16-coefficient
// chunks of one (component, limb):
//   gather  each thread loads 4 taps of one coefficient (coalesced over j),
//           4x4-byte-transposes them with PRMT into digit-planar words and
//           stores them as two 16-byte STS: xt[tap word][j][d]
//   MMA     every A register is one conflict-free 32-bit LDS; KB x (E*MG)
//           mma.sync per 16-row M-tile
//   reduce  in registers: sum over weight digits e, then a 3-step warp
//           reduce-scatter over the 8 digit lanes d (weights 2^(8d)); each
//           lane finishes 1-2 outputs (mod q_l, + bias) and stores them.
#include <algorithm>

#include "common.cuh"

namespace {

constexpr int MW = 4;            // warps per CTA
constexpr int CT = MW * 32;      // threads per CTA
constexpr int CC = 16;           // coefficients per chunk (8 M-tiles of 2 coefficients x 8 digits)
constexpr int CPB = 8;           // chunks per CTA
constexpr int SK = 168;          // 32-bit words per tap-word row (16 coefficients x 8 digits + pad); SK = 8 mod 32

__device__ __forceinline__ int jofs(int j) { return 8 * j + 4 * (j >> 2); }  // conflict-free STS.128 / LDS.32

struct MmaArgs {
    uint64_t *const *out;
    const uint64_t *const *in;
    const int32_t *gcol;     // [G][Tpad] input index, -1 = zero tap
    const int32_t *out_base; // [G]
    const uint32_t *bfrag;   // [KB][E*MG][32][2] weight-digit B fragments, columns n = e*Mpad + m
    const uint64_t *cres;    // [M][ell] constants for component 0, or nullptr
    const ModConst *mc;
    int out_stride, G, gpb, ngb, M, Tpad, KB, ell, logN, l_lo, nl;
};

__device__ __forceinline__ void mma_u8s8(int (&d)[4], const uint32_t (&a)[4], const uint2 b) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b.x), "r"(b.y));
}

// 4x4 byte transpose: out[d] = byte d of w0..w3 packed (w0 in the low byte)
__device__ __forceinline__ void tr4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t (&o)[4]) {
    const uint32_t t0 = __byte_perm(w0, w1, 0x5140), t1 = __byte_perm(w2, w3, 0x5140);
    const uint32_t t2 = __byte_perm(w0, w1, 0x7362), t3 = __byte_perm(w2, w3, 0x7362);
    o[0] = __byte_perm(t0, t1, 0x5410);
    o[1] = __byte_perm(t0, t1, 0x7632);
    o[2] = __byte_perm(t2, t3, 0x5410);
    o[3] = __byte_perm(t2, t3, 0x7632);
}

__device__ __forceinline__ __int128 shfl_xor128(__int128 v, int mask) {
    uint64_t lo = (uint64_t)v, hi = (uint64_t)(v >> 64);
    uint32_t a = __shfl_xor_sync(0xffffffffu, (uint32_t)lo, mask);
    uint32_t b = __shfl_xor_sync(0xffffffffu, (uint32_t)(lo >> 32), mask);
    uint32_t c = __shfl_xor_sync(0xffffffffu, (uint32_t)hi, mask);
    uint32_t d = __shfl_xor_sync(0xffffffffu, (uint32_t)(hi >> 32), mask);
    return (__int128)((((unsigned __int128)(((uint64_t)d << 32) | c)) << 64) | (((uint64_t)b << 32) | a));
}

// exact signed 128-bit -> canonical residue
__device__ __forceinline__ uint64_t mod_i128(__int128 T, const ModConst &c) {
    const int64_t hi = (int64_t)(T >> 64);
    const uint64_t lo = (uint64_t)T;
    uint64_t hic;
    if (hi >= 0) {
        hic = reduce64((uint64_t)hi, c);
    } else {
        const uint64_t r = reduce64((uint64_t)(-hi), c);
        hic = r ? c.q - r : 0;
    }
    const uint64_t t1 = redc(hic, lo, c.q, c.qinv);          // T 2^-64
    return redc(mulhi(t1, c.r2), t1 * c.r2, c.q, c.qinv);    // T
}

template <int E, int MG>
__global__ void __launch_bounds__(CT) k_conv_mma(const MmaArgs a) {
    constexpr int NT = E * MG;        // n-tiles
    constexpr int VR = 4 * MG;        // partial outputs per thread per M-tile
    constexpr int V = VR < 8 ? 8 : VR;  // >= 8 for the 3-step reduce-scatter (padding is zero)
    extern __shared__ __align__(16) uint8_t smraw[];
    uint2 *bfs = (uint2 *)smraw;
    uint32_t *xt = (uint32_t *)(smraw + (size_t)a.KB * NT * 32 * 8);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const int KW = a.Tpad / 4;

    for (int i = tid; i < a.KB * NT * 32; i += CT) bfs[i] = ((const uint2 *)a.bfrag)[i];

    const int N = 1 << a.logN;
    const int pl = blockIdx.y;                     // comp * nl + (limb - l_lo)
    const int l = a.l_lo + pl % a.nl, comp = pl / a.nl;
    const size_t base = ((size_t)comp * a.ell + l) * (size_t)N;
    const ModConst c = a.mc[l];
    const int nbytes = c.q < (1ull << 40) ? 5 : (c.q < (1ull << 48) ? 6 : (c.q < (1ull << 56) ? 7 : 8));
    const int gb = blockIdx.x % a.ngb, cb = blockIdx.x / a.ngb;
    const int g0 = gb * a.gpb, g1 = min(g0 + a.gpb, a.G);

    for (int ch = 0; ch < CPB; ch++) {
        const size_t off0 = base + (size_t)(cb * CPB + ch) * CC;
        for (int g = g0; g < g1; g++) {
            __syncthreads();  // previous readers of xt done (and bfs loaded)
            const int32_t *gc = a.gcol + (size_t)g * a.Tpad;
            // ---- gather + byte transpose: task = (tap word kw, coefficient j)
            for (int t = tid; t < KW * CC; t += CT) {
                const int j = t % CC, kw = t / CC;
                uint64_t x[4];
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const int col = gc[kw * 4 + i];
                    x[i] = col >= 0 ? __ldg(a.in[col] + off0 + j) : 0ull;
                }
                uint32_t lo[4], hi[4];
                tr4((uint32_t)x[0], (uint32_t)x[1], (uint32_t)x[2], (uint32_t)x[3], lo);
                tr4((uint32_t)(x[0] >> 32), (uint32_t)(x[1] >> 32), (uint32_t)(x[2] >> 32), (uint32_t)(x[3] >> 32), hi);
                uint4 *dst = (uint4 *)(xt + kw * SK + jofs(j));
                dst[0] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
                dst[1] = make_uint4(hi[0], hi[1], hi[2], hi[3]);
            }
            __syncthreads();
            const int ob = a.out_base[g];
            for (int mt = warp; mt < CC / 2; mt += MW) {
                const int j0 = 2 * mt;
                int acc[NT][4];
#pragma unroll
                for (int nt = 0; nt < NT; nt++) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0;
                const uint32_t *r0 = xt + jofs(j0) + gid, *r1 = xt + jofs(j0 + 1) + gid;
                for (int kb = 0; kb < a.KB; kb++) {
                    const int w0 = (kb * 8 + tig) * SK, w1 = (kb * 8 + 4 + tig) * SK;
                    const uint32_t af[4] = {r0[w0], r1[w0], r0[w1], r1[w1]};
#pragma unroll
                    for (int nt = 0; nt < NT; nt++) mma_u8s8(acc[nt], af, bfs[(kb * NT + nt) * 32 + lane]);
                }
                // ---- recombine: v[mg*4+q] = sum_e acc[e*MG+mg][q] 2^(8e), q = (m pair bit, j bit)
                __int128 val[V];
#pragma unroll
                for (int i = VR; i < V; i++) val[i] = 0;
#pragma unroll
                for (int mg = 0; mg < MG; mg++)
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        int64_t v = 0;
#pragma unroll
                        for (int e = 0; e < E; e++) v += (int64_t)acc[e * MG + mg][q] << (8 * e);
                        // digit d = gid of this lane: weight 2^(8d); rows of digits >= nbytes are zero
                        val[mg * 4 + q] = (__int128)v << (8 * gid);
                    }
                // ---- reduce-scatter over the 8 digit lanes (lane bits 4, 3, 2 = gid bits 2, 1, 0)
#pragma unroll
                for (int step = 0; step < 3; step++) {
                    const int h = V >> (step + 1);
                    const int bit = (gid >> (2 - step)) & 1;
                    const int mask = 16 >> step;
#pragma unroll
                    for (int t = 0; t < h; t++) {
                        const __int128 mine = bit ? val[t + h] : val[t];
                        const __int128 other = bit ? val[t] : val[t + h];
                        val[t] = mine + shfl_xor128(other, mask);
                    }
                }
                // lane now holds V/8 finished sums; original index of val[t]:
                const int bidx = ((gid >> 2) & 1) * (V / 2) + ((gid >> 1) & 1) * (V / 4) + (gid & 1) * (V / 8);
#pragma unroll
                for (int t = 0; t < V / 8; t++) {
                    const int idx = bidx + t, mg = idx >> 2, q = idx & 3;
                    const int m = mg * 8 + 2 * tig + (q & 1), j = j0 + (q >> 1);
                    if (idx < VR && m < a.M) {
                        uint64_t v = mod_i128(val[t], c);
                        if (a.cres && comp == 0) v = add_mod(v, a.cres[(size_t)m * a.ell + l], c.q);
                        a.out[ob + m * a.out_stride][off0 + j] = v;
                    }
                }
            }
        }
    }
    (void)nbytes;
}

template <int E, int MG>
int launch_mma(dim3 grid, size_t smem, cudaStream_t s, const MmaArgs &a) {
    if (smem > 48 * 1024)
        HE_CHECK_CUDA(cudaFuncSetAttribute(k_conv_mma<E, MG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_conv_mma<E, MG><<<grid, CT, smem, s>>>(a);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

int dispatch_mma(int E, int MG, dim3 grid, size_t smem, cudaStream_t s, const MmaArgs &a) {
#define HE_MMA_CASE(e, mg) \
    if (E == e && MG == mg) return launch_mma<e, mg>(grid, smem, s, a);
    HE_MMA_CASE(1, 1) HE_MMA_CASE(1, 2) HE_MMA_CASE(1, 3) HE_MMA_CASE(1, 4)
    HE_MMA_CASE(2, 1) HE_MMA_CASE(2, 2) HE_MMA_CASE(2, 3) HE_MMA_CASE(2, 4)
    HE_MMA_CASE(3, 1) HE_MMA_CASE(3, 2) HE_MMA_CASE(3, 3) HE_MMA_CASE(3, 4)
    HE_MMA_CASE(4, 1) HE_MMA_CASE(4, 2) HE_MMA_CASE(4, 3)
#undef HE_MMA_CASE
    he_set_error("he_conv_mma: no kernel for E=%d MG=%d", E, MG);
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

// Tensor-core exact conv lincomb: every group g has exactly T tap slots
// (gcol[g][t] = input index or -1), out[out_base[g] + m*out_stride] =
// sum_t weights[m][t] * in[gcol[g][t]] mod q (+ residues[m] on component 0).
// Requires N % 128 == 0, |weights| < 2^31 (E <= 4 signed digits) and
// E * ceil(M/8) <= 12.  Returns HE_EINVAL when a bound does not hold
// (callers fall back to he_lincomb_grouped).
extern "C" int he_conv_mma(he_ctx *c, const uint64_t *const *in, int n_in, uint64_t *const *out, int n_out,
                           int n_groups, const int32_t *gcol, const int32_t *out_base, int out_stride, int M, int T,
                           const int64_t *weights, const uint64_t *residues, int ell, int nc, void *stream) {
    if (!c || n_in < 1 || n_groups < 0 || M < 1 || T < 1 || ell < 1 || ell > c->L || nc < 1 || nc > 3 || !gcol ||
        !out_base || !weights || c->N % (CC * CPB)) {
        he_set_error("he_conv_mma: bad arguments");
        return HE_EINVAL;
    }
    if (!n_groups) return HE_OK;
    int64_t wmax = 0;
    for (int i = 0; i < M * T; i++) wmax = std::max<int64_t>(wmax, weights[i] < 0 ? -weights[i] : weights[i]);
    // balanced E-digit signed base-256 numbers cover |w| <= 127 * (256^E - 1) / 255
    int E = 1;
    int64_t cap = 127;
    while (wmax > cap && E < 4) {
        E++;
        cap = cap * 256 + 127;
    }
    if (wmax > cap) {
        he_set_error("he_conv_mma: weights need more than 4 signed byte digits");
        return HE_EINVAL;
    }
    const int MG = (M + 7) / 8, Mpad = MG * 8, NT = E * MG;
    if (NT > 12 || MG > 4) {
        he_set_error("he_conv_mma: E*ceil(M/8) = %d exceeds 12 n-tiles", NT);
        return HE_EINVAL;
    }
    const int Tpad = (T + 31) / 32 * 32, KB = Tpad / 32;
    for (int g = 0; g < n_groups; g++) {
        if (out_base[g] < 0 || out_base[g] + (M - 1) * out_stride >= n_out) {
            he_set_error("he_conv_mma: outputs of group %d out of range", g);
            return HE_EINVAL;
        }
        for (int t = 0; t < T; t++)
            if (gcol[(size_t)g * T + t] >= n_in) {
                he_set_error("he_conv_mma: group %d tap %d input out of range", g, t);
                return HE_EINVAL;
            }
    }
    if (residues)
        for (int i = 0; i < M * ell; i++)
            if (residues[i] >= c->mod[i % ell]) {
                he_set_error("he_conv_mma: residue not canonical");
                return HE_EINVAL;
            }
    // B fragments: b.x = k in [tig*4, tig*4+4), b.y = k + 16; column n = gid -> (e, m) = (n / Mpad, n % Mpad)
    std::vector<uint32_t> bf((size_t)KB * NT * 32 * 2, 0);
    for (int kb = 0; kb < KB; kb++)
        for (int nt = 0; nt < NT; nt++)
            for (int lane = 0; lane < 32; lane++) {
                const int gid = lane >> 2, tig = lane & 3, n = nt * 8 + gid, e = n / Mpad, m = n % Mpad;
                for (int r = 0; r < 2; r++) {
                    uint32_t reg = 0;
                    for (int i = 0; i < 4; i++) {
                        const int k = kb * 32 + r * 16 + tig * 4 + i;
                        int dg = 0;
                        if (m < M && k < T) dg = digit_s8(weights[(size_t)m * T + k], e);
                        reg |= (uint32_t)(uint8_t)(int8_t)dg << (8 * i);
                    }
                    bf[(((size_t)kb * NT + nt) * 32 + lane) * 2 + r] = reg;
                }
            }
    std::vector<int32_t> gc((size_t)n_groups * Tpad, -1);
    for (int g = 0; g < n_groups; g++)
        for (int t = 0; t < T; t++) gc[(size_t)g * Tpad + t] = gcol[(size_t)g * T + t];
    cudaStream_t s = (cudaStream_t)stream;
    void **din = nullptr, **dout = nullptr;
    HE_TRY(he_upload_ptrs((const void *const *)in, n_in, &din, s));
    HE_TRY(he_upload_ptrs((const void *const *)out, n_out, &dout, s));
    const size_t b_bf = bf.size() * 4, b_gc = gc.size() * 4, b_ob = (size_t)n_groups * 4,
                 b_res = residues ? (size_t)M * ell * 8 : 0;
    char *meta = nullptr;
    HE_TRY(he_scratch_alloc((void **)&meta, b_bf + b_gc + b_ob + b_res + 64, s));
    uint32_t *dbf = (uint32_t *)meta;
    int32_t *dgc = (int32_t *)(meta + b_bf);
    int32_t *dob = (int32_t *)(meta + b_bf + b_gc);
    uint64_t *dres = residues ? (uint64_t *)(meta + ((b_bf + b_gc + b_ob + 7) & ~(size_t)7)) : nullptr;
    HE_CHECK_CUDA(he_h2d(dbf, bf.data(), b_bf, s));
    HE_CHECK_CUDA(he_h2d(dgc, gc.data(), b_gc, s));
    HE_CHECK_CUDA(he_h2d(dob, out_base, b_ob, s));
    if (residues) HE_CHECK_CUDA(he_h2d(dres, residues, b_res, s));
    MmaArgs a;
    a.out = (uint64_t *const *)dout;
    a.in = (const uint64_t *const *)din;
    a.gcol = dgc;
    a.out_base = dob;
    a.bfrag = dbf;
    a.cres = dres;
    a.mc = c->d_mc;
    a.out_stride = out_stride;
    a.G = n_groups;
    a.gpb = std::max(1, std::min(4, n_groups / 64));
    a.ngb = (n_groups + a.gpb - 1) / a.gpb;
    a.M = M;
    a.Tpad = Tpad;
    a.KB = KB;
    a.ell = ell;
    a.logN = c->logN;
    a.l_lo = 0;
    a.nl = ell;
    const size_t smem = (size_t)KB * NT * 32 * 8 + (size_t)(Tpad / 4) * SK * 4;
    int rc = HE_OK;
    if (smem > 220 * 1024) {
        he_set_error("he_conv_mma: %zu bytes of shared memory", smem);
        rc = HE_EINVAL;
    }
    const size_t chunks = (size_t)c->N / (CC * CPB);
    dim3 grid((unsigned)(a.ngb * chunks), (unsigned)(nc * ell));
    if (rc == HE_OK) rc = dispatch_mma(E, MG, grid, smem, s, a);
    he_scratch_free(meta, s);
    he_scratch_free(din, s);
    he_scratch_free(dout, s);
    return rc;
}
