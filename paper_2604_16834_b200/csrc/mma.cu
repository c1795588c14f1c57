// mma.cu -- exact modular feature-major convolution on the tensor cores
// (int8 digit decomposition, mma.sync m16n8k32 u8 x s8 -> s32).
//
// For one output pixel g the conv is a tiny dense product
//     out[m] = sum_k W[m][k] * x_k          (k = the 9p taps, x_k residues < q)
// with W small signed integers (deferred-rescale weights, |W| < 2^23).  Split
//     x_k = sum_d x_{k,d} 256^d   (unsigned bytes: the uint64 residue's own
//                                   little-endian bytes, d < 8)
//     W   = sum_e W_e 256^e       (balanced signed bytes, e < E <= 4)
// then  sum_k W x = sum_{d,e} 256^(d+e) C[(j,d)][(m,e)],
//     C[(j,d)][(m,e)] = sum_k x_{k,j,d} W_e[m][k]      (exact int32)
// is an int8 GEMM with rows (coefficient j, digit d), columns (channel m,
// digit e) and the taps as the reduction.  The epilogue recombines the
// digits exactly in 128 bits and reduces mod q_l (two Montgomery steps), so
// the result is bit-identical to the CUDA-core he_lincomb_grouped.
//
// CTA (4 warps): a group of pixels x a run of 16-coefficient chunks of one
// (component, limb).  Per (pixel, chunk): gather the pixel's taps into
// shared memory [tap][16 coeffs] (zero rows for padding taps), build the A
// fragments with byte permutes, run KB x NT mma.sync per 16-row M-tile,
// stage C in shared memory, recombine + reduce + store (coalesced).
#include <algorithm>

#include "common.cuh"

namespace {

constexpr int MW = 4;            // warps per CTA
constexpr int CT = MW * 32;      // threads per CTA
constexpr int CC = 16;           // coefficients per chunk
constexpr int XS = CC + 2;       // uint64 per gathered row (padding vs bank conflicts)
constexpr int CPB = 8;           // chunks per CTA

struct MmaArgs {
    uint64_t *const *out;
    const uint64_t *const *in;
    const int32_t *gcol;     // [G][Tpad] input index, -1 = zero tap
    const int32_t *out_base; // [G]
    const uint32_t *bfrag;   // [KB][NT][32][2] weight-digit B fragments
    const uint64_t *cres;    // [M][ell] constants for component 0, or nullptr
    const ModConst *mc;
    int out_stride, G, gpb, ngb, M, E, Tpad, KB, ell, logN, l_lo, nl;
};

__device__ __forceinline__ void mma_u8s8(int (&d)[4], const uint32_t (&a)[4], const uint2 b) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b.x), "r"(b.y));
}

// byte `b` (0..3) of the selected 32-bit halves of 4 words -> one packed register
__device__ __forceinline__ uint32_t pack4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t sel) {
    const uint32_t t01 = __byte_perm(w0, w1, sel);
    const uint32_t t23 = __byte_perm(w2, w3, sel);
    return __byte_perm(t01, t23, 0x5410);
}

template <int NT>
__global__ void __launch_bounds__(CT) k_conv_mma(const MmaArgs a) {
    extern __shared__ __align__(16) uint8_t smraw[];
    constexpr int NP = NT * 8;          // padded (channel, digit) columns
    constexpr int JS = NP * 8 + 8;      // int32 per coefficient in the C staging area
    uint2 *bfs = (uint2 *)smraw;
    uint64_t *xs = (uint64_t *)(smraw + (size_t)a.KB * NT * 32 * 8);
    int32_t *cs = (int32_t *)(xs + (size_t)a.Tpad * XS);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;

    for (int i = tid; i < a.KB * NT * 32; i += CT) bfs[i] = ((const uint2 *)a.bfrag)[i];

    const int N = 1 << a.logN;
    const int pl = blockIdx.y;                     // comp * nl + (limb - l_lo)
    const int l = a.l_lo + pl % a.nl, comp = pl / a.nl;
    const size_t base = ((size_t)comp * a.ell + l) * (size_t)N;
    const ModConst c = a.mc[l];
    const int nbytes = c.q < (1ull << 40) ? 5 : (c.q < (1ull << 48) ? 6 : (c.q < (1ull << 56) ? 7 : 8));
    const int gb = blockIdx.x % a.ngb, cb = blockIdx.x / a.ngb;
    const int g0 = gb * a.gpb, g1 = min(g0 + a.gpb, a.G);
    // A-fragment byte selectors: digit d = gid lives in word (d >> 2), byte (d & 3)
    const uint32_t bsel = (uint32_t)(gid & 3);
    const uint32_t sel = bsel | ((4u + bsel) << 4);
    const bool hiword = gid >= 4;

    for (int ch = 0; ch < CPB; ch++) {
        const size_t off0 = base + (size_t)(cb * CPB + ch) * CC;
        for (int g = g0; g < g1; g++) {
            __syncthreads();  // previous users of xs / cs are done (and bfs loaded)
            const int32_t *gc = a.gcol + (size_t)g * a.Tpad;
            for (int i = tid; i < a.Tpad * CC; i += CT) {
                const int k = i / CC, j = i % CC;
                const int col = gc[k];
                xs[k * XS + j] = col >= 0 ? __ldg(a.in[col] + off0 + j) : 0ull;
            }
            __syncthreads();
            for (int mt = warp; mt < CC / 2; mt += MW) {
                int acc[NT][4];
#pragma unroll
                for (int nt = 0; nt < NT; nt++) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0;
                const int j0 = 2 * mt;
                for (int kb = 0; kb < a.KB; kb++) {
                    uint32_t w[2][2][4];  // [half k][coef j][i]
#pragma unroll
                    for (int h = 0; h < 2; h++)
#pragma unroll
                        for (int i = 0; i < 4; i++) {
                            const ulonglong2 v = *(const ulonglong2 *)(xs + (kb * 32 + h * 16 + tig * 4 + i) * XS + j0);
                            w[h][0][i] = hiword ? (uint32_t)(v.x >> 32) : (uint32_t)v.x;
                            w[h][1][i] = hiword ? (uint32_t)(v.y >> 32) : (uint32_t)v.y;
                        }
                    const uint32_t af[4] = {pack4(w[0][0][0], w[0][0][1], w[0][0][2], w[0][0][3], sel),
                                            pack4(w[0][1][0], w[0][1][1], w[0][1][2], w[0][1][3], sel),
                                            pack4(w[1][0][0], w[1][0][1], w[1][0][2], w[1][0][3], sel),
                                            pack4(w[1][1][0], w[1][1][1], w[1][1][2], w[1][1][3], sel)};
#pragma unroll
                    for (int nt = 0; nt < NT; nt++) mma_u8s8(acc[nt], af, bfs[(kb * NT + nt) * 32 + lane]);
                }
                // C rows: (j0, d=gid) and (j0+1, d=gid); columns n = nt*8 + 2*tig (+1)
#pragma unroll
                for (int nt = 0; nt < NT; nt++) {
                    const int n = nt * 8 + 2 * tig;
                    cs[j0 * JS + n * 8 + gid] = acc[nt][0];
                    cs[j0 * JS + (n + 1) * 8 + gid] = acc[nt][1];
                    cs[(j0 + 1) * JS + n * 8 + gid] = acc[nt][2];
                    cs[(j0 + 1) * JS + (n + 1) * 8 + gid] = acc[nt][3];
                }
            }
            __syncthreads();
            // epilogue: out(m, j) = sum_{e,d} 256^(e+d) C[j][m*E+e][d] mod q
            const int ob = a.out_base[g];
            for (int i = tid; i < a.M * CC; i += CT) {
                const int m = i / CC, j = i % CC;
                const int32_t *cp = cs + j * JS + m * a.E * 8;
                int64_t S[11];
#pragma unroll
                for (int s = 0; s < 11; s++) S[s] = 0;
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    if (e < a.E) {
#pragma unroll
                        for (int d = 0; d < 8; d++)
                            if (d < nbytes) S[e + d] += cp[e * 8 + d];
                    }
                }
                // T = sum_s S_s 2^(8s), exact signed 128-bit (|T| < 2^104)
                __int128 T = 0;
#pragma unroll
                for (int s = 0; s < 11; s++) T += (__int128)S[s] << (8 * s);
                const int64_t hi = (int64_t)(T >> 64);
                const uint64_t lo = (uint64_t)T;
                uint64_t hic;  // hi mod q (any sign)
                if (hi >= 0) {
                    hic = reduce64((uint64_t)hi, c);
                } else {
                    const uint64_t r = reduce64((uint64_t)(-hi), c);
                    hic = r ? c.q - r : 0;
                }
                // T mod q = redc(hi, lo) * 2^64 = redc(redc(hi, lo) * r2)
                const uint64_t t1 = redc(hic, lo, c.q, c.qinv);
                uint64_t v = redc(mulhi(t1, c.r2), t1 * c.r2, c.q, c.qinv);
                if (a.cres && comp == 0) v = add_mod(v, a.cres[(size_t)m * a.ell + l], c.q);
                a.out[ob + m * a.out_stride][off0 + j] = v;
            }
        }
    }
}

template <int NT>
int launch_mma(dim3 grid, size_t smem, cudaStream_t s, const MmaArgs &a) {
    if (smem > 48 * 1024)
        HE_CHECK_CUDA(cudaFuncSetAttribute(k_conv_mma<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_conv_mma<NT><<<grid, CT, smem, s>>>(a);
    HE_CHECK_LAUNCH();
    return HE_OK;
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
// ceil(M*E/8) <= 12.  Returns HE_EINVAL when a bound does not hold (callers
// fall back to he_lincomb_grouped).
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
    const int NT = (M * E + 7) / 8;
    if (NT > 12) {
        he_set_error("he_conv_mma: M*E = %d exceeds 96 columns", M * E);
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
    // B fragments: b.x = k in [tig*4, tig*4+4), b.y = k + 16; column n = gid
    std::vector<uint32_t> bf((size_t)KB * NT * 32 * 2, 0);
    for (int kb = 0; kb < KB; kb++)
        for (int nt = 0; nt < NT; nt++)
            for (int lane = 0; lane < 32; lane++) {
                const int gid = lane >> 2, tig = lane & 3, n = nt * 8 + gid, m = n / E, e = n % E;
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
    HE_CHECK_CUDA(cudaMemcpyAsync(dbf, bf.data(), b_bf, cudaMemcpyHostToDevice, s));
    HE_CHECK_CUDA(cudaMemcpyAsync(dgc, gc.data(), b_gc, cudaMemcpyHostToDevice, s));
    HE_CHECK_CUDA(cudaMemcpyAsync(dob, out_base, b_ob, cudaMemcpyHostToDevice, s));
    if (residues) HE_CHECK_CUDA(cudaMemcpyAsync(dres, residues, b_res, cudaMemcpyHostToDevice, s));
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
    a.E = E;
    a.Tpad = Tpad;
    a.KB = KB;
    a.ell = ell;
    a.logN = c->logN;
    a.l_lo = 0;
    a.nl = ell;
    const size_t smem = (size_t)KB * NT * 32 * 8 + (size_t)Tpad * XS * 8 + (size_t)CC * (NT * 8 * 8 + 8) * 4;
    int rc = HE_OK;
    if (smem > 220 * 1024) {
        he_set_error("he_conv_mma: %zu bytes of shared memory", smem);
        rc = HE_EINVAL;
    }
    const size_t chunks = (size_t)c->N / (CC * CPB);
    dim3 grid((unsigned)(a.ngb * chunks), (unsigned)(nc * ell));
    if (rc == HE_OK) {
        switch (NT) {
            case 1: rc = launch_mma<1>(grid, smem, s, a); break;
            case 2: rc = launch_mma<2>(grid, smem, s, a); break;
            case 3: rc = launch_mma<3>(grid, smem, s, a); break;
            case 4: rc = launch_mma<4>(grid, smem, s, a); break;
            case 5: rc = launch_mma<5>(grid, smem, s, a); break;
            case 6: rc = launch_mma<6>(grid, smem, s, a); break;
            case 7: rc = launch_mma<7>(grid, smem, s, a); break;
            case 8: rc = launch_mma<8>(grid, smem, s, a); break;
            case 9: rc = launch_mma<9>(grid, smem, s, a); break;
            case 10: rc = launch_mma<10>(grid, smem, s, a); break;
            case 11: rc = launch_mma<11>(grid, smem, s, a); break;
            default: rc = launch_mma<12>(grid, smem, s, a); break;
        }
    }
    he_scratch_free(meta, s);
    he_scratch_free(din, s);
    he_scratch_free(dout, s);
    return rc;
}
