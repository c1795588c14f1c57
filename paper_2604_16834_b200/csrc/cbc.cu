// cbc.cu -- the batched channel-by-channel (CBC) convolution fold.
//
// The paper's CBC layer (/root/reference/pkg/src/hebatch/conv.py:137-156,
// PAPER.md:309-346) multiplies every tap-aligned input ciphertext by a
// full-width encoded plaintext (the tap weight times the tap's border mask)
// and sums the products per output channel.  The reference folds one
// mult_plain + add at a time; here the whole fold of a layer is ONE kernel:
//
//   out[o][c] = sum_{j < n_in} in[j][c] (.) pt[o][j]     (mod q_l, NTT domain)
//
// for c in {0, 1}, element-wise per (limb, coefficient), exact 128-bit
// accumulation (operands < 2^52: carry-free split accumulator mac52; wider
// primes: mac128) and one reduction per output value.  The caller rescales
// the sums once per output (instead of once per term) and adds the bias.
//
// Work per launch: n_out * n_in * 2 * ell * N modular MACs; bytes: the
// n_out * n_in plaintexts (ell N words each: the dominant stream), the
// n_in aligned inputs once per block of OB outputs, the outputs once.
#include <algorithm>

#include "common.cuh"

namespace {

constexpr int OB = 4;      // outputs per thread (input components are reloaded n_out / OB times)
constexpr int THR = 256;

__device__ __forceinline__ uint64_t reduce_u128(u128 t, const ModConst &c) {
    const uint64_t h = reduce64(t.hi, c);                  // T' = (hi mod q) 2^64 + lo < q 2^64
    const uint64_t r = redc(h, t.lo, c.q, c.qinv);        // T 2^-64 mod q
    return redc(mulhi(r, c.r2), r * c.r2, c.q, c.qinv);  // T mod q
}

template <bool WIDE>
__global__ void __launch_bounds__(THR) k_lincomb_plain(const uint64_t *const *__restrict__ in, int n_in,
                                                       const uint64_t *const *__restrict__ pt,
                                                       uint64_t *const *__restrict__ out, int n_out, int ell,
                                                       int logN, const ModConst *__restrict__ mc) {
    const size_t N = (size_t)1 << logN;
    const size_t k = (size_t)blockIdx.x * THR + threadIdx.x;  // coefficient
    const int l = blockIdx.y;                                  // limb
    const int o0 = blockIdx.z * OB;
    if (k >= N) return;
    const ModConst c = mc[l];
    const size_t off0 = (size_t)l * N + k, off1 = ((size_t)ell + l) * N + k;
    const int nob = min(OB, n_out - o0);
    if (!WIDE) {
        acc52 acc[OB][2];
#pragma unroll
        for (int o = 0; o < OB; o++) acc52_zero(acc[o][0]), acc52_zero(acc[o][1]);
        for (int j = 0; j < n_in; j++) {
            const uint64_t *a = in[j];
            const xsplit a0 = split52(__ldg(a + off0)), a1 = split52(__ldg(a + off1));
#pragma unroll
            for (int o = 0; o < OB; o++) {
                if (o < nob) {
                    const uint64_t w = __ldg(pt[(size_t)(o0 + o) * n_in + j] + off0);
                    mac52(acc[o][0], a0, w);
                    mac52(acc[o][1], a1, w);
                }
            }
        }
#pragma unroll
        for (int o = 0; o < OB; o++)
            if (o < nob) {
                uint64_t *dst = out[o0 + o];
                dst[off0] = reduce_u128(acc52_sum(acc[o][0]), c);
                dst[off1] = reduce_u128(acc52_sum(acc[o][1]), c);
            }
    } else {
        u128 acc[OB][2];
#pragma unroll
        for (int o = 0; o < OB; o++) acc[o][0] = acc[o][1] = u128{0, 0};
        for (int j = 0; j < n_in; j++) {
            const uint64_t *a = in[j];
            const uint64_t a0 = __ldg(a + off0), a1 = __ldg(a + off1);
#pragma unroll
            for (int o = 0; o < OB; o++) {
                if (o < nob) {
                    const uint64_t w = __ldg(pt[(size_t)(o0 + o) * n_in + j] + off0);
                    // n_in q^2 < 2^128 (checked on the host): the 128-bit sum cannot overflow
                    mac128(acc[o][0], a0, w);
                    mac128(acc[o][1], a1, w);
                }
            }
        }
#pragma unroll
        for (int o = 0; o < OB; o++)
            if (o < nob) {
                uint64_t *dst = out[o0 + o];
                dst[off0] = reduce_u128(acc[o][0], c);
                dst[off1] = reduce_u128(acc[o][1], c);
            }
    }
}

}  // namespace

extern "C" int he_lincomb_plain(he_ctx *c, const uint64_t *const *in, int n_in, const uint64_t *const *pts,
                                uint64_t *const *out, int n_out, int ell, void *stream) {
    if (!c || !in || !pts || !out || n_in < 1 || n_out < 1 || ell < 1 || ell > c->L) {
        he_set_error("he_lincomb_plain: bad arguments (n_in=%d n_out=%d ell=%d)", n_in, n_out, ell);
        return HE_EINVAL;
    }
    if (n_in > 1024 || (size_t)n_in * n_out > (1u << 26)) {
        he_set_error("he_lincomb_plain: n_in=%d (<= 1024) x n_out=%d too large", n_in, n_out);
        return HE_EINVAL;
    }
    int bits = 0;
    for (int l = 0; l < ell; l++) bits = std::max(bits, 64 - __builtin_clzll(c->mod[l]));
    const bool wide = bits > 52;
    // exactness of the wide path's 128-bit sums: n_in q^2 < 2^128
    if (wide && (2 * bits >= 128 || n_in >= (1 << std::min(30, 128 - 2 * bits)))) {
        he_set_error("he_lincomb_plain: %d-bit primes limit the fold to %d terms (got %d)", bits,
                     (1 << std::min(30, 128 - 2 * bits)) - 1, n_in);
        return HE_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    void **din = nullptr, **dpt = nullptr, **dout = nullptr;
    HE_TRY(he_upload_ptrs((const void *const *)in, n_in, &din, s));
    HE_TRY(he_upload_ptrs((const void *const *)pts, n_in * n_out, &dpt, s));
    HE_TRY(he_upload_ptrs((const void *const *)out, n_out, &dout, s));
    const dim3 grid((unsigned)((c->N + THR - 1) / THR), (unsigned)ell, (unsigned)((n_out + OB - 1) / OB));
    if (wide)
        k_lincomb_plain<true><<<grid, THR, 0, s>>>((const uint64_t *const *)din, n_in, (const uint64_t *const *)dpt,
                                                   (uint64_t *const *)dout, n_out, ell, c->logN, c->d_mc);
    else
        k_lincomb_plain<false><<<grid, THR, 0, s>>>((const uint64_t *const *)din, n_in, (const uint64_t *const *)dpt,
                                                    (uint64_t *const *)dout, n_out, ell, c->logN, c->d_mc);
    HE_CHECK_LAUNCH();
    he_scratch_free(din, s);
    he_scratch_free(dpt, s);
    he_scratch_free(dout, s);
    return HE_OK;
}
