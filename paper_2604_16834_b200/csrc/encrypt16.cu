// encrypt16.cu -- fused encryption for N = 2^16 (the batched pack_inputs path).
//
// Replaces, for the two-pass ring, the chain encode_finish (14 limb writes of
// m + e) -> forward NTT (two HBM round trips) -> encrypt_finish (re-read of c0)
// of encode.cu with three kernels whose HBM traffic is the c0/c1 output plus
// one int64 plane per ciphertext:
//   k_enc_m16     m_j + e_j as one signed int64 per coefficient (limb-free),
//                 the same float64 operations as encode.cu's k_encode_finish;
//   k_enc16_cols  per (ciphertext, 16-column tile): the int64 plane is loaded
//                 once and every limb's NTT pass 1 (stages 0..7) runs from it;
//   k_enc16_rows  per (ciphertext, limb, 16-row tile): NTT pass 2, then
//                 c1 = a (uniform, NTT domain) and c0 = NTT(m + e) - a s.
// Limbs below 2^42 take the FP64 butterflies (exact integer doubles,
// ntt_core.cuh).  Every output is canonical and equal to the unfused chain's
// (oracle/ckks_oracle.c oc_encrypt; tests/test_gpu_parity.py).
#include "ntt_core.cuh"

namespace {

constexpr int LOGN = 16;
constexpr size_t NN = (size_t)1 << LOGN;

// signed 64-bit -> canonical residue with one high product (reduce64)
__device__ __forceinline__ uint64_t sreduce(int64_t v, const ModConst &c) {
    if (v >= 0) return reduce64((uint64_t)v, c);
    const uint64_t r = reduce64((uint64_t)(-(v + 1)), c);
    return c.q - 1 - r;
}

// m_j (j < n) and m_{j+n} from the normalised, twisted FFT output, plus CBD error
__global__ void k_enc_m16(int64_t *m, const double *re, const double *im, size_t count, double scale,
                          const double *twist, uint64_t seed, uint32_t ct_index0) {
    const size_t n = NN >> 1, tot = count * n;
    const double inv_n = 1.0 / (double)n;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
        const size_t v = i / n, j = i % n;
        const double vr = __dmul_rn(re[i], inv_n), vi = __dmul_rn(im[i], inv_n);
        const double zr = twist[2 * j], zi = twist[2 * j + 1];
        const double ur = __dadd_rn(__dmul_rn(vr, zr), __dmul_rn(vi, zi));
        const double ui = __dsub_rn(__dmul_rn(vi, zr), __dmul_rn(vr, zi));
        int64_t m0 = __double2ll_rn(__dmul_rn(ur, scale));
        int64_t m1 = __double2ll_rn(__dmul_rn(ui, scale));
        m0 += sample_cbd(seed, DOM_ENC_E, ct_index0 + (uint32_t)v, (uint32_t)j);
        m1 += sample_cbd(seed, DOM_ENC_E, ct_index0 + (uint32_t)v, (uint32_t)(j + n));
        m[v * NN + j] = m0;
        m[v * NN + j + n] = m1;
    }
}

// pass 1 of every limb's forward NTT from the shared int64 plane; the result
// (canonical) goes to c0 limb l of out[v]
#ifndef ENC_COLS_CTAS
#define ENC_COLS_CTAS 3
#endif
__global__ void __launch_bounds__(NTT_TPB, ENC_COLS_CTAS) k_enc16_cols(uint64_t *const *out, const int64_t *m, int L,
                                                        const uint64_t *tw, const double *twd, const ModConst *mc) {
    __shared__ uint64_t sm[256 * 16];
    const size_t v = blockIdx.x >> 4;
    const int tid = threadIdx.x, lc = tid & 15, g = tid >> 4;
    const uint32_t col = (blockIdx.x & 15) * 16 + lc;
    const int64_t *mp = m + v * NN + col;
    int64_t mv[16];
#pragma unroll
    for (int j = 0; j < 16; j++) mv[j] = mp[(g + 16 * j) * 256];
    uint64_t *o = out[v];
    for (int l = 0; l < L; l++) {
        const ModConst c = mc[l];
        uint64_t *dst = o + (size_t)l * NN + col;
        if (c.q < FP_QMAX) {
            const double *Wd = twd_fwd(twd, l, LOGN);
            double xd[16];
#pragma unroll
            for (int j = 0; j < 16; j++) xd[j] = u2d(sreduce(mv[j], c));
            fphase_ct<16, 0>(xd, col + 256 * g, Wd, c.qd, c.qid);
#pragma unroll
            for (int j = 0; j < 16; j++) sm[(g + 16 * j) * 16 + lc] = (uint64_t)__double_as_longlong(xd[j]);
            __syncthreads();
#pragma unroll
            for (int j = 0; j < 16; j++) xd[j] = __longlong_as_double((long long)sm[(16 * g + j) * 16 + lc]);
            fphase_ct<16, 4>(xd, col + 4096 * g, Wd, c.qd, c.qid);
#pragma unroll
            for (int j = 0; j < 16; j++) dst[(16 * g + j) * 256] = fcanon(xd[j], c.qd, c.qid);
        } else {
            const ulonglong2 *W2 = tw_fwd(tw, l, LOGN);
            uint64_t x[16];
#pragma unroll
            for (int j = 0; j < 16; j++) x[j] = sreduce(mv[j], c);
            phase_ct<16, 0>(x, col + 256 * g, W2, c.q);
#pragma unroll
            for (int j = 0; j < 16; j++) sm[(g + 16 * j) * 16 + lc] = x[j];
            __syncthreads();
#pragma unroll
            for (int j = 0; j < 16; j++) x[j] = sm[(16 * g + j) * 16 + lc];
            phase_ct<16, 4>(x, col + 4096 * g, W2, c.q);
#pragma unroll
            for (int j = 0; j < 16; j++) dst[(16 * g + j) * 256] = reduce4q(x[j], c.q);
        }
        __syncthreads();  // sm is rewritten by the next limb
    }
}

// pass 2 + encryption epilogue: c1 = a, c0 = x - a s (all canonical)
#ifndef ENC_ROWS_CTAS
#define ENC_ROWS_CTAS 4  // 64 registers: 32 warps per SM (26.0 ms per 3072-ciphertext batch instead of 28.3)
#endif
__global__ void __launch_bounds__(NTT_TPB, ENC_ROWS_CTAS) k_enc16_rows(uint64_t *const *out, int L, const uint64_t *tw,
                                                        const double *twd, const ModConst *mc, const uint64_t *sk,
                                                        uint64_t seed, uint32_t ct_index0) {
    __shared__ uint64_t sm[16 * 272];
    const unsigned cl = blockIdx.x >> 4;  // ciphertext-major, limb-minor
    const int l = (int)(cl % (unsigned)L);
    const size_t v = cl / (unsigned)L;
    const ModConst c = mc[l];
    const int tid = threadIdx.x, g = tid & 15, rl = tid >> 4;
    const uint32_t r = (blockIdx.x & 15) * 16 + rl;
    uint64_t *c0 = out[v] + (size_t)l * NN, *c1 = c0 + (size_t)L * NN;
    uint64_t *row = c0 + r * 256;
    uint64_t *s = sm + rl * 272;
    uint64_t x[16];
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = row[g + 16 * j];
    if (c.q < FP_QMAX) {
        const double *Wd = twd_fwd(twd, l, LOGN);
        double xd[16];
#pragma unroll
        for (int j = 0; j < 16; j++) xd[j] = u2d(x[j]);
        fphase_ct<16, 8>(xd, r * 256 + g, Wd, c.qd, c.qid);
#pragma unroll
        for (int j = 0; j < 16; j++) s[pad16(g + 16 * j)] = (uint64_t)__double_as_longlong(xd[j]);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; j++) xd[j] = __longlong_as_double((long long)s[pad16(16 * g + j)]);
        __syncwarp();
        fphase_ct<16, 12>(xd, r * 256 + 16 * g, Wd, c.qd, c.qid);
#pragma unroll
        for (int j = 0; j < 16; j++) s[pad16(16 * g + j)] = fcanon(xd[j], c.qd, c.qid);
    } else {
        const ulonglong2 *W2 = tw_fwd(tw, l, LOGN);
        phase_ct<16, 8>(x, r * 256 + g, W2, c.q);
#pragma unroll
        for (int j = 0; j < 16; j++) s[pad16(g + 16 * j)] = x[j];
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; j++) x[j] = s[pad16(16 * g + j)];
        __syncwarp();
        phase_ct<16, 12>(x, r * 256 + 16 * g, W2, c.q);
#pragma unroll
        for (int j = 0; j < 16; j++) s[pad16(16 * g + j)] = reduce4q(x[j], c.q);
    }
    __syncwarp();
    const uint64_t *skl = sk + (size_t)l * NN + r * 256;
    const uint32_t obj = ct_index0 + (uint32_t)v;
#pragma unroll 2
    for (int j = 0; j < 16; j += 2) {  // coefficients k and k + 16 share one Philox block
        const int cc = g + 16 * j;
        const uint32_t k = r * 256 + cc;
        uint64_t av[2];
        sample_uniform_pair(seed, DOM_ENC_A, obj, (uint32_t)l, k, c, av[0], av[1]);
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const uint64_t a = av[h];
            const uint64_t sv = skl[cc + 16 * h];
            uint64_t as;
            if (c.q < FP_QMAX)
                as = fcanon(fmulmod(u2d(a), u2d(sv), c.qd, c.qid), c.qd, c.qid);
            else
                as = mul_mod(a, sv, c);
            c1[k + 16 * h] = a;
            row[cc + 16 * h] = sub_mod(s[pad16(cc + 16 * h)], as, c.q);
        }
    }
}

}  // namespace

// Fused encryption of `count` ciphertexts ([2][ell][N] each, out_dev: DEVICE
// array of their addresses) from the FFT output re/im ([count][N/2] each).
int he_encrypt16(he_ctx *c, const double *re, const double *im, int count, double scale, uint32_t ct_index0,
                 int ell, uint64_t *const *out_dev, cudaStream_t s) {
    const size_t n = NN >> 1;
    int64_t *m = nullptr;
    HE_TRY(he_scratch_alloc((void **)&m, (size_t)count * NN * sizeof(int64_t), s));
    const unsigned gm = (unsigned)std::min<size_t>(((size_t)count * n + 255) / 256, (size_t)148 * 32);
    k_enc_m16<<<gm, 256, 0, s>>>(m, re, im, (size_t)count, scale, c->d_twist, c->prm.seed, ct_index0);
    int rc = cudaGetLastError() == cudaSuccess ? HE_OK : HE_ECUDA;
    he_count_launch(1);
    if (rc == HE_OK) {
        k_enc16_cols<<<(unsigned)count * 16, NTT_TPB, 0, s>>>(out_dev, m, ell, c->d_tw, c->d_twd, c->d_mc);
        he_count_launch(1);
        if (cudaGetLastError() != cudaSuccess) rc = HE_ECUDA;
    }
    if (rc == HE_OK) {
        k_enc16_rows<<<(unsigned)count * ell * 16, NTT_TPB, 0, s>>>(out_dev, ell, c->d_tw, c->d_twd, c->d_mc,
                                                                    c->d_sk, c->prm.seed, ct_index0);
        he_count_launch(1);
        if (cudaGetLastError() != cudaSuccess) rc = HE_ECUDA;
    }
    he_scratch_free(m, s);
    if (rc != HE_OK) he_set_error("he_encrypt16: kernel launch failed");
    return rc;
}
