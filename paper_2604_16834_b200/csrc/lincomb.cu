// lincomb.cu -- grouped (register-tiled) feature-major linear combination.
//
// A feature-major 3x3 convolution evaluates, for every output pixel, the SAME
// input gather (the <= 9p valid taps of the window) against every output
// channel's weights.  Grouping outputs by pixel turns the layer into a series
// of tiny dense GEMMs  out[m] = sum_k W[m][tap_k] * in[col_k]  (m < M):
// each thread loads an input residue once and feeds M 128-bit accumulators,
// so the load count per modular MAC drops by M and the kernel becomes
// integer-pipe bound.  Weights (signed integers, shared by all limbs) are
// converted per limb to Montgomery form and staged in shared memory as
// [tap][m] so a thread reads two weights per 128-bit LDS.
//
// Replaces the fold loop of the reference's conv_forward (conv.py:137-156,
// one mult_plain + add per (output, input, tap)) with one launch per layer
// tile.  Output is the exact sum mod q_i (canonical); the caller rescales.
#include <algorithm>

#include "common.cuh"

namespace {

constexpr int LB = 128;  // threads (coefficients) per CTA

__global__ void k_group_weights(uint64_t *wM, const int64_t *w, int M, int MM, int T, int ell, const ModConst *mc) {
    // wM [ell][T][MM] Montgomery; padded m >= M are zero
    size_t tot = (size_t)ell * T * MM;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
        int m = (int)(i % MM);
        int tap = (int)((i / MM) % T);
        int l = (int)(i / ((size_t)MM * T));
        uint64_t v = 0;
        if (m < M) {
            const ModConst c = mc[l];
            uint64_t r = smod64(w[(size_t)m * T + tap], c.q);
            v = redc(mulhi(r, c.r2), r * c.r2, c.q, c.qinv);
        }
        wM[i] = v;
    }
}

template <int MM>
__global__ void __launch_bounds__(LB) k_lincomb_grouped(uint64_t *const *__restrict__ out,
                                                        const uint64_t *const *__restrict__ in,
                                                        const int32_t *__restrict__ term_ptr,
                                                        const int2 *__restrict__ terms,
                                                        const int32_t *__restrict__ out_base, int out_stride, int M,
                                                        int T, const uint64_t *__restrict__ wM, int n_groups, int gpb,
                                                        int ell, int logN, int kmax, const ModConst *mc) {
    extern __shared__ uint64_t wsm[];  // [T][MM]
    const int N = 1 << logN;
    const int cpp = N / LB;
    const int pl = blockIdx.y / cpp;  // comp * ell + limb
    const int l = pl % ell;
    const size_t off = (size_t)pl * N + (size_t)(blockIdx.y % cpp) * LB + threadIdx.x;
    const ModConst c = mc[l];
    const uint64_t *src = wM + (size_t)l * T * MM;
    for (int i = threadIdx.x; i < T * MM; i += LB) wsm[i] = src[i];
    __syncthreads();
    // sums of kmax products < q^2 need a fold to keep hi < q when kmax * q >= 2^64
    const bool fold = (double)kmax * (double)c.q >= 1.8e19;
    const int g0 = blockIdx.x * gpb, g1 = min(g0 + gpb, n_groups);
    for (int g = g0; g < g1; g++) {
        u128 acc[MM];
#pragma unroll
        for (int m = 0; m < MM; m++) acc[m] = {0, 0};
        const int t1 = term_ptr[g + 1];
        for (int t = term_ptr[g]; t < t1; t++) {
            const int2 ct = terms[t];
            const uint64_t x = __ldg(in[ct.x] + off);
            const uint64_t *wr = wsm + ct.y * MM;
#pragma unroll
            for (int m = 0; m < MM; m += 2) {
                const ulonglong2 w2 = *(const ulonglong2 *)(wr + m);
                mac128(acc[m], x, w2.x);
                mac128(acc[m + 1], x, w2.y);
            }
            if (fold) {
#pragma unroll
                for (int m = 0; m < MM; m++)
                    if (acc[m].hi >= c.q) acc[m].hi -= c.q;
            }
        }
        const int ob = out_base[g];
#pragma unroll
        for (int m = 0; m < MM; m++) {
            // hi < q: either folded per term, or kmax * q < 2^64 bounds the sum
            if (m < M) out[ob + m * out_stride][off] = redc(acc[m].hi, acc[m].lo, c.q, c.qinv);
        }
    }
}

template <int MM>
int launch_grouped(dim3 grid, size_t smem, cudaStream_t s, uint64_t *const *out, const uint64_t *const *in,
                   const int32_t *tp, const int2 *terms, const int32_t *ob, int out_stride, int M, int T,
                   const uint64_t *wM, int G, int gpb, int ell, int logN, int kmax, const ModConst *mc) {
    if (smem > 48 * 1024)
        HE_CHECK_CUDA(cudaFuncSetAttribute(k_lincomb_grouped<MM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_lincomb_grouped<MM><<<grid, LB, smem, s>>>(out, in, tp, terms, ob, out_stride, M, T, wM, G, gpb, ell, logN, kmax,
                                                 mc);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

}  // namespace

extern "C" int he_lincomb_grouped(he_ctx *c, const uint64_t *const *in, int n_in, uint64_t *const *out, int n_out,
                                  int n_groups, const int32_t *term_ptr, const int32_t *term_col,
                                  const int32_t *term_tap, const int32_t *out_base, int out_stride, int M, int T,
                                  const int64_t *weights, int ell, int nc, void *stream) {
    if (!c || n_in < 1 || n_out < 0 || n_groups < 0 || M < 1 || M > 32 || T < 1 || ell < 1 || ell > c->L ||
        nc < 1 || nc > 3 || !term_ptr || !term_col || !term_tap || !out_base || !weights) {
        he_set_error("he_lincomb_grouped: bad arguments (M=%d T=%d ell=%d)", M, T, ell);
        return HE_EINVAL;
    }
    if (c->N < LB) {
        he_set_error("he_lincomb_grouped needs N >= %d", LB);
        return HE_EINVAL;
    }
    if (!n_groups) return HE_OK;
    int nnz = term_ptr[n_groups], kmax = 0;
    if (term_ptr[0] != 0 || nnz < 0) {
        he_set_error("he_lincomb_grouped: term_ptr must start at 0");
        return HE_EINVAL;
    }
    for (int g = 0; g < n_groups; g++) {
        int k = term_ptr[g + 1] - term_ptr[g];
        if (k < 0) {
            he_set_error("he_lincomb_grouped: term_ptr not monotone at %d", g);
            return HE_EINVAL;
        }
        kmax = std::max(kmax, k);
        if (out_base[g] < 0 || out_base[g] + (M - 1) * out_stride >= n_out) {
            he_set_error("he_lincomb_grouped: outputs of group %d out of range", g);
            return HE_EINVAL;
        }
    }
    for (int t = 0; t < nnz; t++)
        if (term_col[t] < 0 || term_col[t] >= n_in || term_tap[t] < 0 || term_tap[t] >= T) {
            he_set_error("he_lincomb_grouped: term %d (col %d tap %d) out of range", t, term_col[t], term_tap[t]);
            return HE_EINVAL;
        }
    for (int i = 0; i < M * T; i++)
        if (weights[i] >= ((int64_t)1 << 62) || weights[i] <= -((int64_t)1 << 62)) {
            he_set_error("he_lincomb_grouped: |w| >= 2^62");
            return HE_EINVAL;
        }
    int MM = M <= 2 ? 2 : M <= 4 ? 4 : M <= 8 ? 8 : M <= 16 ? 16 : 32;
    cudaStream_t s = (cudaStream_t)stream;
    void **din = nullptr, **dout = nullptr;
    HE_TRY(he_upload_ptrs((const void *const *)in, n_in, &din, s));
    HE_TRY(he_upload_ptrs((const void *const *)out, n_out, &dout, s));
    std::vector<int2> terms(std::max(nnz, 1));
    for (int t = 0; t < nnz; t++) terms[t] = make_int2(term_col[t], term_tap[t]);
    size_t b_tp = (size_t)(n_groups + 1) * 4, b_terms = (size_t)terms.size() * 8, b_ob = (size_t)n_groups * 4,
           b_w = (size_t)M * T * 8, b_wM = (size_t)ell * T * MM * 8;
    char *meta = nullptr;
    HE_TRY(he_scratch_alloc((void **)&meta, b_wM + b_terms + b_w + b_tp + b_ob + 64, s));
    uint64_t *wM = (uint64_t *)meta;
    int2 *dterms = (int2 *)(meta + b_wM);
    int64_t *dw = (int64_t *)(meta + b_wM + b_terms);
    int32_t *dtp = (int32_t *)(meta + b_wM + b_terms + b_w);
    int32_t *dob = (int32_t *)(meta + b_wM + b_terms + b_w + b_tp);
    HE_CHECK_CUDA(cudaMemcpyAsync(dterms, terms.data(), b_terms, cudaMemcpyHostToDevice, s));
    HE_CHECK_CUDA(cudaMemcpyAsync(dw, weights, b_w, cudaMemcpyHostToDevice, s));
    HE_CHECK_CUDA(cudaMemcpyAsync(dtp, term_ptr, b_tp, cudaMemcpyHostToDevice, s));
    HE_CHECK_CUDA(cudaMemcpyAsync(dob, out_base, b_ob, cudaMemcpyHostToDevice, s));
    k_group_weights<<<ceil_div((size_t)ell * T * MM, 256), 256, 0, s>>>(wM, dw, M, MM, T, ell, c->d_mc);
    HE_CHECK_LAUNCH();
    int gpb = std::max(1, std::min(8, n_groups / 148));
    int cpp = c->N / LB;
    size_t smem = (size_t)T * MM * 8;
    int rc = HE_OK;
    if ((size_t)nc * ell * cpp > 65535) {
        he_set_error("he_lincomb_grouped: grid too large");
        rc = HE_EINVAL;
    }
    if (rc == HE_OK) {
        dim3 grid(ceil_div(n_groups, gpb), (unsigned)(nc * ell * cpp));
        auto O = (uint64_t *const *)dout;
        auto I = (const uint64_t *const *)din;
        switch (MM) {
            case 2: rc = launch_grouped<2>(grid, smem, s, O, I, dtp, dterms, dob, out_stride, M, T, wM, n_groups, gpb, ell, c->logN, kmax, c->d_mc); break;
            case 4: rc = launch_grouped<4>(grid, smem, s, O, I, dtp, dterms, dob, out_stride, M, T, wM, n_groups, gpb, ell, c->logN, kmax, c->d_mc); break;
            case 8: rc = launch_grouped<8>(grid, smem, s, O, I, dtp, dterms, dob, out_stride, M, T, wM, n_groups, gpb, ell, c->logN, kmax, c->d_mc); break;
            case 16: rc = launch_grouped<16>(grid, smem, s, O, I, dtp, dterms, dob, out_stride, M, T, wM, n_groups, gpb, ell, c->logN, kmax, c->d_mc); break;
            default: rc = launch_grouped<32>(grid, smem, s, O, I, dtp, dterms, dob, out_stride, M, T, wM, n_groups, gpb, ell, c->logN, kmax, c->d_mc); break;
        }
    }
    he_scratch_free(meta, s);
    he_scratch_free(din, s);
    he_scratch_free(dout, s);
    return rc;
}
