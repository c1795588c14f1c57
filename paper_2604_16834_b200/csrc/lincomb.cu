// lincomb.cu -- grouped (register-tiled) feature-major linear combination.
//
// A feature-major 3x3 convolution evaluates, for every output pixel, the SAME
// input gather (the <= 9p valid taps of the window) against every output
// channel's weights.  Grouping outputs by pixel turns the layer into a series
// of tiny dense GEMMs  out[m] = sum_k W[m][tap_k] * in[col_k]  (m < M):
// each thread loads an input residue once and feeds M accumulators, so the
// load count per modular MAC drops by M.  Weights (signed integers, shared by
// all limbs) are converted per limb to Montgomery form and staged in shared
// memory as [tap][m] so a thread reads two weights per 128-bit LDS.  Terms
// carry the input's device address directly (no pointer-table indirection)
// and the gather is software-pipelined four terms deep.
//
// Two accumulator variants: for limbs with q < 2^52 (and a bounded term
// count) the split 32-bit accumulator mac52 (~7 instructions per MAC);
// otherwise exact 128-bit mad.lo.cc/madc.hi with a per-term fold.
//
// Replaces the fold loop of the reference's conv_forward (conv.py:137-156,
// one mult_plain + add per (output, input, tap)) with one launch per layer
// tile.  Output is the exact sum mod q_i (canonical); the caller rescales.
#include <algorithm>

#include "common.cuh"

namespace {

constexpr int LB = 128;  // threads (coefficients) per CTA
constexpr int PF = 4;    // gather prefetch depth (terms)

struct __align__(16) Term {
    const uint64_t *p;  // input ciphertext base address
    int32_t tap;
    int32_t pad;
};

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

struct GroupArgs {
    uint64_t *const *out;
    const int32_t *term_ptr;
    const Term *terms;
    const int32_t *out_base;
    const uint64_t *cres;  // [M][ell] constant added to component 0 of output channel m, or nullptr
    const uint64_t *wM;  // [ell][T][WS] Montgomery weights
    const ModConst *mc;
    int out_stride, M, T, WS, n_groups, gpb, ell, logN, kmax;
    int l_lo, nl;        // this launch covers limbs [l_lo, l_lo + nl) of every component
    int m_off;           // first output channel handled by this launch
};

template <bool FAST>
struct Acc;
template <>
struct Acc<true> {
    acc52 a;
    using X = xsplit;
    __device__ __forceinline__ static X prep(uint64_t x) { return split52(x); }
    __device__ __forceinline__ void zero() { acc52_zero(a); }
    __device__ __forceinline__ void mac(const X &x, uint64_t w) { mac52(a, x, w); }
    __device__ __forceinline__ void fold(uint64_t) {}
    __device__ __forceinline__ u128 sum() const { return acc52_sum(a); }
};
template <>
struct Acc<false> {
    u128 a;
    using X = uint64_t;
    __device__ __forceinline__ static X prep(uint64_t x) { return x; }
    __device__ __forceinline__ void zero() { a = {0, 0}; }
    __device__ __forceinline__ void mac(const X &x, uint64_t w) { mac128(a, x, w); }
    __device__ __forceinline__ void fold(uint64_t q) {
        if (a.hi >= q) a.hi -= q;
    }
    __device__ __forceinline__ u128 sum() const { return a; }
};

// FAST: every limb of the launch has q < 2^52 and kmax * q < 2^64 (and
// kmax <= 1024), so the carry-free split accumulator applies and no per-term
// fold is needed.  Dynamic shared memory: weights [T][WS], then the block's
// terms (pointer, tap) so the gather addresses never wait on global loads.
template <int MM, bool FAST>
__global__ void __launch_bounds__(LB) k_lincomb_grouped(const GroupArgs a) {
    extern __shared__ uint64_t wsm[];  // [T][WS] then Term[block terms]
    const int N = 1 << a.logN;
    const int cpp = N / LB;
    const int pl = blockIdx.y / cpp;  // comp * nl + (limb - l_lo)
    const int l = a.l_lo + pl % a.nl;
    const int comp = pl / a.nl;
    const size_t off = ((size_t)comp * a.ell + l) * N + (size_t)(blockIdx.y % cpp) * LB + threadIdx.x;
    const ModConst c = a.mc[l];
    const uint64_t *src = a.wM + (size_t)l * a.T * a.WS;
    for (int i = threadIdx.x; i < a.T * a.WS; i += LB) wsm[i] = src[i];
    const int g0 = blockIdx.x * a.gpb, g1 = min(g0 + a.gpb, a.n_groups);
    const int tb0 = a.term_ptr[g0], tb1 = a.term_ptr[g1];
    Term *tsm = (Term *)(wsm + a.T * a.WS);
    for (int i = threadIdx.x; i < tb1 - tb0; i += LB) tsm[i] = a.terms[tb0 + i];
    __syncthreads();
    // sums of kmax products < q^2 need a fold to keep hi < q when kmax * q >= 2^64
    const bool fold = !FAST && (double)a.kmax * (double)c.q >= 1.8e19;
    for (int g = g0; g < g1; g++) {
        const int t0 = a.term_ptr[g] - tb0, t1 = a.term_ptr[g + 1] - tb0;
        const int ob = a.out_base[g] + a.m_off * a.out_stride;
        Acc<FAST> acc[MM];
#pragma unroll
        for (int m = 0; m < MM; m++) acc[m].zero();
        for (int t = t0; t < t1; t += PF) {
            uint64_t xs[PF];
            int taps[PF];
#pragma unroll
            for (int u = 0; u < PF; u++) {  // issue all gathers first
                if (t + u < t1) {
                    const Term tm = tsm[t + u];
                    xs[u] = __ldg(tm.p + off);
                    taps[u] = tm.tap;
                } else {
                    xs[u] = 0;
                    taps[u] = 0;
                }
            }
#pragma unroll
            for (int u = 0; u < PF; u++) {
                const uint64_t *wr = wsm + taps[u] * a.WS + a.m_off;
                const typename Acc<FAST>::X xv = Acc<FAST>::prep(xs[u]);
#pragma unroll
                for (int m = 0; m < MM; m += 2) {
                    const ulonglong2 w2 = *(const ulonglong2 *)(wr + m);
                    acc[m].mac(xv, w2.x);
                    acc[m + 1].mac(xv, w2.y);
                }
                if (fold) {
#pragma unroll
                    for (int m = 0; m < MM; m++) acc[m].fold(c.q);
                }
            }
        }
#pragma unroll
        for (int m = 0; m < MM; m++) {
            // hi < q: either folded per term, or kmax * q < 2^64 bounds the sum
            if (a.m_off + m < a.M) {
                const u128 sm = acc[m].sum();
                uint64_t v = redc(sm.hi, sm.lo, c.q, c.qinv);
                if (a.cres && comp == 0) v = add_mod(v, a.cres[(size_t)(a.m_off + m) * a.ell + l], c.q);
                a.out[ob + m * a.out_stride][off] = v;
            }
        }
    }
}

template <int MM, bool FAST>
int launch_grouped(dim3 grid, size_t smem, cudaStream_t s, const GroupArgs &a) {
    if (smem > 48 * 1024)
        HE_CHECK_CUDA(cudaFuncSetAttribute(k_lincomb_grouped<MM, FAST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem));
    k_lincomb_grouped<MM, FAST><<<grid, LB, smem, s>>>(a);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

int dispatch_grouped(int MM, bool fast, dim3 grid, size_t smem, cudaStream_t s, const GroupArgs &a) {
    if (fast) {
        switch (MM) {
            case 2: return launch_grouped<2, true>(grid, smem, s, a);
            case 4: return launch_grouped<4, true>(grid, smem, s, a);
            default: return launch_grouped<8, true>(grid, smem, s, a);
        }
    }
    switch (MM) {
        case 2: return launch_grouped<2, false>(grid, smem, s, a);
        case 4: return launch_grouped<4, false>(grid, smem, s, a);
        case 8: return launch_grouped<8, false>(grid, smem, s, a);
        case 16: return launch_grouped<16, false>(grid, smem, s, a);
        default: return launch_grouped<32, false>(grid, smem, s, a);
    }
}

// Sum of squares over groups (lazy degree-2 activation fused with the pool /
// GAP sum):  out[o] = sum_{t in row o} in[col_t] (x) in[col_t]  + cres[o],
// where (x) is the tensor product (d0, d1, d2) = (x0^2, 2 x0 x1, x1^2) and
// cres is added to d0.  Bit-identical to he_tensor + he_add_const per input
// followed by the unit-weight he_lincomb (all steps are exact mod q).
// One thread = one (limb, coefficient) of one output; inputs [2][ell][N],
// outputs [3][ell][N].
__global__ void __launch_bounds__(LB) k_square_sum(uint64_t *const *out, const uint64_t *const *in,
                                                   const int32_t *row_ptr, const int32_t *col, const uint64_t *cres,
                                                   int n_out, int ell, int logN, int kmax, const ModConst *mc) {
    const size_t N = (size_t)1 << logN;
    const int cpp = (int)(N / LB);
    const int l = blockIdx.y / cpp;
    const size_t k = (size_t)(blockIdx.y % cpp) * LB + threadIdx.x;
    const size_t o0 = (size_t)l * N + k, o1 = ((size_t)ell + l) * N + k;
    const ModConst c = mc[l];
    const bool fold = (double)(2 * kmax) * (double)c.q >= 1.8e19;
    const int o = blockIdx.x;
    u128 a0 = {0, 0}, a1 = {0, 0}, a2 = {0, 0};
    for (int t = row_ptr[o]; t < row_ptr[o + 1]; t++) {
        const uint64_t *x = in[col[t]];
        const uint64_t x0 = __ldg(x + o0), x1 = __ldg(x + o1);
        mac128(a0, x0, x0);
        mac128(a1, x0, x1);
        mac128(a1, x0, x1);
        mac128(a2, x1, x1);
        if (fold) {
            if (a0.hi >= c.q) a0.hi -= c.q;
            if (a1.hi >= c.q) a1.hi -= c.q;
            if (a1.hi >= c.q) a1.hi -= c.q;
            if (a2.hi >= c.q) a2.hi -= c.q;
        }
    }
    // redc gives sum * 2^-64; one more Montgomery product with R^2 restores it
    uint64_t d[3] = {redc(a0.hi, a0.lo, c.q, c.qinv), redc(a1.hi, a1.lo, c.q, c.qinv),
                     redc(a2.hi, a2.lo, c.q, c.qinv)};
    uint64_t *O = out[o];
#pragma unroll
    for (int j = 0; j < 3; j++) {
        uint64_t v = redc(mulhi(d[j], c.r2), d[j] * c.r2, c.q, c.qinv);
        if (j == 0 && cres) v = add_mod(v, cres[(size_t)o * ell + l], c.q);
        O[((size_t)j * ell + l) * N + k] = v;
    }
}

}  // namespace

extern "C" int he_square_sum(he_ctx *c, const uint64_t *const *in, int n_in, uint64_t *const *out, int n_out,
                             const int32_t *row_ptr, const int32_t *col, const uint64_t *residues, int ell,
                             void *stream) {
    if (!c || n_in < 1 || n_out < 0 || ell < 1 || ell > c->L || !row_ptr || !col || c->N < LB) {
        he_set_error("he_square_sum: bad arguments");
        return HE_EINVAL;
    }
    if (!n_out) return HE_OK;
    const int nnz = row_ptr[n_out];
    int kmax = 0;
    for (int o = 0; o < n_out; o++) {
        if (row_ptr[o + 1] < row_ptr[o]) {
            he_set_error("he_square_sum: row_ptr not monotone");
            return HE_EINVAL;
        }
        kmax = std::max(kmax, row_ptr[o + 1] - row_ptr[o]);
    }
    for (int t = 0; t < nnz; t++)
        if (col[t] < 0 || col[t] >= n_in) {
            he_set_error("he_square_sum: col[%d] out of range", t);
            return HE_EINVAL;
        }
    if (residues)
        for (int i = 0; i < n_out * ell; i++)
            if (residues[i] >= c->mod[i % ell]) {
                he_set_error("he_square_sum: residue %d not canonical", i);
                return HE_EINVAL;
            }
    cudaStream_t s = (cudaStream_t)stream;
    void **din = nullptr, **dout = nullptr;
    HE_TRY(he_upload_ptrs((const void *const *)in, n_in, &din, s));
    HE_TRY(he_upload_ptrs((const void *const *)out, n_out, &dout, s));
    char *meta = nullptr;
    size_t b_rp = (size_t)(n_out + 1) * 4, b_col = (size_t)std::max(nnz, 1) * 4, b_res = (size_t)n_out * ell * 8;
    HE_TRY(he_scratch_alloc((void **)&meta, b_res + b_rp + b_col + 64, s));
    uint64_t *dres = residues ? (uint64_t *)meta : nullptr;
    int32_t *drp = (int32_t *)(meta + b_res), *dcol = (int32_t *)(meta + b_res + b_rp);
    if (residues) HE_CHECK_CUDA(he_h2d(dres, residues, b_res, s));
    HE_CHECK_CUDA(he_h2d(drp, row_ptr, b_rp, s));
    HE_CHECK_CUDA(he_h2d(dcol, col, (size_t)nnz * 4, s));
    int rc = HE_OK;
    const int cpp = c->N / LB;
    for (int o0 = 0; o0 < n_out && rc == HE_OK; o0 += 65535) {
        const int cnt = std::min(65535, n_out - o0);
        dim3 grid((unsigned)cnt, (unsigned)(ell * cpp));
        k_square_sum<<<grid, LB, 0, s>>>((uint64_t *const *)dout + o0, (const uint64_t *const *)din, drp + o0, dcol,
                                         dres ? dres + (size_t)o0 * ell : nullptr, cnt, ell, c->logN, kmax, c->d_mc);
        he_count_launch(1);
        if (cudaGetLastError() != cudaSuccess) rc = HE_ECUDA;
    }
    he_scratch_free(meta, s);
    he_scratch_free(din, s);
    he_scratch_free(dout, s);
    return rc;
}

extern "C" int he_lincomb_grouped(he_ctx *c, const uint64_t *const *in, int n_in, uint64_t *const *out, int n_out,
                                  int n_groups, const int32_t *term_ptr, const int32_t *term_col,
                                  const int32_t *term_tap, const int32_t *out_base, int out_stride, int M, int T,
                                  const int64_t *weights, const uint64_t *residues, int ell, int nc,
                                  void *stream) {
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
    std::vector<Term> terms(std::max(nnz, 1));
    for (int t = 0; t < nnz; t++) {
        if (term_col[t] < 0 || term_col[t] >= n_in || term_tap[t] < 0 || term_tap[t] >= T) {
            he_set_error("he_lincomb_grouped: term %d (col %d tap %d) out of range", t, term_col[t], term_tap[t]);
            return HE_EINVAL;
        }
        terms[t].p = in[term_col[t]];
        terms[t].tap = term_tap[t];
        terms[t].pad = 0;
    }
    for (int i = 0; i < M * T; i++)
        if (weights[i] >= ((int64_t)1 << 62) || weights[i] <= -((int64_t)1 << 62)) {
            he_set_error("he_lincomb_grouped: |w| >= 2^62");
            return HE_EINVAL;
        }
    const int MM = M <= 2 ? 2 : M <= 4 ? 4 : M <= 8 ? 8 : M <= 16 ? 16 : 32;
    cudaStream_t s = (cudaStream_t)stream;
    void **dout = nullptr;
    HE_TRY(he_upload_ptrs((const void *const *)out, n_out, &dout, s));
    if (residues)
        for (int i = 0; i < M * ell; i++)
            if (residues[i] >= c->mod[i % ell]) {
                he_set_error("he_lincomb_grouped: residue %d not canonical", i);
                return HE_EINVAL;
            }
    size_t b_tp = (size_t)(n_groups + 1) * 4, b_terms = terms.size() * sizeof(Term), b_ob = (size_t)n_groups * 4,
           b_w = (size_t)M * T * 8, b_wM = (size_t)ell * T * MM * 8, b_res = (size_t)M * ell * 8;
    char *meta = nullptr;
    HE_TRY(he_scratch_alloc((void **)&meta, b_wM + b_terms + b_w + b_tp + b_ob + b_res + 64, s));
    uint64_t *dres =
        residues ? (uint64_t *)(meta + ((b_wM + b_terms + b_w + b_tp + b_ob + 7) & ~(size_t)7)) : nullptr;
    if (residues) HE_CHECK_CUDA(he_h2d(dres, residues, b_res, s));
    uint64_t *wM = (uint64_t *)meta;
    Term *dterms = (Term *)(meta + b_wM);
    int64_t *dw = (int64_t *)(meta + b_wM + b_terms);
    int32_t *dtp = (int32_t *)(meta + b_wM + b_terms + b_w);
    int32_t *dob = (int32_t *)(meta + b_wM + b_terms + b_w + b_tp);
    HE_CHECK_CUDA(he_h2d(dterms, terms.data(), b_terms, s));
    HE_CHECK_CUDA(he_h2d(dw, weights, b_w, s));
    HE_CHECK_CUDA(he_h2d(dtp, term_ptr, b_tp, s));
    HE_CHECK_CUDA(he_h2d(dob, out_base, b_ob, s));
    k_group_weights<<<ceil_div((size_t)ell * T * MM, 256), 256, 0, s>>>(wM, dw, M, MM, T, ell, c->d_mc);
    HE_CHECK_LAUNCH();
    const int gpb = std::max(1, std::min(8, n_groups / 148));
    const int cpp = c->N / LB;
    int max_block_terms = 0;
    for (int g0 = 0; g0 < n_groups; g0 += gpb)
        max_block_terms = std::max(max_block_terms, term_ptr[std::min(g0 + gpb, n_groups)] - term_ptr[g0]);
    const size_t smem = (size_t)T * MM * 8 + (size_t)max_block_terms * sizeof(Term);
    if (smem > 200 * 1024) {
        he_set_error("he_lincomb_grouped: %zu bytes of shared memory needed (T=%d, M=%d)", smem, T, M);
        he_scratch_free(meta, s);
        he_scratch_free(dout, s);
        return HE_EINVAL;
    }
    int rc = HE_OK;
    if ((size_t)nc * ell * cpp > 65535) {
        he_set_error("he_lincomb_grouped: grid too large");
        rc = HE_EINVAL;
    }
    GroupArgs a;
    a.out = (uint64_t *const *)dout;
    a.term_ptr = dtp;
    a.terms = dterms;
    a.out_base = dob;
    a.wM = wM;
    a.mc = c->d_mc;
    a.cres = dres;
    a.out_stride = out_stride;
    a.M = M;
    a.T = T;
    a.WS = MM;
    a.n_groups = n_groups;
    a.gpb = gpb;
    a.ell = ell;
    a.logN = c->logN;
    a.kmax = kmax;
    // runs of consecutive limbs that share the accumulator variant
    auto fast_ok = [&](int l) {
        return c->mod[l] < (1ull << 52) && (double)kmax * (double)c->mod[l] < 1.8e19 && kmax <= 1024;
    };
    for (int l0 = 0; l0 < ell && rc == HE_OK;) {
        const bool fast = fast_ok(l0);
        int l1 = l0 + 1;
        while (l1 < ell && fast_ok(l1) == fast) l1++;
        a.l_lo = l0;
        a.nl = l1 - l0;
        dim3 grid(ceil_div(n_groups, gpb), (unsigned)(nc * a.nl * cpp));
        const int mm = fast ? std::min(MM, 8) : MM;
        for (int m0 = 0; m0 < M && rc == HE_OK; m0 += mm) {
            a.m_off = m0;
            rc = dispatch_grouped(mm, fast, grid, smem, s, a);
        }
        l0 = l1;
    }
    he_scratch_free(meta, s);
    he_scratch_free(dout, s);
    return rc;
}
