// ops.cu -- ciphertext arithmetic for sm_100a: element-wise ops, tensor,
// rescale, hybrid key switching (relinearisation, rotation) and the
// feature-major linear combination.
//
// Reference operations replaced (all in /root/reference/pkg/src/hebatch):
//   add / add_plain            engine.py:285-295   -> k_add / k_add_const
//   mult_plain (+ level -1)    engine.py:297-304   -> k_mul_const + rescale
//   mult_ct (+ level -1)       engine.py:306-313   -> tensor + relin + rescale
//   rotate                     engine.py:276-283   -> automorphism + key switch
//   conv_forward k=1 fold loop conv.py:137-156     -> k_lincomb (one launch)
// Arithmetic contract: DESIGN.md section 2; oracle/ckks_oracle.c restates it.
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace {

constexpr int EW = 256;          // threads per CTA for element-wise kernels
constexpr size_t SCRATCH_BUDGET = (size_t)6 << 30;  // bytes of temporaries per chunk

__device__ __forceinline__ int limb_of(size_t idx, int logN, int ell) { return (int)((idx >> logN) % ell); }

// ---------------------------------------------------------------- element-wise
__global__ void k_addsub(uint64_t *const *out, const uint64_t *const *a, const uint64_t *const *b, int count,
                         int ell, int nc, int logN, const ModConst *mc, int sub) {
    size_t per = (size_t)nc * ell << logN;
    for (int ct = blockIdx.y; ct < count; ct += gridDim.y) {
        const uint64_t *A = a[ct], *B = b[ct];
        uint64_t *O = out[ct];
        for (size_t i = 2 * (blockIdx.x * (size_t)blockDim.x + threadIdx.x); i < per; i += 2 * (size_t)gridDim.x * blockDim.x) {
            uint64_t q = mc[limb_of(i, logN, ell)].q;
            ulonglong2 x = *(const ulonglong2 *)(A + i), y = *(const ulonglong2 *)(B + i);
            ulonglong2 r;
            r.x = sub ? sub_mod(x.x, y.x, q) : add_mod(x.x, y.x, q);
            r.y = sub ? sub_mod(x.y, y.y, q) : add_mod(x.y, y.y, q);
            *(ulonglong2 *)(O + i) = r;
        }
    }
}

// res: device [count][ell] residues.  add: constant added to component 0 only.
__global__ void k_const(uint64_t *const *out, const uint64_t *const *in, int count, int ell, int nc, int logN,
                        const ModConst *mc, const uint64_t *res, int mul) {
    size_t per = (size_t)nc * ell << logN;
    size_t c0 = (size_t)ell << logN;
    for (int ct = blockIdx.y; ct < count; ct += gridDim.y) {
        const uint64_t *A = in[ct];
        uint64_t *O = out[ct];
        for (size_t i = 2 * (blockIdx.x * (size_t)blockDim.x + threadIdx.x); i < per; i += 2 * (size_t)gridDim.x * blockDim.x) {
            int l = limb_of(i, logN, ell);
            const ModConst m = mc[l];
            uint64_t r = res[(size_t)ct * ell + l];
            ulonglong2 x = *(const ulonglong2 *)(A + i);
            if (mul) {
                uint64_t rM = redc(mulhi(r, m.r2), r * m.r2, m.q, m.qinv);  // r * 2^64 mod q
                x.x = redc(mulhi(x.x, rM), x.x * rM, m.q, m.qinv);
                x.y = redc(mulhi(x.y, rM), x.y * rM, m.q, m.qinv);
            } else if (i < c0) {
                x.x = add_mod(x.x, r, m.q);
                x.y = add_mod(x.y, r, m.q);
            }
            *(ulonglong2 *)(O + i) = x;
        }
    }
}

__global__ void k_mul_plain(uint64_t *const *out, const uint64_t *const *in, const uint64_t *pt, int count, int ell,
                            int nc, int logN, const ModConst *mc) {
    size_t per = (size_t)nc * ell << logN, poly = (size_t)ell << logN;
    for (int ct = blockIdx.y; ct < count; ct += gridDim.y) {
        const uint64_t *A = in[ct];
        uint64_t *O = out[ct];
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < per; i += (size_t)gridDim.x * blockDim.x)
            O[i] = mul_mod(A[i], pt[i % poly], mc[limb_of(i, logN, ell)]);
    }
}

__global__ void k_drop(uint64_t *const *out, const uint64_t *const *in, int count, int ell_in, int ell_out, int nc,
                       int logN) {
    size_t per = (size_t)nc * ell_out << logN;
    for (int ct = blockIdx.y; ct < count; ct += gridDim.y) {
        const uint64_t *A = in[ct];
        uint64_t *O = out[ct];
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < per; i += (size_t)gridDim.x * blockDim.x) {
            size_t comp = i / ((size_t)ell_out << logN), rem = i % ((size_t)ell_out << logN);
            O[i] = A[comp * ((size_t)ell_in << logN) + rem];
        }
    }
}

__global__ void k_tensor(uint64_t *const *out, const uint64_t *const *a, const uint64_t *const *b, int count, int ell,
                         int logN, const ModConst *mc) {
    size_t P = (size_t)ell << logN;
    for (int ct = blockIdx.y; ct < count; ct += gridDim.y) {
        const uint64_t *A = a[ct], *B = b[ct];
        uint64_t *O = out[ct];
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < P; i += (size_t)gridDim.x * blockDim.x) {
            const ModConst m = mc[i >> logN];
            uint64_t a0 = A[i], a1 = A[P + i], b0 = B[i], b1 = B[P + i];
            // exact 128-bit sums, one Montgomery pass, then fix the R^-1 factor
            u128 t0 = {0, 0}, t1 = {0, 0}, t2 = {0, 0};
            mac128(t0, a0, b0);
            mac128(t1, a0, b1);
            mac128(t1, a1, b0);
            mac128(t2, a1, b1);
            if (t1.hi >= m.q) t1.hi -= m.q;
            uint64_t d0 = redc(t0.hi, t0.lo, m.q, m.qinv);
            uint64_t d1 = redc(t1.hi, t1.lo, m.q, m.qinv);
            uint64_t d2 = redc(t2.hi, t2.lo, m.q, m.qinv);
            O[i] = redc(mulhi(d0, m.r2), d0 * m.r2, m.q, m.qinv);
            O[P + i] = redc(mulhi(d1, m.r2), d1 * m.r2, m.q, m.qinv);
            O[2 * P + i] = redc(mulhi(d2, m.r2), d2 * m.r2, m.q, m.qinv);
        }
    }
}

__device__ __forceinline__ uint32_t galois_src(uint32_t k, uint32_t g, int logN) {
    uint32_t e = 2u * (__brev(k) >> (32 - logN)) + 1u;
    uint32_t e2 = (uint32_t)(((uint64_t)e * g) & ((2ull << logN) - 1));
    return __brev((e2 - 1u) >> 1) >> (32 - logN);
}

// out (contiguous [count][npoly][N]) from pointer-array input
__global__ void k_automorph_ptrs(uint64_t *const *out, const uint64_t *const *in, int count, int npoly, int logN,
                                 uint32_t g) {
    size_t per = (size_t)npoly << logN, N = (size_t)1 << logN;
    for (int ct = blockIdx.y; ct < count; ct += gridDim.y) {
        const uint64_t *A = in[ct];
        uint64_t *O = out[ct];
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < per; i += (size_t)gridDim.x * blockDim.x) {
            size_t p = i >> logN;
            O[i] = A[p * N + galois_src((uint32_t)(i & (N - 1)), g, logN)];
        }
    }
}

// ---------------------------------------------------------------- rescale pieces
// gather the last limb of every (ct, comp) into r [count*nc][N]
__global__ void k_gather_last(uint64_t *r, const uint64_t *const *in, int count, int ell, int nc, int logN) {
    size_t N = (size_t)1 << logN, tot = (size_t)count * nc * N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
        size_t pc = i >> logN;
        int ct = (int)(pc / nc), comp = (int)(pc % nc);
        r[i] = in[ct][((size_t)comp * ell + ell - 1) * N + (i & (N - 1))];
    }
}
// t [count*nc][ell-1][N] = centered(r) mod q_i
__global__ void k_expand_centered(uint64_t *t, const uint64_t *r, size_t npc, int lm1, int logN, const ModConst *mc,
                                  uint64_t ql) {
    size_t N = (size_t)1 << logN, tot = npc * lm1 * N;
    uint64_t half = (ql - 1) >> 1;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
        size_t pc = i / ((size_t)lm1 * N);
        int l = (int)((i >> logN) % lm1);
        uint64_t v = r[pc * N + (i & (N - 1))];
        const ModConst m = mc[l];
        t[i] = v > half ? sub_mod(0, reduce64(ql - v, m), m.q) : reduce64(v, m);
    }
}
// out[i] = (x_i - t_i) * ql^-1 mod q_i
__global__ void k_rescale_final(uint64_t *const *out, const uint64_t *const *in, const uint64_t *t, int count, int ell,
                                int nc, int logN, const ModConst *mc, const uint64_t *qlinv /*[ell-1][2]*/) {
    int lm1 = ell - 1;
    size_t N = (size_t)1 << logN, per = (size_t)nc * lm1 * N;
    for (int ct = blockIdx.y; ct < count; ct += gridDim.y) {
        const uint64_t *X = in[ct];
        uint64_t *O = out[ct];
        const uint64_t *T = t + (size_t)ct * per;
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < per; i += (size_t)gridDim.x * blockDim.x) {
            size_t comp = i / ((size_t)lm1 * N);
            int l = (int)((i >> logN) % lm1);
            uint64_t q = mc[l].q;
            uint64_t x = X[(comp * ell + l) * N + (i & (N - 1))];
            O[i] = shoup(sub_mod(x, T[i], q), qlinv[2 * l], qlinv[2 * l + 1], q);
        }
    }
}

// ---------------------------------------------------------------- key switching pieces
// dc [B][ell][N] <- d pointers (copy, then INTT in place)
__global__ void k_gather_polys(uint64_t *dst, const uint64_t *const *src, int count, size_t per_words) {
    for (int ct = blockIdx.y; ct < count; ct += gridDim.y) {
        const uint64_t *S = src[ct];
        uint64_t *D = dst + (size_t)ct * per_words;
        for (size_t i = 2 * (blockIdx.x * (size_t)blockDim.x + threadIdx.x); i < per_words; i += 2 * (size_t)gridDim.x * blockDim.x)
            *(ulonglong2 *)(D + i) = *(const ulonglong2 *)(S + i);
    }
}

// ModUp basis conversion for digit j: from dc[b][S_j][N] (coefficient domain)
// into ext[b][j][pos][N] for every target pos not in S_j.
// tab layout: [ns] qhat^-1, [ns] Shoup, [nd][ns] (qhat mod t) * 2^64 mod t
__global__ void k_modup_bconv(uint64_t *ext, const uint64_t *dc, int B, int ell, int ext_n, int beta, int j, int s0,
                              int ns, int nd, const uint64_t *tab, const int32_t *src_mod, const int32_t *dst_mod,
                              const ModConst *mc, int logN, int L) {
    size_t N = (size_t)1 << logN;
    size_t tot = (size_t)B * N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
        size_t b = i >> logN, k = i & (N - 1);
        uint64_t v[8];
        const uint64_t *D = dc + b * ell * N;
        for (int s = 0; s < ns; s++) {
            uint64_t qs = mc[src_mod[s]].q;
            v[s] = shoup(D[(size_t)(s0 + s) * N + k], tab[s], tab[ns + s], qs);
        }
        uint64_t *E = ext + ((b * beta + j) * (size_t)ext_n) * N;
        for (int d = 0; d < nd; d++) {
            int m = dst_mod[d];
            const ModConst mcd = mc[m];
            const uint64_t *row = tab + 2 * ns + (size_t)d * ns;
            u128 acc = {0, 0};
            for (int s = 0; s < ns; s++) {
                mac128(acc, v[s], row[s]);  // v < 2^61, row < q_t: keep hi < q_t
                if (acc.hi >= mcd.q) acc.hi -= mcd.q;
            }
            int pos = m < L ? m : ell + (m - L);
            E[(size_t)pos * N + k] = redc(acc.hi, acc.lo, mcd.q, mcd.qinv);
        }
    }
}

// inner product with the switch key.  ext positions in S_j come from d itself.
// acc [B][2][ext_n][N] canonical.
__global__ void k_ks_inner(uint64_t *acc, const uint64_t *ext, const uint64_t *const *d, const uint64_t *key, int B,
                           int ell, int ext_n, int beta, int alpha, int L, int K, int logN, const ModConst *mc) {
    size_t N = (size_t)1 << logN;
    size_t M = (size_t)(L + K);
    size_t tot = (size_t)B * ext_n * N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
        size_t b = i / ((size_t)ext_n * N);
        int t = (int)((i >> logN) % ext_n);
        size_t k = i & (N - 1);
        int m = t < ell ? t : L + (t - ell);
        const ModConst c = mc[m];
        u128 a0 = {0, 0}, a1 = {0, 0};
        int jt = t < ell ? t / alpha : -1;
        for (int j = 0; j < beta; j++) {
            uint64_t e = (j == jt) ? d[b][(size_t)t * N + k] : ext[(((b * beta + j) * (size_t)ext_n) + t) * N + k];
            const uint64_t *kb = key + ((size_t)j * 2 * M + m) * N + k;
            mac128(a0, e, kb[0]);
            mac128(a1, e, kb[M * N]);
            if (a0.hi >= c.q) a0.hi -= c.q;
            if (a1.hi >= c.q) a1.hi -= c.q;
        }
        size_t o = (b * 2 * ext_n + t) * N + k;
        acc[o] = redc(a0.hi, a0.lo, c.q, c.qinv);
        acc[o + (size_t)ext_n * N] = redc(a1.hi, a1.lo, c.q, c.qinv);
    }
}

// ModDown basis conversion: P limbs of acc (coefficient domain) -> conv [B][2][ell][N]
__global__ void k_moddown_bconv(uint64_t *conv, const uint64_t *acc, int B, int ell, int ext_n, int K,
                                const uint64_t *tab, const int32_t *src_mod, const ModConst *mc, int logN) {
    size_t N = (size_t)1 << logN;
    size_t tot = (size_t)B * 2 * N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
        size_t bc = i >> logN, k = i & (N - 1);
        const uint64_t *A = acc + bc * ext_n * N;
        uint64_t v[16];
        for (int s = 0; s < K; s++) {
            uint64_t qs = mc[src_mod[s]].q;
            v[s] = shoup(A[(size_t)(ell + s) * N + k], tab[s], tab[K + s], qs);
        }
        uint64_t *C = conv + bc * ell * N;
        for (int d = 0; d < ell; d++) {
            const ModConst mcd = mc[d];
            const uint64_t *row = tab + 2 * K + (size_t)d * K;
            u128 a = {0, 0};
            for (int s = 0; s < K; s++) {
                mac128(a, v[s], row[s]);
                if (a.hi >= mcd.q) a.hi -= mcd.q;
            }
            C[(size_t)d * N + k] = redc(a.hi, a.lo, mcd.q, mcd.qinv);
        }
    }
}

// out_c[i] = (acc_c[i] - conv_c[i]) * P^-1 (+ add_c[i])
__global__ void k_moddown_final(uint64_t *const *out0, uint64_t *const *out1, const uint64_t *const *add0,
                                const uint64_t *const *add1, const uint64_t *acc, const uint64_t *conv, int B, int ell,
                                int ext_n, int logN, const ModConst *mc, const uint64_t *pinv) {
    size_t N = (size_t)1 << logN, per = (size_t)ell * N;
    for (int b = blockIdx.y; b < B; b += gridDim.y) {
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < 2 * per; i += (size_t)gridDim.x * blockDim.x) {
            int c = (int)(i / per);
            size_t r = i % per;
            int l = (int)(r >> logN);
            uint64_t q = mc[l].q;
            uint64_t x = acc[((size_t)b * 2 + c) * ext_n * N + r];
            uint64_t y = conv[((size_t)b * 2 + c) * per + r];
            uint64_t v = shoup(sub_mod(x, y, q), pinv[2 * l], pinv[2 * l + 1], q);
            const uint64_t *const *add = c == 0 ? add0 : add1;
            if (add) v = add_mod(v, add[b][r], q);
            (c == 0 ? out0 : out1)[b][r] = v;
        }
    }
}

// ---------------------------------------------------------------- lincomb
// wM [nnz][ell] = (w mod q_i) * 2^64 mod q_i
__global__ void k_lincomb_weights(uint64_t *wM, const int64_t *w, int nnz, int ell, const ModConst *mc) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= (size_t)nnz * ell) return;
    int l = (int)(i % ell);
    const ModConst m = mc[l];
    uint64_t r = smod64(w[i / ell], m.q);
    wM[i] = redc(mulhi(r, m.r2), r * m.r2, m.q, m.qinv);
}

// grid.x = (comp, limb, coefficient block of 256); grid.y = output tile of `tile` outputs
__global__ void __launch_bounds__(256) k_lincomb(uint64_t *const *out, const uint64_t *const *in, const int32_t *row_ptr,
                                                 const int32_t *col, const uint64_t *wM, int n_out, int tile, int ell,
                                                 int logN, const ModConst *mc) {
    size_t N = (size_t)1 << logN;
    int cpp = (int)(N / blockDim.x);  // coefficient blocks per limb-poly
    int pl = blockIdx.x / cpp;  // comp * ell + limb
    int l = pl % ell;
    size_t off = (size_t)pl * N + (size_t)(blockIdx.x % cpp) * blockDim.x + threadIdx.x;
    const ModConst m = mc[l];
    int o0 = blockIdx.y * tile, o1 = min(o0 + tile, n_out);
    for (int o = o0; o < o1; o++) {
        u128 acc = {0, 0};
        int t1 = row_ptr[o + 1];
        for (int t = row_ptr[o]; t < t1; t++) {
            uint64_t x = __ldg(in[col[t]] + off);
            mac128(acc, x, wM[(size_t)t * ell + l]);
            if (acc.hi >= m.q) acc.hi -= m.q;
        }
        out[o][off] = redc(acc.hi, acc.lo, m.q, m.qinv);
    }
}

// ---------------------------------------------------------------- launch helpers
inline dim3 grid_ew(size_t per_ct_words, int count, int vec = 1) {
    size_t threads = (per_ct_words / vec + EW - 1) / EW;
    unsigned gx = (unsigned)std::min<size_t>(threads, 4096);
    unsigned gy = (unsigned)std::min(count, 65535);
    return dim3(gx ? gx : 1, gy ? gy : 1);
}
inline unsigned grid_flat(size_t n) { return (unsigned)std::min<size_t>((n + EW - 1) / EW, (size_t)148 * 64); }

struct DevPtrs {
    void **p = nullptr;
    cudaStream_t s;
    explicit DevPtrs(cudaStream_t st) : s(st) {}
    ~DevPtrs() { he_scratch_free(p, s); }
    int up(const void *const *h, int n) { return he_upload_ptrs(h, n, &p, s); }
    template <class T>
    T **as() const { return (T **)p; }
};

struct Scratch {
    void *p = nullptr;
    cudaStream_t s;
    explicit Scratch(cudaStream_t st) : s(st) {}
    ~Scratch() { he_scratch_free(p, s); }
    int alloc(size_t bytes) { return he_scratch_alloc(&p, bytes, s); }
    uint64_t *u() const { return (uint64_t *)p; }
};

int check_basic(he_ctx *c, int count, int ell, int nc, const char *fn) {
    if (!c) {
        he_set_error("%s: null context", fn);
        return HE_EINVAL;
    }
    if (count < 0 || ell < 1 || ell > c->L || nc < 1 || nc > 5) {
        he_set_error("%s: bad shape count=%d ell=%d n_comp=%d (L=%d)", fn, count, ell, nc, c->L);
        return HE_EINVAL;
    }
    return HE_OK;
}

// chunk size so that `bytes_per_ct` temporaries stay within the budget
inline int chunk_of(size_t bytes_per_ct, int count) {
    size_t ch = std::max<size_t>(1, SCRATCH_BUDGET / std::max<size_t>(bytes_per_ct, 1));
    return (int)std::min<size_t>(ch, (size_t)count);
}

// Hybrid key switch of d (ell limbs, NTT) for a chunk of B ciphertexts held
// in device pointer arrays (already offset to the chunk).  Writes
// out_c = KS_c(d) (+ add_c).  Scratch is allocated per call.
int keyswitch_chunk(he_ctx *c, const uint64_t *key, uint64_t *const *d_dev, int B, int ell, uint64_t *const *out0,
                    uint64_t *const *out1, const uint64_t *const *add0, const uint64_t *const *add1, cudaStream_t s) {
    const int N = c->N, L = c->L, K = c->K, alpha = c->alpha, logN = c->logN;
    const int beta = (ell + alpha - 1) / alpha, ext_n = ell + K;
    const size_t Nw = (size_t)N;
    size_t w_dc = (size_t)B * ell * Nw, w_ext = (size_t)B * beta * ext_n * Nw, w_acc = (size_t)B * 2 * ext_n * Nw,
           w_conv = (size_t)B * 2 * ell * Nw;
    Scratch sc(s);
    HE_TRY(sc.alloc((w_dc + w_ext + w_acc + w_conv) * 8));
    uint64_t *dc = sc.u(), *ext = dc + w_dc, *acc = ext + w_ext, *conv = acc + w_acc;
    // 1. coefficient-domain copy of d
    k_gather_polys<<<grid_ew(ell * Nw, B, 2), EW, 0, s>>>(dc, (const uint64_t *const *)d_dev, B, ell * Nw);
    HE_CHECK_LAUNCH();
    HE_TRY(he_ntt_inv(c, dc, B * ell, c->d_ident, ell, s));
    // 2. ModUp per digit, then NTT the extended limbs
    std::vector<uint8_t> map((size_t)beta * ext_n, 0xFF);
    for (int j = 0; j < beta; j++) {
        const BconvTable *tab;
        HE_TRY(he_get_modup_table(c, ell, j, &tab));
        int s0 = j * alpha;
        k_modup_bconv<<<grid_flat((size_t)B * Nw), EW, 0, s>>>(ext, dc, B, ell, ext_n, beta, j, s0, tab->n_src,
                                                              tab->n_dst, tab->d, tab->d_src_mod, tab->d_dst_mod,
                                                              c->d_mc, logN, L);
        HE_CHECK_LAUNCH();
        int s1 = std::min(s0 + alpha, ell);
        for (int t = 0; t < ext_n; t++) {
            bool in_s = t >= s0 && t < s1;
            map[(size_t)j * ext_n + t] = in_s ? 0xFF : (uint8_t)(t < ell ? t : L + (t - ell));
        }
    }
    Scratch dmap(s);
    HE_TRY(dmap.alloc(map.size()));
    HE_CHECK_CUDA(he_h2d(dmap.p, map.data(), map.size(), s));
    HE_TRY(he_ntt_fwd(c, ext, B * beta * ext_n, (const uint8_t *)dmap.p, beta * ext_n, s));
    // 3. inner product with the key
    k_ks_inner<<<grid_flat((size_t)B * ext_n * Nw), EW, 0, s>>>(acc, ext, (const uint64_t *const *)d_dev, key, B, ell,
                                                               ext_n, beta, alpha, L, K, logN, c->d_mc);
    HE_CHECK_LAUNCH();
    // 4. ModDown: INTT the P limbs, convert to Q, NTT, subtract and scale by P^-1
    std::vector<uint8_t> pmap((size_t)2 * ext_n, 0xFF);
    for (int k = 0; k < K; k++) {
        pmap[ell + k] = (uint8_t)(L + k);
        pmap[ext_n + ell + k] = (uint8_t)(L + k);
    }
    Scratch dpmap(s);
    HE_TRY(dpmap.alloc(pmap.size()));
    HE_CHECK_CUDA(he_h2d(dpmap.p, pmap.data(), pmap.size(), s));
    HE_TRY(he_ntt_inv(c, acc, B * 2 * ext_n, (const uint8_t *)dpmap.p, 2 * ext_n, s));
    const BconvTable *dt;
    HE_TRY(he_get_moddown_table(c, ell, &dt));
    k_moddown_bconv<<<grid_flat((size_t)B * 2 * Nw), EW, 0, s>>>(conv, acc, B, ell, ext_n, K, dt->d, dt->d_src_mod,
                                                                c->d_mc, logN);
    HE_CHECK_LAUNCH();
    HE_TRY(he_ntt_fwd(c, conv, B * 2 * ell, c->d_ident, ell, s));
    k_moddown_final<<<grid_ew(2 * ell * Nw, B), EW, 0, s>>>(out0, out1, add0, add1, acc, conv, B, ell, ext_n, logN,
                                                            c->d_mc, c->d_pinv);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

size_t ks_bytes_per_ct(he_ctx *c, int ell) {
    int beta = (ell + c->alpha - 1) / c->alpha, ext_n = ell + c->K;
    return ((size_t)ell + (size_t)beta * ext_n + 2 * ext_n + 2 * ell) * c->N * 8;
}

// rescale a chunk: in/out device pointer arrays (offset to the chunk)
int rescale_chunk(he_ctx *c, const uint64_t *const *in, uint64_t *const *out, int B, int ell, int nc, cudaStream_t s) {
    const int N = c->N, logN = c->logN, lm1 = ell - 1;
    size_t npc = (size_t)B * nc;
    Scratch sc(s);
    HE_TRY(sc.alloc((npc * N + npc * lm1 * N) * 8));
    uint64_t *r = sc.u(), *t = r + npc * N;
    k_gather_last<<<grid_flat(npc * N), EW, 0, s>>>(r, in, B, ell, nc, logN);
    HE_CHECK_LAUNCH();
    HE_TRY(he_ntt_inv(c, r, (int)npc, c->d_ident + lm1, 1, s));
    k_expand_centered<<<grid_flat(npc * lm1 * N), EW, 0, s>>>(t, r, npc, lm1, logN, c->d_mc, c->mod[lm1]);
    HE_CHECK_LAUNCH();
    HE_TRY(he_ntt_fwd(c, t, (int)(npc * lm1), c->d_ident, lm1, s));
    k_rescale_final<<<grid_ew((size_t)nc * lm1 * N, B), EW, 0, s>>>(out, in, t, B, ell, nc, logN, c->d_mc,
                                                                    c->d_qlinv + (size_t)lm1 * c->L * 2);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

}  // namespace

// ================================================================ C-ABI
extern "C" int he_add(he_ctx *c, const uint64_t *const *a, const uint64_t *const *b, uint64_t *const *out, int count,
                      int ell, int nc, void *stream) {
    HE_TRY(check_basic(c, count, ell, nc, "he_add"));
    if (!count) return HE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    DevPtrs A(s), B(s), O(s);
    HE_TRY(A.up((const void *const *)a, count));
    HE_TRY(B.up((const void *const *)b, count));
    HE_TRY(O.up((const void *const *)out, count));
    k_addsub<<<grid_ew((size_t)nc * ell * c->N, count, 2), EW, 0, s>>>(O.as<uint64_t>(), A.as<const uint64_t>(),
                                                                        B.as<const uint64_t>(), count, ell, nc, c->logN,
                                                                        c->d_mc, 0);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

extern "C" int he_sub(he_ctx *c, const uint64_t *const *a, const uint64_t *const *b, uint64_t *const *out, int count,
                      int ell, int nc, void *stream) {
    HE_TRY(check_basic(c, count, ell, nc, "he_sub"));
    if (!count) return HE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    DevPtrs A(s), B(s), O(s);
    HE_TRY(A.up((const void *const *)a, count));
    HE_TRY(B.up((const void *const *)b, count));
    HE_TRY(O.up((const void *const *)out, count));
    k_addsub<<<grid_ew((size_t)nc * ell * c->N, count, 2), EW, 0, s>>>(O.as<uint64_t>(), A.as<const uint64_t>(),
                                                                        B.as<const uint64_t>(), count, ell, nc, c->logN,
                                                                        c->d_mc, 1);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

static int const_op(he_ctx *c, const uint64_t *const *in, uint64_t *const *out, int count, int ell, int nc,
                    const uint64_t *res, void *stream, int mul, const char *fn) {
    HE_TRY(check_basic(c, count, ell, nc, fn));
    if (!count) return HE_OK;
    if (!res) {
        he_set_error("%s: null residues", fn);
        return HE_EINVAL;
    }
    for (int i = 0; i < count * ell; i++)
        if (res[i] >= c->mod[i % ell]) {
            he_set_error("%s: residue %d not canonical", fn, i);
            return HE_EINVAL;
        }
    cudaStream_t s = (cudaStream_t)stream;
    DevPtrs I(s), O(s);
    HE_TRY(I.up((const void *const *)in, count));
    HE_TRY(O.up((const void *const *)out, count));
    Scratch R(s);
    HE_TRY(R.alloc((size_t)count * ell * 8));
    HE_CHECK_CUDA(he_h2d(R.p, res, (size_t)count * ell * 8, s));
    k_const<<<grid_ew((size_t)nc * ell * c->N, count, 2), EW, 0, s>>>(O.as<uint64_t>(), I.as<const uint64_t>(), count,
                                                                       ell, nc, c->logN, c->d_mc, R.u(), mul);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

extern "C" int he_add_const(he_ctx *c, const uint64_t *const *in, uint64_t *const *out, int count, int ell, int nc,
                            const uint64_t *res, void *stream) {
    return const_op(c, in, out, count, ell, nc, res, stream, 0, "he_add_const");
}

extern "C" int he_mul_const(he_ctx *c, const uint64_t *const *in, uint64_t *const *out, int count, int ell, int nc,
                            const uint64_t *res, void *stream) {
    return const_op(c, in, out, count, ell, nc, res, stream, 1, "he_mul_const");
}

extern "C" int he_mul_plain(he_ctx *c, const uint64_t *const *in, const uint64_t *pt, uint64_t *const *out, int count,
                            int ell, int nc, void *stream) {
    HE_TRY(check_basic(c, count, ell, nc, "he_mul_plain"));
    if (!count) return HE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    DevPtrs I(s), O(s);
    HE_TRY(I.up((const void *const *)in, count));
    HE_TRY(O.up((const void *const *)out, count));
    k_mul_plain<<<grid_ew((size_t)nc * ell * c->N, count), EW, 0, s>>>(O.as<uint64_t>(), I.as<const uint64_t>(), pt,
                                                                        count, ell, nc, c->logN, c->d_mc);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

extern "C" int he_drop_limbs(he_ctx *c, const uint64_t *const *in, uint64_t *const *out, int count, int ell_in,
                             int ell_out, int nc, void *stream) {
    HE_TRY(check_basic(c, count, ell_in, nc, "he_drop_limbs"));
    if (ell_out < 1 || ell_out > ell_in) {
        he_set_error("he_drop_limbs: ell_out=%d not in [1, %d]", ell_out, ell_in);
        return HE_EINVAL;
    }
    if (!count) return HE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    DevPtrs I(s), O(s);
    HE_TRY(I.up((const void *const *)in, count));
    HE_TRY(O.up((const void *const *)out, count));
    k_drop<<<grid_ew((size_t)nc * ell_out * c->N, count), EW, 0, s>>>(O.as<uint64_t>(), I.as<const uint64_t>(), count,
                                                                       ell_in, ell_out, nc, c->logN);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// ---------------------------------------------------------------- bootstrapping: ModRaise
// limb 0 (q_0) of both components -> t[2 ct + comp] (coefficient domain after the INTT)
__global__ void k_take_limb0(uint64_t *t, const uint64_t *const *in, int count, int ell_in, int logN) {
    const size_t N = (size_t)1 << logN;
    for (int ct = blockIdx.y; ct < count; ct += gridDim.y)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < 2 * N; i += (size_t)gridDim.x * blockDim.x) {
            const size_t comp = i >> logN, k = i & (N - 1);
            t[((size_t)ct * 2 + comp) * N + k] = in[ct][comp * ((size_t)ell_in << logN) + k];
        }
}

// centred lift of a residue mod q_0 to every limb of the output chain:
// v in [0, q_0) -> v - q_0 [v > q_0 / 2] -> mod q_l  (coefficient domain)
__global__ void k_mod_raise_lift(uint64_t *const *out, const uint64_t *t, int count, int ell_out, int logN,
                                 const ModConst *mc) {
    const size_t N = (size_t)1 << logN;
    const uint64_t q0 = mc[0].q;
    for (int ct = blockIdx.y; ct < count; ct += gridDim.y)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < 2 * N; i += (size_t)gridDim.x * blockDim.x) {
            const size_t comp = i >> logN, k = i & (N - 1);
            const uint64_t v = t[((size_t)ct * 2 + comp) * N + k];
            const int64_t cv = v > (q0 >> 1) ? (int64_t)v - (int64_t)q0 : (int64_t)v;
            uint64_t *O = out[ct] + comp * ((size_t)ell_out << logN) + k;
            for (int l = 0; l < ell_out; l++) O[(size_t)l << logN] = smod64(cv, mc[l].q);
        }
}

// ModRaise (the first step of CKKS bootstrapping): a ciphertext read at level 0
// (limb q_0 of `in`, which may hold more limbs) is reinterpreted over the full
// chain q_0 .. q_{ell_out-1}: INTT of limb 0, centred lift of each coefficient
// into every limb, NTT.  Decrypts to m + q_0 I(X) with a small integer
// polynomial I; the EvalMod step of the bootstrap circuit removes q_0 I.
extern "C" int he_mod_raise(he_ctx *c, const uint64_t *const *in, int ell_in, uint64_t *const *out, int count,
                            int ell_out, void *stream) {
    HE_TRY(check_basic(c, count, ell_out, 2, "he_mod_raise"));
    if (ell_in < 1 || ell_in > c->L) {
        he_set_error("he_mod_raise: ell_in=%d not in [1, %d]", ell_in, c->L);
        return HE_EINVAL;
    }
    if (!count) return HE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    DevPtrs I(s), O(s), O2(s);
    HE_TRY(I.up((const void *const *)in, count));
    HE_TRY(O.up((const void *const *)out, count));
    std::vector<const uint64_t *> halves(2 * (size_t)count);
    for (int i = 0; i < count; i++) {
        halves[2 * i] = out[i];
        halves[2 * i + 1] = out[i] + (size_t)ell_out * c->N;
    }
    HE_TRY(O2.up((const void *const *)halves.data(), 2 * count));
    Scratch t(s);
    HE_TRY(t.alloc((size_t)count * 2 * c->N * 8));
    k_take_limb0<<<grid_ew(2 * (size_t)c->N, count), EW, 0, s>>>(t.u(), I.as<const uint64_t>(), count, ell_in, c->logN);
    HE_CHECK_LAUNCH();
    HE_TRY(he_ntt_inv(c, t.u(), 2 * count, c->d_ident, 1, s));
    k_mod_raise_lift<<<grid_ew(2 * (size_t)c->N, count), EW, 0, s>>>(O.as<uint64_t>(), t.u(), count, ell_out, c->logN,
                                                                      c->d_mc);
    HE_CHECK_LAUNCH();
    HE_TRY(he_ntt_fwd_ptrs(c, O2.as<uint64_t>(), 2 * count, ell_out, c->d_ident, s));
    return HE_OK;
}

extern "C" int he_tensor(he_ctx *c, const uint64_t *const *a, const uint64_t *const *b, uint64_t *const *out,
                         int count, int ell, void *stream) {
    HE_TRY(check_basic(c, count, ell, 2, "he_tensor"));
    if (!count) return HE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    DevPtrs A(s), B(s), O(s);
    HE_TRY(A.up((const void *const *)a, count));
    HE_TRY(B.up((const void *const *)b, count));
    HE_TRY(O.up((const void *const *)out, count));
    k_tensor<<<grid_ew((size_t)ell * c->N, count), EW, 0, s>>>(O.as<uint64_t>(), A.as<const uint64_t>(),
                                                                B.as<const uint64_t>(), count, ell, c->logN, c->d_mc);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

extern "C" int he_keyswitch(he_ctx *c, uint32_t g, const uint64_t *const *d, uint64_t *const *out0,
                            uint64_t *const *out1, int count, int ell, void *stream) {
    HE_TRY(check_basic(c, count, ell, 1, "he_keyswitch"));
    const uint64_t *key = he_get_key(c, g);
    if (!key) {
        he_set_error("no switch key for galois element %u", g);
        return HE_ENOKEY;
    }
    if (!count) return HE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    DevPtrs D(s), O0(s), O1(s);
    HE_TRY(D.up((const void *const *)d, count));
    HE_TRY(O0.up((const void *const *)out0, count));
    HE_TRY(O1.up((const void *const *)out1, count));
    int ch = chunk_of(ks_bytes_per_ct(c, ell), count);
    for (int b0 = 0; b0 < count; b0 += ch) {
        int B = std::min(ch, count - b0);
        if (c->logN == 16)
            HE_TRY(he_keyswitch_fused(c, key, d + b0, D.as<const uint64_t>() + b0, B, ell, out0 + b0, out1 + b0,
                                      nullptr, nullptr, s));
        else
            HE_TRY(keyswitch_chunk(c, key, D.as<uint64_t>() + b0, B, ell, O0.as<uint64_t>() + b0,
                                   O1.as<uint64_t>() + b0, nullptr, nullptr, s));
    }
    return HE_OK;
}

extern "C" int he_relin(he_ctx *c, const uint64_t *const *d3, uint64_t *const *out, int count, int ell, void *stream) {
    HE_TRY(check_basic(c, count, ell, 3, "he_relin"));
    const uint64_t *key = he_get_key(c, 0);
    if (!key) {
        he_set_error("relinearisation key not generated");
        return HE_ENOKEY;
    }
    if (!count) return HE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    size_t P = (size_t)ell * c->N;
    std::vector<const uint64_t *> p0(count), p1(count), p2(count);
    std::vector<uint64_t *> q0(count), q1(count);
    for (int i = 0; i < count; i++) {
        p0[i] = d3[i];
        p1[i] = d3[i] + P;
        p2[i] = d3[i] + 2 * P;
        q0[i] = out[i];
        q1[i] = out[i] + P;
    }
    DevPtrs D0(s), D1(s), D2(s), O0(s), O1(s);
    HE_TRY(D0.up((const void *const *)p0.data(), count));
    HE_TRY(D1.up((const void *const *)p1.data(), count));
    HE_TRY(D2.up((const void *const *)p2.data(), count));
    HE_TRY(O0.up((const void *const *)q0.data(), count));
    HE_TRY(O1.up((const void *const *)q1.data(), count));
    int ch = chunk_of(ks_bytes_per_ct(c, ell), count);
    for (int b0 = 0; b0 < count; b0 += ch) {
        int B = std::min(ch, count - b0);
        if (c->logN == 16)
            HE_TRY(he_keyswitch_fused(c, key, p2.data() + b0, D2.as<const uint64_t>() + b0, B, ell, q0.data() + b0,
                                      q1.data() + b0, p0.data() + b0, p1.data() + b0, s));
        else
            HE_TRY(keyswitch_chunk(c, key, D2.as<uint64_t>() + b0, B, ell, O0.as<uint64_t>() + b0,
                                   O1.as<uint64_t>() + b0, D0.as<const uint64_t>() + b0, D1.as<const uint64_t>() + b0,
                                   s));
    }
    return HE_OK;
}

extern "C" int he_relin_rescale_n(he_ctx *c, const uint64_t *const *d, uint64_t *const *out, int count, int ell,
                                  int extra, int nc, void *stream) {
    if (nc != 3 && nc != 5) {
        he_set_error("he_relin_rescale_n: nc=%d (3 or 5 components)", nc);
        return HE_EINVAL;
    }
    HE_TRY(check_basic(c, count, ell, nc, "he_relin_rescale_n"));
    if (extra < 0 || extra >= ell || extra > 8) {
        he_set_error("he_relin_rescale: extra=%d must be in [0, min(ell-1, 8)] (ell=%d)", extra, ell);
        return HE_ELEVEL;
    }
    if (c->logN != 16) {
        he_set_error("he_relin_rescale: the joint ModDown is implemented for N = 2^16 only (log_n=%d)", c->logN);
        return HE_EINVAL;
    }
    const int nk = nc - 2;
    const uint64_t *keys[3] = {nullptr, nullptr, nullptr};
    for (int k = 0; k < nk; k++) {  // s^2: code 0; s^3, s^4: codes 2, 4
        keys[k] = he_get_key(c, k == 0 ? 0u : 2u * (uint32_t)k);
        if (!keys[k]) {
            he_set_error(k == 0 ? "relinearisation key not generated" : "power key s^%d not generated", k + 2);
            return HE_ENOKEY;
        }
    }
    if (!count) return HE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    size_t P = (size_t)ell * c->N;
    int ch = chunk_of((size_t)nk * ks_bytes_per_ct(c, ell), count);
    std::vector<const uint64_t *> pk((size_t)nk * ch);
    for (int b0 = 0; b0 < count; b0 += ch) {
        int B = std::min(ch, count - b0);
        for (int k = 0; k < nk; k++)
            for (int b = 0; b < B; b++) pk[(size_t)k * B + b] = d[b0 + b] + (size_t)(2 + k) * P;
        DevPtrs DK(s);
        HE_TRY(DK.up((const void *const *)pk.data(), nk * B));
        HE_TRY(he_relin_rescale_fused(c, keys, nk, d + b0, DK.as<const uint64_t>(), B, ell, extra, out + b0, s));
    }
    return HE_OK;
}

extern "C" int he_relin_rescale(he_ctx *c, const uint64_t *const *d3, uint64_t *const *out, int count, int ell,
                                int extra, void *stream) {
    return he_relin_rescale_n(c, d3, out, count, ell, extra, 3, stream);
}

extern "C" int he_rescale(he_ctx *c, const uint64_t *const *in, uint64_t *const *out, int count, int ell, int nc,
                          void *stream) {
    HE_TRY(check_basic(c, count, ell, nc, "he_rescale"));
    if (ell < 2) {
        he_set_error("he_rescale: level exhausted (ell=%d)", ell);
        return HE_ELEVEL;
    }
    if (!count) return HE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    DevPtrs I(s), O(s);
    HE_TRY(I.up((const void *const *)in, count));
    HE_TRY(O.up((const void *const *)out, count));
    int ch = chunk_of((size_t)nc * ell * c->N * 8, count);
    for (int b0 = 0; b0 < count; b0 += ch) {
        int B = std::min(ch, count - b0);
        if (c->logN == 16)
            HE_TRY(he_rescale_fused(c, in + b0, out + b0, B, ell, nc, s));
        else
            HE_TRY(rescale_chunk(c, I.as<const uint64_t>() + b0, O.as<uint64_t>() + b0, B, ell, nc, s));
    }
    return HE_OK;
}

extern "C" int he_mult_ct(he_ctx *c, const uint64_t *const *a, const uint64_t *const *b, uint64_t *const *out,
                          int count, int ell, void *stream) {
    HE_TRY(check_basic(c, count, ell, 2, "he_mult_ct"));
    if (ell < 2) {
        he_set_error("he_mult_ct: level exhausted (ell=%d)", ell);
        return HE_ELEVEL;
    }
    const uint64_t *key = he_get_key(c, 0);
    if (!key) {
        he_set_error("relinearisation key not generated");
        return HE_ENOKEY;
    }
    if (!count) return HE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const size_t P = (size_t)ell * c->N;
    DevPtrs A(s), B(s), O(s);
    HE_TRY(A.up((const void *const *)a, count));
    HE_TRY(B.up((const void *const *)b, count));
    HE_TRY(O.up((const void *const *)out, count));
    size_t per_ct = ks_bytes_per_ct(c, ell) + 5 * P * 8 + 2 * P * 8;
    int ch = chunk_of(per_ct, count);
    for (int b0 = 0; b0 < count; b0 += ch) {
        int Bn = std::min(ch, count - b0);
        Scratch sc(s);
        HE_TRY(sc.alloc((size_t)Bn * 5 * P * 8));
        uint64_t *d3 = sc.u(), *rl = d3 + (size_t)Bn * 3 * P;
        std::vector<uint64_t *> pd0(Bn), pd1(Bn), pd2(Bn), pd3(Bn), pr0(Bn), pr1(Bn), prl(Bn);
        for (int i = 0; i < Bn; i++) {
            pd3[i] = d3 + (size_t)i * 3 * P;
            pd0[i] = pd3[i];
            pd1[i] = pd3[i] + P;
            pd2[i] = pd3[i] + 2 * P;
            prl[i] = rl + (size_t)i * 2 * P;
            pr0[i] = prl[i];
            pr1[i] = prl[i] + P;
        }
        DevPtrs D3(s), D0(s), D1(s), D2(s), R0(s), R1(s), RL(s);
        HE_TRY(D3.up((const void *const *)pd3.data(), Bn));
        HE_TRY(D0.up((const void *const *)pd0.data(), Bn));
        HE_TRY(D1.up((const void *const *)pd1.data(), Bn));
        HE_TRY(D2.up((const void *const *)pd2.data(), Bn));
        HE_TRY(R0.up((const void *const *)pr0.data(), Bn));
        HE_TRY(R1.up((const void *const *)pr1.data(), Bn));
        HE_TRY(RL.up((const void *const *)prl.data(), Bn));
        k_tensor<<<grid_ew(P, Bn), EW, 0, s>>>(D3.as<uint64_t>(), A.as<const uint64_t>() + b0,
                                               B.as<const uint64_t>() + b0, Bn, ell, c->logN, c->d_mc);
        HE_CHECK_LAUNCH();
        if (c->logN == 16) {
            HE_TRY(he_keyswitch_fused(c, key, pd2.data(), D2.as<const uint64_t>(), Bn, ell, pr0.data(), pr1.data(),
                                      pd0.data(), pd1.data(), s));
            HE_TRY(he_rescale_fused(c, prl.data(), out + b0, Bn, ell, 2, s));
        } else {
            HE_TRY(keyswitch_chunk(c, key, D2.as<uint64_t>(), Bn, ell, R0.as<uint64_t>(), R1.as<uint64_t>(),
                                   D0.as<const uint64_t>(), D1.as<const uint64_t>(), s));
            HE_TRY(rescale_chunk(c, RL.as<const uint64_t>(), O.as<uint64_t>() + b0, Bn, ell, 2, s));
        }
    }
    return HE_OK;
}

extern "C" int he_automorphism(he_ctx *c, uint32_t g, const uint64_t *const *in, uint64_t *const *out, int count,
                               int ell, int nc, void *stream) {
    HE_TRY(check_basic(c, count, ell, nc, "he_automorphism"));
    if (g % 2 == 0 || g >= 2u * (uint32_t)c->N) {
        he_set_error("galois element %u must be odd and < 2N", g);
        return HE_EINVAL;
    }
    if (!count) return HE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    DevPtrs I(s), O(s);
    HE_TRY(I.up((const void *const *)in, count));
    HE_TRY(O.up((const void *const *)out, count));
    k_automorph_ptrs<<<grid_ew((size_t)nc * ell * c->N, count), EW, 0, s>>>(O.as<uint64_t>(), I.as<const uint64_t>(),
                                                                              count, nc * ell, c->logN, g);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

extern "C" int he_rotate(he_ctx *c, uint32_t g, const uint64_t *const *in, uint64_t *const *out, int count, int ell,
                         void *stream) {
    HE_TRY(check_basic(c, count, ell, 2, "he_rotate"));
    const uint64_t *key = he_get_key(c, g);
    if (!key) {
        he_set_error("no rotation key for galois element %u", g);
        return HE_ENOKEY;
    }
    if (!count) return HE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const size_t P = (size_t)ell * c->N;
    DevPtrs I(s);
    HE_TRY(I.up((const void *const *)in, count));
    int ch = chunk_of(ks_bytes_per_ct(c, ell) + 2 * P * 8, count);
    for (int b0 = 0; b0 < count; b0 += ch) {
        int Bn = std::min(ch, count - b0);
        Scratch sc(s);
        HE_TRY(sc.alloc((size_t)Bn * 2 * P * 8));
        std::vector<uint64_t *> pt(Bn), p0(Bn), p1(Bn), o0(Bn), o1(Bn);
        for (int i = 0; i < Bn; i++) {
            pt[i] = sc.u() + (size_t)i * 2 * P;
            p0[i] = pt[i];
            p1[i] = pt[i] + P;
            o0[i] = out[b0 + i];
            o1[i] = out[b0 + i] + P;
        }
        DevPtrs T(s), T0(s), T1(s), O0(s), O1(s);
        HE_TRY(T.up((const void *const *)pt.data(), Bn));
        HE_TRY(T0.up((const void *const *)p0.data(), Bn));
        HE_TRY(T1.up((const void *const *)p1.data(), Bn));
        HE_TRY(O0.up((const void *const *)o0.data(), Bn));
        HE_TRY(O1.up((const void *const *)o1.data(), Bn));
        k_automorph_ptrs<<<grid_ew(2 * P, Bn), EW, 0, s>>>(T.as<uint64_t>(), I.as<const uint64_t>() + b0, Bn, 2 * ell,
                                                            c->logN, g);
        HE_CHECK_LAUNCH();
        if (c->logN == 16)
            HE_TRY(he_keyswitch_fused(c, key, p1.data(), T1.as<const uint64_t>(), Bn, ell, o0.data(), o1.data(),
                                      p0.data(), nullptr, s));
        else
            HE_TRY(keyswitch_chunk(c, key, T1.as<uint64_t>(), Bn, ell, O0.as<uint64_t>(), O1.as<uint64_t>(),
                                   T0.as<const uint64_t>(), nullptr, s));
    }
    return HE_OK;
}

// Hoisted rotations of `count` ciphertexts by R Galois elements (oracle
// oc_rotate_hoisted): KS of the unrotated c1 with each hoisting key, + c0, then
// sigma_g.  N = 2^16 shares one ModUp of c1 among the R rotations.
// out: HOST array [R][count] of device [2][ell][N] outputs.
extern "C" int he_rotate_hoisted(he_ctx *c, const uint32_t *gs, int R, const uint64_t *const *in,
                                 uint64_t *const *out, int count, int ell, void *stream) {
    HE_TRY(check_basic(c, count, ell, 2, "he_rotate_hoisted"));
    if (R < 1 || !gs) {
        he_set_error("he_rotate_hoisted: no rotations");
        return HE_EINVAL;
    }
    std::vector<const uint64_t *> hk(R);
    for (int r = 0; r < R; r++) {
        if (!he_get_key(c, gs[r])) {
            he_set_error("no rotation key for galois element %u", gs[r]);
            return HE_ENOKEY;
        }
        HE_TRY(he_gen_hoist_key(c, gs[r], stream));
        hk[r] = he_get_key(c, HE_HOIST_CODE | gs[r]);
    }
    if (!count) return HE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const size_t P = (size_t)ell * c->N;
    int ch = chunk_of(ks_bytes_per_ct(c, ell) + (size_t)R * 2 * P * 8, count);
    for (int b0 = 0; b0 < count; b0 += ch) {
        const int Bn = std::min(ch, count - b0);
        Scratch sc(s);  // t_r for every rotation of the chunk: [R][Bn][2][ell][N]
        HE_TRY(sc.alloc((size_t)R * Bn * 2 * P * 8));
        std::vector<const uint64_t *> c0(Bn), c1(Bn);
        std::vector<uint64_t *> t(R * (size_t)Bn), t0(R * (size_t)Bn), t1(R * (size_t)Bn), o(R * (size_t)Bn);
        for (int i = 0; i < Bn; i++) {
            c0[i] = in[b0 + i];
            c1[i] = in[b0 + i] + P;
        }
        for (int r = 0; r < R; r++)
            for (int i = 0; i < Bn; i++) {
                const size_t k = (size_t)r * Bn + i;
                t[k] = t0[k] = sc.u() + k * 2 * P;
                t1[k] = t0[k] + P;
                o[k] = out[(size_t)r * count + b0 + i];
            }
        DevPtrs C1(s);
        HE_TRY(C1.up((const void *const *)c1.data(), Bn));
        if (c->logN == 16) {
            HE_TRY(he_hoisted_ks_fused(c, hk.data(), R, c0.data(), c1.data(), C1.as<const uint64_t>(), Bn, ell,
                                       t0.data(), t1.data(), s));
        } else {
            DevPtrs C0(s);
            HE_TRY(C0.up((const void *const *)c0.data(), Bn));
            for (int r = 0; r < R; r++) {
                DevPtrs T0(s), T1(s);
                HE_TRY(T0.up((const void *const *)(t0.data() + (size_t)r * Bn), Bn));
                HE_TRY(T1.up((const void *const *)(t1.data() + (size_t)r * Bn), Bn));
                HE_TRY(keyswitch_chunk(c, hk[r], (uint64_t *const *)C1.as<uint64_t>(), Bn, ell, T0.as<uint64_t>(),
                                       T1.as<uint64_t>(), C0.as<const uint64_t>(), nullptr, s));
            }
        }
        for (int r = 0; r < R; r++) {  // sigma_g on both components of every t_r
            DevPtrs T(s), O(s);
            HE_TRY(T.up((const void *const *)(t.data() + (size_t)r * Bn), Bn));
            HE_TRY(O.up((const void *const *)(o.data() + (size_t)r * Bn), Bn));
            k_automorph_ptrs<<<grid_ew(2 * P, Bn), EW, 0, s>>>(O.as<uint64_t>(), T.as<const uint64_t>(), Bn, 2 * ell,
                                                                c->logN, gs[r]);
            HE_CHECK_LAUNCH();
        }
    }
    return HE_OK;
}

extern "C" int he_lincomb(he_ctx *c, const uint64_t *const *in, int n_in, uint64_t *const *out, int n_out,
                          const int32_t *row_ptr, const int32_t *col, const int64_t *w, int ell, int nc, void *stream) {
    HE_TRY(check_basic(c, n_out, ell, nc, "he_lincomb"));
    if (n_in < 1 || !row_ptr || !col || !w) {
        he_set_error("he_lincomb: bad arguments");
        return HE_EINVAL;
    }
    if (!n_out) return HE_OK;
    int nnz = row_ptr[n_out];
    if (row_ptr[0] != 0 || nnz < 0) {
        he_set_error("he_lincomb: row_ptr must start at 0");
        return HE_EINVAL;
    }
    for (int o = 0; o < n_out; o++)
        if (row_ptr[o + 1] < row_ptr[o]) {
            he_set_error("he_lincomb: row_ptr not monotone at %d", o);
            return HE_EINVAL;
        }
    for (int t = 0; t < nnz; t++) {
        if (col[t] < 0 || col[t] >= n_in) {
            he_set_error("he_lincomb: col[%d]=%d out of range [0,%d)", t, col[t], n_in);
            return HE_EINVAL;
        }
        if (w[t] >= ((int64_t)1 << 62) || w[t] <= -((int64_t)1 << 62)) {
            he_set_error("he_lincomb: |w[%d]| >= 2^62", t);
            return HE_EINVAL;
        }
    }
    cudaStream_t s = (cudaStream_t)stream;
    DevPtrs I(s), O(s);
    HE_TRY(I.up((const void *const *)in, n_in));
    HE_TRY(O.up((const void *const *)out, n_out));
    Scratch meta(s);
    size_t nz = (size_t)std::max(nnz, 1);
    HE_TRY(meta.alloc(((size_t)n_out + 1) * 4 + nz * 4 + nz * 8 + nz * ell * 8 + 64));
    char *base = (char *)meta.p;
    int64_t *dw = (int64_t *)base;
    uint64_t *wM = (uint64_t *)(base + nz * 8);
    int32_t *drp = (int32_t *)(base + nz * 8 + nz * ell * 8);
    int32_t *dcol = drp + n_out + 1;
    HE_CHECK_CUDA(he_h2d(dw, w, (size_t)nnz * 8, s));
    HE_CHECK_CUDA(he_h2d(drp, row_ptr, ((size_t)n_out + 1) * 4, s));
    HE_CHECK_CUDA(he_h2d(dcol, col, (size_t)nnz * 4, s));
    if (nnz) {
        k_lincomb_weights<<<ceil_div((size_t)nnz * ell, EW), EW, 0, s>>>(wM, dw, nnz, ell, c->d_mc);
        HE_CHECK_LAUNCH();
    }
    int tile = n_out > 4096 ? 16 : (n_out > 256 ? 4 : 1);
    int bs = std::min(c->N, 256);
    unsigned gx = (unsigned)(nc * ell * (c->N / bs));
    for (int o0 = 0; o0 < n_out; o0 += 65535 * tile) {
        int cnt = std::min(n_out - o0, 65535 * tile);
        dim3 grid(gx, ceil_div(cnt, tile));
        k_lincomb<<<grid, bs, 0, s>>>(O.as<uint64_t>() + o0, I.as<const uint64_t>(), drp + o0, dcol, wM, cnt, tile,
                                       ell, c->logN, c->d_mc);
        HE_CHECK_LAUNCH();
    }
    return HE_OK;
}
