/*
 * ckks_oracle.c -- CPU restatement of the RNS-CKKS convention contract.
 *
 * TEST INFRASTRUCTURE ONLY (see ckks_oracle.h).  Written to be obviously
 * correct rather than fast: every modular product is a 128-bit product
 * followed by a hardware divide, every basis conversion is the textbook
 * formula.  OpenMP is used only across independent polynomials.
 *
 * What each function restates (DESIGN.md section 2 is the full contract):
 *   - rotation direction: rotate(ct, k) left-shifts slots, output slot i holds
 *     input slot i+k  (reference engine.py:13-15, engine.py:283 np.roll(-k));
 *     realised as X -> X^{5^k mod 2N}.
 *   - one level per multiplication (engine.py:297-313): mult_plain / mult_ct
 *     are followed by exactly one rescale that drops the last Q limb.
 *   - add at min level (engine.py:289): callers drop limbs before calling add.
 *   - constants over the occupied span (conv.py:160-166, packing.py:146-151)
 *     become constant polynomials: the same residue at every NTT point.
 */
#include "ckks_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;
typedef __int128 i128;

#define MAXM 64
enum { DOM_SK = 1, DOM_ENC_A = 2, DOM_ENC_E = 3, DOM_KSK_A = 4, DOM_KSK_E = 5 };

struct oc_ctx {
    oc_params prm;
    int N, logN, L, K, alpha, dnum, nslots;
    uint64_t mod[MAXM];
    uint64_t psi[MAXM];
    uint64_t *psi_brv[MAXM], *psi_brv_sh[MAXM];      /* forward twiddles + Shoup */
    uint64_t *ipsi_brv[MAXM], *ipsi_brv_sh[MAXM];    /* inverse twiddles + Shoup */
    uint64_t ninv[MAXM];
    uint64_t *sk;                                    /* [L+K][N] NTT domain      */
    double *wr, *wi;                                 /* omega^k, k < nslots      */
    double *zr, *zi;                                 /* zeta^j, j < nslots       */
    int32_t *pos;                                    /* slot i -> FFT index t    */
};

/* ---------------------------------------------------------------- modular */

static inline uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q) {
    /* requires a, b < q so the 128-bit product's high word is < q */
    uint64_t hi, lo, quo, rem;
    __asm__("mulq %3" : "=a"(lo), "=d"(hi) : "a"(a), "rm"(b));
    __asm__("divq %4" : "=a"(quo), "=d"(rem) : "a"(lo), "d"(hi), "rm"(q));
    (void)quo;
    return rem;
}
static inline uint64_t addmod(uint64_t a, uint64_t b, uint64_t q) {
    uint64_t s = a + b;
    return s >= q ? s - q : s;
}
static inline uint64_t submod(uint64_t a, uint64_t b, uint64_t q) { return a >= b ? a - b : a + q - b; }
static uint64_t powmod(uint64_t a, uint64_t e, uint64_t q) {
    uint64_t r = 1 % q;
    a %= q;
    while (e) {
        if (e & 1) r = mulmod(r, a, q);
        a = mulmod(a, a, q);
        e >>= 1;
    }
    return r;
}
static uint64_t invmod(uint64_t a, uint64_t q) { return powmod(a, q - 2, q); } /* q prime */
static inline uint64_t shoup_pre(uint64_t w, uint64_t q) { return (uint64_t)(((u128)w << 64) / q); }
static inline uint64_t mulmod_shoup(uint64_t a, uint64_t w, uint64_t wp, uint64_t q) {
    uint64_t qt = (uint64_t)(((u128)a * wp) >> 64);
    uint64_t r = a * w - qt * q;
    return r >= q ? r - q : r;
}
/* signed int64 -> canonical residue mod q */
static inline uint64_t smod(int64_t v, uint64_t q) {
    if (v >= 0) return (uint64_t)v % q;
    uint64_t r = ((uint64_t)(-(v + 1))) % q; /* |v|-1 mod q, safe for INT64_MIN */
    return q - 1 - r;
}

static int is_prime(uint64_t n) {
    static const uint64_t bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return 0;
    for (int i = 0; i < 12; i++) {
        if (n == bases[i]) return 1;
        if (n % bases[i] == 0) return 0;
    }
    uint64_t d = n - 1;
    int s = 0;
    while (!(d & 1)) { d >>= 1; s++; }
    for (int i = 0; i < 12; i++) {
        uint64_t x = powmod(bases[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int comp = 1;
        for (int r = 1; r < s; r++) {
            x = mulmod(x, x, n);
            if (x == n - 1) { comp = 0; break; }
        }
        if (comp) return 0;
    }
    return 1;
}

static uint32_t brv(uint32_t x, int bits) {
    uint32_t r = 0;
    for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

/* ---------------------------------------------------------------- philox */

void oc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; r++) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* stream word block: counter = (idx, limb, obj, domain), key = seed */
static void rnd4(const oc_ctx *c, uint32_t dom, uint32_t obj, uint32_t limb, uint32_t idx, uint32_t o[4]) {
    uint32_t ctr[4] = {idx, limb, obj, dom};
    uint32_t key[2] = {(uint32_t)c->prm.seed, (uint32_t)(c->prm.seed >> 32)};
    oc_philox(ctr, key, o);
}
static int64_t sample_cbd(const oc_ctx *c, uint32_t dom, uint32_t obj, uint32_t j) {
    uint32_t r[4];
    rnd4(c, dom, obj, 0, j, r);
    return (int64_t)__builtin_popcount(r[0] & 0x1FFFFFu) - (int64_t)__builtin_popcount(r[1] & 0x1FFFFFu);
}
/* Uniform residue k of (dom, obj, limb).  One Philox block serves the pair of indices that
 * differ in bit 4: block index = k with bit 4 removed, words (r0, r1) for bit 4 clear, (r2, r3)
 * for bit 4 set.  A 64-bit draw x is accepted when x < q floor(2^64 / q) and reduced mod q; a
 * rejected draw is replaced by words (r0, r1) of block (k, limb, obj, dom + 16 t), t = 1, 2, ... */
static uint64_t sample_uniform(const oc_ctx *c, uint32_t dom, uint32_t obj, uint32_t limb, uint32_t k,
                               uint64_t q) {
    uint32_t r[4];
    rnd4(c, dom, obj, limb, ((k >> 5) << 4) | (k & 15u), r);
    uint64_t x = (k & 16u) ? ((uint64_t)r[2] | ((uint64_t)r[3] << 32)) : ((uint64_t)r[0] | ((uint64_t)r[1] << 32));
    const uint64_t T = (uint64_t)((((u128)1 << 64) / q) * q);
    for (uint32_t t = 1; x >= T; t++) {
        rnd4(c, dom + 16u * t, obj, limb, k, r);
        x = (uint64_t)r[0] | ((uint64_t)r[1] << 32);
    }
    return x % q;
}
/* secret coefficient j: dense ternary (r mod 3) - 1, or, for sk_hamming = h > 0,
 * nonzero with probability h / N (a second Philox draw below floor(h 2^32 / N))
 * and sign from the low bit of the first draw */
static int64_t sample_ternary(const oc_ctx *c, uint32_t j) {
    uint32_t r[4];
    rnd4(c, DOM_SK, 0, 0, j >> 2, r);
    if (c->prm.sk_hamming <= 0) return (int64_t)(r[j & 3] % 3u) - 1;
    uint32_t r2[4];
    rnd4(c, DOM_SK, 1, 0, j >> 2, r2);
    uint64_t t = ((uint64_t)c->prm.sk_hamming << 32) / (uint64_t)c->N;
    uint32_t thr = t > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)t;
    if (r2[j & 3] >= thr) return 0;
    return (r[j & 3] & 1u) ? 1 : -1;
}

/* ---------------------------------------------------------------- setup */

static void gen_moduli(oc_ctx *c) {
    int total = c->L + c->K;
    uint64_t twoN = 2 * (uint64_t)c->N;
    for (int m = 0; m < total; m++) {
        int bits = m < c->L ? c->prm.q_bits[m] : c->prm.p_bits[m - c->L];
        uint64_t top = (uint64_t)1 << bits;
        for (uint64_t k = 1;; k++) {
            uint64_t cand = top - k * twoN + 1;
            int used = 0;
            for (int u = 0; u < m; u++) used |= (c->mod[u] == cand);
            if (!used && is_prime(cand)) { c->mod[m] = cand; break; }
        }
    }
}

static uint64_t find_psi(uint64_t q, int N) {
    uint64_t e = (q - 1) / (2 * (uint64_t)N);
    for (uint64_t g = 2;; g++) {
        uint64_t psi = powmod(g, e, q);
        if (powmod(psi, (uint64_t)N, q) == q - 1) return psi;
    }
}

oc_ctx *oc_create(const oc_params *p) {
    oc_ctx *c = (oc_ctx *)calloc(1, sizeof(oc_ctx));
    c->prm = *p;
    c->logN = p->log_n;
    c->N = 1 << p->log_n;
    c->L = p->n_q;
    c->K = p->n_p;
    c->alpha = p->alpha;
    c->dnum = (c->L + c->alpha - 1) / c->alpha;
    c->nslots = c->N / 2;
    gen_moduli(c);
    int N = c->N, total = c->L + c->K;
    for (int m = 0; m < total; m++) {
        uint64_t q = c->mod[m];
        uint64_t psi = find_psi(q, N), ipsi = invmod(psi, q);
        c->psi[m] = psi;
        c->psi_brv[m] = (uint64_t *)malloc(8 * N);
        c->psi_brv_sh[m] = (uint64_t *)malloc(8 * N);
        c->ipsi_brv[m] = (uint64_t *)malloc(8 * N);
        c->ipsi_brv_sh[m] = (uint64_t *)malloc(8 * N);
        uint64_t pw = 1, ipw = 1;
        for (int i = 0; i < N; i++) {
            uint32_t r = brv((uint32_t)i, c->logN);
            c->psi_brv[m][r] = pw;
            c->ipsi_brv[m][r] = ipw;
            pw = mulmod(pw, psi, q);
            ipw = mulmod(ipw, ipsi, q);
        }
        for (int i = 0; i < N; i++) {
            c->psi_brv_sh[m][i] = shoup_pre(c->psi_brv[m][i], q);
            c->ipsi_brv_sh[m][i] = shoup_pre(c->ipsi_brv[m][i], q);
        }
        c->ninv[m] = invmod((uint64_t)N % q, q);
    }
    /* FFT tables for the canonical embedding */
    int n = c->nslots;
    c->wr = (double *)malloc(sizeof(double) * n);
    c->wi = (double *)malloc(sizeof(double) * n);
    c->zr = (double *)malloc(sizeof(double) * n);
    c->zi = (double *)malloc(sizeof(double) * n);
    c->pos = (int32_t *)malloc(sizeof(int32_t) * n);
    const double PI = 3.14159265358979323846;
    for (int k = 0; k < n; k++) {
        c->wr[k] = cos(2.0 * PI * (double)k / (double)n);
        c->wi[k] = sin(2.0 * PI * (double)k / (double)n);
        c->zr[k] = cos(PI * (double)k / (double)N);
        c->zi[k] = sin(PI * (double)k / (double)N);
    }
    uint64_t g = 1, twoN = 2 * (uint64_t)N;
    for (int i = 0; i < n; i++) {
        c->pos[i] = (int32_t)((g - 1) / 4);
        g = (g * 5) % twoN;
    }
    /* secret key: ternary coefficients, NTT per modulus */
    c->sk = (uint64_t *)malloc(8 * (size_t)total * N);
    int64_t *s = (int64_t *)malloc(8 * N);
    for (int j = 0; j < N; j++) s[j] = sample_ternary(c, (uint32_t)j);
    for (int m = 0; m < total; m++) {
        uint64_t *dst = c->sk + (size_t)m * N;
        for (int j = 0; j < N; j++) dst[j] = smod(s[j], c->mod[m]);
        oc_ntt(c, dst, m);
    }
    free(s);
    return c;
}

void oc_destroy(oc_ctx *c) {
    if (!c) return;
    for (int m = 0; m < c->L + c->K; m++) {
        free(c->psi_brv[m]); free(c->psi_brv_sh[m]);
        free(c->ipsi_brv[m]); free(c->ipsi_brv_sh[m]);
    }
    free(c->sk); free(c->wr); free(c->wi); free(c->zr); free(c->zi); free(c->pos);
    free(c);
}

/* Coefficient view: the same moduli with N = n evaluation points and no tables.
 * Every element-wise operation in the NTT domain (add, sub, add_const, mul_const,
 * mul_plain, tensor, tensor_sq, lincomb) acts on each evaluation point
 * independently, so running them on n sampled points of [nc][ell][N] ciphertexts
 * (packed as [nc][ell][n]) gives exactly those points of the full result.  NTT,
 * key switching, rescale and encryption need the tables and must not be called
 * on a view (the Python wrapper refuses them).  Free with oc_destroy. */
oc_ctx *oc_coeff_view(const oc_ctx *c, int n) {
    oc_ctx *v = (oc_ctx *)calloc(1, sizeof(oc_ctx));
    v->prm = c->prm;
    v->logN = c->logN;
    v->N = n;
    v->L = c->L;
    v->K = c->K;
    v->alpha = c->alpha;
    v->dnum = c->dnum;
    v->nslots = 0;
    memcpy(v->mod, c->mod, sizeof(c->mod));
    memcpy(v->psi, c->psi, sizeof(c->psi));
    return v;
}

void oc_moduli(const oc_ctx *c, uint64_t *moduli, uint64_t *psi) {
    for (int m = 0; m < c->L + c->K; m++) {
        if (moduli) moduli[m] = c->mod[m];
        if (psi) psi[m] = c->psi[m];
    }
}

void oc_secret_key(const oc_ctx *c, uint64_t *sk_out) {
    memcpy(sk_out, c->sk, 8 * (size_t)(c->L + c->K) * c->N);
}

/* ---------------------------------------------------------------- NTT */

/* forward negacyclic NTT, Cooley-Tukey, natural order in, bit-reversed out:
 * out[k] = a(psi^(2*brv(k)+1)) mod q */
void oc_ntt(const oc_ctx *c, uint64_t *a, int m) {
    int N = c->N;
    uint64_t q = c->mod[m];
    const uint64_t *W = c->psi_brv[m], *Wp = c->psi_brv_sh[m];
    int t = N;
    for (int mm = 1; mm < N; mm <<= 1) {
        t >>= 1;
        for (int i = 0; i < mm; i++) {
            int j1 = 2 * i * t;
            uint64_t w = W[mm + i], wp = Wp[mm + i];
            for (int j = j1; j < j1 + t; j++) {
                uint64_t u = a[j], v = mulmod_shoup(a[j + t], w, wp, q);
                a[j] = addmod(u, v, q);
                a[j + t] = submod(u, v, q);
            }
        }
    }
}

/* inverse, Gentleman-Sande, bit-reversed in, natural out, times N^-1 */
void oc_intt(const oc_ctx *c, uint64_t *a, int m) {
    int N = c->N;
    uint64_t q = c->mod[m];
    const uint64_t *W = c->ipsi_brv[m], *Wp = c->ipsi_brv_sh[m];
    int t = 1;
    for (int mm = N; mm > 1; mm >>= 1) {
        int h = mm >> 1, j1 = 0;
        for (int i = 0; i < h; i++) {
            uint64_t w = W[h + i], wp = Wp[h + i];
            for (int j = j1; j < j1 + t; j++) {
                uint64_t u = a[j], v = a[j + t];
                a[j] = addmod(u, v, q);
                a[j + t] = mulmod_shoup(submod(u, v, q), w, wp, q);
            }
            j1 += 2 * t;
        }
        t <<= 1;
    }
    uint64_t ni = c->ninv[m], nip = shoup_pre(ni, q);
    for (int j = 0; j < N; j++) a[j] = mulmod_shoup(a[j], ni, nip, q);
}

/* ---------------------------------------------------------------- FFT */

/* iterative radix-2 DIT, bit-reversed input permutation, no normalisation.
 * sign = -1: X_j = sum_t x_t w^{-jt};  sign = +1: sum_t x_t w^{+jt}.
 * The operation order here is part of the contract (bit-exact with the GPU). */
static void fft(const oc_ctx *c, double *re, double *im, int sign) {
    int n = c->nslots, bits = c->logN - 1;
    for (int i = 0; i < n; i++) {
        int r = (int)brv((uint32_t)i, bits);
        if (r > i) {
            double t = re[i]; re[i] = re[r]; re[r] = t;
            t = im[i]; im[i] = im[r]; im[r] = t;
        }
    }
    for (int len = 2; len <= n; len <<= 1) {
        int half = len >> 1, step = n / len;
        for (int s = 0; s < n; s += len) {
            for (int k = 0; k < half; k++) {
                double wr = c->wr[k * step];
                double wi = sign < 0 ? -c->wi[k * step] : c->wi[k * step];
                double vr0 = re[s + k + half], vi0 = im[s + k + half];
                double t1 = vr0 * wr, t2 = vi0 * wi;
                double vr = t1 - t2;
                double t3 = vr0 * wi, t4 = vi0 * wr;
                double vi = t3 + t4;
                double ur = re[s + k], ui = im[s + k];
                re[s + k] = ur + vr;
                im[s + k] = ui + vi;
                re[s + k + half] = ur - vr;
                im[s + k + half] = ui - vi;
            }
        }
    }
}

void oc_encode(const oc_ctx *c, const double *vals, int nvals, double scale, int64_t *m_out) {
    oc_encode_c(c, vals, NULL, nvals, scale, m_out);
}

/* complex slots z_i = vals[i] + j vals_im[i] (vals_im may be NULL): the same
 * inverse canonical embedding; used by the bootstrap circuit's DFT diagonals */
void oc_encode_c(const oc_ctx *c, const double *vals, const double *vals_im, int nvals, double scale,
                 int64_t *m_out) {
    int n = c->nslots;
    double *re = (double *)calloc(n, sizeof(double));
    double *im = (double *)calloc(n, sizeof(double));
    for (int i = 0; i < nvals && i < n; i++) {
        re[c->pos[i]] = vals[i];
        if (vals_im) im[c->pos[i]] = vals_im[i];
    }
    fft(c, re, im, -1);
    double inv_n = 1.0 / (double)n; /* exact: n is a power of two */
    for (int j = 0; j < n; j++) {
        double vr = re[j] * inv_n, vi = im[j] * inv_n;
        double a1 = vr * c->zr[j], a2 = vi * c->zi[j];
        double ur = a1 + a2;
        double b1 = vi * c->zr[j], b2 = vr * c->zi[j];
        double ui = b1 - b2;
        m_out[j] = (int64_t)llrint(ur * scale);
        m_out[j + n] = (int64_t)llrint(ui * scale);
    }
    free(re);
    free(im);
}

void oc_decode(const oc_ctx *c, const double *coeffs, double scale, double *slots_out) {
    int n = c->nslots;
    double *re = (double *)malloc(sizeof(double) * n);
    double *im = (double *)malloc(sizeof(double) * n);
    for (int j = 0; j < n; j++) {
        double ur = coeffs[j] / scale, ui = coeffs[j + n] / scale;
        double a1 = ur * c->zr[j], a2 = ui * c->zi[j];
        double b1 = ur * c->zi[j], b2 = ui * c->zr[j];
        re[j] = a1 - a2;
        im[j] = b1 + b2;
    }
    fft(c, re, im, +1);
    for (int i = 0; i < n; i++) slots_out[i] = re[c->pos[i]];
    free(re);
    free(im);
}

/* ---------------------------------------------------------------- keys */

static uint32_t key_obj(uint32_t g, int j) { return g * 64u + (uint32_t)j; }

/* evaluation-point permutation of X -> X^g in bit-reversed NTT order */
static void automorph_poly(const oc_ctx *c, const uint64_t *in, uint32_t g, uint64_t *out) {
    int N = c->N, logN = c->logN;
    uint64_t twoN = 2 * (uint64_t)N;
    for (int k = 0; k < N; k++) {
        uint64_t e = 2 * (uint64_t)brv((uint32_t)k, logN) + 1;
        uint64_t e2 = (e * g) % twoN;
        out[k] = in[brv((uint32_t)((e2 - 1) / 2), logN)];
    }
}

static uint64_t prod_p_mod(const oc_ctx *c, uint64_t q) {
    uint64_t r = 1 % q;
    for (int k = 0; k < c->K; k++) r = mulmod(r, c->mod[c->L + k] % q, q);
    return r;
}

void oc_gen_switch_key(const oc_ctx *c, uint32_t g, uint64_t *key) {
    int N = c->N, L = c->L, K = c->K, total = L + K;
    size_t poly = N, comp = (size_t)total * N;
    /* s' = s^2 (g = 0, relin), s^(g/2+2) (even g: the power keys of 5-component
     * relinearisation, s^3 at g = 2, s^4 at g = 4) or sigma_g(s) (odd g, galois),
     * NTT domain per modulus */
    uint64_t *sp = (uint64_t *)malloc(8 * comp);
    for (int m = 0; m < L; m++) {
        const uint64_t *s = c->sk + (size_t)m * N;
        if (g % 2 == 0) {
            const int power = g == 0 ? 2 : (int)(g / 2) + 2;
            for (int k = 0; k < N; k++) {
                uint64_t v = s[k];
                for (int e = 1; e < power; e++) v = mulmod(v, s[k], c->mod[m]);
                sp[m * poly + k] = v;
            }
        } else {
            automorph_poly(c, s, g, sp + m * poly);
        }
    }
    int64_t *e = (int64_t *)malloc(8 * N);
    uint64_t *tmp = (uint64_t *)malloc(8 * N);
    for (int j = 0; j < c->dnum; j++) {
        uint32_t obj = key_obj(g, j);
        for (int k = 0; k < N; k++) e[k] = sample_cbd(c, DOM_KSK_E, obj, (uint32_t)k);
        uint64_t *B = key + (size_t)j * 2 * comp, *A = B + comp;
        for (int m = 0; m < total; m++) {
            uint64_t q = c->mod[m];
            for (int k = 0; k < N; k++) tmp[k] = smod(e[k], q);
            oc_ntt(c, tmp, m);
            int in_digit = (m < L) && (m >= j * c->alpha) && (m < (j + 1) * c->alpha);
            uint64_t pm = in_digit ? prod_p_mod(c, q) : 0;
            const uint64_t *s = c->sk + (size_t)m * N;
            for (int k = 0; k < N; k++) {
                uint64_t a = sample_uniform(c, DOM_KSK_A, obj, (uint32_t)m, (uint32_t)k, q);
                uint64_t b = submod(tmp[k], mulmod(a, s[k], q), q);
                if (in_digit) b = addmod(b, mulmod(pm, sp[m * poly + k], q), q);
                A[m * poly + k] = a;
                B[m * poly + k] = b;
            }
        }
    }
    free(e);
    free(tmp);
    free(sp);
}

/* ---------------------------------------------------------------- enc/dec */

void oc_encrypt(const oc_ctx *c, const double *vals, int nvals, double scale, uint32_t ct_index,
                uint64_t *ct) {
    int N = c->N, L = c->L;
    int64_t *m = (int64_t *)malloc(8 * N);
    oc_encode(c, vals, nvals, scale, m);
    for (int j = 0; j < N; j++) m[j] += sample_cbd(c, DOM_ENC_E, ct_index, (uint32_t)j);
    uint64_t *c0 = ct, *c1 = ct + (size_t)L * N;
    for (int i = 0; i < L; i++) {
        uint64_t q = c->mod[i];
        uint64_t *p0 = c0 + (size_t)i * N, *p1 = c1 + (size_t)i * N;
        for (int j = 0; j < N; j++) p0[j] = smod(m[j], q);
        oc_ntt(c, p0, i);
        const uint64_t *s = c->sk + (size_t)i * N;
        for (int j = 0; j < N; j++) {
            uint64_t a = sample_uniform(c, DOM_ENC_A, ct_index, (uint32_t)i, (uint32_t)j, q);
            p1[j] = a;
            p0[j] = submod(p0[j], mulmod(a, s[j], q), q);
        }
    }
    free(m);
}

static double i128_to_double(i128 v) {
    if (v >= -((i128)1 << 62) && v < ((i128)1 << 62)) return (double)(int64_t)v;
    int64_t hi = (int64_t)(v >> 64);
    uint64_t lo = (uint64_t)v;
    return (double)hi * 18446744073709551616.0 + (double)lo;
}

void oc_decrypt_coeffs(const oc_ctx *c, const uint64_t *ct, int ell, double *out) {
    int N = c->N, D = ell < 2 ? ell : 2;
    uint64_t *x[2];
    for (int i = 0; i < D; i++) {
        uint64_t q = c->mod[i];
        x[i] = (uint64_t *)malloc(8 * N);
        const uint64_t *c0 = ct + (size_t)i * N, *c1 = ct + (size_t)(ell + i) * N, *s = c->sk + (size_t)i * N;
        for (int j = 0; j < N; j++) x[i][j] = addmod(c0[j], mulmod(c1[j], s[j], q), q);
        oc_intt(c, x[i], i);
    }
    uint64_t q0 = c->mod[0];
    for (int j = 0; j < N; j++) {
        i128 v;
        if (D == 1) {
            uint64_t r = x[0][j];
            v = r > (q0 - 1) / 2 ? (i128)r - (i128)q0 : (i128)r;
        } else {
            uint64_t q1 = c->mod[1];
            uint64_t x0 = x[0][j], x1 = x[1][j];
            uint64_t d = mulmod(submod(x1, x0 % q1, q1), invmod(q0 % q1, q1), q1);
            u128 Q = (u128)q0 * q1;
            u128 r = (u128)x0 + (u128)q0 * d;
            v = r > (Q - 1) / 2 ? (i128)r - (i128)Q : (i128)r;
        }
        out[j] = i128_to_double(v);
    }
    for (int i = 0; i < D; i++) free(x[i]);
}

void oc_decrypt(const oc_ctx *c, const uint64_t *ct, int ell, double scale, double *slots) {
    double *co = (double *)malloc(sizeof(double) * c->N);
    oc_decrypt_coeffs(c, ct, ell, co);
    oc_decode(c, co, scale, slots);
    free(co);
}

/* ---------------------------------------------------------------- arithmetic */

void oc_add(const oc_ctx *c, const uint64_t *a, const uint64_t *b, uint64_t *out, int ell, int nc) {
    size_t N = c->N;
    for (int p = 0; p < nc; p++)
        for (int i = 0; i < ell; i++) {
            size_t o = ((size_t)p * ell + i) * N;
            for (size_t k = 0; k < N; k++) out[o + k] = addmod(a[o + k], b[o + k], c->mod[i]);
        }
}

void oc_sub(const oc_ctx *c, const uint64_t *a, const uint64_t *b, uint64_t *out, int ell, int nc) {
    size_t N = c->N;
    for (int p = 0; p < nc; p++)
        for (int i = 0; i < ell; i++) {
            size_t o = ((size_t)p * ell + i) * N;
            for (size_t k = 0; k < N; k++) out[o + k] = submod(a[o + k], b[o + k], c->mod[i]);
        }
}

void oc_add_const(const oc_ctx *c, const uint64_t *ct, const uint64_t *res, uint64_t *out, int ell) {
    size_t N = c->N;
    memcpy(out, ct, 8 * 2 * (size_t)ell * N);
    for (int i = 0; i < ell; i++)
        for (size_t k = 0; k < N; k++) out[i * N + k] = addmod(ct[i * N + k], res[i], c->mod[i]);
}

void oc_mul_const(const oc_ctx *c, const uint64_t *ct, const uint64_t *res, uint64_t *out, int ell, int nc) {
    size_t N = c->N;
    for (int p = 0; p < nc; p++)
        for (int i = 0; i < ell; i++) {
            size_t o = ((size_t)p * ell + i) * N;
            for (size_t k = 0; k < N; k++) out[o + k] = mulmod(ct[o + k], res[i], c->mod[i]);
        }
}

void oc_mul_plain(const oc_ctx *c, const uint64_t *ct, const uint64_t *pt, uint64_t *out, int ell, int nc) {
    size_t N = c->N;
    for (int p = 0; p < nc; p++)
        for (int i = 0; i < ell; i++) {
            size_t o = ((size_t)p * ell + i) * N;
            for (size_t k = 0; k < N; k++) out[o + k] = mulmod(ct[o + k], pt[i * N + k], c->mod[i]);
        }
}

void oc_plain_to_ntt(const oc_ctx *c, const int64_t *m, uint64_t *pt, int ell) {
    size_t N = c->N;
    for (int i = 0; i < ell; i++) {
        for (size_t k = 0; k < N; k++) pt[i * N + k] = smod(m[k], c->mod[i]);
        oc_ntt(c, pt + i * N, i);
    }
}

void oc_tensor(const oc_ctx *c, const uint64_t *a, const uint64_t *b, uint64_t *out, int ell) {
    size_t N = c->N, P = (size_t)ell * N;
    const uint64_t *a0 = a, *a1 = a + P, *b0 = b, *b1 = b + P;
    uint64_t *d0 = out, *d1 = out + P, *d2 = out + 2 * P;
    for (int i = 0; i < ell; i++) {
        uint64_t q = c->mod[i];
        for (size_t k = i * N; k < (i + 1) * N; k++) {
            d0[k] = mulmod(a0[k], b0[k], q);
            d1[k] = addmod(mulmod(a0[k], b1[k], q), mulmod(a1[k], b0[k], q), q);
            d2[k] = mulmod(a1[k], b1[k], q);
        }
    }
}

/* square of an nc-component ciphertext: out_k = sum_{i+j=k} a_i a_j, 2nc-1 components */
void oc_tensor_sq(const oc_ctx *c, const uint64_t *a, int nc, uint64_t *out, int ell) {
    size_t N = c->N, P = (size_t)ell * N;
    for (int k = 0; k < 2 * nc - 1; k++)
        for (int i = 0; i < ell; i++) {
            uint64_t q = c->mod[i];
            for (size_t x = i * N; x < (i + 1) * N; x++) {
                uint64_t v = 0;
                for (int u = 0; u < nc; u++) {
                    const int w = k - u;
                    if (w < 0 || w >= nc) continue;
                    v = addmod(v, mulmod(a[u * P + x], a[w * P + x], q), q);
                }
                out[k * P + x] = v;
            }
        }
}

/* fast basis conversion of coefficient-domain limbs src (moduli sidx[0..ns))
 * to target modulus tq: y = sum_s [x_s * qhat_s^-1]_{q_s} * (qhat_s mod tq) mod tq */
static void bconv(const oc_ctx *c, const uint64_t *const *src, const int *sidx, int ns, uint64_t tq,
                  uint64_t *dst) {
    int N = c->N;
    uint64_t qhinv[MAXM], qhmod[MAXM];
    for (int s = 0; s < ns; s++) {
        uint64_t qs = c->mod[sidx[s]], h = 1 % qs, ht = 1 % tq;
        for (int u = 0; u < ns; u++) {
            if (u == s) continue;
            h = mulmod(h, c->mod[sidx[u]] % qs, qs);
            ht = mulmod(ht, c->mod[sidx[u]] % tq, tq);
        }
        qhinv[s] = invmod(h, qs);
        qhmod[s] = ht;
    }
    for (int k = 0; k < N; k++) {
        u128 acc = 0;
        for (int s = 0; s < ns; s++) {
            uint64_t v = mulmod(src[s][k], qhinv[s], c->mod[sidx[s]]);
            acc += (u128)v * qhmod[s];
        }
        dst[k] = (uint64_t)(acc % tq);
    }
}

/* ModUp of d + inner product with the key: acc [2][ell+K][N] (NTT domain,
 * limbs Q_0..Q_{ell-1} then P_0..P_{K-1}); caller frees */
static uint64_t *ks_inner(const oc_ctx *c, const uint64_t *d, const uint64_t *key, int ell) {
    int N = c->N, L = c->L, K = c->K, total = L + K;
    size_t comp = (size_t)total * N;
    int ext = ell + K;
    int midx[MAXM];
    for (int t = 0; t < ell; t++) midx[t] = t;
    for (int k = 0; k < K; k++) midx[ell + k] = L + k;
    uint64_t *dc = (uint64_t *)malloc(8 * (size_t)ell * N);
    memcpy(dc, d, 8 * (size_t)ell * N);
    for (int i = 0; i < ell; i++) oc_intt(c, dc + (size_t)i * N, i);
    uint64_t *acc = (uint64_t *)calloc(2 * (size_t)ext * N, 8);
    uint64_t *tmp = (uint64_t *)malloc(8 * (size_t)N);
    int beta = (ell + c->alpha - 1) / c->alpha;
    for (int j = 0; j < beta; j++) {
        int s0 = j * c->alpha, s1 = (j + 1) * c->alpha < ell ? (j + 1) * c->alpha : ell;
        const uint64_t *src[MAXM];
        int sidx[MAXM];
        for (int s = s0; s < s1; s++) { src[s - s0] = dc + (size_t)s * N; sidx[s - s0] = s; }
        const uint64_t *B = key + (size_t)j * 2 * comp, *A = B + comp;
        for (int t = 0; t < ext; t++) {
            int m = midx[t];
            uint64_t q = c->mod[m];
            const uint64_t *dt;
            if (t >= s0 && t < s1) {
                dt = d + (size_t)t * N;
            } else {
                bconv(c, src, sidx, s1 - s0, q, tmp);
                oc_ntt(c, tmp, m);
                dt = tmp;
            }
            uint64_t *a0 = acc + (size_t)t * N, *a1 = acc + (size_t)(ext + t) * N;
            const uint64_t *kb = B + (size_t)m * N, *ka = A + (size_t)m * N;
            for (int k = 0; k < N; k++) {
                a0[k] = addmod(a0[k], mulmod(dt[k], kb[k], q), q);
                a1[k] = addmod(a1[k], mulmod(dt[k], ka[k], q), q);
            }
        }
    }
    free(dc);
    free(tmp);
    return acc;
}

/* Relinearisation fused with `extra` rescales (one joint ModDown):
 *   X_c = acc_c + [P]_{q_i} d_c on Q limbs, X_c = acc_c on P limbs;
 *   S = {q_{ell-extra} .. q_{ell-1}} u P;  y_s = INTT(X_c[s]) for s in S;
 *   out_c[i] = (X_c[i] - NTT_i(BConv_{S -> q_i}(y))) * (prod S)^-1,  i < ell - extra.
 * d3 [3][ell][N] -> out [2][ell-extra][N]. */
void oc_relin_rescale(const oc_ctx *c, const uint64_t *d3, const uint64_t *key, uint64_t *out, int ell, int extra) {
    const uint64_t *keys[1] = {key};
    oc_relin_rescale_n(c, d3, 3, keys, out, ell, extra);
}

/* nc-component form (nc = 3 or 5): component k >= 2 is key-switched with
 * keys[k-2] (the s^k key) and the inner products are summed in the extended
 * basis before the one joint ModDown:  acc = sum_k ks_inner(d_k, keys[k-2]). */
void oc_relin_rescale_n(const oc_ctx *c, const uint64_t *d3, int nc, const uint64_t *const *keys, uint64_t *out,
                        int ell, int extra) {
    int N = c->N, L = c->L, K = c->K, ext = ell + K, lo = ell - extra;
    size_t P = (size_t)ell * N;
    uint64_t *acc = ks_inner(c, d3 + 2 * P, keys[0], ell);
    for (int k = 3; k < nc; k++) {
        uint64_t *a2 = ks_inner(c, d3 + (size_t)k * P, keys[k - 2], ell);
        for (int t = 0; t < ext; t++) {
            const int m = t < ell ? t : L + (t - ell);
            const uint64_t q = c->mod[m];
            for (int cc = 0; cc < 2; cc++) {
                uint64_t *x = acc + ((size_t)cc * ext + t) * N;
                const uint64_t *y = a2 + ((size_t)cc * ext + t) * N;
                for (int j = 0; j < N; j++) x[j] = addmod(x[j], y[j], q);
            }
        }
        free(a2);
    }
    uint64_t *tmp = (uint64_t *)malloc(8 * (size_t)N);
    for (int cc = 0; cc < 2; cc++) {
        uint64_t *X = acc + (size_t)cc * ext * N;
        const uint64_t *dcc = d3 + (size_t)cc * P;
        for (int i = 0; i < ell; i++) {
            uint64_t q = c->mod[i], pm = prod_p_mod(c, q);
            for (int k = 0; k < N; k++) X[(size_t)i * N + k] = addmod(X[(size_t)i * N + k], mulmod(dcc[(size_t)i * N + k], pm, q), q);
        }
        const uint64_t *src[MAXM];
        int sidx[MAXM], ns = 0;
        for (int s = lo; s < ell; s++) {
            oc_intt(c, X + (size_t)s * N, s);
            src[ns] = X + (size_t)s * N;
            sidx[ns++] = s;
        }
        for (int k = 0; k < K; k++) {
            oc_intt(c, X + (size_t)(ell + k) * N, L + k);
            src[ns] = X + (size_t)(ell + k) * N;
            sidx[ns++] = L + k;
        }
        for (int i = 0; i < lo; i++) {
            uint64_t q = c->mod[i];
            bconv(c, src, sidx, ns, q, tmp);
            oc_ntt(c, tmp, i);
            uint64_t prod = prod_p_mod(c, q);
            for (int s = lo; s < ell; s++) prod = mulmod(prod, c->mod[s] % q, q);
            uint64_t inv = invmod(prod, q);
            const uint64_t *x = X + (size_t)i * N;
            uint64_t *o = out + ((size_t)cc * lo + i) * N;
            for (int k = 0; k < N; k++) o[k] = mulmod(submod(x[k], tmp[k], q), inv, q);
        }
    }
    free(acc);
    free(tmp);
}

void oc_keyswitch(const oc_ctx *c, const uint64_t *d, const uint64_t *key, int ell, uint64_t *out0,
                  uint64_t *out1) {
    int N = c->N, L = c->L, K = c->K, total = L + K;
    size_t comp = (size_t)total * N;
    int ext = ell + K; /* extended basis: Q_0..Q_{ell-1}, P_0..P_{K-1} */
    int midx[MAXM];
    for (int t = 0; t < ell; t++) midx[t] = t;
    for (int k = 0; k < K; k++) midx[ell + k] = L + k;
    uint64_t *dc = (uint64_t *)malloc(8 * (size_t)ell * N);
    memcpy(dc, d, 8 * (size_t)ell * N);
    for (int i = 0; i < ell; i++) oc_intt(c, dc + (size_t)i * N, i);
    uint64_t *acc = (uint64_t *)calloc(2 * (size_t)ext * N, 8); /* [2][ext][N] */
    uint64_t *tmp = (uint64_t *)malloc(8 * (size_t)N);
    int beta = (ell + c->alpha - 1) / c->alpha;
    for (int j = 0; j < beta; j++) {
        int s0 = j * c->alpha, s1 = (j + 1) * c->alpha < ell ? (j + 1) * c->alpha : ell;
        const uint64_t *src[MAXM];
        int sidx[MAXM];
        for (int s = s0; s < s1; s++) { src[s - s0] = dc + (size_t)s * N; sidx[s - s0] = s; }
        const uint64_t *B = key + (size_t)j * 2 * comp, *A = B + comp;
        for (int t = 0; t < ext; t++) {
            int m = midx[t];
            uint64_t q = c->mod[m];
            const uint64_t *dt;
            if (t >= s0 && t < s1) {
                dt = d + (size_t)t * N;
            } else {
                bconv(c, src, sidx, s1 - s0, q, tmp);
                oc_ntt(c, tmp, m);
                dt = tmp;
            }
            uint64_t *a0 = acc + (size_t)t * N, *a1 = acc + (size_t)(ext + t) * N;
            const uint64_t *kb = B + (size_t)m * N, *ka = A + (size_t)m * N;
            for (int k = 0; k < N; k++) {
                a0[k] = addmod(a0[k], mulmod(dt[k], kb[k], q), q);
                a1[k] = addmod(a1[k], mulmod(dt[k], ka[k], q), q);
            }
        }
    }
    /* ModDown: (x_Q - BConv_{P->Q}(x_P)) * P^-1 */
    for (int cc = 0; cc < 2; cc++) {
        uint64_t *ac = acc + (size_t)cc * ext * N;
        uint64_t *outc = cc == 0 ? out0 : out1;
        const uint64_t *src[MAXM];
        int sidx[MAXM];
        for (int k = 0; k < K; k++) {
            oc_intt(c, ac + (size_t)(ell + k) * N, L + k);
            src[k] = ac + (size_t)(ell + k) * N;
            sidx[k] = L + k;
        }
        for (int i = 0; i < ell; i++) {
            uint64_t q = c->mod[i];
            bconv(c, src, sidx, K, q, tmp);
            oc_ntt(c, tmp, i);
            uint64_t pinv = invmod(prod_p_mod(c, q), q);
            const uint64_t *x = ac + (size_t)i * N;
            for (int k = 0; k < N; k++) outc[(size_t)i * N + k] = mulmod(submod(x[k], tmp[k], q), pinv, q);
        }
    }
    free(dc);
    free(acc);
    free(tmp);
}

void oc_relin(const oc_ctx *c, const uint64_t *d3, const uint64_t *key, uint64_t *out, int ell) {
    size_t P = (size_t)ell * c->N;
    uint64_t *k0 = (uint64_t *)malloc(8 * P), *k1 = (uint64_t *)malloc(8 * P);
    oc_keyswitch(c, d3 + 2 * P, key, ell, k0, k1);
    oc_add(c, d3, k0, out, ell, 1);
    oc_add(c, d3 + P, k1, out + P, ell, 1);
    free(k0);
    free(k1);
}

void oc_rescale(const oc_ctx *c, const uint64_t *in, uint64_t *out, int ell, int nc) {
    int N = c->N;
    int l = ell - 1;
    uint64_t ql = c->mod[l], half = (ql - 1) / 2;
    uint64_t *r = (uint64_t *)malloc(8 * (size_t)N), *t = (uint64_t *)malloc(8 * (size_t)N);
    for (int p = 0; p < nc; p++) {
        const uint64_t *x = in + (size_t)p * ell * N;
        uint64_t *y = out + (size_t)p * l * N;
        memcpy(r, x + (size_t)l * N, 8 * (size_t)N);
        oc_intt(c, r, l);
        for (int i = 0; i < l; i++) {
            uint64_t q = c->mod[i];
            for (int k = 0; k < N; k++)
                t[k] = r[k] > half ? submod(0, (ql - r[k]) % q, q) : r[k] % q;
            oc_ntt(c, t, i);
            uint64_t inv = invmod(ql % q, q);
            for (int k = 0; k < N; k++)
                y[(size_t)i * N + k] = mulmod(submod(x[(size_t)i * N + k], t[k], q), inv, q);
        }
    }
    free(r);
    free(t);
}

void oc_automorphism(const oc_ctx *c, const uint64_t *in, uint32_t g, uint64_t *out, int n_polys) {
    for (int p = 0; p < n_polys; p++)
        automorph_poly(c, in + (size_t)p * c->N, g, out + (size_t)p * c->N);
}

void oc_rotate(const oc_ctx *c, const uint64_t *ct, uint32_t g, const uint64_t *key, uint64_t *out, int ell) {
    size_t P = (size_t)ell * c->N;
    uint64_t *s = (uint64_t *)malloc(8 * 2 * P);
    oc_automorphism(c, ct, g, s, 2 * ell);
    uint64_t *k0 = (uint64_t *)malloc(8 * P), *k1 = (uint64_t *)malloc(8 * P);
    oc_keyswitch(c, s + P, key, ell, k0, k1);
    oc_add(c, s, k0, out, ell, 1);
    memcpy(out + P, k1, 8 * P);
    free(s);
    free(k0);
    free(k1);
}

/* Hoisting key for Galois element g: every polynomial of the switch key moved by
 * sigma_{g^-1} (the inverse automorphism, g g^-1 = 1 mod 2N).  key -> hkey, both
 * [dnum][2][L+K][N]. */
void oc_hoist_key(const oc_ctx *c, const uint64_t *key, uint32_t g, uint64_t *hkey) {
    const uint64_t twoN = 2 * (uint64_t)c->N;
    uint32_t gi = 1;
    while (((uint64_t)gi * g) % twoN != 1) gi += 2; /* g odd: an inverse exists */
    const int np = c->dnum * 2 * (c->L + c->K);
    for (int p = 0; p < np; p++) automorph_poly(c, key + (size_t)p * c->N, gi, hkey + (size_t)p * c->N);
}

/* Hoisted rotation (the contract of he_rotate_hoisted): ModUp of the UNROTATED c1,
 * inner product with the hoisting key sigma_g^-1(key_g), ModDown, add c0, then
 * sigma_g on both components:
 *   (t0, t1) = (c0 + KS(c1, hkey).0, KS(c1, hkey).1),  out = (sigma_g t0, sigma_g t1).
 * t0 + t1 sigma_g^-1(s) = c0 + c1 s, so out decrypts to sigma_g(m) under s.  The
 * basis extension of c1 is shared by every rotation of the same ciphertext. */
void oc_rotate_hoisted(const oc_ctx *c, const uint64_t *ct, uint32_t g, const uint64_t *hkey, uint64_t *out,
                       int ell) {
    size_t P = (size_t)ell * c->N;
    uint64_t *t = (uint64_t *)malloc(8 * 2 * P);
    uint64_t *k0 = (uint64_t *)malloc(8 * P);
    oc_keyswitch(c, ct + P, hkey, ell, k0, t + P);
    oc_add(c, ct, k0, t, ell, 1);
    oc_automorphism(c, t, g, out, 2 * ell);
    free(t);
    free(k0);
}

void oc_mult_ct(const oc_ctx *c, const uint64_t *a, const uint64_t *b, const uint64_t *rk, uint64_t *out,
                int ell) {
    size_t P = (size_t)ell * c->N;
    uint64_t *d3 = (uint64_t *)malloc(8 * 3 * P), *r = (uint64_t *)malloc(8 * 2 * P);
    oc_tensor(c, a, b, d3, ell);
    oc_relin(c, d3, rk, r, ell);
    oc_rescale(c, r, out, ell, 2);
    free(d3);
    free(r);
}

void oc_lincomb(const oc_ctx *c, const uint64_t *const *in, uint64_t *const *out, int n_out,
                const int32_t *row_ptr, const int32_t *col, const int64_t *w, int ell, int nc,
                int n_threads) {
    int N = c->N;
#ifdef _OPENMP
    if (n_threads <= 0) n_threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(n_threads)
#endif
    for (int o = 0; o < n_out; o++) {
        for (int p = 0; p < nc; p++)
            for (int i = 0; i < ell; i++) {
                uint64_t q = c->mod[i];
                uint64_t *y = out[o] + ((size_t)p * ell + i) * N;
                /* exact 128-bit sums of (x * (w mod q)), reduced every 32 terms (x, w < 2^61:
                 * 32 products < 2^127) -- the same residue as adding mulmod() terms one by one */
                const int CH = N < 256 ? N : 256;
                for (int k0 = 0; k0 < N; k0 += CH) {
                    u128 acc[256];
                    uint64_t part[256];
                    for (int k = 0; k < CH; k++) { acc[k] = 0; part[k] = 0; }
                    int cnt = 0;
                    for (int t = row_ptr[o]; t < row_ptr[o + 1]; t++) {
                        uint64_t wq = smod(w[t], q);
                        const uint64_t *x = in[col[t]] + ((size_t)p * ell + i) * N + k0;
                        for (int k = 0; k < CH; k++) acc[k] += (u128)x[k] * wq;
                        if (++cnt == 32) {
                            for (int k = 0; k < CH; k++) { part[k] = addmod(part[k], (uint64_t)(acc[k] % q), q); acc[k] = 0; }
                            cnt = 0;
                        }
                    }
                    for (int k = 0; k < CH; k++) y[k0 + k] = addmod(part[k], (uint64_t)(acc[k] % q), q);
                }
            }
    }
    (void)n_threads;
}
