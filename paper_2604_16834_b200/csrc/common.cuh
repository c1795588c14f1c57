// common.cuh -- shared host/device definitions for libhe_sm100.so.
//
// Modular arithmetic on 64-bit residues (q < 2^62):
//   * Shoup products for constant multipliers (twiddles, q_l^-1, P^-1):
//     one 64x64 high product + two low products, result in [0, 2q) (lazy).
//   * Montgomery REDC for sums of products against stored constants whose
//     table entries are pre-multiplied by R = 2^64 (BConv tables, key-switch
//     keys, lincomb weights): accumulate exact 128-bit sums, reduce once.
// Every kernel boundary leaves residues canonical in [0, q): that is the
// bit-exact contract with oracle/ckks_oracle.c.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/he_sm100.h"

#define HE_MAXM 64

struct ModConst {
    uint64_t q;
    uint64_t qinv;      // q^-1 mod 2^64 (Montgomery)
    uint64_t r2;        // 2^128 mod q  (redc(x * r2) = x * 2^64 mod q)
    uint64_t ninv;      // N^-1 mod q
    uint64_t ninv_sh;   // Shoup(ninv)
    uint64_t ratio;     // floor((2^64 - 1) / q): reduce64
    double qd, qid;     // q and 1/q as doubles (FP64 butterflies for q < 2^42)
};

// x mod q for any 64-bit x (one high product + one conditional subtract)
__device__ __forceinline__ uint64_t reduce64(uint64_t x, const ModConst &mc) {
    uint64_t r = x - __umul64hi(x, mc.ratio) * mc.q;
    return r >= mc.q ? r - mc.q : r;
}

// Per-(level, digit) ModUp table and per-level ModDown table, device resident.
struct BconvTable {
    int n_src, n_dst;
    std::vector<uint64_t> h_qhinv;  // host copy: qhat_s^-1 mod q_s
    std::vector<int> h_dst_mod;     // host copy: target modulus indices
    uint64_t *d;        // [n_src] qhat_inv, [n_src] Shoup(qhat_inv), [n_src][n_dst] qhat mod dst (Montgomery form)
    int32_t *d_src_mod; // [n_src] modulus index of each source
    int32_t *d_dst_mod; // [n_dst] modulus index of each target
};

constexpr uint32_t HE_HOIST_CODE = 0x80000000u;  // key-map code of a hoisting key

struct he_ctx {
    he_params prm;
    int N, logN, L, K, alpha, dnum, nslots, device;
    std::vector<uint64_t> mod, psi;
    ModConst *d_mc = nullptr;        // [L+K]
    uint64_t *d_tw = nullptr;        // [L+K][fwd|inv][N][2]  (psi^brv(i), Shoup) pairs
    double *d_twd = nullptr;         // [L+K][fwd|inv][N]     psi^brv(i) as doubles (FP64 butterflies)
    double *d_twdc = nullptr;        // [L+K][fwd|inv][N]     the same, centred into (-q/2, q/2] (q < 2^50 path)
    bool fp50 = false;               // every modulus < 2^50: standalone NTTs use the centred FP64 path
    double *d_rinvd = nullptr;       // [L+K]  2^-64 mod q as doubles (undo Montgomery factors on the FP64 path)
    uint64_t *d_sk = nullptr;        // [L+K][N]     canonical, NTT domain
    double *d_fftw = nullptr;        // [nslots][2]  omega^k
    double *d_twist = nullptr;       // [nslots][2]  zeta^j
    int32_t *d_slot_brv = nullptr;   // [nslots]     brv(pos[i]): slot i <-> FFT input index
    int32_t *d_slot_inv = nullptr;   // [nslots]     the inverse permutation: FFT input index -> slot
    uint8_t *d_ident = nullptr;      // [HE_MAXM]    identity modulus map
    std::map<uint32_t, uint64_t *> keys;            // [dnum][2][L+K][N] Montgomery form (HE_HOIST_CODE | g: hoisting keys)
    std::map<uint64_t, BconvTable> modup_tab;       // key = ell*64 + digit
    std::map<int, BconvTable> moddown_tab;          // key = ell
    std::vector<uint64_t> h_pmodq, h_pinv;          // P mod q_i, P^-1 mod q_i (i < L)
    uint64_t *d_pinv = nullptr;                     // [L] P^-1 mod q_i and Shoup  ([L][2])
    uint64_t *d_qlinv = nullptr;                    // [L][L][2] q_l^-1 mod q_i, Shoup
    std::vector<uint64_t> h_qlinv;                  // host copy of d_qlinv
    std::vector<uint64_t> h_ninv;                   // N^-1 mod every modulus
    std::mutex mu;
};

// host-side modular helpers (context.cu)
uint64_t he_h_mulmod(uint64_t a, uint64_t b, uint64_t q);
uint64_t he_h_shoup(uint64_t w, uint64_t q);
uint64_t he_h_inv(uint64_t a, uint64_t q);
// fused N = 2^16 key switching / rescale (fused.cu); pointer lists are HOST arrays
int he_keyswitch_fused(he_ctx *c, const uint64_t *key, const uint64_t *const *d, const uint64_t *const *d_dev, int B,
                       int ell, uint64_t *const *out0, uint64_t *const *out1, const uint64_t *const *add0,
                       const uint64_t *const *add1, cudaStream_t s);
int he_rescale_fused(he_ctx *c, const uint64_t *const *in, uint64_t *const *out, int B, int ell, int nc,
                     cudaStream_t s);
int he_hoisted_ks_fused(he_ctx *c, const uint64_t *const *hkeys, int R, const uint64_t *const *c0,
                        const uint64_t *const *c1, const uint64_t *const *c1_dev, int B, int ell,
                        uint64_t *const *t0, uint64_t *const *t1, cudaStream_t s);

// ---------------------------------------------------------------- errors

void he_set_error(const char *fmt, ...);
void he_count_launch(int n);  // process-wide kernel launch counter (he_launch_count)
#define HE_CHECK_CUDA(call)                                                            \
    do {                                                                               \
        cudaError_t _e = (call);                                                       \
        if (_e != cudaSuccess) {                                                       \
            he_set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(_e)); \
            return HE_ECUDA;                                                           \
        }                                                                              \
    } while (0)
#define HE_CHECK_LAUNCH()         \
    do {                          \
        he_count_launch(1);       \
        HE_CHECK_CUDA(cudaGetLastError()); \
    } while (0)
#define HE_TRY(x)                     \
    do {                              \
        int _r = (x);                 \
        if (_r != HE_OK) return _r;   \
    } while (0)

// ---------------------------------------------------------------- device math

__device__ __forceinline__ uint64_t mulhi(uint64_t a, uint64_t b) { return __umul64hi(a, b); }

// Shoup: w * a mod q with wp = floor(w 2^64 / q); lazy result in [0, 2q)
__device__ __forceinline__ uint64_t shoup_lazy(uint64_t a, uint64_t w, uint64_t wp, uint64_t q) {
    return a * w - mulhi(a, wp) * q;
}
__device__ __forceinline__ uint64_t shoup(uint64_t a, uint64_t w, uint64_t wp, uint64_t q) {
    uint64_t r = shoup_lazy(a, w, wp, q);
    return r >= q ? r - q : r;
}
__device__ __forceinline__ uint64_t add_mod(uint64_t a, uint64_t b, uint64_t q) {
    uint64_t s = a + b;
    return s >= q ? s - q : s;
}
__device__ __forceinline__ uint64_t sub_mod(uint64_t a, uint64_t b, uint64_t q) {
    return a >= b ? a - b : a + q - b;
}

struct u128 {
    uint64_t lo, hi;
};
// acc += a * b  (exact 128-bit)
__device__ __forceinline__ void mac128(u128 &acc, uint64_t a, uint64_t b) {
    asm("mad.lo.cc.u64 %0, %2, %3, %0;\n\t"
        "madc.hi.u64 %1, %2, %3, %1;"
        : "+l"(acc.lo), "+l"(acc.hi)
        : "l"(a), "l"(b));
}
// Carry-free split accumulator for moduli q < 2^52 (operands < 2^52) and at
// most 1024 terms: with x = xh 2^32 + xl1 2^16 + xl0 and w = wh 2^32 + wl,
//   x w = xl0 wl + 2^16 xl1 wl + 2^32 (xh wl + xl wh) + 2^64 xh wh,
// and every column sum fits its 64-bit accumulator (xl0 wl, xl1 wl < 2^48;
// xh wl, xl wh < 2^52; xh wh < 2^40), so one MAC is five IMAD.WIDE.U32 with
// 64-bit accumulate and no carry propagation.  The x split (xl0, xl1, xh) is
// done once per input and shared by every output of the group.
struct xsplit {
    uint32_t l0, l1, l, h;
};
__device__ __forceinline__ xsplit split52(uint64_t x) {
    xsplit s;
    s.l = (uint32_t)x;
    s.h = (uint32_t)(x >> 32);
    s.l0 = s.l & 0xFFFFu;
    s.l1 = s.l >> 16;
    return s;
}
struct acc52 {
    uint64_t L0, L1, M, H;
};
__device__ __forceinline__ void acc52_zero(acc52 &a) { a.L0 = a.L1 = a.M = a.H = 0; }
__device__ __forceinline__ void mac52(acc52 &a, const xsplit &x, uint64_t w) {
    const uint32_t wl = (uint32_t)w, wh = (uint32_t)(w >> 32);
    // mad.wide.u32 = one IMAD.WIDE.U32 with 64-bit accumulate (ptxas does not
    // always form it from the C expression)
    asm("mad.wide.u32 %0, %4, %6, %0;\n\t"
        "mad.wide.u32 %1, %5, %6, %1;\n\t"
        "mad.wide.u32 %2, %7, %6, %2;\n\t"
        "mad.wide.u32 %2, %8, %9, %2;\n\t"
        "mad.wide.u32 %3, %7, %9, %3;"
        : "+l"(a.L0), "+l"(a.L1), "+l"(a.M), "+l"(a.H)
        : "r"(x.l0), "r"(x.l1), "r"(wl), "r"(x.h), "r"(x.l), "r"(wh));
}
// collapse to a 128-bit (hi, lo)
__device__ __forceinline__ u128 acc52_sum(const acc52 &a) {
    u128 r;
    const uint64_t l1s = a.L1 << 16, ms = a.M << 32;
    uint64_t lo = a.L0 + l1s;
    uint64_t hi = a.H + (a.L1 >> 48) + (a.M >> 32) + (lo < l1s ? 1 : 0);
    r.lo = lo + ms;
    r.hi = hi + (r.lo < ms ? 1 : 0);
    return r;
}

// Montgomery reduction of T = hi 2^64 + lo < q 2^64: returns T 2^-64 mod q in [0, q)
__device__ __forceinline__ uint64_t redc(uint64_t hi, uint64_t lo, uint64_t q, uint64_t qinv) {
    uint64_t m = lo * qinv;
    uint64_t mh = mulhi(m, q);
    uint64_t t = hi - mh;
    return hi < mh ? t + q : t;
}
// exact a * b mod q for canonical a, b: two Montgomery reductions
__device__ __forceinline__ uint64_t mul_mod(uint64_t a, uint64_t b, const ModConst &mc) {
    uint64_t t = redc(mulhi(a, b), a * b, mc.q, mc.qinv);  // a b R^-1
    return redc(mulhi(t, mc.r2), t * mc.r2, mc.q, mc.qinv);  // (a b R^-1)(R^2) R^-1
}
// signed int64 -> canonical residue
__device__ __forceinline__ uint64_t smod64(int64_t v, uint64_t q) {
    if (v >= 0) return (uint64_t)v % q;
    uint64_t r = ((uint64_t)(-(v + 1))) % q;
    return q - 1 - r;
}

// ---------------------------------------------------------------- philox
__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; r++) {
        uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
        uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
        uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = lo1;
        c[2] = n2;
        c[3] = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}
enum { DOM_SK = 1, DOM_ENC_A = 2, DOM_ENC_E = 3, DOM_KSK_A = 4, DOM_KSK_E = 5 };
__device__ __forceinline__ void rnd4(uint64_t seed, uint32_t dom, uint32_t obj, uint32_t limb, uint32_t idx,
                                     uint32_t o[4]) {
    o[0] = idx;
    o[1] = limb;
    o[2] = obj;
    o[3] = dom;
    philox4x32_10(o, (uint32_t)seed, (uint32_t)(seed >> 32));
}
__device__ __forceinline__ int64_t sample_cbd(uint64_t seed, uint32_t dom, uint32_t obj, uint32_t j) {
    uint32_t r[4];
    rnd4(seed, dom, obj, 0, j, r);
    return (int64_t)__popc(r[0] & 0x1FFFFFu) - (int64_t)__popc(r[1] & 0x1FFFFFu);
}
// Uniform residues mod q.  One Philox block serves the PAIR of indices k0
// (bit 4 clear) and k0 | 16: its counter index is k with bit 4 removed, words (r0, r1) are the
// 64-bit draw of k0 and (r2, r3) that of k0 | 16.  A draw x is accepted when x < q floor(2^64 / q)
// and reduced mod q (exactly uniform); a rejected draw (probability < q / 2^64) is replaced by
// words (r0, r1) of block (k, limb, obj, dom + 16 t), t = 1, 2, ...
__device__ __forceinline__ uint64_t uniform_accept(uint64_t x, uint64_t seed, uint32_t dom, uint32_t obj, uint32_t limb,
                                                   uint32_t k, const ModConst &mc) {
    const uint64_t T = mc.ratio * mc.q;  // ratio = floor((2^64 - 1) / q) = floor(2^64 / q) for odd q
    uint32_t t = 0;
    while (x >= T) {
        uint32_t r[4];
        rnd4(seed, dom + 16u * ++t, obj, limb, k, r);
        x = (uint64_t)r[0] | ((uint64_t)r[1] << 32);
    }
    return reduce64(x, mc);
}
__device__ __forceinline__ void sample_uniform_pair(uint64_t seed, uint32_t dom, uint32_t obj, uint32_t limb, uint32_t k0,
                                                    const ModConst &mc, uint64_t &a0, uint64_t &a1) {
    uint32_t r[4];
    rnd4(seed, dom, obj, limb, ((k0 >> 5) << 4) | (k0 & 15u), r);
    a0 = uniform_accept((uint64_t)r[0] | ((uint64_t)r[1] << 32), seed, dom, obj, limb, k0, mc);
    a1 = uniform_accept((uint64_t)r[2] | ((uint64_t)r[3] << 32), seed, dom, obj, limb, k0 | 16u, mc);
}
__device__ __forceinline__ uint64_t sample_uniform(uint64_t seed, uint32_t dom, uint32_t obj, uint32_t limb,
                                                   uint32_t k, const ModConst &mc) {
    uint32_t r[4];
    rnd4(seed, dom, obj, limb, ((k >> 5) << 4) | (k & 15u), r);
    const uint64_t x = (k & 16u) ? (uint64_t)r[2] | ((uint64_t)r[3] << 32) : (uint64_t)r[0] | ((uint64_t)r[1] << 32);
    return uniform_accept(x, seed, dom, obj, limb, k, mc);
}

// ---------------------------------------------------------------- host helpers (defined in context.cu)
int he_upload_ptrs(const void *const *host_ptrs, int count, void ***dev_out, cudaStream_t s);
// host -> device copy through the pinned staging ring (returns immediately; src may be reused)
cudaError_t he_h2d(void *dst, const void *src, size_t bytes, cudaStream_t s);
int he_scratch_alloc(void **p, size_t bytes, cudaStream_t s);
void he_scratch_free(void *p, cudaStream_t s);
int he_get_modup_table(he_ctx *ctx, int ell, int digit, const BconvTable **out);
int he_get_moddown_table(he_ctx *ctx, int ell, const BconvTable **out);
int he_get_moddown_table_x(he_ctx *ctx, int ell, int extra, const BconvTable **out);
int he_relin_rescale_fused(he_ctx *c, const uint64_t *const *keys, int nk, const uint64_t *const *d3,
                           const uint64_t *const *dk_dev, int B, int ell, int extra, uint64_t *const *out,
                           cudaStream_t s);
const uint64_t *he_get_key(he_ctx *ctx, uint32_t galois_elt);
// fused N = 2^16 encryption from the encode FFT output (encrypt16.cu); out_dev: device pointer array
int he_encrypt16(he_ctx *c, const double *re, const double *im, int count, double scale, uint32_t ct_index0,
                 int ell, uint64_t *const *out_dev, cudaStream_t s);

// NTT launchers (ntt.cu).  Polys: data + p*N for p in [0, n_polys); the
// modulus of poly p is mod_map[p % per] (0xFF: skip the poly).
int he_ntt_fwd(he_ctx *ctx, uint64_t *data, int n_polys, const uint8_t *mod_map, int per, cudaStream_t s);
int he_ntt_inv(he_ctx *ctx, uint64_t *data, int n_polys, const uint8_t *mod_map, int per, cudaStream_t s);
// pointer-array form: poly p = ptrs[p / per] + (p % per) * N (ptrs in device memory)
int he_ntt_fwd_ptrs(he_ctx *ctx, uint64_t *const *ptrs, int count, int per, const uint8_t *mod_map, cudaStream_t s);
int he_ntt_inv_ptrs(he_ctx *ctx, uint64_t *const *ptrs, int count, int per, const uint8_t *mod_map, cudaStream_t s);

static inline unsigned ceil_div(size_t a, size_t b) { return (unsigned)((a + b - 1) / b); }
