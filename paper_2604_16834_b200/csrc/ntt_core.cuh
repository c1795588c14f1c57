// ntt_core.cuh -- register-resident radix-16 NTT phases shared by ntt.cu and fused.cu.
//
// Each thread keeps 16 residues x[j] whose global indices are e0 + j*estride.
// A phase runs four butterfly stages on them.  Forward stages are
// Cooley-Tukey with Harvey lazy reduction (values in [0, 4q)); inverse stages
// are Gentleman-Sande (values in [0, 2q)).  In stage s (j-distance d) the
// butterflies of each run of 2d consecutive j share one twiddle, index
// (1<<lm) + (e0 >> (LOGN-lm)) + run (forward) -- every call site keeps
// e0 mod 2t below the element stride -- so a phase needs 15 twiddle pairs,
// each one 16-byte (twiddle, Shoup) load.
#pragma once
#include "common.cuh"

constexpr int NTT_TPB = 256;  // threads per CTA, 16 residues each = 4096 per CTA

__device__ __forceinline__ uint64_t reduce4q(uint64_t x, uint64_t q) {
    uint64_t q2 = 2 * q;
    x = x >= q2 ? x - q2 : x;
    return x >= q ? x - q : x;
}
__device__ __forceinline__ uint64_t reduce2q(uint64_t x, uint64_t q) { return x >= q ? x - q : x; }

// NC ("no correction", primes q < 2^58 only): skip Harvey's u >= 2q
// correction.  Shoup's lazy product is in [0, 2q) for ANY 64-bit input, so a
// value that enters a stage below B*q leaves it below (B+2)*q: a pass of 8
// stages from [0, 17q) ends below 33q < 2^64, and the pass's consumer reduces
// once with reduce64 instead of once per butterfly.
template <int LOGN, int LM, int D, bool NC = false>
__device__ __forceinline__ void stage_ct(uint64_t (&x)[16], uint32_t e0, const ulonglong2 *__restrict__ W2, uint64_t q) {
    const uint64_t q2 = 2 * q;
    const uint32_t base = (1u << LM) + (e0 >> (LOGN - LM));
#pragma unroll
    for (int k = 0; k < 8 / D; k++) {
        const ulonglong2 tw = __ldg(W2 + base + k);
#pragma unroll
        for (int jj = 0; jj < D; jj++) {
            uint64_t u = x[2 * D * k + jj];
            if (!NC) u = u >= q2 ? u - q2 : u;
            const uint64_t v = shoup_lazy(x[2 * D * k + jj + D], tw.x, tw.y, q);
            x[2 * D * k + jj] = u + v;
            x[2 * D * k + jj + D] = u - v + q2;
        }
    }
}
template <int LOGN, int LM0, bool NC = false>
__device__ __forceinline__ void phase_ct(uint64_t (&x)[16], uint32_t e0, const ulonglong2 *__restrict__ W2, uint64_t q) {
    stage_ct<LOGN, LM0, 8, NC>(x, e0, W2, q);
    stage_ct<LOGN, LM0 + 1, 4, NC>(x, e0, W2, q);
    stage_ct<LOGN, LM0 + 2, 2, NC>(x, e0, W2, q);
    stage_ct<LOGN, LM0 + 3, 1, NC>(x, e0, W2, q);
}

// LOGB >= 0 selects the no-correction form (primes q < 2^46 only): inputs of
// the stage are below 2^LOGB * q, the sum is left unreduced (bound doubles)
// and the difference adds 2^LOGB * q before Shoup's lazy product (< 2q).
// Two passes of 8 stages from canonical input stay below 2^16 q < 2^62.
template <int LOGN, int LT, int D, int LOGB = -1>
__device__ __forceinline__ void stage_gs(uint64_t (&x)[16], uint32_t e0, const ulonglong2 *__restrict__ W2, uint64_t q) {
    const uint64_t q2 = 2 * q, qb = LOGB >= 0 ? (q << (LOGB >= 0 ? LOGB : 0)) : q2;
    const uint32_t base = (1u << (LOGN - 1 - LT)) + (e0 >> (LT + 1));
#pragma unroll
    for (int k = 0; k < 8 / D; k++) {
        const ulonglong2 tw = __ldg(W2 + base + k);
#pragma unroll
        for (int jj = 0; jj < D; jj++) {
            const uint64_t u = x[2 * D * k + jj], v = x[2 * D * k + jj + D];
            uint64_t sm = u + v;
            if (LOGB < 0) sm = sm >= q2 ? sm - q2 : sm;
            x[2 * D * k + jj] = sm;
            x[2 * D * k + jj + D] = shoup_lazy(u - v + qb, tw.x, tw.y, q);
        }
    }
}
template <int LOGN, int LT0, int LOGB = -1>
__device__ __forceinline__ void phase_gs(uint64_t (&x)[16], uint32_t e0, const ulonglong2 *__restrict__ W2, uint64_t q) {
    stage_gs<LOGN, LT0, 1, LOGB>(x, e0, W2, q);
    stage_gs<LOGN, LT0 + 1, 2, (LOGB < 0 ? -1 : LOGB + 1)>(x, e0, W2, q);
    stage_gs<LOGN, LT0 + 2, 4, (LOGB < 0 ? -1 : LOGB + 2)>(x, e0, W2, q);
    stage_gs<LOGN, LT0 + 3, 8, (LOGB < 0 ? -1 : LOGB + 3)>(x, e0, W2, q);
}

// ---------------------------------------------------------------- FP64 butterflies
// For primes q < 2^42 the butterflies run on the FP64 pipe (twice the
// integer-Shoup rate on B200, scripts/mb_modmul.cu).  Residues are held as
// doubles that are EXACT integers (|x| < 2^53):
//   a*w mod q:  h = a*w (rounded), l = fma(a, w, -h) (exact error, integer),
//               e = rint(h / q), r = fma(-e, q, h) + l = a*w - e*q exactly,
//   with |a| < 2^51 the estimate e is off by < 2 so r lies in (-3q, 3q) and
//   every intermediate is an integer below 2^53 (no rounding anywhere).
// Forward: |x| grows by < 3q per stage; inverse: the sum path doubles per
// stage -- 8 stages from canonical input stay below 2^51 for q < 2^42.  Each
// pass converts canonical uint64 -> double on entry and canonicalises on exit,
// so the bits at every kernel boundary are those of the integer path.
constexpr uint64_t FP_QMAX = 1ull << 42;
constexpr double FP_MAGIC = 4503599627370496.0;  // 2^52

__device__ __forceinline__ double u2d(uint64_t x) {  // exact for x < 2^52
    return __longlong_as_double((long long)(x | 0x4330000000000000ull)) - FP_MAGIC;
}
__device__ __forceinline__ uint64_t d2u(double r) {  // r an integer in [0, 2^52)
    return (uint64_t)__double_as_longlong(r + FP_MAGIC) - 0x4330000000000000ull;
}
__device__ __forceinline__ double fmulmod(double a, double w, double q, double qi) {
    const double h = a * w;
    const double l = fma(a, w, -h);
    const double e = rint(h * qi);
    return fma(-e, q, h) + l;
}
// exact integer |x| < 2^52 -> canonical residue (as an integer-valued double)
__device__ __forceinline__ double fcanond(double x, double q, double qi) {
    const double e = floor(x * qi);
    double r = fma(-e, q, x);
    r = r < 0.0 ? r + q : r;
    return r >= q ? r - q : r;
}
// exact integer |x| < 2^52 -> canonical residue as uint64
__device__ __forceinline__ uint64_t fcanon(double x, double q, double qi) {
    const double e = floor(x * qi);
    double r = fma(-e, q, x);
    r = r < 0.0 ? r + q : r;
    r = r >= q ? r - q : r;
    return d2u(r);
}

template <int LOGN, int LM, int D>
__device__ __forceinline__ void fstage_ct(double (&x)[16], uint32_t e0, const double *__restrict__ W, double q,
                                          double qi) {
    const uint32_t base = (1u << LM) + (e0 >> (LOGN - LM));
#pragma unroll
    for (int k = 0; k < 8 / D; k++) {
        const double w = __ldg(W + base + k);
#pragma unroll
        for (int jj = 0; jj < D; jj++) {
            const double u = x[2 * D * k + jj], v = fmulmod(x[2 * D * k + jj + D], w, q, qi);
            x[2 * D * k + jj] = u + v;
            x[2 * D * k + jj + D] = u - v;
        }
    }
}
template <int LOGN, int LM0>
__device__ __forceinline__ void fphase_ct(double (&x)[16], uint32_t e0, const double *__restrict__ W, double q,
                                          double qi) {
    fstage_ct<LOGN, LM0, 8>(x, e0, W, q, qi);
    fstage_ct<LOGN, LM0 + 1, 4>(x, e0, W, q, qi);
    fstage_ct<LOGN, LM0 + 2, 2>(x, e0, W, q, qi);
    fstage_ct<LOGN, LM0 + 3, 1>(x, e0, W, q, qi);
}
template <int LOGN, int LT, int D>
__device__ __forceinline__ void fstage_gs(double (&x)[16], uint32_t e0, const double *__restrict__ W, double q,
                                          double qi) {
    const uint32_t base = (1u << (LOGN - 1 - LT)) + (e0 >> (LT + 1));
#pragma unroll
    for (int k = 0; k < 8 / D; k++) {
        const double w = __ldg(W + base + k);
#pragma unroll
        for (int jj = 0; jj < D; jj++) {
            const double u = x[2 * D * k + jj], v = x[2 * D * k + jj + D];
            x[2 * D * k + jj] = u + v;
            x[2 * D * k + jj + D] = fmulmod(u - v, w, q, qi);
        }
    }
}
template <int LOGN, int LT0>
__device__ __forceinline__ void fphase_gs(double (&x)[16], uint32_t e0, const double *__restrict__ W, double q,
                                          double qi) {
    fstage_gs<LOGN, LT0, 1>(x, e0, W, q, qi);
    fstage_gs<LOGN, LT0 + 1, 2>(x, e0, W, q, qi);
    fstage_gs<LOGN, LT0 + 2, 4>(x, e0, W, q, qi);
    fstage_gs<LOGN, LT0 + 3, 8>(x, e0, W, q, qi);
}
// ---------------------------------------------------------------- centred FP64 butterflies, q < 2^50
// For primes below 2^50 the residues are integer-valued doubles kept small by
// CENTRED reductions, and rounding to the nearest integer uses the 1.5*2^52
// magic constant (FP64 pipe, no FRND on the XU pipe):
//   fmulmod_c(a, w): w centred (|w| <= q/2), |a| < 2^52: h = a w, l = fma(a, w, -h),
//     e = round(h / q) (|h/q| < 2^51, so the magic add rounds exactly), r = fma(-e, q, h) + l
//     = a w - e q exactly, |r| < 1.01 q; every intermediate is an integer below 2^53.
//   fred_c(x): x - round(x/q) q, |x| < 2^53 -> |x| <= q/2 + 1.
// Forward (CT): u +- v grows by < 1.01 q per stage; reducing after every second
// stage keeps multiply inputs below 2.02 q and sums below 3.03 q < 2^53.
// Inverse (GS): the sum is reduced every stage, the difference (< 2.02 q) feeds
// the product.  Kernels convert canonical uint64 on entry and canonicalise on
// exit, so the bits at kernel boundaries are those of the integer path.
constexpr double FP_RND = 6755399441055744.0;  // 1.5 * 2^52
__device__ __forceinline__ double fmulmod_c(double a, double w, double q, double qi) {
    const double h = a * w;
    const double l = fma(a, w, -h);
    const double e = fma(h, qi, FP_RND) - FP_RND;
    return fma(-e, q, h) + l;
}
__device__ __forceinline__ double fred_c(double x, double q, double qi) {
    const double e = fma(x, qi, FP_RND) - FP_RND;
    return fma(-e, q, x);
}
template <int LOGN, int LM, int D, bool RED>
__device__ __forceinline__ void fstage_ct_c(double (&x)[16], uint32_t e0, const double *__restrict__ W, double q,
                                            double qi) {
    const uint32_t base = (1u << LM) + (e0 >> (LOGN - LM));
#pragma unroll
    for (int k = 0; k < 8 / D; k++) {
        const double w = __ldg(W + base + k);
#pragma unroll
        for (int jj = 0; jj < D; jj++) {
            const double u = x[2 * D * k + jj], v = fmulmod_c(x[2 * D * k + jj + D], w, q, qi);
            const double a = u + v, b = u - v;
            x[2 * D * k + jj] = RED ? fred_c(a, q, qi) : a;
            x[2 * D * k + jj + D] = RED ? fred_c(b, q, qi) : b;
        }
    }
}
template <int LOGN, int LM0>
__device__ __forceinline__ void fphase_ct_c(double (&x)[16], uint32_t e0, const double *__restrict__ W, double q,
                                            double qi) {
    fstage_ct_c<LOGN, LM0, 8, false>(x, e0, W, q, qi);
    fstage_ct_c<LOGN, LM0 + 1, 4, true>(x, e0, W, q, qi);
    fstage_ct_c<LOGN, LM0 + 2, 2, false>(x, e0, W, q, qi);
    fstage_ct_c<LOGN, LM0 + 3, 1, true>(x, e0, W, q, qi);
}
template <int LOGN, int LT, int D>
__device__ __forceinline__ void fstage_gs_c(double (&x)[16], uint32_t e0, const double *__restrict__ W, double q,
                                            double qi) {
    const uint32_t base = (1u << (LOGN - 1 - LT)) + (e0 >> (LT + 1));
#pragma unroll
    for (int k = 0; k < 8 / D; k++) {
        const double w = __ldg(W + base + k);
#pragma unroll
        for (int jj = 0; jj < D; jj++) {
            const double u = x[2 * D * k + jj], v = x[2 * D * k + jj + D];
            x[2 * D * k + jj] = fred_c(u + v, q, qi);
            x[2 * D * k + jj + D] = fmulmod_c(u - v, w, q, qi);
        }
    }
}
template <int LOGN, int LT0>
__device__ __forceinline__ void fphase_gs_c(double (&x)[16], uint32_t e0, const double *__restrict__ W, double q,
                                            double qi) {
    fstage_gs_c<LOGN, LT0, 1>(x, e0, W, q, qi);
    fstage_gs_c<LOGN, LT0 + 1, 2>(x, e0, W, q, qi);
    fstage_gs_c<LOGN, LT0 + 2, 4>(x, e0, W, q, qi);
    fstage_gs_c<LOGN, LT0 + 3, 8>(x, e0, W, q, qi);
}

__device__ __forceinline__ const double *twd_fwd(const double *twd, int m, int logN) {
    return twd + ((size_t)m << (logN + 1));
}
__device__ __forceinline__ const double *twd_inv(const double *twd, int m, int logN) {
    return twd + ((size_t)m << (logN + 1)) + ((size_t)1 << logN);
}

__device__ __forceinline__ int pad16(int e) { return e + (e >> 4); }

// twiddle pair tables of modulus m (layout of he_ctx::d_tw)
__device__ __forceinline__ const ulonglong2 *tw_fwd(const uint64_t *tw, int m, int logN) {
    return (const ulonglong2 *)(tw + ((size_t)m << (logN + 2)));
}
__device__ __forceinline__ const ulonglong2 *tw_inv(const uint64_t *tw, int m, int logN) {
    return (const ulonglong2 *)(tw + ((size_t)m << (logN + 2)) + ((size_t)2 << logN));
}
