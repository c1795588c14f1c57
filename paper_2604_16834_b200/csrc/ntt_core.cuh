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

__device__ __forceinline__ int pad16(int e) { return e + (e >> 4); }

// twiddle pair tables of modulus m (layout of he_ctx::d_tw)
__device__ __forceinline__ const ulonglong2 *tw_fwd(const uint64_t *tw, int m, int logN) {
    return (const ulonglong2 *)(tw + ((size_t)m << (logN + 2)));
}
__device__ __forceinline__ const ulonglong2 *tw_inv(const uint64_t *tw, int m, int logN) {
    return (const ulonglong2 *)(tw + ((size_t)m << (logN + 2)) + ((size_t)2 << logN));
}
