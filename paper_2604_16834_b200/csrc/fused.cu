// fused.cu -- key switching and rescale with their conversions fused into the
// NTT passes (N = 2^16).
//
// Unfused, one hybrid key switch at level l streams every intermediate
// through HBM: INTT(d) -> BConv -> NTT -> inner product -> INTT(P) -> BConv ->
// NTT -> subtract/scale.  Here each NTT pass is driven by a per-polynomial job
// descriptor whose loader/epilogue absorbs the neighbouring element-wise step:
//
//   INTT of d       pass 2 multiplies by N^-1 * qhat_s^-1   (ModUp's Shoup step)
//   ModUp NTT       pass 1 loads sum_s v_s * qhat_s (BConv, Montgomery REDC)
//   ModUp NTT pass 2 + key inner product: one kernel per (ct, target limb)
//                   runs pass 2 of every digit and accumulates e_j * key_j
//                   in registers -- the extended digits never return to HBM
//   INTT of P limbs pass 2 multiplies by N^-1 * phat_k^-1
//   ModDown NTT     pass 1 loads the P->Q BConv, pass 2 writes
//                   (acc - conv) * P^-1 (+ d0/d1 for relinearisation)
//   rescale         INTT(last limb); pass 1 loads the centred lift into each
//                   q_i; pass 2 writes (x_i - t_i) * q_l^-1
//
// Every stage computes exactly the values of the unfused definition
// (oracle/ckks_oracle.c), so results stay bit-exact.
#include <algorithm>
#include <vector>

#include "ntt_core.cuh"

namespace {

// FP64 phases for any prime below 2^50: the lazy (non-reducing) form below
// 2^42, the centred form (ntt_core.cuh fphase_*_c) from 2^42 to 2^50.  Both
// take canonical or centred inputs and take centred twiddles (he_ctx::d_twdc).
constexpr uint64_t FP_QMAX50 = 1ull << 50;
template <int LOGN, int LM0>
__device__ __forceinline__ void fphase_ct_any(double (&x)[16], uint32_t e0, const double *W, const ModConst &c) {
    if (c.q < FP_QMAX)
        fphase_ct<LOGN, LM0>(x, e0, W, c.qd, c.qid);
    else
        fphase_ct_c<LOGN, LM0>(x, e0, W, c.qd, c.qid);
}
template <int LOGN, int LT0>
__device__ __forceinline__ void fphase_gs_any(double (&x)[16], uint32_t e0, const double *W, const ModConst &c) {
    if (c.q < FP_QMAX)
        fphase_gs<LOGN, LT0>(x, e0, W, c.qd, c.qid);
    else
        fphase_gs_c<LOGN, LT0>(x, e0, W, c.qd, c.qid);
}

constexpr int LOGN = 16;
constexpr size_t NN = (size_t)1 << LOGN;
// primes below these bounds take the no-correction butterflies (ntt_core.cuh):
// forward passes end below 33q, inverse passes below 2^17 q -- both < 2^64
constexpr uint64_t NC_FWD = 1ull << 58, NC_INV = 1ull << 46;

struct Job {
    const uint64_t *src;  // pass-1 input: direct poly / first BConv source limb / centred source
    uint64_t *dst;        // pass-1 output (and pass-2 in-place buffer)
    uint64_t *out;        // pass-2 epilogue destination
    const uint64_t *aux;  // epilogue operand (acc limb / rescale input limb)
    const uint64_t *add;  // epilogue addend (relin d0/d1 limb) or nullptr
    const uint64_t *tab;  // BConv Montgomery constants [ns]
    uint64_t cw, cwp;     // Shoup constant: inverse final scale / epilogue scale
    uint64_t ql;          // centred-lift source modulus
    const uint64_t *src2; // inverse pass-1 addend: input = src + c2 * src2 (or nullptr)
    const uint64_t *aux2; // epilogue: operand = aux + c2 * aux2 (or nullptr)
    uint64_t c2, c2p;     // Shoup constant for src2 / aux2 (P mod q for the joint ModDown)
    int32_t mod;          // modulus index of this polynomial
    int32_t ns;           // BConv source count
    int32_t wide;         // L_BCONV_FP: bit s set when source s is a prime >= 2^42 (split in 30-bit halves)
    int32_t pad_;
};

enum { L_DIRECT = 0, L_BCONV = 1, L_CENTER = 2, L_BCONV_FP = 3, L_BCONV_FPW = 4 };  // FPW: wide sources allowed
enum { E_STORE = 0, E_SUBSCALE = 1 };

// 8-byte cp.async (global -> shared, no register staging) and its group fences
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

// ---------------------------------------------------------------- forward pass 1 (columns)
template <int LD>
__global__ void __launch_bounds__(NTT_TPB) kf_cols(const Job *__restrict__ jobs, const uint64_t *tw,
                                                  const double *twd, const ModConst *mc, const double *rinvd) {
    __shared__ uint64_t sm[256 * 16];
    const Job jb = jobs[blockIdx.x >> 4];
    const ModConst c = mc[jb.mod];
    const ulonglong2 *W2 = tw_fwd(tw, jb.mod, LOGN);
    const int tid = threadIdx.x, lc = tid & 15, g = tid >> 4;
    const uint32_t col = (blockIdx.x & 15) * 16 + lc;
    if (LD == L_BCONV_FP || LD == L_BCONV_FPW) {
        // target below 2^42: the BConv is FP64 modular products against the
        // Montgomery-form table (sum < 4 ns q), one R^-1 product, and the NTT
        // runs on the FP64 pipe without leaving doubles.  A source residue from a
        // prime >= 2^42 is split v = hi 2^30 + lo (both exact, < 2^31) and takes
        // two products, the high one against t 2^30 mod q.
        const double *Wd = twd_fwd(twd, jb.mod, LOGN);
        double xd[16];
#pragma unroll
        for (int j = 0; j < 16; j++) xd[j] = 0.0;
        for (int s = 0; s < jb.ns; s++) {
            const double t = u2d(__ldg(jb.tab + s));
            const uint64_t *src = jb.src + (size_t)s * NN + col;
            uint64_t v[16];
#pragma unroll
            for (int j = 0; j < 16; j++) v[j] = __ldg(src + (g + 16 * j) * 256);
            if (LD == L_BCONV_FPW && ((jb.wide >> s) & 1)) {
                const double t30 = fmulmod(t, 1073741824.0, c.qd, c.qid);
#pragma unroll
                for (int j = 0; j < 16; j++)
                    xd[j] += fmulmod(u2d(v[j] & 0x3FFFFFFFull), t, c.qd, c.qid) +
                             fmulmod(u2d(v[j] >> 30), t30, c.qd, c.qid);
            } else {
#pragma unroll
                for (int j = 0; j < 16; j++) xd[j] += fmulmod(u2d(v[j]), t, c.qd, c.qid);
            }
        }
        const double ri = rinvd[jb.mod];  // 2^-64 mod q
#pragma unroll
        for (int j = 0; j < 16; j++) xd[j] = fmulmod(xd[j], ri, c.qd, c.qid);  // |x| < 2q
        fphase_ct<16, 0>(xd, col + 256 * g, Wd, c.qd, c.qid);
#pragma unroll
        for (int j = 0; j < 16; j++) sm[(g + 16 * j) * 16 + lc] = (uint64_t)__double_as_longlong(xd[j]);
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 16; j++) xd[j] = __longlong_as_double((long long)sm[(16 * g + j) * 16 + lc]);
        fphase_ct<16, 4>(xd, col + 4096 * g, Wd, c.qd, c.qid);
#pragma unroll
        for (int j = 0; j < 16; j++) jb.dst[(16 * g + j) * 256 + col] = fcanon(xd[j], c.qd, c.qid);
        return;
    }
    uint64_t x[16];
    if (LD == L_DIRECT) {
#pragma unroll
        for (int j = 0; j < 16; j++) x[j] = jb.src[(g + 16 * j) * 256 + col];
    } else if (LD == L_BCONV) {
        // source-major, double-buffered: source s+1's 16 values per thread stream
        // into shared memory with cp.async while source s is multiplied (each
        // thread reads back only what it copied: no block barrier); with
        // v_s, t_s < q < 2^61 each product adds < q/8 to the high word, so
        // ns <= 8 terms keep hi < q without folding (redc's precondition)
        extern __shared__ uint64_t stage[];  // [2][16 x 256]: this thread's slots (g + 16 j) * 16 + lc
        auto issue = [&](int s) {
            const uint64_t *src = jb.src + (size_t)s * NN + col;
            uint64_t *dstp = stage + (s & 1) * 4096 + lc;
#pragma unroll
            for (int j = 0; j < 16; j++) cp_async8(dstp + (g + 16 * j) * 16, src + (g + 16 * j) * 256);
            cp_async_commit();
        };
        u128 acc[16];
#pragma unroll
        for (int j = 0; j < 16; j++) acc[j] = u128{0, 0};
        issue(0);
        for (int s = 0; s < jb.ns; s++) {
            const uint64_t t = __ldg(jb.tab + s);
            if (s + 1 < jb.ns) {
                issue(s + 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            const uint64_t *vs = stage + (s & 1) * 4096 + lc;
            uint64_t v[16];
#pragma unroll
            for (int j = 0; j < 16; j++) v[j] = vs[(g + 16 * j) * 16];
#pragma unroll
            for (int j = 0; j < 16; j++) mac128(acc[j], v[j], t);
            if ((s & 7) == 7)  // more than 8 sources: fold (hi < 2q -> < q)
#pragma unroll
                for (int j = 0; j < 16; j++) acc[j].hi = acc[j].hi >= c.q ? acc[j].hi - c.q : acc[j].hi;
        }
        if (jb.ns > 8 && (jb.ns & 7))
#pragma unroll
            for (int j = 0; j < 16; j++) acc[j].hi = acc[j].hi >= c.q ? acc[j].hi - c.q : acc[j].hi;
#pragma unroll
        for (int j = 0; j < 16; j++) x[j] = redc(acc[j].hi, acc[j].lo, c.q, c.qinv);
    } else {
        const uint64_t half = (jb.ql - 1) >> 1;
#pragma unroll
        for (int j = 0; j < 16; j++) {
            const uint64_t v = jb.src[(g + 16 * j) * 256 + col];
            x[j] = v > half ? sub_mod(0, reduce64(jb.ql - v, c), c.q) : reduce64(v, c);
        }
    }
    if (c.q < FP_QMAX50) {  // FP64 butterflies; canonical output
        const double *Wd = twd_fwd(twd, jb.mod, LOGN);
        double xd[16];
#pragma unroll
        for (int j = 0; j < 16; j++) xd[j] = u2d(x[j]);
        fphase_ct_any<16, 0>(xd, col + 256 * g, Wd, c);
#pragma unroll
        for (int j = 0; j < 16; j++) sm[(g + 16 * j) * 16 + lc] = (uint64_t)__double_as_longlong(xd[j]);
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 16; j++) xd[j] = __longlong_as_double((long long)sm[(16 * g + j) * 16 + lc]);
        fphase_ct_any<16, 4>(xd, col + 4096 * g, Wd, c);
#pragma unroll
        for (int j = 0; j < 16; j++) jb.dst[(16 * g + j) * 256 + col] = fcanon(xd[j], c.qd, c.qid);
        return;
    }
    const bool nc = c.q < NC_FWD;  // no per-butterfly correction: output < 17q, else < 4q
    if (nc)
        phase_ct<16, 0, true>(x, col + 256 * g, W2, c.q);
    else
        phase_ct<16, 0>(x, col + 256 * g, W2, c.q);
#pragma unroll
    for (int j = 0; j < 16; j++) sm[(g + 16 * j) * 16 + lc] = x[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = sm[(16 * g + j) * 16 + lc];
    if (nc)
        phase_ct<16, 4, true>(x, col + 4096 * g, W2, c.q);
    else
        phase_ct<16, 4>(x, col + 4096 * g, W2, c.q);
#pragma unroll
    for (int j = 0; j < 16; j++) jb.dst[(16 * g + j) * 256 + col] = x[j];  // lazy
}

// ---------------------------------------------------------------- forward pass 2 (rows)
// E_SUBSCALE: the epilogue operands (aux, and aux2 or add) stream into shared
// memory with cp.async while the NTT phases run (dynamic smem [2][16][256]):
// each thread prefetches exactly the 16 + 16 words it will consume.
template <int EP>
__global__ void __launch_bounds__(NTT_TPB) kf_rows(const Job *__restrict__ jobs, const uint64_t *tw,
                                                  const double *twd, const ModConst *mc) {
    __shared__ uint64_t sm[16 * 272];
    extern __shared__ uint64_t pre[];
    const Job jb = jobs[blockIdx.x >> 4];
    const ModConst c = mc[jb.mod];
    const ulonglong2 *W2 = tw_fwd(tw, jb.mod, LOGN);
    const int tid = threadIdx.x, g = tid & 15, rl = tid >> 4;
    const uint32_t r = (blockIdx.x & 15) * 16 + rl;
    uint64_t *row = jb.dst + r * 256;
    uint64_t *s = sm + rl * 272;
    const uint64_t *second = jb.aux2 ? jb.aux2 : jb.add;
    uint64_t *pa = pre + rl * 256, *pb = pre + 4096 + rl * 256;
    if (EP == E_SUBSCALE) {
#pragma unroll
        for (int j = 0; j < 16; j++) cp_async8(pa + g + 16 * j, jb.aux + r * 256 + g + 16 * j);
        if (second)
#pragma unroll
            for (int j = 0; j < 16; j++) cp_async8(pb + g + 16 * j, second + r * 256 + g + 16 * j);
        cp_async_commit();
    }
    uint64_t x[16];
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = row[g + 16 * j];
    const bool nc = c.q < NC_FWD;
    if (c.q < FP_QMAX50) {
        const double *Wd = twd_fwd(twd, jb.mod, LOGN);
        double xd[16];
#pragma unroll
        for (int j = 0; j < 16; j++) xd[j] = u2d(x[j]);
        fphase_ct_any<16, 8>(xd, r * 256 + g, Wd, c);
#pragma unroll
        for (int j = 0; j < 16; j++) s[pad16(g + 16 * j)] = (uint64_t)__double_as_longlong(xd[j]);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; j++) xd[j] = __longlong_as_double((long long)s[pad16(16 * g + j)]);
        __syncwarp();
        fphase_ct_any<16, 12>(xd, r * 256 + 16 * g, Wd, c);
#pragma unroll
        for (int j = 0; j < 16; j++) s[pad16(16 * g + j)] = fcanon(xd[j], c.qd, c.qid);
    } else {
    if (nc)
        phase_ct<16, 8, true>(x, r * 256 + g, W2, c.q);
    else
        phase_ct<16, 8>(x, r * 256 + g, W2, c.q);
#pragma unroll
    for (int j = 0; j < 16; j++) s[pad16(g + 16 * j)] = x[j];
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = s[pad16(16 * g + j)];
    __syncwarp();
    if (nc) {
        phase_ct<16, 12, true>(x, r * 256 + 16 * g, W2, c.q);
#pragma unroll
        for (int j = 0; j < 16; j++) s[pad16(16 * g + j)] = reduce64(x[j], c);  // < 33q
    } else {
        phase_ct<16, 12>(x, r * 256 + 16 * g, W2, c.q);
#pragma unroll
        for (int j = 0; j < 16; j++) s[pad16(16 * g + j)] = reduce4q(x[j], c.q);
    }
    }
    __syncwarp();
    if (EP == E_SUBSCALE) cp_async_wait<0>();
#pragma unroll
    for (int j = 0; j < 16; j++) {
        const int cc = g + 16 * j;
        const uint64_t v = s[pad16(cc)];
        if (EP == E_STORE) {
            row[cc] = v;
        } else {
            const size_t idx = r * 256 + cc;
            uint64_t base = pa[cc];
            if (jb.aux2) base = add_mod(base, shoup(pb[cc], jb.c2, jb.c2p, c.q), c.q);
            uint64_t y = shoup(sub_mod(base, v, c.q), jb.cw, jb.cwp, c.q);
            if (jb.add) y = add_mod(y, jb.aux2 ? jb.add[idx] : pb[cc], c.q);
            jb.out[idx] = y;
        }
    }
}

// ---------------------------------------------------------------- inverse passes
// ---------------------------------------------------------------- async-pipelined passes
// Persistent form of the row passes: each CTA walks tiles (job, 16-row tile)
// with stride gridDim.x and keeps KS tiles in flight with cp.async (8-byte
// copies straight into the padded shared layout, no register staging), so a
// CTA computes one tile while the next ones stream in.

constexpr int KS = 3;            // tiles in flight per CTA
constexpr int TILE_W = 16 * 272;  // padded words per 16-row tile

__device__ __forceinline__ void ki_rows_issue(const Job *jobs, int ntiles, int tile, uint64_t *st) {
    if (tile < ntiles) {
        const Job &jb = jobs[tile >> 4];
        const int tid = threadIdx.x, g = tid & 15, rl = tid >> 4;
        const uint64_t *in = jb.src + ((tile & 15) * 16 + rl) * 256;
        uint64_t *s = st + rl * 272;
#pragma unroll
        for (int j = 0; j < 16; j++) cp_async8(s + pad16(g + 16 * j), in + g + 16 * j);
    }
    cp_async_commit();  // (empty groups keep the wait counts uniform)
}

__global__ void __launch_bounds__(NTT_TPB, 2) ki_rows_p(const Job *__restrict__ jobs, int ntiles, const uint64_t *tw,
                                                       const double *twd, const ModConst *mc) {
    extern __shared__ uint64_t ring[];  // [KS][TILE_W]
    const int tid = threadIdx.x, g = tid & 15, rl = tid >> 4;
#pragma unroll
    for (int k = 0; k < KS - 1; k++) ki_rows_issue(jobs, ntiles, blockIdx.x + k * gridDim.x, ring + k * TILE_W);
    for (int i = 0;; i++) {
        const int tile = blockIdx.x + i * gridDim.x;
        if (tile >= ntiles) break;
        ki_rows_issue(jobs, ntiles, tile + (KS - 1) * gridDim.x, ring + ((i + KS - 1) % KS) * TILE_W);
        cp_async_wait<KS - 1>();
        __syncthreads();
        const Job jb = jobs[tile >> 4];
        const ModConst c = mc[jb.mod];
        const ulonglong2 *W2 = tw_inv(tw, jb.mod, LOGN);
        const uint32_t r = (tile & 15) * 16 + rl;
        uint64_t *s = ring + (i % KS) * TILE_W + rl * 272;
        uint64_t x[16];
        if (jb.src2) {  // joint ModDown: X = acc + (P mod q) * d on the dropped Q limbs
            const uint64_t *in2 = jb.src2 + r * 256;
#pragma unroll
            for (int j = 0; j < 16; j++)
                s[pad16(g + 16 * j)] = add_mod(s[pad16(g + 16 * j)], shoup(in2[g + 16 * j], jb.c2, jb.c2p, c.q), c.q);
            __syncwarp();
        }
#pragma unroll
        for (int j = 0; j < 16; j++) x[j] = s[pad16(16 * g + j)];
        if (c.q < FP_QMAX50) {  // FP64 butterflies, canonical output
            const double *Wd = twd_inv(twd, jb.mod, LOGN);
            double xd[16];
#pragma unroll
            for (int j = 0; j < 16; j++) xd[j] = u2d(x[j]);
            fphase_gs_any<16, 0>(xd, r * 256 + 16 * g, Wd, c);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 16; j++) s[pad16(16 * g + j)] = (uint64_t)__double_as_longlong(xd[j]);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 16; j++) xd[j] = __longlong_as_double((long long)s[pad16(g + 16 * j)]);
            fphase_gs_any<16, 4>(xd, r * 256 + g, Wd, c);
#pragma unroll
            for (int j = 0; j < 16; j++) x[j] = fcanon(xd[j], c.qd, c.qid);
        } else {
        const bool nc = c.q < NC_INV;
        if (nc)
            phase_gs<16, 0, 1>(x, r * 256 + 16 * g, W2, c.q);
        else
            phase_gs<16, 0>(x, r * 256 + 16 * g, W2, c.q);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; j++) s[pad16(16 * g + j)] = x[j];
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 16; j++) x[j] = s[pad16(g + 16 * j)];
        if (nc)
            phase_gs<16, 4, 5>(x, r * 256 + g, W2, c.q);
        else
            phase_gs<16, 4>(x, r * 256 + g, W2, c.q);
        }
        uint64_t *out = jb.dst + r * 256;
#pragma unroll
        for (int j = 0; j < 16; j++) out[g + 16 * j] = x[j];
        __syncthreads();  // the stage is refilled by the next iteration's issue
    }
    cp_async_wait<0>();
}

// pass 2 (columns): in place on dst, GS stages 8..15, times (cw, cwp) = N^-1 * extra
__global__ void __launch_bounds__(NTT_TPB) ki_cols(const Job *__restrict__ jobs, const uint64_t *tw,
                                                  const double *twd, const ModConst *mc) {
    __shared__ uint64_t sm[256 * 16];
    const Job jb = jobs[blockIdx.x >> 4];
    const ModConst c = mc[jb.mod];
    const ulonglong2 *W2 = tw_inv(tw, jb.mod, LOGN);
    const int tid = threadIdx.x, lc = tid & 15, g = tid >> 4;
    const uint32_t col = (blockIdx.x & 15) * 16 + lc;
    uint64_t x[16];
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = jb.dst[(16 * g + j) * 256 + col];
    if (c.q < FP_QMAX50) {  // FP64 butterflies; the final scale is one more FP64 product
        const double *Wd = twd_inv(twd, jb.mod, LOGN);
        double xd[16];
#pragma unroll
        for (int j = 0; j < 16; j++) xd[j] = u2d(x[j]);
        fphase_gs_any<16, 8>(xd, col + 4096 * g, Wd, c);
#pragma unroll
        for (int j = 0; j < 16; j++) sm[(16 * g + j) * 16 + lc] = (uint64_t)__double_as_longlong(xd[j]);
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 16; j++) xd[j] = __longlong_as_double((long long)sm[(g + 16 * j) * 16 + lc]);
        fphase_gs_any<16, 12>(xd, col + 256 * g, Wd, c);
        const double cwd = u2d(jb.cw);
#pragma unroll
        for (int j = 0; j < 16; j++)
            jb.dst[(g + 16 * j) * 256 + col] = fcanon(fmulmod(xd[j], cwd, c.qd, c.qid), c.qd, c.qid);
        return;
    }
    const bool nc = c.q < NC_INV;  // inputs < 2^9 q (ki_rows), output < 2^17 q, then Shoup -> canonical
    if (nc)
        phase_gs<16, 8, 9>(x, col + 4096 * g, W2, c.q);
    else
        phase_gs<16, 8>(x, col + 4096 * g, W2, c.q);
#pragma unroll
    for (int j = 0; j < 16; j++) sm[(16 * g + j) * 16 + lc] = x[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = sm[(g + 16 * j) * 16 + lc];
    if (nc)
        phase_gs<16, 12, 13>(x, col + 256 * g, W2, c.q);
    else
        phase_gs<16, 12>(x, col + 256 * g, W2, c.q);
#pragma unroll
    for (int j = 0; j < 16; j++) jb.dst[(g + 16 * j) * 256 + col] = shoup(x[j], jb.cw, jb.cwp, c.q);
}

// ---------------------------------------------------------------- ModUp pass 2 + inner product
constexpr int KS_MAXC = 3;  // key-switched components per inner product (s^2, s^3, s^4)
struct IpArgs {
    const uint64_t *ext;  // [nk][B][beta][ext_n][N] ModUp pass-1 outputs
    const uint64_t *const *d;  // [nk][B] device pointers to the switched components (NTT domain, [ell][N])
    const uint64_t *key[KS_MAXC];  // per component: [dnum][2][M][N] Montgomery form
    int nk;               // components summed into one accumulator
    uint64_t *acc;        // [B][2][ext_n][N]
    const uint64_t *tw;
    const double *twd;
    const ModConst *mc;
    const double *rinvd;  // [M] 2^-64 mod q (as doubles): undoes the key's Montgomery factor
    const int32_t *tlist; // targets handled by this launch (indices into the extended basis)
    int ell, ext_n, beta, alpha, L, M, B;
};

// FP64 form for targets with q < 2^42: pass 2 of every digit's NTT on the
// FP64 pipe, inner product as exact FP64 modular products against the
// Montgomery-form key (|sum| < 6 nk beta q < 2^51, exact), one R^-1 product and one
// canonicalisation at the end.  Half the registers of the 128-bit integer
// accumulators (no spills) and twice the multiply rate.
__global__ void __launch_bounds__(NTT_TPB, 2) k_modup_ip_fp(const IpArgs a) {
    __shared__ uint64_t sm[16 * 272];
    const int b = blockIdx.x % a.B, rest = blockIdx.x / a.B;
    const int rt = rest & 15, t = a.tlist[rest >> 4];
    const int m = t < a.ell ? t : a.L + (t - a.ell);
    const ModConst c = a.mc[m];
    const double *Wd = twd_fwd(a.twd, m, LOGN);
    const int tid = threadIdx.x, g = tid & 15, rl = tid >> 4;
    const uint32_t r = rt * 16 + rl;
    const int jt = t < a.ell ? t / a.alpha : -1;
    uint64_t *s = sm + rl * 272;
    double acc0[16], acc1[16];
#pragma unroll
    for (int j = 0; j < 16; j++) acc0[j] = acc1[j] = 0.0;
    for (int kc = 0; kc < a.nk; kc++)
    for (int dj = 0; dj < a.beta; dj++) {
        const int bk = kc * a.B + b;
        const uint64_t *kbase = kc == 0 ? a.key[0] : kc == 1 ? a.key[1] : a.key[2];  // (no param-array indexing)
        double xd[16];
        if (dj == jt) {
            const uint64_t *dp = a.d[bk] + (size_t)t * NN + r * 256;
#pragma unroll
            for (int j = 0; j < 16; j++) xd[j] = u2d(dp[g + 16 * j]);
        } else {
            const uint64_t *row = a.ext + ((((size_t)bk * a.beta + dj) * a.ext_n + t) << LOGN) + r * 256;
#pragma unroll
            for (int j = 0; j < 16; j++) xd[j] = u2d(row[g + 16 * j]);
            fphase_ct_any<16, 8>(xd, r * 256 + g, Wd, c);
#pragma unroll
            for (int j = 0; j < 16; j++) s[pad16(g + 16 * j)] = (uint64_t)__double_as_longlong(xd[j]);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 16; j++) xd[j] = __longlong_as_double((long long)s[pad16(16 * g + j)]);
            __syncwarp();
            fphase_ct_any<16, 12>(xd, r * 256 + 16 * g, Wd, c);  // < 2^42: |x| < 17q, no reduction needed
#pragma unroll
            for (int j = 0; j < 16; j++) s[pad16(16 * g + j)] = (uint64_t)__double_as_longlong(xd[j]);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 16; j++) xd[j] = __longlong_as_double((long long)s[pad16(g + 16 * j)]);
            __syncwarp();
        }
        const uint64_t *k0 = kbase + (((size_t)dj * 2 * a.M + m) << LOGN) + r * 256;
        const uint64_t *k1 = k0 + ((size_t)a.M << LOGN);
#pragma unroll
        for (int j = 0; j < 16; j++) {
            const int cc = g + 16 * j;
            const double w0 = u2d(__ldg(k0 + cc)), w1 = u2d(__ldg(k1 + cc));
            acc0[j] += fmulmod(xd[j], w0, c.qd, c.qid);
            acc1[j] += fmulmod(xd[j], w1, c.qd, c.qid);
        }
        if (c.q >= FP_QMAX)  // 2^42 .. 2^50: each product < 1.01 q, keep the sums centred
#pragma unroll
            for (int j = 0; j < 16; j++) {
                acc0[j] = fred_c(acc0[j], c.qd, c.qid);
                acc1[j] = fred_c(acc1[j], c.qd, c.qid);
            }
    }
    const double ri = a.rinvd[m];
    uint64_t *o0 = a.acc + ((((size_t)b * 2) * a.ext_n + t) << LOGN) + r * 256;
    uint64_t *o1 = o0 + ((size_t)a.ext_n << LOGN);
#pragma unroll
    for (int j = 0; j < 16; j++) {
        o0[g + 16 * j] = fcanon(fmulmod(acc0[j], ri, c.qd, c.qid), c.qd, c.qid);
        o1[g + 16 * j] = fcanon(fmulmod(acc1[j], ri, c.qd, c.qid), c.qd, c.qid);
    }
}

__global__ void __launch_bounds__(NTT_TPB, 2) k_modup_ip(const IpArgs a) {
    __shared__ uint64_t sm[16 * 272];
    // ciphertext-fastest order: CTAs resident together read the same key rows
    // (dnum x 2 x 16 rows of limb t), so the key streams from L2, not HBM
    const int b = blockIdx.x % a.B, rest = blockIdx.x / a.B;
    const int rt = rest & 15, t = a.tlist[rest >> 4];
    const int m = t < a.ell ? t : a.L + (t - a.ell);
    const ModConst c = a.mc[m];
    const ulonglong2 *W2 = tw_fwd(a.tw, m, LOGN);
    const int tid = threadIdx.x, g = tid & 15, rl = tid >> 4;
    const uint32_t r = rt * 16 + rl;
    const int jt = t < a.ell ? t / a.alpha : -1;
    uint64_t *s = sm + rl * 272;
    // inner product with the Montgomery-form key: one REDC per product, canonical
    // accumulators (64-bit: these wide-prime targets keep the register budget)
    uint64_t acc0[16], acc1[16];
#pragma unroll
    for (int j = 0; j < 16; j++) acc0[j] = acc1[j] = 0;
    for (int kc = 0; kc < a.nk; kc++)
    for (int dj = 0; dj < a.beta; dj++) {
        const int bk = kc * a.B + b;
        const uint64_t *kbase = kc == 0 ? a.key[0] : kc == 1 ? a.key[1] : a.key[2];
        uint64_t x[16];
        if (dj == jt) {
            const uint64_t *dp = a.d[bk] + (size_t)t * NN + r * 256;
#pragma unroll
            for (int j = 0; j < 16; j++) x[j] = dp[g + 16 * j];
        } else {
            const uint64_t *row = a.ext + ((((size_t)bk * a.beta + dj) * a.ext_n + t) << LOGN) + r * 256;
#pragma unroll
            for (int j = 0; j < 16; j++) x[j] = row[g + 16 * j];
            const bool nc = c.q < NC_FWD;  // (targets below 2^42 go to k_modup_ip_fp)
            if (nc)
                phase_ct<16, 8, true>(x, r * 256 + g, W2, c.q);
            else
                phase_ct<16, 8>(x, r * 256 + g, W2, c.q);
#pragma unroll
            for (int j = 0; j < 16; j++) s[pad16(g + 16 * j)] = x[j];
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 16; j++) x[j] = s[pad16(16 * g + j)];
            __syncwarp();
            if (nc) {
                phase_ct<16, 12, true>(x, r * 256 + 16 * g, W2, c.q);
#pragma unroll
                for (int j = 0; j < 16; j++) s[pad16(16 * g + j)] = reduce64(x[j], c);
            } else {
                phase_ct<16, 12>(x, r * 256 + 16 * g, W2, c.q);
#pragma unroll
                for (int j = 0; j < 16; j++) s[pad16(16 * g + j)] = reduce4q(x[j], c.q);
            }
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 16; j++) x[j] = s[pad16(g + 16 * j)];
            __syncwarp();
        }
        const uint64_t *k0 = kbase + (((size_t)dj * 2 * a.M + m) << LOGN) + r * 256;
        const uint64_t *k1 = k0 + ((size_t)a.M << LOGN);
#pragma unroll
        for (int j = 0; j < 16; j++) {
            const int cc = g + 16 * j;
            const uint64_t w0 = __ldg(k0 + cc), w1 = __ldg(k1 + cc);
            acc0[j] = add_mod(acc0[j], redc(mulhi(x[j], w0), x[j] * w0, c.q, c.qinv), c.q);
            acc1[j] = add_mod(acc1[j], redc(mulhi(x[j], w1), x[j] * w1, c.q, c.qinv), c.q);
        }
    }
    uint64_t *o0 = a.acc + ((((size_t)b * 2) * a.ext_n + t) << LOGN) + r * 256;
    uint64_t *o1 = o0 + ((size_t)a.ext_n << LOGN);
#pragma unroll
    for (int j = 0; j < 16; j++) {
        o0[g + 16 * j] = acc0[j];
        o1[g + 16 * j] = acc1[j];
    }
}

// ---------------------------------------------------------------- host plumbing
struct JobBuf {
    Job *d = nullptr;
    cudaStream_t s;
    explicit JobBuf(cudaStream_t st) : s(st) {}
    ~JobBuf() { he_scratch_free(d, s); }
    int up(const std::vector<Job> &v) {
        HE_TRY(he_scratch_alloc((void **)&d, v.size() * sizeof(Job), s));
        HE_CHECK_CUDA(he_h2d(d, v.data(), v.size() * sizeof(Job), s));
        return HE_OK;
    }
};

int run_inverse(he_ctx *c, const std::vector<Job> &jobs, cudaStream_t s) {
    if (jobs.empty()) return HE_OK;
    JobBuf jb(s);
    HE_TRY(jb.up(jobs));
    unsigned g = (unsigned)jobs.size() * 16;
    static int sms = 0;
    if (!sms) {
        HE_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
        HE_CHECK_CUDA(cudaFuncSetAttribute(ki_rows_p, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(KS * TILE_W * sizeof(uint64_t))));
    }
    const unsigned gp = std::min<unsigned>(g, 2u * (unsigned)sms);
    ki_rows_p<<<gp, NTT_TPB, KS * TILE_W * sizeof(uint64_t), s>>>(jb.d, (int)g, c->d_tw, c->d_twdc, c->d_mc);
    HE_CHECK_LAUNCH();
    ki_cols<<<g, NTT_TPB, 0, s>>>(jb.d, c->d_tw, c->d_twdc, c->d_mc);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

constexpr size_t KF_STAGE_BYTES = (size_t)2 * 4096 * sizeof(uint64_t);  // kf_cols<L_BCONV> source double buffer

// kf_cols launch; the integer BConv loader stages its sources in 64 KB of dynamic smem
template <int LD>
int launch_kf_cols(unsigned grid, const Job *jobs, he_ctx *c, cudaStream_t s) {
    const size_t smem = LD == L_BCONV ? KF_STAGE_BYTES : 0;
    if (LD == L_BCONV) {
        static bool attr = false;
        if (!attr) {
            HE_CHECK_CUDA(cudaFuncSetAttribute(kf_cols<L_BCONV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)KF_STAGE_BYTES));
            attr = true;
        }
    }
    kf_cols<LD><<<grid, NTT_TPB, smem, s>>>(jobs, c->d_tw, c->d_twdc, c->d_mc, c->d_rinvd);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

template <int LD, int EP>
int run_forward(he_ctx *c, const std::vector<Job> &jobs_in, cudaStream_t s) {
    if (jobs_in.empty()) return HE_OK;
    // BConv passes: targets below 2^42 take the FP64 loader (own launch), listed first
    std::vector<Job> jobs;
    size_t nfp = 0;
    if (LD == L_BCONV) {
        for (const Job &j : jobs_in)
            if (c->mod[j.mod] < FP_QMAX) jobs.push_back(j);
        nfp = jobs.size();
        for (const Job &j : jobs_in)
            if (c->mod[j.mod] >= FP_QMAX) jobs.push_back(j);
    } else {
        jobs = jobs_in;
    }
    JobBuf jb(s);
    HE_TRY(jb.up(jobs));
    if (nfp) {
        kf_cols<L_BCONV_FPW><<<(unsigned)nfp * 16, NTT_TPB, 0, s>>>(jb.d, c->d_tw, c->d_twdc, c->d_mc, c->d_rinvd);
        HE_CHECK_LAUNCH();
    }
    if (jobs.size() > nfp) HE_TRY(launch_kf_cols<LD>((unsigned)(jobs.size() - nfp) * 16, jb.d + nfp, c, s));
    const size_t pre_bytes = EP == E_SUBSCALE ? (size_t)2 * 4096 * sizeof(uint64_t) : 0;
    static bool attr = false;
    if (EP == E_SUBSCALE && !attr) {
        HE_CHECK_CUDA(cudaFuncSetAttribute(kf_rows<E_SUBSCALE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)pre_bytes));
        attr = true;
    }
    kf_rows<EP><<<(unsigned)jobs.size() * 16, NTT_TPB, pre_bytes, s>>>(jb.d, c->d_tw, c->d_twdc, c->d_mc);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

Job blank() {
    Job j;
    memset(&j, 0, sizeof j);
    return j;
}

}  // namespace

// ModUp of nk components + key inner products summed into one accumulator:
// acc [B][2][ell+K][N] (NTT domain) = sum_k ModUp(d_k) . keys[k].  d (HOST) and
// d_dev (DEVICE) list the components [nk][B]; dcv [nk][B][ell][N] and ext
// [nk][B][beta][ell+K][N] are caller-provided scratch.
// ModUp steps 1-2 (INTT of d with the per-source q-hat^-1 folded in, BConv + NTT
// pass 1 of every extended limb into ext).  ext is not modified by step 3, so
// one ModUp serves every key applied to the same d (hoisted rotations).
static int modup_prep(he_ctx *c, int nk, const uint64_t *const *d, int B, int ell, uint64_t *dcv, uint64_t *ext,
                      cudaStream_t s) {
    const int L = c->L, K = c->K, alpha = c->alpha;
    const int beta = (ell + alpha - 1) / alpha, ext_n = ell + K;
    int rc = HE_OK;
    std::vector<const BconvTable *> up(beta);
    for (int j = 0; j < beta && rc == HE_OK; j++) rc = he_get_modup_table(c, ell, j, &up[j]);
    // 1. v = INTT(d) * qhat_s^-1 (ModUp's per-source Shoup step folded into INTT's N^-1)
    if (rc == HE_OK) {
        std::vector<Job> jobs;
        for (int b = 0; b < nk * B; b++)
            for (int i = 0; i < ell; i++) {
                Job j = blank();
                j.src = d[b] + (size_t)i * NN;
                j.dst = dcv + ((size_t)b * ell + i) * NN;
                j.mod = i;
                const int dj = i / alpha, si = i - dj * alpha;
                j.cw = he_h_mulmod(c->h_ninv[i], up[dj]->h_qhinv[si], c->mod[i]);
                j.cwp = he_h_shoup(j.cw, c->mod[i]);
                jobs.push_back(j);
            }
        rc = run_inverse(c, jobs, s);
    }
    // 2. ModUp pass 1: BConv loaded straight into the NTT of every target limb
    //    (FP64 loader for targets below 2^42)
    if (rc == HE_OK) {
        std::vector<Job> jobs, jobs_fp;
        for (int b = 0; b < nk * B; b++)
            for (int dj = 0; dj < beta; dj++) {
                const BconvTable *tb = up[dj];
                const int s0 = dj * alpha, ns = tb->n_src;
                int wide = 0;
                for (int k = 0; k < ns; k++) wide |= (c->mod[s0 + k] >= FP_QMAX ? 1 : 0) << k;
                for (int dst = 0; dst < tb->n_dst; dst++) {
                    const int m = tb->h_dst_mod[dst];
                    const int t = m < L ? m : ell + (m - L);
                    Job j = blank();
                    j.src = dcv + ((size_t)b * ell + s0) * NN;
                    j.ns = ns;
                    j.tab = tb->d + 2 * ns + (size_t)dst * ns;
                    j.mod = m;
                    j.dst = ext + (((size_t)b * beta + dj) * ext_n + t) * NN;
                    if (c->mod[m] < FP_QMAX) {
                        j.wide = wide;
                        jobs_fp.push_back(j);
                    } else {
                        jobs.push_back(j);
                    }
                }
            }
        if (!jobs_fp.empty()) {  // narrow-source jobs first (64-register instantiation), then wide
            std::stable_partition(jobs_fp.begin(), jobs_fp.end(), [](const Job &j) { return j.wide == 0; });
            size_t nn = 0;
            while (nn < jobs_fp.size() && jobs_fp[nn].wide == 0) nn++;
            JobBuf jb(s);
            rc = jb.up(jobs_fp);
            if (rc == HE_OK && nn) {
                kf_cols<L_BCONV_FP><<<(unsigned)nn * 16, NTT_TPB, 0, s>>>(jb.d, c->d_tw, c->d_twdc, c->d_mc,
                                                                         c->d_rinvd);
                he_count_launch(1);
                if (cudaGetLastError() != cudaSuccess) rc = HE_ECUDA;
            }
            if (rc == HE_OK && jobs_fp.size() > nn) {
                kf_cols<L_BCONV_FPW><<<(unsigned)(jobs_fp.size() - nn) * 16, NTT_TPB, 0, s>>>(
                    jb.d + nn, c->d_tw, c->d_twdc, c->d_mc, c->d_rinvd);
                he_count_launch(1);
                if (cudaGetLastError() != cudaSuccess) rc = HE_ECUDA;
            }
        }
        if (rc == HE_OK && !jobs.empty()) {
            JobBuf jb(s);
            rc = jb.up(jobs);
            if (rc == HE_OK) {
                rc = launch_kf_cols<L_BCONV>((unsigned)jobs.size() * 16, jb.d, c, s);  // counts the launch
            }
        }
    }
    return rc;
}

// ModUp step 3: NTT pass 2 of every extended limb fused with the inner product
// against `keys` (sum over the nk components of d), into acc [B][2][ext_n][N].
static int modup_ip3(he_ctx *c, const uint64_t *const *keys, int nk, const uint64_t *const *d_dev, int B, int ell,
                     uint64_t *ext, uint64_t *acc, cudaStream_t s) {
    const int L = c->L, K = c->K, alpha = c->alpha, M = L + K;
    const int beta = (ell + alpha - 1) / alpha, ext_n = ell + K;
    int rc = HE_OK;
    {
        IpArgs a;
        a.ext = ext;
        a.d = d_dev;
        a.nk = nk;
        for (int k = 0; k < KS_MAXC; k++) a.key[k] = keys[k < nk ? k : 0];
        a.acc = acc;
        a.tw = c->d_tw;
        a.twd = c->d_twdc;
        a.mc = c->d_mc;
        a.ell = ell;
        a.ext_n = ext_n;
        a.beta = beta;
        a.alpha = alpha;
        a.L = L;
        a.M = M;
        a.B = B;
        a.rinvd = c->d_rinvd;
        // targets split by prime size: FP64 kernel below 2^50, integer kernel otherwise
        std::vector<int32_t> tl;
        int nfp = 0;
        for (int pass = 0; pass < 2; pass++)
            for (int t = 0; t < ext_n; t++) {
                const int m = t < ell ? t : L + (t - ell);
                if ((c->mod[m] < FP_QMAX50) == (pass == 0)) {
                    tl.push_back(t);
                    nfp += pass == 0;
                }
            }
        int32_t *dtl = nullptr;
        rc = he_scratch_alloc((void **)&dtl, tl.size() * 4, s);
        if (rc == HE_OK && he_h2d(dtl, tl.data(), tl.size() * 4, s) != cudaSuccess)
            rc = HE_ECUDA;
        if (rc == HE_OK && nfp) {
            a.tlist = dtl;
            k_modup_ip_fp<<<(unsigned)(B * nfp * 16), NTT_TPB, 0, s>>>(a);
            he_count_launch(1);
            if (cudaGetLastError() != cudaSuccess) rc = HE_ECUDA;
        }
        if (rc == HE_OK && nfp < ext_n) {
            a.tlist = dtl + nfp;
            k_modup_ip<<<(unsigned)(B * (ext_n - nfp) * 16), NTT_TPB, 0, s>>>(a);
            he_count_launch(1);
            if (cudaGetLastError() != cudaSuccess) rc = HE_ECUDA;
        }
        he_scratch_free(dtl, s);
    }
    return rc;
}

static int modup_ip(he_ctx *c, const uint64_t *const *keys, int nk, const uint64_t *const *d,
                    const uint64_t *const *d_dev, int B, int ell, uint64_t *dcv, uint64_t *ext, uint64_t *acc,
                    cudaStream_t s) {
    HE_TRY(modup_prep(c, nk, d, B, ell, dcv, ext, s));
    return modup_ip3(c, keys, nk, d_dev, B, ell, ext, acc, s);
}

// ModDown of acc [B][2][ext_n][N]: INTT of the P limbs (times N^-1 phat_k^-1),
// then the P -> Q BConv NTT whose epilogue writes (acc - conv) P^-1 (+ add0/add1)
// to out0 / out1 (HOST arrays of device addresses; md: scratch [B][2][ell][N]).
static int moddown_add(he_ctx *c, const BconvTable *dn, uint64_t *acc, uint64_t *md, int B, int ell,
                       uint64_t *const *out0, uint64_t *const *out1, const uint64_t *const *add0,
                       const uint64_t *const *add1, cudaStream_t s) {
    const int L = c->L, K = c->K, ext_n = ell + K;
    int rc = HE_OK;
    if (rc == HE_OK) {
        std::vector<Job> jobs;
        for (int b = 0; b < B; b++)
            for (int cc = 0; cc < 2; cc++)
                for (int k = 0; k < K; k++) {
                    Job j = blank();
                    j.src = j.dst = acc + (((size_t)b * 2 + cc) * ext_n + ell + k) * NN;
                    j.mod = L + k;
                    j.cw = he_h_mulmod(c->h_ninv[L + k], dn->h_qhinv[k], c->mod[L + k]);
                    j.cwp = he_h_shoup(j.cw, c->mod[L + k]);
                    jobs.push_back(j);
                }
        rc = run_inverse(c, jobs, s);
    }
    if (rc == HE_OK) {
        std::vector<Job> jobs;
        for (int b = 0; b < B; b++)
            for (int cc = 0; cc < 2; cc++) {
                const uint64_t *const *addv = cc == 0 ? add0 : add1;
                uint64_t *const *outv = cc == 0 ? out0 : out1;
                for (int i = 0; i < ell; i++) {
                    Job j = blank();
                    j.src = acc + (((size_t)b * 2 + cc) * ext_n + ell) * NN;
                    j.ns = K;
                    j.tab = dn->d + 2 * K + (size_t)i * K;
                    for (int k = 0; k < K; k++) j.wide |= (c->mod[L + k] >= FP_QMAX ? 1 : 0) << k;
                    j.mod = i;
                    j.dst = md + (((size_t)b * 2 + cc) * ell + i) * NN;
                    j.aux = acc + (((size_t)b * 2 + cc) * ext_n + i) * NN;
                    j.add = addv ? addv[b] + (size_t)i * NN : nullptr;
                    j.out = outv[b] + (size_t)i * NN;
                    j.cw = c->h_pinv[2 * i];
                    j.cwp = c->h_pinv[2 * i + 1];
                    jobs.push_back(j);
                }
            }
        rc = run_forward<L_BCONV, E_SUBSCALE>(c, jobs, s);
    }
    return rc;
}

// Fused hybrid key switch for B ciphertexts (N = 2^16).  Pointer arguments are
// HOST arrays of device addresses; d_dev is the same list of d pointers in
// device memory (read by the inner-product kernel).
int he_keyswitch_fused(he_ctx *c, const uint64_t *key, const uint64_t *const *d, const uint64_t *const *d_dev, int B,
                       int ell, uint64_t *const *out0, uint64_t *const *out1, const uint64_t *const *add0,
                       const uint64_t *const *add1, cudaStream_t s) {
    const int L = c->L, K = c->K, alpha = c->alpha;
    const int beta = (ell + alpha - 1) / alpha, ext_n = ell + K;
    const size_t w_dc = (size_t)B * ell * NN, w_ext = (size_t)B * beta * ext_n * NN, w_acc = (size_t)B * 2 * ext_n * NN,
                 w_md = (size_t)B * 2 * ell * NN;
    void *scr = nullptr;
    HE_TRY(he_scratch_alloc(&scr, (w_dc + w_ext + w_acc + w_md) * 8, s));
    uint64_t *dcv = (uint64_t *)scr, *ext = dcv + w_dc, *acc = ext + w_ext, *md = acc + w_acc;
    const BconvTable *dn = nullptr;
    int rc = he_get_moddown_table(c, ell, &dn);
    const uint64_t *keys[1] = {key};
    if (rc == HE_OK) rc = modup_ip(c, keys, 1, d, d_dev, B, ell, dcv, ext, acc, s);
    if (rc == HE_OK) rc = moddown_add(c, dn, acc, md, B, ell, out0, out1, add0, add1, s);
    he_scratch_free(scr, s);
    return rc;
}

// Hoisted rotations, step 1 of he_rotate_hoisted (N = 2^16): for R hoisting keys,
// t_r = (c0 + KS(c1, hkey_r).0, KS(c1, hkey_r).1) with ONE ModUp of c1 shared by
// every rotation (oracle oc_rotate_hoisted; the caller applies sigma_g to t_r).
// c0, c1: HOST arrays [B]; c1_dev: device array [B]; t0, t1: HOST arrays [R][B].
int he_hoisted_ks_fused(he_ctx *c, const uint64_t *const *hkeys, int R, const uint64_t *const *c0,
                        const uint64_t *const *c1, const uint64_t *const *c1_dev, int B, int ell,
                        uint64_t *const *t0, uint64_t *const *t1, cudaStream_t s) {
    const int K = c->K, alpha = c->alpha;
    const int beta = (ell + alpha - 1) / alpha, ext_n = ell + K;
    const size_t w_dc = (size_t)B * ell * NN, w_ext = (size_t)B * beta * ext_n * NN, w_acc = (size_t)B * 2 * ext_n * NN,
                 w_md = (size_t)B * 2 * ell * NN;
    void *scr = nullptr;
    HE_TRY(he_scratch_alloc(&scr, (w_dc + w_ext + w_acc + w_md) * 8, s));
    uint64_t *dcv = (uint64_t *)scr, *ext = dcv + w_dc, *acc = ext + w_ext, *md = acc + w_acc;
    const BconvTable *dn = nullptr;
    int rc = he_get_moddown_table(c, ell, &dn);
    if (rc == HE_OK) rc = modup_prep(c, 1, c1, B, ell, dcv, ext, s);
    for (int r = 0; r < R && rc == HE_OK; r++) {
        const uint64_t *keys[1] = {hkeys[r]};
        rc = modup_ip3(c, keys, 1, c1_dev, B, ell, ext, acc, s);
        if (rc == HE_OK)
            rc = moddown_add(c, dn, acc, md, B, ell, t0 + (size_t)r * B, t1 + (size_t)r * B, c0, nullptr, s);
    }
    he_scratch_free(scr, s);
    return rc;
}

// Relinearisation + `extra` rescales as one ModDown over S = {dropped Q limbs}
// u P (oracle: oc_relin_rescale_n).  d3: HOST array of [nc][ell][N] device
// ciphertexts (nc = nk + 2; component k >= 2 switched with keys[k-2], the s^k
// key), dk_dev: device array [nk][B] of their component pointers d3 + k ell N,
// out: HOST array of [2][ell-extra][N].
int he_relin_rescale_fused(he_ctx *c, const uint64_t *const *keys, int nk, const uint64_t *const *d3,
                           const uint64_t *const *dk_dev, int B, int ell, int extra, uint64_t *const *out,
                           cudaStream_t s) {
    const int L = c->L, K = c->K, alpha = c->alpha, lo = ell - extra, ns = extra + K;
    const int beta = (ell + alpha - 1) / alpha, ext_n = ell + K;
    const size_t P = (size_t)ell * NN;
    const size_t w_dc = (size_t)nk * B * ell * NN, w_ext = (size_t)nk * B * beta * ext_n * NN,
                 w_acc = (size_t)B * 2 * ext_n * NN, w_md = (size_t)B * 2 * lo * NN;
    void *scr = nullptr;
    HE_TRY(he_scratch_alloc(&scr, (w_dc + w_ext + w_acc + w_md) * 8, s));
    uint64_t *dcv = (uint64_t *)scr, *ext = dcv + w_dc, *acc = ext + w_ext, *md = acc + w_acc;
    std::vector<const uint64_t *> dk((size_t)nk * B);
    for (int k = 0; k < nk; k++)
        for (int b = 0; b < B; b++) dk[(size_t)k * B + b] = d3[b] + (size_t)(2 + k) * P;
    const BconvTable *dn = nullptr;
    int rc = he_get_moddown_table_x(c, ell, extra, &dn);
    if (rc == HE_OK) rc = modup_ip(c, keys, nk, dk.data(), dk_dev, B, ell, dcv, ext, acc, s);
    // joint ModDown, step 1: y_s = INTT(X_s) * N^-1 * shat_s^-1 for s in S, with
    // X_s = acc_s + [P]_{q_s} d_s on the dropped Q limbs (acc's S limbs are contiguous)
    if (rc == HE_OK) {
        std::vector<Job> jobs;
        for (int b = 0; b < B; b++)
            for (int cc = 0; cc < 2; cc++)
                for (int si = 0; si < ns; si++) {
                    const int t = lo + si, m = t < ell ? t : L + (t - ell);
                    Job j = blank();
                    j.src = j.dst = acc + (((size_t)b * 2 + cc) * ext_n + t) * NN;
                    if (t < ell) {
                        j.src2 = d3[b] + (size_t)cc * P + (size_t)t * NN;
                        j.c2 = c->h_pmodq[t];
                        j.c2p = he_h_shoup(j.c2, c->mod[t]);
                    }
                    j.mod = m;
                    j.cw = he_h_mulmod(c->h_ninv[m], dn->h_qhinv[si], c->mod[m]);
                    j.cwp = he_h_shoup(j.cw, c->mod[m]);
                    jobs.push_back(j);
                }
        rc = run_inverse(c, jobs, s);
    }
    // step 2: out_c[i] = (acc_i + [P] d_i - NTT_i(BConv_S(y))) * (prod S)^-1, i < ell - extra
    if (rc == HE_OK) {
        std::vector<Job> jobs;
        for (int b = 0; b < B; b++)
            for (int cc = 0; cc < 2; cc++)
                for (int i = 0; i < lo; i++) {
                    const uint64_t q = c->mod[i];
                    uint64_t prod = c->h_pmodq[i];
                    for (int t = lo; t < ell; t++) prod = he_h_mulmod(prod, c->mod[t] % q, q);
                    Job j = blank();
                    j.src = acc + (((size_t)b * 2 + cc) * ext_n + lo) * NN;
                    j.ns = ns;
                    j.tab = dn->d + 2 * ns + (size_t)i * ns;
                    for (int si = 0; si < ns; si++) {  // sources: dropped Q limbs, then P
                        const int sm_ = si < extra ? lo + si : L + (si - extra);
                        j.wide |= (c->mod[sm_] >= FP_QMAX ? 1 : 0) << si;
                    }
                    j.mod = i;
                    j.dst = md + (((size_t)b * 2 + cc) * lo + i) * NN;
                    j.aux = acc + (((size_t)b * 2 + cc) * ext_n + i) * NN;
                    j.aux2 = d3[b] + (size_t)cc * P + (size_t)i * NN;
                    j.c2 = c->h_pmodq[i];
                    j.c2p = he_h_shoup(j.c2, q);
                    j.out = out[b] + ((size_t)cc * lo + i) * NN;
                    j.cw = he_h_inv(prod, q);
                    j.cwp = he_h_shoup(j.cw, q);
                    jobs.push_back(j);
                }
        rc = run_forward<L_BCONV, E_SUBSCALE>(c, jobs, s);
    }
    he_scratch_free(scr, s);
    return rc;
}

// Fused rescale for B ciphertexts of nc components at ell limbs (N = 2^16).
// in / out: HOST arrays of device addresses ([nc][ell][N] -> [nc][ell-1][N]).
int he_rescale_fused(he_ctx *c, const uint64_t *const *in, uint64_t *const *out, int B, int ell, int nc,
                     cudaStream_t s) {
    const int lm1 = ell - 1;
    const size_t npc = (size_t)B * nc;
    void *scr = nullptr;
    HE_TRY(he_scratch_alloc(&scr, (npc + npc * lm1) * NN * 8, s));
    uint64_t *r = (uint64_t *)scr, *tmp = r + npc * NN;
    int rc = HE_OK;
    {
        std::vector<Job> jobs;
        for (int b = 0; b < B; b++)
            for (int cc = 0; cc < nc; cc++) {
                Job j = blank();
                j.src = in[b] + ((size_t)cc * ell + lm1) * NN;
                j.dst = r + ((size_t)b * nc + cc) * NN;
                j.mod = lm1;
                j.cw = c->h_ninv[lm1];
                j.cwp = he_h_shoup(j.cw, c->mod[lm1]);
                jobs.push_back(j);
            }
        rc = run_inverse(c, jobs, s);
    }
    if (rc == HE_OK) {
        std::vector<Job> jobs;
        for (int b = 0; b < B; b++)
            for (int cc = 0; cc < nc; cc++)
                for (int i = 0; i < lm1; i++) {
                    Job j = blank();
                    j.src = r + ((size_t)b * nc + cc) * NN;
                    j.ql = c->mod[lm1];
                    j.mod = i;
                    j.dst = tmp + (((size_t)b * nc + cc) * lm1 + i) * NN;
                    j.aux = in[b] + ((size_t)cc * ell + i) * NN;
                    j.out = out[b] + ((size_t)cc * lm1 + i) * NN;
                    j.cw = c->h_qlinv[((size_t)lm1 * c->L + i) * 2];
                    j.cwp = c->h_qlinv[((size_t)lm1 * c->L + i) * 2 + 1];
                    jobs.push_back(j);
                }
        rc = run_forward<L_CENTER, E_SUBSCALE>(c, jobs, s);
    }
    he_scratch_free(scr, s);
    return rc;
}
