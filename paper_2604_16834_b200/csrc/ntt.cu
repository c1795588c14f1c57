// ntt.cu -- batched negacyclic NTT / INTT for sm_100a.
//
// Contract: forward is Cooley-Tukey, natural order in,
// bit-reversed order out, out[k] = a(psi^(2 brv(k) + 1)); inverse is
// Gentleman-Sande, bit-reversed in, natural out, scaled by N^-1.  Outputs are
// canonical, so the result is the unique NTT and bit-exact with any other
// correct implementation (oracle/ckks_oracle.c oc_ntt / oc_intt).
//
// Structure: every thread keeps 16 residues in registers and runs radix-16
// "phases" of 4 butterfly stages; phases exchange data through shared memory.
//   N = 2^16: two kernels (two HBM round trips), 4096 residues per CTA:
//     pass "cols": stages 0..7 on 16 columns x 256 rows (stride-256 column
//     sub-transforms), pass "rows": stages 8..15 on 16 contiguous rows of 256.
//   N = 2^12: one kernel, one CTA per limb-polynomial, three phases.
// Butterflies use Harvey's lazy reduction (values in [0, 4q) forward,
// [0, 2q) inverse) with Shoup twiddles read through the read-only cache.
#include <algorithm>

#include "ntt_core.cuh"

namespace {

constexpr int TPB = NTT_TPB;

struct PolyInfo {
    uint64_t *p;
    const ulonglong2 *W2;  // (twiddle, Shoup) pairs
    uint64_t q;
    const ModConst *mc;
};

// Polys live either contiguously (data + poly*N) or, when ptrs != nullptr, in
// per-ciphertext allocations: poly p = ptrs[p / per] + (p % per) * N.
struct PolySrc {
    uint64_t *data;
    uint64_t *const *ptrs;
};

__device__ __forceinline__ bool poly_info(PolyInfo &pi, PolySrc src, size_t poly, const uint8_t *mod_map, int per,
                                          const uint64_t *tw, const ModConst *mc, int logN, bool inverse) {
    int m = mod_map[poly % per];
    if (m == 0xFF) return false;
    size_t N = (size_t)1 << logN;
    pi.p = src.ptrs ? src.ptrs[poly / per] + (poly % per) * N : src.data + poly * N;
    pi.W2 = (const ulonglong2 *)(tw + (size_t)m * 4 * N + (inverse ? 2 * N : 0));
    pi.q = mc[m].q;
    pi.mc = mc + m;
    return true;
}

// ---------------------------------------------------------------- N = 2^16
// pass 1 forward: 16 columns x 256 rows, stages 0..7
__global__ void __launch_bounds__(TPB) k_fwd16_cols(PolySrc data, const uint8_t *mod_map, int per, const uint64_t *tw,
                                                    const ModConst *mc) {
    __shared__ uint64_t sm[256 * 16];
    PolyInfo pi;
    if (!poly_info(pi, data, blockIdx.x >> 4, mod_map, per, tw, mc, 16, false)) return;
    const int tid = threadIdx.x, lc = tid & 15, g = tid >> 4;
    const uint32_t col = (blockIdx.x & 15) * 16 + lc;
    uint64_t x[16];
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = pi.p[(g + 16 * j) * 256 + col];
    phase_ct<16, 0>(x, col + 256 * g, pi.W2, pi.q);
#pragma unroll
    for (int j = 0; j < 16; j++) sm[(g + 16 * j) * 16 + lc] = x[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = sm[(16 * g + j) * 16 + lc];
    phase_ct<16, 4>(x, col + 4096 * g, pi.W2, pi.q);
#pragma unroll
    for (int j = 0; j < 16; j++) pi.p[(16 * g + j) * 256 + col] = x[j];  // lazy [0,4q) between passes
}

// pass 2 forward: 16 rows of 256, stages 8..15, canonical output
__global__ void __launch_bounds__(TPB) k_fwd16_rows(PolySrc data, const uint8_t *mod_map, int per, const uint64_t *tw,
                                                    const ModConst *mc) {
    __shared__ uint64_t sm[16 * 272];
    PolyInfo pi;
    if (!poly_info(pi, data, blockIdx.x >> 4, mod_map, per, tw, mc, 16, false)) return;
    const int tid = threadIdx.x, g = tid & 15, rl = tid >> 4;
    const uint32_t r = (blockIdx.x & 15) * 16 + rl;
    uint64_t *row = pi.p + r * 256;
    uint64_t x[16];
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = row[g + 16 * j];
    phase_ct<16, 8>(x, r * 256 + g, pi.W2, pi.q);
    uint64_t *s = sm + rl * 272;
#pragma unroll
    for (int j = 0; j < 16; j++) s[pad16(g + 16 * j)] = x[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = s[pad16(16 * g + j)];
    phase_ct<16, 12>(x, r * 256 + 16 * g, pi.W2, pi.q);
#pragma unroll
    for (int j = 0; j < 16; j++) s[pad16(16 * g + j)] = reduce4q(x[j], pi.q);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) row[g + 16 * j] = s[pad16(g + 16 * j)];
}

// pass 1 inverse: 16 rows of 256, GS stages 0..7
__global__ void __launch_bounds__(TPB) k_inv16_rows(PolySrc data, const uint8_t *mod_map, int per, const uint64_t *tw,
                                                    const ModConst *mc) {
    __shared__ uint64_t sm[16 * 272];
    PolyInfo pi;
    if (!poly_info(pi, data, blockIdx.x >> 4, mod_map, per, tw, mc, 16, true)) return;
    const int tid = threadIdx.x, g = tid & 15, rl = tid >> 4;
    const uint32_t r = (blockIdx.x & 15) * 16 + rl;
    uint64_t *row = pi.p + r * 256;
    uint64_t *s = sm + rl * 272;
    uint64_t x[16];
#pragma unroll
    for (int j = 0; j < 16; j++) s[pad16(g + 16 * j)] = row[g + 16 * j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = s[pad16(16 * g + j)];
    phase_gs<16, 0>(x, r * 256 + 16 * g, pi.W2, pi.q);
#pragma unroll
    for (int j = 0; j < 16; j++) s[pad16(16 * g + j)] = x[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = s[pad16(g + 16 * j)];
    phase_gs<16, 4>(x, r * 256 + g, pi.W2, pi.q);
#pragma unroll
    for (int j = 0; j < 16; j++) row[g + 16 * j] = x[j];  // lazy [0,2q)
}

// pass 2 inverse: 16 columns x 256 rows, GS stages 8..15, times N^-1, canonical
__global__ void __launch_bounds__(TPB) k_inv16_cols(PolySrc data, const uint8_t *mod_map, int per, const uint64_t *tw,
                                                    const ModConst *mc) {
    __shared__ uint64_t sm[256 * 16];
    PolyInfo pi;
    if (!poly_info(pi, data, blockIdx.x >> 4, mod_map, per, tw, mc, 16, true)) return;
    const int tid = threadIdx.x, lc = tid & 15, g = tid >> 4;
    const uint32_t col = (blockIdx.x & 15) * 16 + lc;
    uint64_t x[16];
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = pi.p[(16 * g + j) * 256 + col];
    phase_gs<16, 8>(x, col + 4096 * g, pi.W2, pi.q);
#pragma unroll
    for (int j = 0; j < 16; j++) sm[(16 * g + j) * 16 + lc] = x[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = sm[(g + 16 * j) * 16 + lc];
    phase_gs<16, 12>(x, col + 256 * g, pi.W2, pi.q);
    const uint64_t ni = pi.mc->ninv, nip = pi.mc->ninv_sh;
#pragma unroll
    for (int j = 0; j < 16; j++) pi.p[(g + 16 * j) * 256 + col] = shoup(x[j], ni, nip, pi.q);
}

// ---------------------------------------------------------------- N = 2^16, centred FP64 (q < 2^50)
// The same two-pass structure on the FP64 pipe (ntt_core.cuh fphase_*_c).
// Between the passes the buffer holds centred residues as raw double bits
// (private to the pair of kernels); both passes' outer boundaries are
// canonical uint64.
struct FpInfo {
    uint64_t *p;
    const double *W;
    double q, qi;
    const ModConst *mc;
};
__device__ __forceinline__ bool fp_info(FpInfo &fi, PolySrc src, size_t poly, const uint8_t *mod_map, int per,
                                        const double *twdc, const ModConst *mc, bool inverse) {
    const int m = mod_map[poly % per];
    if (m == 0xFF) return false;
    constexpr size_t N = (size_t)1 << 16;
    fi.p = src.ptrs ? src.ptrs[poly / per] + (poly % per) * N : src.data + poly * N;
    fi.W = inverse ? twd_inv(twdc, m, 16) : twd_fwd(twdc, m, 16);
    fi.q = mc[m].qd;
    fi.qi = mc[m].qid;
    fi.mc = mc + m;
    return true;
}

__global__ void __launch_bounds__(TPB) k_fwd16_cols_c(PolySrc data, const uint8_t *mod_map, int per,
                                                      const double *twdc, const ModConst *mc) {
    __shared__ double sm[256 * 16];
    FpInfo fi;
    if (!fp_info(fi, data, blockIdx.x >> 4, mod_map, per, twdc, mc, false)) return;
    const int tid = threadIdx.x, lc = tid & 15, g = tid >> 4;
    const uint32_t col = (blockIdx.x & 15) * 16 + lc;
    double x[16];
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = u2d(fi.p[(g + 16 * j) * 256 + col]);
    fphase_ct_c<16, 0>(x, col + 256 * g, fi.W, fi.q, fi.qi);
#pragma unroll
    for (int j = 0; j < 16; j++) sm[(g + 16 * j) * 16 + lc] = x[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = sm[(16 * g + j) * 16 + lc];
    fphase_ct_c<16, 4>(x, col + 4096 * g, fi.W, fi.q, fi.qi);
    double *pd = (double *)fi.p;
#pragma unroll
    for (int j = 0; j < 16; j++) pd[(16 * g + j) * 256 + col] = x[j];  // centred doubles between passes
}

__global__ void __launch_bounds__(TPB) k_fwd16_rows_c(PolySrc data, const uint8_t *mod_map, int per,
                                                      const double *twdc, const ModConst *mc) {
    __shared__ double sm[16 * 272];
    FpInfo fi;
    if (!fp_info(fi, data, blockIdx.x >> 4, mod_map, per, twdc, mc, false)) return;
    const int tid = threadIdx.x, g = tid & 15, rl = tid >> 4;
    const uint32_t r = (blockIdx.x & 15) * 16 + rl;
    uint64_t *row = fi.p + r * 256;
    const double *rowd = (const double *)row;
    double x[16];
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = rowd[g + 16 * j];
    fphase_ct_c<16, 8>(x, r * 256 + g, fi.W, fi.q, fi.qi);
    double *s = sm + rl * 272;
#pragma unroll
    for (int j = 0; j < 16; j++) s[pad16(g + 16 * j)] = x[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = s[pad16(16 * g + j)];
    fphase_ct_c<16, 12>(x, r * 256 + 16 * g, fi.W, fi.q, fi.qi);
#pragma unroll
    for (int j = 0; j < 16; j++) s[pad16(16 * g + j)] = x[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) row[g + 16 * j] = fcanon(s[pad16(g + 16 * j)], fi.q, fi.qi);
}

__global__ void __launch_bounds__(TPB) k_inv16_rows_c(PolySrc data, const uint8_t *mod_map, int per,
                                                      const double *twdc, const ModConst *mc) {
    __shared__ double sm[16 * 272];
    FpInfo fi;
    if (!fp_info(fi, data, blockIdx.x >> 4, mod_map, per, twdc, mc, true)) return;
    const int tid = threadIdx.x, g = tid & 15, rl = tid >> 4;
    const uint32_t r = (blockIdx.x & 15) * 16 + rl;
    uint64_t *row = fi.p + r * 256;
    double *s = sm + rl * 272;
    double x[16];
#pragma unroll
    for (int j = 0; j < 16; j++) s[pad16(g + 16 * j)] = u2d(row[g + 16 * j]);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = s[pad16(16 * g + j)];
    fphase_gs_c<16, 0>(x, r * 256 + 16 * g, fi.W, fi.q, fi.qi);
#pragma unroll
    for (int j = 0; j < 16; j++) s[pad16(16 * g + j)] = x[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = s[pad16(g + 16 * j)];
    fphase_gs_c<16, 4>(x, r * 256 + g, fi.W, fi.q, fi.qi);
    double *rowd = (double *)row;
#pragma unroll
    for (int j = 0; j < 16; j++) rowd[g + 16 * j] = x[j];  // centred doubles between passes
}

__global__ void __launch_bounds__(TPB) k_inv16_cols_c(PolySrc data, const uint8_t *mod_map, int per,
                                                      const double *twdc, const ModConst *mc) {
    __shared__ double sm[256 * 16];
    FpInfo fi;
    if (!fp_info(fi, data, blockIdx.x >> 4, mod_map, per, twdc, mc, true)) return;
    const int tid = threadIdx.x, lc = tid & 15, g = tid >> 4;
    const uint32_t col = (blockIdx.x & 15) * 16 + lc;
    const double *pd = (const double *)fi.p;
    double x[16];
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = pd[(16 * g + j) * 256 + col];
    fphase_gs_c<16, 8>(x, col + 4096 * g, fi.W, fi.q, fi.qi);
#pragma unroll
    for (int j = 0; j < 16; j++) sm[(16 * g + j) * 16 + lc] = x[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = sm[(g + 16 * j) * 16 + lc];
    fphase_gs_c<16, 12>(x, col + 256 * g, fi.W, fi.q, fi.qi);
    const uint64_t ni = fi.mc->ninv, qq = fi.mc->q;
    const double nic = ni > qq / 2 ? -(double)(qq - ni) : (double)ni;  // centred N^-1
    __syncthreads();  // all reads of sm done before it is reused for the coalesced store
#pragma unroll
    for (int j = 0; j < 16; j++) sm[(g + 16 * j) * 16 + lc] = fmulmod_c(x[j], nic, fi.q, fi.qi);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) fi.p[(g + 16 * j) * 256 + col] = fcanon(sm[(g + 16 * j) * 16 + lc], fi.q, fi.qi);
}

// ---------------------------------------------------------------- N = 2^12, one CTA per poly
__global__ void __launch_bounds__(TPB) k_fwd12(PolySrc data, const uint8_t *mod_map, int per, const uint64_t *tw,
                                               const ModConst *mc) {
    __shared__ uint64_t sm[4096 + 256];
    PolyInfo pi;
    if (!poly_info(pi, data, blockIdx.x, mod_map, per, tw, mc, 12, false)) return;
    const int g = threadIdx.x;
    uint64_t x[16];
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = pi.p[g + 256 * j];
    phase_ct<12, 0>(x, g, pi.W2, pi.q);
#pragma unroll
    for (int j = 0; j < 16; j++) sm[pad16(g + 256 * j)] = x[j];
    __syncthreads();
    const uint32_t e1 = (g & 15) + 256 * (g >> 4);
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = sm[pad16(e1 + 16 * j)];
    phase_ct<12, 4>(x, e1, pi.W2, pi.q);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) sm[pad16(e1 + 16 * j)] = x[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = sm[pad16(16 * g + j)];
    phase_ct<12, 8>(x, 16 * g, pi.W2, pi.q);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) sm[pad16(16 * g + j)] = reduce4q(x[j], pi.q);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) pi.p[g + 256 * j] = sm[pad16(g + 256 * j)];
}

__global__ void __launch_bounds__(TPB) k_inv12(PolySrc data, const uint8_t *mod_map, int per, const uint64_t *tw,
                                               const ModConst *mc) {
    __shared__ uint64_t sm[4096 + 256];
    PolyInfo pi;
    if (!poly_info(pi, data, blockIdx.x, mod_map, per, tw, mc, 12, true)) return;
    const int g = threadIdx.x;
    uint64_t x[16];
#pragma unroll
    for (int j = 0; j < 16; j++) sm[pad16(g + 256 * j)] = pi.p[g + 256 * j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = sm[pad16(16 * g + j)];
    phase_gs<12, 0>(x, 16 * g, pi.W2, pi.q);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) sm[pad16(16 * g + j)] = x[j];
    __syncthreads();
    const uint32_t e1 = (g & 15) + 256 * (g >> 4);
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = sm[pad16(e1 + 16 * j)];
    phase_gs<12, 4>(x, e1, pi.W2, pi.q);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) sm[pad16(e1 + 16 * j)] = x[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; j++) x[j] = sm[pad16(g + 256 * j)];
    phase_gs<12, 8>(x, g, pi.W2, pi.q);
    const uint64_t ni = pi.mc->ninv, nip = pi.mc->ninv_sh;
#pragma unroll
    for (int j = 0; j < 16; j++) pi.p[g + 256 * j] = shoup(x[j], ni, nip, pi.q);
}

// ---------------------------------------------------------------- generic N <= 2^14
// One CTA per polynomial, radix-2 stages in shared memory.  Used for the small
// rings of the API-level tests (SPEC.md examples at n = 4 ... 8192 slots).
__global__ void k_ntt_generic(PolySrc data, const uint8_t *mod_map, int per, const uint64_t *tw, const ModConst *mc,
                              int logN, int inverse) {
    extern __shared__ uint64_t sg[];
    PolyInfo pi;
    if (!poly_info(pi, data, blockIdx.x, mod_map, per, tw, mc, logN, inverse)) return;
    const int N = 1 << logN, half = N >> 1;
    for (int i = threadIdx.x; i < N; i += blockDim.x) sg[i] = pi.p[i];
    __syncthreads();
    const uint64_t q = pi.q;
    if (!inverse) {
        for (int lm = 0; lm < logN; lm++) {
            int t = half >> lm;
            for (int b = threadIdx.x; b < half; b += blockDim.x) {
                int i = b / t, j = 2 * i * t + (b % t);
                const ulonglong2 tw = pi.W2[(1 << lm) + i];
                uint64_t u = sg[j], v = shoup(sg[j + t], tw.x, tw.y, q);
                sg[j] = add_mod(u, v, q);
                sg[j + t] = sub_mod(u, v, q);
            }
            __syncthreads();
        }
    } else {
        for (int lt = 0; lt < logN; lt++) {
            int t = 1 << lt;
            for (int b = threadIdx.x; b < half; b += blockDim.x) {
                int i = b / t, j = 2 * i * t + (b % t);
                int idx = (N >> (lt + 1)) + i;
                uint64_t u = sg[j], v = sg[j + t];
                sg[j] = add_mod(u, v, q);
                sg[j + t] = shoup(sub_mod(u, v, q), pi.W2[idx].x, pi.W2[idx].y, q);
            }
            __syncthreads();
        }
        for (int i = threadIdx.x; i < N; i += blockDim.x) sg[i] = shoup(sg[i], pi.mc->ninv, pi.mc->ninv_sh, q);
        __syncthreads();
    }
    for (int i = threadIdx.x; i < N; i += blockDim.x) pi.p[i] = sg[i];
}

// ---------------------------------------------------------------- N = 2^15 (and any N > 2^14)
// The transform splits into 2^(logN-14) independent sub-blocks of 2^14 after the first
// logN - 14 forward stages (before the last ones inverse): those stages run over global
// memory (k_ntt_gstage), the other 14 per sub-block in shared memory (k_ntt_sub, the
// k_ntt_generic butterflies with the sub-block's twiddle-block offset).  Same butterflies in
// the same order as the one-CTA kernel, canonical output.
constexpr int SUBLOG = 14;

__global__ void k_ntt_gstage(PolySrc data, const uint8_t *mod_map, int per, const uint64_t *tw, const ModConst *mc,
                             int logN, size_t n_polys, int stage, int inverse, int scale) {
    const size_t N = (size_t)1 << logN, half = N >> 1;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < n_polys * half;
         idx += (size_t)gridDim.x * blockDim.x) {
        const size_t poly = idx / half, b = idx % half;
        PolyInfo pi;
        if (!poly_info(pi, data, poly, mod_map, per, tw, mc, logN, inverse)) continue;
        const uint64_t q = pi.q;
        if (!inverse) {
            const size_t t = half >> stage, i = b / t, j = 2 * i * t + (b % t);
            const ulonglong2 w = pi.W2[((size_t)1 << stage) + i];
            const uint64_t u = pi.p[j], v = shoup(pi.p[j + t], w.x, w.y, q);
            pi.p[j] = add_mod(u, v, q);
            pi.p[j + t] = sub_mod(u, v, q);
        } else {
            const size_t t = (size_t)1 << stage, i = b / t, j = 2 * i * t + (b % t);
            const size_t wi = (N >> (stage + 1)) + i;
            const uint64_t u = pi.p[j], v = pi.p[j + t];
            uint64_t x0 = add_mod(u, v, q), x1 = shoup(sub_mod(u, v, q), pi.W2[wi].x, pi.W2[wi].y, q);
            if (scale) {
                x0 = shoup(x0, pi.mc->ninv, pi.mc->ninv_sh, q);
                x1 = shoup(x1, pi.mc->ninv, pi.mc->ninv_sh, q);
            }
            pi.p[j] = x0;
            pi.p[j + t] = x1;
        }
    }
}

// stages lm = logN-14 .. logN-1 (forward) or lt = 0 .. 13 (inverse, no scaling) of sub-block
// blockIdx.x % nsub of polynomial blockIdx.x / nsub
__global__ void k_ntt_sub(PolySrc data, const uint8_t *mod_map, int per, const uint64_t *tw, const ModConst *mc,
                          int logN, int inverse) {
    extern __shared__ uint64_t sg[];
    const int nsub = 1 << (logN - SUBLOG);
    const size_t sb = blockIdx.x % nsub;
    PolyInfo pi;
    if (!poly_info(pi, data, blockIdx.x / nsub, mod_map, per, tw, mc, logN, inverse)) return;
    const int S = 1 << SUBLOG, half = S >> 1, lm0 = logN - SUBLOG;
    uint64_t *p = pi.p + sb * S;
    for (int i = threadIdx.x; i < S; i += blockDim.x) sg[i] = p[i];
    __syncthreads();
    const uint64_t q = pi.q;
    if (!inverse) {
        for (int ls = 0; ls < SUBLOG; ls++) {
            const int lm = lm0 + ls, t = half >> ls;
            for (int b = threadIdx.x; b < half; b += blockDim.x) {
                const int i = b / t, j = 2 * i * t + (b % t);
                const ulonglong2 w = pi.W2[((size_t)1 << lm) + (sb << ls) + i];
                const uint64_t u = sg[j], v = shoup(sg[j + t], w.x, w.y, q);
                sg[j] = add_mod(u, v, q);
                sg[j + t] = sub_mod(u, v, q);
            }
            __syncthreads();
        }
    } else {
        const size_t N = (size_t)1 << logN;
        for (int lt = 0; lt < SUBLOG; lt++) {
            const int t = 1 << lt;
            for (int b = threadIdx.x; b < half; b += blockDim.x) {
                const int i = b / t, j = 2 * i * t + (b % t);
                const size_t wi = (N >> (lt + 1)) + (sb << (SUBLOG - 1 - lt)) + i;
                const uint64_t u = sg[j], v = sg[j + t];
                sg[j] = add_mod(u, v, q);
                sg[j + t] = shoup(sub_mod(u, v, q), pi.W2[wi].x, pi.W2[wi].y, q);
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < S; i += blockDim.x) p[i] = sg[i];
}

}  // namespace

static int ntt_big(he_ctx *c, PolySrc src, int n_polys, const uint8_t *mod_map, int per, bool inv, cudaStream_t s) {
    const int logN = c->logN, G = logN - SUBLOG;
    const size_t smem = ((size_t)1 << SUBLOG) * 8;
    static bool attr = false;
    if (!attr) {
        HE_CHECK_CUDA(cudaFuncSetAttribute(k_ntt_sub, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    const size_t tot = (size_t)n_polys * ((size_t)c->N >> 1);
    const unsigned gg = (unsigned)std::min<size_t>((tot + 255) / 256, (size_t)148 * 32);
    const unsigned gs = (unsigned)n_polys << G;
    if (!inv) {
        for (int st = 0; st < G; st++) {
            k_ntt_gstage<<<gg, 256, 0, s>>>(src, mod_map, per, c->d_tw, c->d_mc, logN, (size_t)n_polys, st, 0, 0);
            HE_CHECK_LAUNCH();
        }
        k_ntt_sub<<<gs, 1024, smem, s>>>(src, mod_map, per, c->d_tw, c->d_mc, logN, 0);
        HE_CHECK_LAUNCH();
    } else {
        k_ntt_sub<<<gs, 1024, smem, s>>>(src, mod_map, per, c->d_tw, c->d_mc, logN, 1);
        HE_CHECK_LAUNCH();
        for (int st = SUBLOG; st < logN; st++) {
            k_ntt_gstage<<<gg, 256, 0, s>>>(src, mod_map, per, c->d_tw, c->d_mc, logN, (size_t)n_polys, st, 1,
                                           st == logN - 1);
            HE_CHECK_LAUNCH();
        }
    }
    return HE_OK;
}

static int ntt_launch(he_ctx *c, PolySrc src, int n_polys, const uint8_t *mod_map, int per, bool inv, cudaStream_t s) {
    if (n_polys <= 0) return HE_OK;
    if (c->logN == 16 && c->fp50) {  // every modulus < 2^50: centred FP64 butterflies
        unsigned g = (unsigned)n_polys * 16;
        if (!inv) {
            k_fwd16_cols_c<<<g, TPB, 0, s>>>(src, mod_map, per, c->d_twdc, c->d_mc);
            k_fwd16_rows_c<<<g, TPB, 0, s>>>(src, mod_map, per, c->d_twdc, c->d_mc);
        } else {
            k_inv16_rows_c<<<g, TPB, 0, s>>>(src, mod_map, per, c->d_twdc, c->d_mc);
            k_inv16_cols_c<<<g, TPB, 0, s>>>(src, mod_map, per, c->d_twdc, c->d_mc);
        }
        he_count_launch(1);
    } else if (c->logN == 16) {
        unsigned g = (unsigned)n_polys * 16;
        if (!inv) {
            k_fwd16_cols<<<g, TPB, 0, s>>>(src, mod_map, per, c->d_tw, c->d_mc);
            k_fwd16_rows<<<g, TPB, 0, s>>>(src, mod_map, per, c->d_tw, c->d_mc);
            he_count_launch(1);
        } else {
            k_inv16_rows<<<g, TPB, 0, s>>>(src, mod_map, per, c->d_tw, c->d_mc);
            k_inv16_cols<<<g, TPB, 0, s>>>(src, mod_map, per, c->d_tw, c->d_mc);
            he_count_launch(1);
        }
    } else if (c->logN > SUBLOG) {
        return ntt_big(c, src, n_polys, mod_map, per, inv, s);
    } else if (c->logN == 12) {
        if (!inv)
            k_fwd12<<<(unsigned)n_polys, TPB, 0, s>>>(src, mod_map, per, c->d_tw, c->d_mc);
        else
            k_inv12<<<(unsigned)n_polys, TPB, 0, s>>>(src, mod_map, per, c->d_tw, c->d_mc);
    } else {
        int N = c->N, threads = std::min(std::max(N / 2, 32), 512);
        size_t smem = (size_t)N * 8;
        if (smem > 48 * 1024)
            HE_CHECK_CUDA(cudaFuncSetAttribute(k_ntt_generic, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_ntt_generic<<<(unsigned)n_polys, threads, smem, s>>>(src, mod_map, per, c->d_tw, c->d_mc, c->logN, inv);
    }
    HE_CHECK_LAUNCH();
    return HE_OK;
}

int he_ntt_fwd(he_ctx *c, uint64_t *data, int n_polys, const uint8_t *mod_map, int per, cudaStream_t s) {
    return ntt_launch(c, PolySrc{data, nullptr}, n_polys, mod_map, per, false, s);
}
int he_ntt_inv(he_ctx *c, uint64_t *data, int n_polys, const uint8_t *mod_map, int per, cudaStream_t s) {
    return ntt_launch(c, PolySrc{data, nullptr}, n_polys, mod_map, per, true, s);
}
int he_ntt_fwd_ptrs(he_ctx *c, uint64_t *const *ptrs, int count, int per, const uint8_t *mod_map, cudaStream_t s) {
    return ntt_launch(c, PolySrc{nullptr, ptrs}, count * per, mod_map, per, false, s);
}
int he_ntt_inv_ptrs(he_ctx *c, uint64_t *const *ptrs, int count, int per, const uint8_t *mod_map, cudaStream_t s) {
    return ntt_launch(c, PolySrc{nullptr, ptrs}, count * per, mod_map, per, true, s);
}

extern "C" int he_ntt(he_ctx *c, uint64_t *data, int batch, int ell, int inverse, void *stream) {
    if (!c || !data || batch < 0 || ell < 1 || ell > c->L) {
        he_set_error("he_ntt: bad arguments (batch=%d ell=%d)", batch, ell);
        return HE_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    return inverse ? he_ntt_inv(c, data, batch * ell, c->d_ident, ell, s)
                   : he_ntt_fwd(c, data, batch * ell, c->d_ident, ell, s);
}
