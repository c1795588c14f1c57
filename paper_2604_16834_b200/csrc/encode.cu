#include <vector>
// encode.cu -- canonical-embedding encode/decode, encryption and decryption.
//
// Replaces SimulatorEngine.encrypt / decrypt (engine.py:257-268) and the
// per-channel encrypt loop of pack_inputs (packing.py:119-123) with real
// RNS-CKKS.  The float64 FFT below performs exactly the operations of
// oracle/ckks_oracle.c fft() in the same order, with __dmul_rn/__dadd_rn
// (no FMA contraction), so encodings and decodings are bit-identical to the
// oracle.  The whole file is compiled with -fmad=false too.
#include "common.cuh"

namespace {

constexpr int EW = 256;

__device__ __forceinline__ uint32_t brvb(uint32_t x, int bits) { return __brev(x) >> (32 - bits); }

// one radix-2 DIT stage over `count` vectors of n complex values (SoA re/im)
// One radix-2 DIT butterfly with twiddle index tw: the operation order is part of
// the bit-exact contract (oracle/ckks_oracle.c oc_fft, -ffp-contract=off here
// via __dmul_rn / __dadd_rn), shared by every FFT kernel below.
__device__ __forceinline__ void fft_bfly(double &ur, double &ui, double &vr0, double &vi0, const double *w, size_t tw,
                                         int sign) {
    const double wr = w[2 * tw];
    const double wi = sign < 0 ? -w[2 * tw + 1] : w[2 * tw + 1];
    const double t1 = __dmul_rn(vr0, wr), t2 = __dmul_rn(vi0, wi);
    const double vr = __dsub_rn(t1, t2);
    const double t3 = __dmul_rn(vr0, wi), t4 = __dmul_rn(vi0, wr);
    const double vi = __dadd_rn(t3, t4);
    const double a = ur, b = ui;
    ur = __dadd_rn(a, vr);
    ui = __dadd_rn(b, vi);
    vr0 = __dsub_rn(a, vr);
    vi0 = __dsub_rn(b, vi);
}

// fft_bfly with the twiddle (sign already applied) passed in: identical operations
__device__ __forceinline__ void fft_bfly_w(double &ur, double &ui, double &vr0, double &vi0, const double wr,
                                           const double wi) {
    const double t1 = __dmul_rn(vr0, wr), t2 = __dmul_rn(vi0, wi);
    const double vr = __dsub_rn(t1, t2);
    const double t3 = __dmul_rn(vr0, wi), t4 = __dmul_rn(vi0, wr);
    const double vi = __dadd_rn(t3, t4);
    const double a = ur, b = ui;
    ur = __dadd_rn(a, vr);
    ui = __dadd_rn(b, vi);
    vr0 = __dsub_rn(a, vr);
    vi0 = __dsub_rn(b, vi);
}

__global__ void k_fft_stage(double *re, double *im, size_t count, int logn, int len, int sign, const double *w) {
    size_t n = (size_t)1 << logn, halfn = n >> 1, tot = count * halfn;
    int half = len >> 1;
    size_t step = n / len;
    for (size_t b = blockIdx.x * (size_t)blockDim.x + threadIdx.x; b < tot; b += (size_t)gridDim.x * blockDim.x) {
        size_t v = b / halfn, r = b % halfn;
        size_t s = (r / half) * len, k = r % half;
        double *R = re + v * n, *I = im + v * n;
        fft_bfly(R[s + k], I[s + k], R[s + k + half], I[s + k + half], w, k * step, sign);
    }
}

// Stages len = 2 .. 2^B of every aligned 2^B-element chunk in shared memory
// (one CTA per chunk): the same butterflies as k_fft_stage, one HBM pass.
constexpr int FFT_B = 11, FFT_TPB = 256;
// gvals != nullptr: the chunk's inputs are GATHERED from the slot values (the encoder's
// scatter V[brv(pos[i])] = vals[i] read backwards through the inverse permutation; zero
// imaginary parts and zero padding beyond nvals) instead of read from re / im
__global__ void __launch_bounds__(FFT_TPB) k_fft_chunk(double *re, double *im, int logn, int B, int sign,
                                                       const double *w, const double *gvals = nullptr,
                                                       int nvals = 0, const int32_t *ginv = nullptr) {
    __shared__ double sr[1 << FFT_B], si[1 << FFT_B];
    // the chunk stages only use twiddles w[k (n >> lg)], lg <= B: the 2^(B-1) entries of stride
    // n >> B, staged once per CTA (sign applied) instead of two global loads per butterfly
    __shared__ double swr[1 << (FFT_B - 1)], swi[1 << (FFT_B - 1)];
    const size_t n = (size_t)1 << logn, csz = (size_t)1 << B;
    const size_t base = (size_t)blockIdx.x * csz;  // chunks of consecutive polynomials tile the batch
    const size_t wst = n >> B;
    for (int i = threadIdx.x; i < (int)(csz >> 1); i += FFT_TPB) {
        swr[i] = w[2 * (i * wst)];
        swi[i] = sign < 0 ? -w[2 * (i * wst) + 1] : w[2 * (i * wst) + 1];
    }
    if (gvals) {
        const size_t v = base >> logn, t0 = base & (n - 1);
        for (int i = threadIdx.x; i < (int)csz; i += FFT_TPB) {
            const int sl = __ldg(ginv + t0 + i);
            sr[i] = sl < nvals ? __ldg(gvals + v * (size_t)nvals + sl) : 0.0;
            si[i] = 0.0;
        }
    } else {
        for (int i = threadIdx.x; i < (int)csz; i += FFT_TPB) {
            sr[i] = re[base + i];
            si[i] = im[base + i];
        }
    }
    __syncthreads();
    // stages in register groups of up to three (radix-8 passes): a thread owns the
    // 2^nst elements gbase + j 2^(lg0-1), closed under stages lg0 .. lg0+nst-1;
    // every butterfly is the one k_fft_stage computes, in the same stage order
    for (int lg0 = 1; lg0 <= B; lg0 += 3) {
        const int nst = B - lg0 + 1 < 3 ? B - lg0 + 1 : 3, m = 1 << nst, h = 1 << (lg0 - 1);
        for (int grp = threadIdx.x; grp < (int)(csz >> nst); grp += FFT_TPB) {
            const int gbase = (grp & (h - 1)) + ((grp >> (lg0 - 1)) << (lg0 - 1 + nst));
            double xr[8], xi[8];
#pragma unroll
            for (int j = 0; j < 8; j++)
                if (j < m) {
                    xr[j] = sr[gbase + j * h];
                    xi[j] = si[gbase + j * h];
                }
#pragma unroll
            for (int st = 0; st < 3; st++) {
                if (st >= nst) break;
                const int lg = lg0 + st;
                const size_t step = n >> lg;
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    if (j >= m || (j >> st) & 1) continue;
                    const int k = (gbase & (h - 1)) + (j & ((1 << st) - 1)) * h;  // index inside the half
                    const int ti = (int)(((size_t)k * step) / wst);           // = k 2^(B - lg)
                    fft_bfly_w(xr[j], xi[j], xr[j + (1 << st)], xi[j + (1 << st)], swr[ti], swi[ti]);
                }
            }
#pragma unroll
            for (int j = 0; j < 8; j++)
                if (j < m) {
                    sr[gbase + j * h] = xr[j];
                    si[gbase + j * h] = xi[j];
                }
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < (int)csz; i += FFT_TPB) {
        re[base + i] = sr[i];
        im[base + i] = si[i];
    }
}

// Stages len = 2^(B+1) .. n (R = logn - B <= 4 of them) in registers: thread
// (polynomial v, k0 < 2^B) owns the 2^R elements k0 + j 2^B, closed under those
// stages.
__global__ void k_fft_high(double *re, double *im, size_t count, int logn, int B, int sign, const double *w) {
    const size_t n = (size_t)1 << logn, grp = (size_t)1 << B, tot = count * grp;
    const int R = logn - B, m = 1 << R;
    for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < tot; g += (size_t)gridDim.x * blockDim.x) {
        const size_t v = g / grp, k0 = g % grp;
        double *Rp = re + v * n + k0, *Ip = im + v * n + k0;
        double xr[16], xi[16];
#pragma unroll
        for (int j = 0; j < 16; j++)
            if (j < m) {
                xr[j] = Rp[(size_t)j << B];
                xi[j] = Ip[(size_t)j << B];
            }
#pragma unroll
        for (int r = 0; r < 4; r++) {
            if (r >= R) break;
            const size_t step = n >> (B + r + 1);
#pragma unroll
            for (int j = 0; j < 16; j++) {
                if (j >= m || (j >> r) & 1) continue;
                const size_t k = k0 + ((size_t)(j & ((1 << r) - 1)) << B);  // index inside the half
                fft_bfly(xr[j], xi[j], xr[j + (1 << r)], xi[j + (1 << r)], w, k * step, sign);
            }
        }
#pragma unroll
        for (int j = 0; j < 16; j++)
            if (j < m) {
                Rp[(size_t)j << B] = xr[j];
                Ip[(size_t)j << B] = xi[j];
            }
    }
}

// encoder FFT of `count` slot vectors vals [count][nvals] gathered straight into the first
// pass (no zero fill, no scatter pass); N = 2^16 layout only (chunk + high stages)
static int run_fft_gather(he_ctx *c, const double *vals, int nvals, double *re, double *im, size_t count,
                          cudaStream_t s) {
    const int logn = c->logN - 1;
    const size_t n = (size_t)1 << logn;
    const int B = FFT_B;
    k_fft_chunk<<<(unsigned)(count * (n >> B)), FFT_TPB, 0, s>>>(re, im, logn, B, -1, c->d_fftw, vals, nvals,
                                                                c->d_slot_inv);
    HE_CHECK_LAUNCH();
    const size_t tot = count << B;
    unsigned grid = (unsigned)std::min<size_t>((tot + EW - 1) / EW, (size_t)148 * 32);
    k_fft_high<<<grid, EW, 0, s>>>(re, im, count, logn, B, -1, c->d_fftw);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

int run_fft(he_ctx *c, double *re, double *im, size_t count, int sign, cudaStream_t s) {
    const int logn = c->logN - 1;
    const size_t n = (size_t)1 << logn;
    const int B = logn < FFT_B ? logn : FFT_B;
    if (logn - B > 4) {  // (not reached for N <= 2^16) one launch per stage
        unsigned grid = (unsigned)std::min<size_t>((count * (n / 2) + EW - 1) / EW, (size_t)148 * 32);
        for (int len = 2; len <= (int)n; len <<= 1) {
            k_fft_stage<<<grid, EW, 0, s>>>(re, im, count, logn, len, sign, c->d_fftw);
            HE_CHECK_LAUNCH();
        }
        return HE_OK;
    }
    if (B >= 1) {
        k_fft_chunk<<<(unsigned)(count * (n >> B)), FFT_TPB, 0, s>>>(re, im, logn, B, sign, c->d_fftw);
        HE_CHECK_LAUNCH();
    }
    if (logn > B) {
        const size_t tot = count << B;
        unsigned grid = (unsigned)std::min<size_t>((tot + EW - 1) / EW, (size_t)148 * 32);
        k_fft_high<<<grid, EW, 0, s>>>(re, im, count, logn, B, sign, c->d_fftw);
        HE_CHECK_LAUNCH();
    }
    return HE_OK;
}

// V[brv(pos[i])] = vals[i] (the FFT's bit-reversal folded into the scatter)
__global__ void k_scatter_slots2(double *re, const double *vals, size_t count, int nvals, int n, const int32_t *slot_brv) {
    size_t tot = count * (size_t)nvals;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
        size_t v = i / nvals;
        int s = (int)(i % nvals);
        re[v * n + slot_brv[s]] = vals[i];
    }
}

// m_j, m_{j+n} = rint(Delta * conj-twisted, normalised FFT output) (+ CBD error)
// written as signed residues into c0 limbs of each output ct.
__global__ void k_encode_finish(uint64_t *const *out, const double *re, const double *im, size_t count, int logN,
                                int L, double scale, const double *twist, const ModConst *mc, uint64_t seed,
                                uint32_t ct_index0, int add_error) {
    size_t N = (size_t)1 << logN, n = N >> 1, tot = count * n;
    double inv_n = 1.0 / (double)n;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
        size_t v = i / n, j = i % n;
        double vr = __dmul_rn(re[i], inv_n), vi = __dmul_rn(im[i], inv_n);
        double zr = twist[2 * j], zi = twist[2 * j + 1];
        double ur = __dadd_rn(__dmul_rn(vr, zr), __dmul_rn(vi, zi));
        double ui = __dsub_rn(__dmul_rn(vi, zr), __dmul_rn(vr, zi));
        int64_t m0 = __double2ll_rn(__dmul_rn(ur, scale));
        int64_t m1 = __double2ll_rn(__dmul_rn(ui, scale));
        if (add_error) {
            m0 += sample_cbd(seed, DOM_ENC_E, ct_index0 + (uint32_t)v, (uint32_t)j);
            m1 += sample_cbd(seed, DOM_ENC_E, ct_index0 + (uint32_t)v, (uint32_t)(j + n));
        }
        uint64_t *O = out[v];
        for (int l = 0; l < L; l++) {
            uint64_t q = mc[l].q;
            O[(size_t)l * N + j] = smod64(m0, q);
            O[(size_t)l * N + j + n] = smod64(m1, q);
        }
    }
}

// c1 = a (uniform, NTT domain), c0 = NTT(m + e) - a s
__global__ void k_encrypt_finish(uint64_t *const *out, size_t count, int logN, int L, const uint64_t *sk,
                                 const ModConst *mc, uint64_t seed, uint32_t ct_index0) {
    size_t N = (size_t)1 << logN, per = (size_t)L * N, tot = count * per;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
        size_t v = i / per, r = i % per;
        int l = (int)(r >> logN);
        uint32_t k = (uint32_t)(r & (N - 1));
        const ModConst m = mc[l];
        uint64_t a = sample_uniform(seed, DOM_ENC_A, ct_index0 + (uint32_t)v, (uint32_t)l, k, m);
        uint64_t *O = out[v];
        O[per + r] = a;
        O[r] = sub_mod(O[r], mul_mod(a, sk[r], m), m.q);
    }
}

// x [count][D][N] = c0 + c1 s on the first D limbs
__global__ void k_dec_phase(uint64_t *x, const uint64_t *const *cts, size_t count, int ell, int D, int logN,
                            const uint64_t *sk, const ModConst *mc) {
    size_t N = (size_t)1 << logN, per = (size_t)D * N, tot = count * per;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
        size_t v = i / per, r = i % per;
        int l = (int)(r >> logN);
        const ModConst m = mc[l];
        const uint64_t *C = cts[v];
        x[i] = add_mod(C[r], mul_mod(C[(size_t)ell * N + r], sk[r], m), m.q);
    }
}

__device__ __forceinline__ double i128_to_double(__int128 v) {
    const __int128 lim = (__int128)1 << 62;
    if (v >= -lim && v < lim) return __ll2double_rn((long long)v);
    long long hi = (long long)(v >> 64);
    unsigned long long lo = (unsigned long long)v;
    return __dadd_rn(__dmul_rn(__ll2double_rn(hi), 18446744073709551616.0), __ull2double_rn(lo));
}

// CRT of D in {1,2} limbs -> centered integer -> double
__global__ void k_crt(double *out, const uint64_t *x, size_t count, int D, int logN, uint64_t q0, uint64_t q1,
                      uint64_t q0inv_mod_q1) {
    size_t N = (size_t)1 << logN, tot = count * N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
        size_t v = i >> logN, k = i & (N - 1);
        const uint64_t *X = x + v * D * N;
        __int128 val;
        if (D == 1) {
            uint64_t r = X[k];
            val = r > (q0 - 1) / 2 ? (__int128)r - (__int128)q0 : (__int128)r;
        } else {
            uint64_t x0 = X[k], x1 = X[N + k];
            uint64_t t = x1 >= x0 % q1 ? x1 - x0 % q1 : x1 + q1 - x0 % q1;
            uint64_t d = (uint64_t)(((unsigned __int128)t * q0inv_mod_q1) % q1);
            unsigned __int128 Q = (unsigned __int128)q0 * q1;
            unsigned __int128 r = (unsigned __int128)x0 + (unsigned __int128)q0 * d;
            val = r > (Q - 1) / 2 ? (__int128)r - (__int128)Q : (__int128)r;
        }
        out[i] = i128_to_double(val);
    }
}

// decode prologue: u = coeff/scale, v = u * zeta^j, scattered bit-reversed
__global__ void k_decode_twist(double *re, double *im, const double *coeffs, size_t count, int logN,
                               const double *scales, const double *twist) {
    size_t N = (size_t)1 << logN, n = N >> 1, tot = count * n;
    int logn = logN - 1;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
        size_t v = i / n, j = i % n;
        double sc = scales[v];
        double ur = __ddiv_rn(coeffs[v * N + j], sc), ui = __ddiv_rn(coeffs[v * N + j + n], sc);
        double zr = twist[2 * j], zi = twist[2 * j + 1];
        size_t d = v * n + brvb((uint32_t)j, logn);
        re[d] = __dsub_rn(__dmul_rn(ur, zr), __dmul_rn(ui, zi));
        im[d] = __dadd_rn(__dmul_rn(ur, zi), __dmul_rn(ui, zr));
    }
}

__global__ void k_gather_slots(double *out, const double *re, size_t count, int logn, const int32_t *slot_brv) {
    size_t n = (size_t)1 << logn, tot = count * n;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
        size_t v = i / n, s = i % n;
        out[i] = re[v * n + brvb((uint32_t)slot_brv[s], logn)];
    }
}

inline unsigned gridn(size_t n) { return (unsigned)std::min<size_t>((n + EW - 1) / EW, (size_t)148 * 32); }

struct Buf {
    void *p = nullptr;
    cudaStream_t s;
    explicit Buf(cudaStream_t st) : s(st) {}
    ~Buf() { he_scratch_free(p, s); }
};

// encode `count` vectors into c0-limb residues of `out` cts (L limbs each)
int encode_into(he_ctx *c, const double *vals, int count, int nvals, double scale, uint64_t *const *out_dev, int L,
                int add_error, uint32_t ct_index0, cudaStream_t s, const double *vals_im = nullptr) {
    size_t n = c->nslots;
    Buf b(s);
    HE_TRY(he_scratch_alloc(&b.p, (size_t)count * n * 16, s));
    double *re = (double *)b.p, *im = re + (size_t)count * n;
    HE_CHECK_CUDA(cudaMemsetAsync(re, 0, (size_t)count * n * 16, s));
    if (nvals > 0) {
        k_scatter_slots2<<<gridn((size_t)count * nvals), EW, 0, s>>>(re, vals, count, nvals, (int)n, c->d_slot_brv);
        HE_CHECK_LAUNCH();
        if (vals_im) {  // complex slots: the imaginary parts go through the same scatter
            k_scatter_slots2<<<gridn((size_t)count * nvals), EW, 0, s>>>(im, vals_im, count, nvals, (int)n,
                                                                         c->d_slot_brv);
            HE_CHECK_LAUNCH();
        }
    }
    HE_TRY(run_fft(c, re, im, count, -1, s));
    k_encode_finish<<<gridn((size_t)count * n), EW, 0, s>>>(out_dev, re, im, count, c->logN, L, scale, c->d_twist,
                                                           c->d_mc, c->prm.seed, ct_index0, add_error);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

int upload_map(const std::vector<uint8_t> &m, Buf &b, cudaStream_t s) {
    HE_TRY(he_scratch_alloc(&b.p, m.size(), s));
    HE_CHECK_CUDA(he_h2d(b.p, m.data(), m.size(), s));
    return HE_OK;
}

int decrypt_to_coeffs(he_ctx *c, const uint64_t *const *cts, int count, int ell, double *coeffs, cudaStream_t s) {
    int D = ell < 2 ? ell : 2;
    size_t N = c->N;
    Buf ptrs(s), x(s);
    HE_TRY(he_upload_ptrs((const void *const *)cts, count, (void ***)&ptrs.p, s));
    HE_TRY(he_scratch_alloc(&x.p, (size_t)count * D * N * 8, s));
    k_dec_phase<<<gridn((size_t)count * D * N), EW, 0, s>>>((uint64_t *)x.p, (const uint64_t *const *)ptrs.p, count,
                                                           ell, D, c->logN, c->d_sk, c->d_mc);
    HE_CHECK_LAUNCH();
    HE_TRY(he_ntt_inv(c, (uint64_t *)x.p, count * D, c->d_ident, D, s));
    uint64_t q0 = c->mod[0], q1 = D > 1 ? c->mod[1] : 1;
    uint64_t q0inv = 0;
    if (D > 1) {  // (q0 mod q1)^-1 mod q1 by Fermat
        unsigned __int128 r = 1, a = q0 % q1;
        uint64_t e = q1 - 2;
        while (e) {
            if (e & 1) r = r * a % q1;
            a = a * a % q1;
            e >>= 1;
        }
        q0inv = (uint64_t)r;
    }
    k_crt<<<gridn((size_t)count * N), EW, 0, s>>>(coeffs, (const uint64_t *)x.p, count, D, c->logN, q0, q1, q0inv);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

}  // namespace

extern "C" int he_encrypt(he_ctx *c, const double *vals, int count, int nvals, double scale, uint32_t ct_index0,
                          uint64_t *const *out, void *stream) {
    if (!c) {
        he_set_error("he_encrypt: bad arguments");
        return HE_EINVAL;
    }
    return he_encrypt_level(c, vals, count, nvals, scale, ct_index0, c->L, out, stream);
}

extern "C" int he_encrypt_level(he_ctx *c, const double *vals, int count, int nvals, double scale,
                                uint32_t ct_index0, int ell, uint64_t *const *out, void *stream) {
    if (!c || count < 0 || nvals < 0 || (nvals > 0 && !vals) || !(scale > 0) || ell < 1 || ell > c->L) {
        he_set_error("he_encrypt: bad arguments");
        return HE_EINVAL;
    }
    if (nvals > c->nslots) {
        he_set_error("%d values > %d slots", nvals, c->nslots);
        return HE_ELENGTH;
    }
    if (!count) return HE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    Buf ptrs(s), map(s);
    HE_TRY(he_upload_ptrs((const void *const *)out, count, (void ***)&ptrs.p, s));
    uint64_t *const *op = (uint64_t *const *)ptrs.p;
    if (c->logN == 16) {  // fused encode -> NTT -> encrypt (encrypt16.cu)
        const size_t n = c->nslots;
        Buf f(s);
        HE_TRY(he_scratch_alloc(&f.p, (size_t)count * n * 16, s));
        double *re = (double *)f.p, *im = re + (size_t)count * n;
        if (nvals > 0) {
            HE_TRY(run_fft_gather(c, vals, nvals, re, im, count, s));  // scatter folded into the first pass
        } else {
            HE_CHECK_CUDA(cudaMemsetAsync(re, 0, (size_t)count * n * 16, s));
            HE_TRY(run_fft(c, re, im, count, -1, s));
        }
        return he_encrypt16(c, re, im, count, scale, ct_index0, ell, op, s);
    }
    HE_TRY(encode_into(c, vals, count, nvals, scale, op, ell, 1, ct_index0, s));
    std::vector<uint8_t> m(2 * (size_t)ell, 0xFF);
    for (int l = 0; l < ell; l++) m[l] = (uint8_t)l;
    HE_TRY(upload_map(m, map, s));
    HE_TRY(he_ntt_fwd_ptrs(c, op, count, 2 * ell, (const uint8_t *)map.p, s));
    k_encrypt_finish<<<gridn((size_t)count * ell * c->N), EW, 0, s>>>(op, count, c->logN, ell, c->d_sk, c->d_mc,
                                                                       c->prm.seed, ct_index0);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

extern "C" int he_encode_plain(he_ctx *c, const double *vals, int nvals, double scale, int ell, uint64_t *pt_out,
                               void *stream) {
    if (!c || nvals < 0 || ell < 1 || ell > c->L || !pt_out || !(scale > 0)) {
        he_set_error("he_encode_plain: bad arguments");
        return HE_EINVAL;
    }
    if (nvals > c->nslots) {
        he_set_error("%d values > %d slots", nvals, c->nslots);
        return HE_ELENGTH;
    }
    cudaStream_t s = (cudaStream_t)stream;
    Buf ptrs(s);
    const uint64_t *h[1] = {pt_out};
    HE_TRY(he_upload_ptrs((const void *const *)h, 1, (void ***)&ptrs.p, s));
    HE_TRY(encode_into(c, vals, 1, nvals, scale, (uint64_t *const *)ptrs.p, ell, 0, 0, s));
    HE_TRY(he_ntt_fwd(c, pt_out, ell, c->d_ident, ell, s));
    return HE_OK;
}

// count full-width plaintexts at once: vals [count][nvals] (device), pt_out [count][ell][N]
extern "C" int he_encode_plain_batch(he_ctx *c, const double *vals, int count, int nvals, double scale, int ell,
                                     uint64_t *pt_out, void *stream) {
    if (!c || count < 0 || nvals < 0 || ell < 1 || ell > c->L || !pt_out || !(scale > 0)) {
        he_set_error("he_encode_plain_batch: bad arguments");
        return HE_EINVAL;
    }
    if (nvals > c->nslots) {
        he_set_error("%d values > %d slots", nvals, c->nslots);
        return HE_ELENGTH;
    }
    if (!count) return HE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<const uint64_t *> h(count);
    for (int i = 0; i < count; i++) h[i] = pt_out + (size_t)i * ell * c->N;
    Buf ptrs(s);
    HE_TRY(he_upload_ptrs((const void *const *)h.data(), count, (void ***)&ptrs.p, s));
    HE_TRY(encode_into(c, vals, count, nvals, scale, (uint64_t *const *)ptrs.p, ell, 0, 0, s));
    HE_TRY(he_ntt_fwd(c, pt_out, count * ell, c->d_ident, ell, s));
    return HE_OK;
}

// complex slot vectors (bootstrapping's CoeffToSlot / SlotToCoeff diagonals):
// slot i = re[i] + j im[i]; otherwise identical to he_encode_plain_batch
extern "C" int he_encode_plain_batch_c(he_ctx *c, const double *re, const double *im, int count, int nvals,
                                       double scale, int ell, uint64_t *pt_out, void *stream) {
    if (!c || count < 0 || nvals < 0 || ell < 1 || ell > c->L || !pt_out || !(scale > 0) || (nvals && (!re || !im))) {
        he_set_error("he_encode_plain_batch_c: bad arguments");
        return HE_EINVAL;
    }
    if (nvals > c->nslots) {
        he_set_error("%d values > %d slots", nvals, c->nslots);
        return HE_ELENGTH;
    }
    if (!count) return HE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<const uint64_t *> h(count);
    for (int i = 0; i < count; i++) h[i] = pt_out + (size_t)i * ell * c->N;
    Buf ptrs(s);
    HE_TRY(he_upload_ptrs((const void *const *)h.data(), count, (void ***)&ptrs.p, s));
    HE_TRY(encode_into(c, re, count, nvals, scale, (uint64_t *const *)ptrs.p, ell, 0, 0, s, im));
    HE_TRY(he_ntt_fwd(c, pt_out, count * ell, c->d_ident, ell, s));
    return HE_OK;
}

extern "C" int he_decrypt_coeffs(he_ctx *c, const uint64_t *const *cts, int count, int ell, double *out, void *stream) {
    if (!c || count < 0 || ell < 1 || ell > c->L || !out) {
        he_set_error("he_decrypt_coeffs: bad arguments");
        return HE_EINVAL;
    }
    if (!count) return HE_OK;
    return decrypt_to_coeffs(c, cts, count, ell, out, (cudaStream_t)stream);
}

extern "C" int he_decrypt(he_ctx *c, const uint64_t *const *cts, int count, int ell, const double *scales,
                          double *slots_out, void *stream) {
    if (!c || count < 0 || ell < 1 || ell > c->L || !slots_out || !scales) {
        he_set_error("he_decrypt: bad arguments");
        return HE_EINVAL;
    }
    if (!count) return HE_OK;
    cudaStream_t s = (cudaStream_t)stream;
    size_t N = c->N, n = c->nslots;
    Buf co(s), sc(s), fft(s);
    HE_TRY(he_scratch_alloc(&co.p, (size_t)count * N * 8, s));
    HE_TRY(decrypt_to_coeffs(c, cts, count, ell, (double *)co.p, s));
    HE_TRY(he_scratch_alloc(&sc.p, (size_t)count * 8, s));
    HE_CHECK_CUDA(he_h2d(sc.p, scales, (size_t)count * 8, s));
    HE_TRY(he_scratch_alloc(&fft.p, (size_t)count * n * 16, s));
    double *re = (double *)fft.p, *im = re + (size_t)count * n;
    k_decode_twist<<<gridn((size_t)count * n), EW, 0, s>>>(re, im, (const double *)co.p, count, c->logN,
                                                          (const double *)sc.p, c->d_twist);
    HE_CHECK_LAUNCH();
    HE_TRY(run_fft(c, re, im, count, +1, s));
    k_gather_slots<<<gridn((size_t)count * n), EW, 0, s>>>(slots_out, re, count, c->logN - 1, c->d_slot_brv);
    HE_CHECK_LAUNCH();
    return HE_OK;
}
