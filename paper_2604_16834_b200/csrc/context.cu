#include <algorithm>
// context.cu -- parameter generation, device tables, keys, scratch memory.
//
// Replaces the reference's EngineContext + SimulatorEngine construction
// (engine.py:36-63, :237-243) and RotationKeySet's key material
// (engine.py:93-136, :343-360).  Prime generation, psi selection, Philox
// streams and key layout follow DESIGN.md section 2; oracle/ckks_oracle.c is
// an independent restatement of the same contract.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include "common.cuh"

typedef unsigned __int128 hu128;

static thread_local char g_err[512];

void he_set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}
extern "C" const char *he_last_error(void) { return g_err; }

#include <atomic>
#include <deque>
static std::atomic<unsigned long long> g_launches{0};
void he_count_launch(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }
extern "C" unsigned long long he_launch_count(void) { return g_launches.load(); }
extern "C" int he_abi_version(void) { return HE_ABI_VERSION; }

// ---------------------------------------------------------------- host modular helpers
static uint64_t h_mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)((hu128)a * b % q); }
static uint64_t h_pow(uint64_t a, uint64_t e, uint64_t q) {
    uint64_t r = 1 % q;
    a %= q;
    while (e) {
        if (e & 1) r = h_mulmod(r, a, q);
        a = h_mulmod(a, a, q);
        e >>= 1;
    }
    return r;
}
static uint64_t h_inv(uint64_t a, uint64_t q) { return h_pow(a % q, q - 2, q); }
static uint64_t h_shoup(uint64_t w, uint64_t q) { return (uint64_t)(((hu128)w << 64) / q); }
uint64_t he_h_mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)((hu128)a * b % q); }
uint64_t he_h_shoup(uint64_t w, uint64_t q) { return h_shoup(w, q); }
uint64_t he_h_inv(uint64_t a, uint64_t q) { return h_inv(a, q); }
static uint64_t h_mont(uint64_t w, uint64_t q) { return (uint64_t)(((hu128)(w % q) << 64) % q); }
static bool h_is_prime(uint64_t n) {
    static const uint64_t B[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return false;
    for (uint64_t p : B) {
        if (n == p) return true;
        if (n % p == 0) return false;
    }
    uint64_t d = n - 1;
    int s = 0;
    while (!(d & 1)) d >>= 1, s++;
    for (uint64_t a : B) {
        uint64_t x = h_pow(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int r = 1; r < s && comp; r++) {
            x = h_mulmod(x, x, n);
            if (x == n - 1) comp = false;
        }
        if (comp) return false;
    }
    return true;
}
static uint32_t h_brv(uint32_t x, int bits) {
    uint32_t r = 0;
    for (int i = 0; i < bits; i++) r = (r << 1) | ((x >> i) & 1);
    return r;
}

// ---------------------------------------------------------------- pinned staging ring
// Every small host->device upload (pointer tables, job lists, weights) goes
// through one process-wide pinned ring: the bytes are copied into the ring at
// call time and the DMA is queued on the stream, so the host never waits for
// the GPU to drain (a pageable cudaMemcpyAsync stages synchronously in stream
// order).  A region is reused only after the event recorded behind its copy
// has completed; ring allocation is sequential, so the regions to retire are
// always at the front of the FIFO.
namespace {
struct Staging {
    std::mutex mu;
    char *buf = nullptr;
    size_t cap = 0, head = 0;
    bool tried = false;
    struct Ent {
        size_t lo, hi;
        cudaEvent_t ev;
    };
    std::deque<Ent> fifo;
    std::vector<cudaEvent_t> spare;
};
Staging g_stage;

// The ring is mapped into the device address space and the upload is a small
// kernel reading it over PCIe (zero-copy), NOT a copy-engine DMA: a large
// host->device DMA on another stream (bench.py's e2e images, 805 MB) would
// otherwise hold the H2D copy engine for ~15 ms and every small upload queued
// behind it -- and the kernels that wait for those uploads -- would stall.
__global__ void k_stage_copy(uint8_t *__restrict__ dst, const uint8_t *__restrict__ src, size_t bytes) {
    const size_t n16 = ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0) ? bytes / 16 : 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
        ((uint4 *)dst)[i] = ((const uint4 *)src)[i];
    for (size_t i = n16 * 16 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < bytes;
         i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}
}  // namespace

cudaError_t he_h2d(void *dst, const void *src, size_t bytes, cudaStream_t s) {
    if (!bytes) return cudaSuccess;
    std::lock_guard<std::mutex> lk(g_stage.mu);
    if (!g_stage.tried) {
        g_stage.tried = true;
        if (cudaHostAlloc((void **)&g_stage.buf, (size_t)256 << 20, cudaHostAllocMapped) == cudaSuccess)
            g_stage.cap = (size_t)256 << 20;
        else
            g_stage.buf = nullptr;
    }
    if (!g_stage.buf || bytes > g_stage.cap / 4) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
    size_t lo = (g_stage.head + 15) & ~(size_t)15;
    if (lo + bytes > g_stage.cap) lo = 0;
    const size_t hi = lo + bytes;
    while (!g_stage.fifo.empty()) {  // retire completed copies; wait only on overlapping ones
        Staging::Ent &f = g_stage.fifo.front();
        const bool overlap = f.lo < hi && lo < f.hi;
        if (!overlap && cudaEventQuery(f.ev) != cudaSuccess) break;
        if (overlap) cudaEventSynchronize(f.ev);
        g_stage.spare.push_back(f.ev);
        g_stage.fifo.pop_front();
    }
    memcpy(g_stage.buf + lo, src, bytes);
    void *dsrc = nullptr;
    cudaError_t e = cudaHostGetDevicePointer(&dsrc, g_stage.buf + lo, 0);
    if (e != cudaSuccess) return e;
    const unsigned blocks = (unsigned)std::min<size_t>((bytes + 4095) / 4096, 64);
    k_stage_copy<<<blocks, 256, 0, s>>>((uint8_t *)dst, (const uint8_t *)dsrc, bytes);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    cudaEvent_t ev;
    if (g_stage.spare.empty()) {
        e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
    } else {
        ev = g_stage.spare.back();
        g_stage.spare.pop_back();
    }
    e = cudaEventRecord(ev, s);
    g_stage.fifo.push_back({lo, hi, ev});
    g_stage.head = hi;
    return e;
}

// ---------------------------------------------------------------- scratch / pointer upload
int he_scratch_alloc(void **p, size_t bytes, cudaStream_t s) {
    if (bytes == 0) bytes = 8;
    cudaError_t e = cudaMallocAsync(p, bytes, s);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();  // not sticky: clear it so the caller can free memory and retry
        he_set_error("cudaMallocAsync(%zu bytes): %s", bytes, cudaGetErrorString(e));
        return HE_ENOMEM;
    }
    return HE_OK;
}
void he_scratch_free(void *p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}
int he_upload_ptrs(const void *const *host_ptrs, int count, void ***dev_out, cudaStream_t s) {
    HE_TRY(he_scratch_alloc((void **)dev_out, sizeof(void *) * (size_t)(count > 0 ? count : 1), s));
    if (count > 0)
        HE_CHECK_CUDA(he_h2d(*dev_out, host_ptrs, sizeof(void *) * count, s));
    return HE_OK;
}

// ---------------------------------------------------------------- key kernels
// secret coefficient j (oracle sample_ternary): dense ternary, or for h > 0 nonzero
// with probability h / N (second draw below thr = floor(h 2^32 / N)), sign = low bit
__global__ void k_sk_fill(uint64_t *sk, const ModConst *mc, int N, int M, uint64_t seed, int h, uint32_t thr) {
    size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (idx >= (size_t)M * N) return;
    int m = (int)(idx / N), j = (int)(idx % N);
    uint32_t r[4];
    rnd4(seed, DOM_SK, 0, 0, (uint32_t)j >> 2, r);
    int64_t s;
    if (h <= 0) {
        s = (int64_t)(r[j & 3] % 3u) - 1;
    } else {
        uint32_t r2[4];
        rnd4(seed, DOM_SK, 1, 0, (uint32_t)j >> 2, r2);
        s = r2[j & 3] >= thr ? 0 : ((r[j & 3] & 1u) ? 1 : -1);
    }
    sk[idx] = smod64(s, mc[m].q);
}

__global__ void k_ksk_err(uint64_t *buf, const ModConst *mc, int N, int M, int dnum, uint32_t g, uint64_t seed) {
    size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (idx >= (size_t)dnum * M * N) return;
    int j = (int)(idx / ((size_t)M * N));
    int m = (int)((idx / N) % M), k = (int)(idx % N);
    int64_t e = sample_cbd(seed, DOM_KSK_E, g * 64u + (uint32_t)j, (uint32_t)k);
    buf[idx] = smod64(e, mc[m].q);
}

// sprime: [L][N] NTT-domain target secret (s^2 or sigma_g(s)) for Q limbs
__global__ void k_ksk_final(uint64_t *key, const uint64_t *err, const uint64_t *sk, const uint64_t *sprime,
                            const ModConst *mc, const uint64_t *pmodq, int N, int L, int K, int alpha, int dnum,
                            uint32_t g, uint64_t seed) {
    int M = L + K;
    size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (idx >= (size_t)dnum * M * N) return;
    int j = (int)(idx / ((size_t)M * N));
    int m = (int)((idx / N) % M), k = (int)(idx % N);
    const ModConst c = mc[m];
    uint64_t a = sample_uniform(seed, DOM_KSK_A, g * 64u + (uint32_t)j, (uint32_t)m, (uint32_t)k, c);
    uint64_t s = sk[(size_t)m * N + k];
    uint64_t b = sub_mod(err[idx], mul_mod(a, s, c), c.q);
    bool in_digit = m < L && m >= j * alpha && m < (j + 1) * alpha;
    if (in_digit) b = add_mod(b, mul_mod(pmodq[m], sprime[(size_t)m * N + k], c), c.q);
    // Montgomery form for the inner product (redc(x * kM) = x * k)
    size_t base = ((size_t)j * 2) * M * N + (size_t)m * N + k;
    uint64_t bM = redc(mulhi(b, c.r2), b * c.r2, c.q, c.qinv);
    uint64_t aM = redc(mulhi(a, c.r2), a * c.r2, c.q, c.qinv);
    key[base] = bM;
    key[base + (size_t)M * N] = aM;
}

// s^power (NTT domain, Q limbs): the relinearisation target s^2 and the power
// keys s^3, s^4 of 5-component relinearisation (oracle: oc_gen_switch_key, even g)
__global__ void k_sk_power(uint64_t *out, const uint64_t *sk, const ModConst *mc, int N, int L, int power) {
    size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (idx >= (size_t)L * N) return;
    int m = (int)(idx / N);
    uint64_t v = sk[idx];
    for (int e = 1; e < power; e++) v = mul_mod(v, sk[idx], mc[m]);
    out[idx] = v;
}

// X -> X^g in bit-reversed evaluation order: out[k] = in[brv((e*g mod 2N - 1)/2)], e = 2 brv(k) + 1
__device__ __forceinline__ uint32_t galois_src(uint32_t k, uint32_t g, int logN) {
    uint32_t e = 2u * (__brev(k) >> (32 - logN)) + 1u;
    uint32_t e2 = (uint32_t)(((uint64_t)e * g) & ((2ull << logN) - 1));
    return __brev((e2 - 1u) >> 1) >> (32 - logN);
}
__global__ void k_automorph(uint64_t *out, const uint64_t *in, size_t n_polys, int logN, uint32_t g) {
    size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    size_t N = (size_t)1 << logN;
    if (idx >= n_polys * N) return;
    size_t p = idx >> logN;
    uint32_t k = (uint32_t)(idx & (N - 1));
    out[idx] = in[p * N + galois_src(k, g, logN)];
}

__global__ void k_from_mont(uint64_t *out, const uint64_t *in, const ModConst *mc, int N, int M, size_t total) {
    size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (idx >= total) return;
    int m = (int)((idx / N) % M);
    out[idx] = redc(0, in[idx], mc[m].q, mc[m].qinv);
}

// ---------------------------------------------------------------- context
static int build_tables(he_ctx *c) {
    int N = c->N, M = c->L + c->K;
    uint64_t twoN = 2 * (uint64_t)N;
    // moduli: for each requested bit size, the largest unused prime q < 2^bits with q = 1 mod 2N
    for (int m = 0; m < M; m++) {
        int bits = m < c->L ? c->prm.q_bits[m] : c->prm.p_bits[m - c->L];
        if (bits < 20 || bits > 61) {
            he_set_error("prime size %d bits outside [20, 61]", bits);
            return HE_EINVAL;
        }
        uint64_t top = 1ull << bits;
        for (uint64_t k = 1;; k++) {
            uint64_t cand = top - k * twoN + 1;
            bool used = false;
            for (int u = 0; u < m; u++) used |= c->mod[u] == cand;
            if (!used && h_is_prime(cand)) {
                c->mod[m] = cand;
                break;
            }
        }
        uint64_t q = c->mod[m], e = (q - 1) / twoN;
        for (uint64_t g = 2;; g++) {
            uint64_t psi = h_pow(g, e, q);
            if (h_pow(psi, N, q) == q - 1) {
                c->psi[m] = psi;
                break;
            }
        }
    }
    // twiddles: per modulus [fwd|inv][N] pairs (psi^brv(i), Shoup) -- one 16-byte load each
    std::vector<uint64_t> tw((size_t)M * 4 * N);
    std::vector<ModConst> mc(M);
    for (int m = 0; m < M; m++) {
        uint64_t q = c->mod[m], psi = c->psi[m], ipsi = h_inv(psi, q);
        uint64_t *T = &tw[(size_t)m * 4 * N];
        uint64_t pw = 1, ipw = 1;
        for (int i = 0; i < N; i++) {
            uint32_t r = h_brv((uint32_t)i, c->logN);
            T[2 * r] = pw;
            T[2 * r + 1] = h_shoup(pw, q);
            T[2 * N + 2 * r] = ipw;
            T[2 * N + 2 * r + 1] = h_shoup(ipw, q);
            pw = h_mulmod(pw, psi, q);
            ipw = h_mulmod(ipw, ipsi, q);
        }
        ModConst &k = mc[m];
        memset(&k, 0, sizeof k);
        k.q = q;
        uint64_t inv = 1;  // Newton iteration for q^-1 mod 2^64
        for (int it = 0; it < 7; it++) inv *= 2 - q * inv;
        k.qinv = inv;
        k.r2 = (uint64_t)(((hu128)h_mont(1, q) << 64) % q);  // R^2 mod q
        k.ninv = h_inv((uint64_t)N % q, q);
        c->h_ninv.push_back(k.ninv);
        k.ninv_sh = h_shoup(k.ninv, q);
        k.ratio = UINT64_MAX / q;
        k.qd = (double)q;
        k.qid = 1.0 / (double)q;
    }
    HE_CHECK_CUDA(cudaMalloc(&c->d_tw, tw.size() * 8));
    HE_CHECK_CUDA(cudaMemcpy(c->d_tw, tw.data(), tw.size() * 8, cudaMemcpyHostToDevice));
    {   // the same twiddles as doubles (exact: every value < q < 2^61 < 2^53 only matters for q < 2^42)
        std::vector<double> twd((size_t)M * 2 * N);
        for (size_t i = 0; i < twd.size(); i++) twd[i] = (double)tw[2 * i];
        HE_CHECK_CUDA(cudaMalloc(&c->d_twd, twd.size() * 8));
        HE_CHECK_CUDA(cudaMemcpy(c->d_twd, twd.data(), twd.size() * 8, cudaMemcpyHostToDevice));
        // centred copy for the q < 2^50 FP64 NTT (ntt_core.cuh fphase_ct_c / fphase_gs_c)
        c->fp50 = true;
        for (int m = 0; m < M; m++) c->fp50 = c->fp50 && c->mod[m] < (1ull << 50);
        std::vector<double> twdc(twd.size());
        for (size_t i = 0; i < twd.size(); i++) {
            const uint64_t q = c->mod[i / (2 * (size_t)N)], w = tw[2 * i];
            twdc[i] = w > q / 2 ? -(double)(q - w) : (double)w;
        }
        HE_CHECK_CUDA(cudaMalloc(&c->d_twdc, twdc.size() * 8));
        HE_CHECK_CUDA(cudaMemcpy(c->d_twdc, twdc.data(), twdc.size() * 8, cudaMemcpyHostToDevice));
        std::vector<double> rinv(M);
        for (int m = 0; m < M; m++) {
            const uint64_t q = c->mod[m], R = (uint64_t)(((hu128)1 << 64) % q);
            rinv[m] = (double)h_inv(R, q);
        }
        HE_CHECK_CUDA(cudaMalloc(&c->d_rinvd, M * sizeof(double)));
        HE_CHECK_CUDA(cudaMemcpy(c->d_rinvd, rinv.data(), M * sizeof(double), cudaMemcpyHostToDevice));
    }
    HE_CHECK_CUDA(cudaMalloc(&c->d_mc, sizeof(ModConst) * M));
    HE_CHECK_CUDA(cudaMemcpy(c->d_mc, mc.data(), sizeof(ModConst) * M, cudaMemcpyHostToDevice));
    // rescale constants q_l^-1 mod q_i, and P constants
    std::vector<uint64_t> qlinv((size_t)c->L * c->L * 2, 0);
    for (int l = 1; l < c->L; l++)
        for (int i = 0; i < l; i++) {
            uint64_t v = h_inv(c->mod[l] % c->mod[i], c->mod[i]);
            qlinv[((size_t)l * c->L + i) * 2] = v;
            qlinv[((size_t)l * c->L + i) * 2 + 1] = h_shoup(v, c->mod[i]);
        }
    c->h_qlinv = qlinv;
    HE_CHECK_CUDA(cudaMalloc(&c->d_qlinv, qlinv.size() * 8));
    HE_CHECK_CUDA(cudaMemcpy(c->d_qlinv, qlinv.data(), qlinv.size() * 8, cudaMemcpyHostToDevice));
    c->h_pmodq.assign(c->L, 0);
    c->h_pinv.assign((size_t)c->L * 2, 0);
    for (int i = 0; i < c->L; i++) {
        uint64_t q = c->mod[i], p = 1 % q;
        for (int k = 0; k < c->K; k++) p = h_mulmod(p, c->mod[c->L + k] % q, q);
        c->h_pmodq[i] = p;
        uint64_t pi = c->K ? h_inv(p, q) : 1;
        c->h_pinv[2 * i] = pi;
        c->h_pinv[2 * i + 1] = h_shoup(pi, q);
    }
    HE_CHECK_CUDA(cudaMalloc(&c->d_pinv, c->h_pinv.size() * 8));
    HE_CHECK_CUDA(cudaMemcpy(c->d_pinv, c->h_pinv.data(), c->h_pinv.size() * 8, cudaMemcpyHostToDevice));
    // FFT tables for the canonical embedding (libm cos/sin: same values as the oracle)
    int n = c->nslots;
    std::vector<double> w(2 * (size_t)n), z(2 * (size_t)n);
    std::vector<int32_t> sb(n);
    const double PI = 3.14159265358979323846;
    for (int k = 0; k < n; k++) {
        w[2 * k] = cos(2.0 * PI * (double)k / (double)n);
        w[2 * k + 1] = sin(2.0 * PI * (double)k / (double)n);
        z[2 * k] = cos(PI * (double)k / (double)N);
        z[2 * k + 1] = sin(PI * (double)k / (double)N);
    }
    uint64_t g = 1;
    for (int i = 0; i < n; i++) {
        sb[i] = (int32_t)h_brv((uint32_t)((g - 1) / 4), c->logN - 1);
        g = (g * 5) % twoN;
    }
    HE_CHECK_CUDA(cudaMalloc(&c->d_fftw, w.size() * 8));
    HE_CHECK_CUDA(cudaMemcpy(c->d_fftw, w.data(), w.size() * 8, cudaMemcpyHostToDevice));
    HE_CHECK_CUDA(cudaMalloc(&c->d_twist, z.size() * 8));
    HE_CHECK_CUDA(cudaMemcpy(c->d_twist, z.data(), z.size() * 8, cudaMemcpyHostToDevice));
    HE_CHECK_CUDA(cudaMalloc(&c->d_slot_brv, sb.size() * 4));
    HE_CHECK_CUDA(cudaMemcpy(c->d_slot_brv, sb.data(), sb.size() * 4, cudaMemcpyHostToDevice));
    std::vector<int32_t> inv(n);
    for (int i = 0; i < n; i++) inv[sb[i]] = i;
    HE_CHECK_CUDA(cudaMalloc(&c->d_slot_inv, inv.size() * 4));
    HE_CHECK_CUDA(cudaMemcpy(c->d_slot_inv, inv.data(), inv.size() * 4, cudaMemcpyHostToDevice));
    uint8_t ident[HE_MAXM];
    for (int i = 0; i < HE_MAXM; i++) ident[i] = (uint8_t)i;
    HE_CHECK_CUDA(cudaMalloc(&c->d_ident, HE_MAXM));
    HE_CHECK_CUDA(cudaMemcpy(c->d_ident, ident, HE_MAXM, cudaMemcpyHostToDevice));
    return HE_OK;
}

extern "C" int he_ctx_create(const he_params *p, int device, he_ctx **out) {
    if (!p || !out) {
        he_set_error("he_ctx_create: null argument");
        return HE_EINVAL;
    }
    if (p->log_n < 3 || p->log_n > 16) {
        he_set_error("log_n=%d unsupported (N = 2^3 .. 2^16)", p->log_n);
        return HE_EINVAL;
    }
    if (p->n_q < 1 || p->n_q > 48 || p->n_p < 1 || p->n_p > 16 || p->n_q + p->n_p > HE_MAXM || p->alpha < 1 ||
        p->alpha > p->n_q || p->alpha > 8) {
        he_set_error("bad parameter counts: n_q=%d n_p=%d alpha=%d", p->n_q, p->n_p, p->alpha);
        return HE_EINVAL;
    }
    HE_CHECK_CUDA(cudaSetDevice(device));
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    he_ctx *c = new he_ctx();
    c->prm = *p;
    c->device = device;
    c->logN = p->log_n;
    c->N = 1 << p->log_n;
    c->L = p->n_q;
    c->K = p->n_p;
    c->alpha = p->alpha;
    c->dnum = (c->L + c->alpha - 1) / c->alpha;
    c->nslots = c->N / 2;
    c->mod.assign(c->L + c->K, 0);
    c->psi.assign(c->L + c->K, 0);
    int r = build_tables(c);
    if (r != HE_OK) {
        he_ctx_destroy(c);
        return r;
    }
    // secret key
    int M = c->L + c->K;
    size_t tot = (size_t)M * c->N;
    if (cudaMalloc(&c->d_sk, tot * 8) != cudaSuccess) {
        he_set_error("cudaMalloc secret key failed");
        he_ctx_destroy(c);
        return HE_ENOMEM;
    }
    {
        const uint64_t t = p->sk_hamming > 0 ? ((uint64_t)p->sk_hamming << 32) / (uint64_t)c->N : 0;
        const uint32_t thr = t > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)t;
        k_sk_fill<<<ceil_div(tot, 256), 256>>>(c->d_sk, c->d_mc, c->N, M, p->seed, p->sk_hamming, thr);
    }
    r = he_ntt_fwd(c, c->d_sk, M, c->d_ident, M, 0);
    if (r == HE_OK && cudaDeviceSynchronize() != cudaSuccess) {
        he_set_error("secret key generation failed: %s", cudaGetErrorString(cudaGetLastError()));
        r = HE_ECUDA;
    }
    if (r != HE_OK) {
        he_ctx_destroy(c);
        return r;
    }
    *out = c;
    return HE_OK;
}

static void free_table(BconvTable &t) {
    cudaFree(t.d);
    cudaFree(t.d_src_mod);
    cudaFree(t.d_dst_mod);
}

extern "C" int he_ctx_destroy(he_ctx *c) {
    if (!c) return HE_OK;
    cudaDeviceSynchronize();
    for (auto &kv : c->keys) cudaFree(kv.second);
    for (auto &kv : c->modup_tab) free_table(kv.second);
    for (auto &kv : c->moddown_tab) free_table(kv.second);
    cudaFree(c->d_mc);
    cudaFree(c->d_tw);
    cudaFree(c->d_twd);
    cudaFree(c->d_twdc);
    cudaFree(c->d_rinvd);
    cudaFree(c->d_sk);
    cudaFree(c->d_fftw);
    cudaFree(c->d_twist);
    cudaFree(c->d_slot_brv);
    cudaFree(c->d_slot_inv);
    cudaFree(c->d_ident);
    cudaFree(c->d_pinv);
    cudaFree(c->d_qlinv);
    delete c;
    return HE_OK;
}

extern "C" int he_ctx_moduli(const he_ctx *c, uint64_t *moduli, uint64_t *psi) {
    if (!c) return HE_EINVAL;
    for (int m = 0; m < c->L + c->K; m++) {
        if (moduli) moduli[m] = c->mod[m];
        if (psi) psi[m] = c->psi[m];
    }
    return HE_OK;
}

// ---------------------------------------------------------------- BConv tables
static int make_table(he_ctx *c, const std::vector<int> &src, const std::vector<int> &dst, BconvTable &t) {
    int ns = (int)src.size(), nd = (int)dst.size();
    std::vector<uint64_t> h((size_t)2 * ns + (size_t)ns * nd);
    for (int s = 0; s < ns; s++) {
        uint64_t qs = c->mod[src[s]], hh = 1 % qs;
        for (int u = 0; u < ns; u++)
            if (u != s) hh = h_mulmod(hh, c->mod[src[u]] % qs, qs);
        uint64_t inv = h_inv(hh, qs);
        h[s] = inv;
        h[ns + s] = h_shoup(inv, qs);
    }
    for (int d = 0; d < nd; d++) {
        uint64_t qt = c->mod[dst[d]];
        for (int s = 0; s < ns; s++) {
            uint64_t hh = 1 % qt;
            for (int u = 0; u < ns; u++)
                if (u != s) hh = h_mulmod(hh, c->mod[src[u]] % qt, qt);
            h[2 * ns + (size_t)d * ns + s] = h_mont(hh, qt);
        }
    }
    t.n_src = ns;
    t.n_dst = nd;
    t.h_qhinv.assign(h.begin(), h.begin() + ns);
    t.h_dst_mod = dst;
    HE_CHECK_CUDA(cudaMalloc(&t.d, h.size() * 8));
    HE_CHECK_CUDA(cudaMemcpy(t.d, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
    HE_CHECK_CUDA(cudaMalloc(&t.d_src_mod, 4 * ns));
    HE_CHECK_CUDA(cudaMemcpy(t.d_src_mod, src.data(), 4 * ns, cudaMemcpyHostToDevice));
    HE_CHECK_CUDA(cudaMalloc(&t.d_dst_mod, 4 * nd));
    HE_CHECK_CUDA(cudaMemcpy(t.d_dst_mod, dst.data(), 4 * nd, cudaMemcpyHostToDevice));
    return HE_OK;
}

int he_get_modup_table(he_ctx *c, int ell, int j, const BconvTable **out) {
    std::lock_guard<std::mutex> g(c->mu);
    uint64_t key = (uint64_t)ell * 64 + j;
    auto it = c->modup_tab.find(key);
    if (it == c->modup_tab.end()) {
        int s0 = j * c->alpha, s1 = std::min((j + 1) * c->alpha, ell);
        std::vector<int> src, dst;
        for (int s = s0; s < s1; s++) src.push_back(s);
        for (int t = 0; t < ell; t++)
            if (t < s0 || t >= s1) dst.push_back(t);
        for (int k = 0; k < c->K; k++) dst.push_back(c->L + k);
        BconvTable t;
        HE_TRY(make_table(c, src, dst, t));
        it = c->modup_tab.emplace(key, t).first;
    }
    *out = &it->second;
    return HE_OK;
}

int he_get_moddown_table(he_ctx *c, int ell, const BconvTable **out) { return he_get_moddown_table_x(c, ell, 0, out); }

// ModDown over S = {q_{ell-extra} .. q_{ell-1}} u P -> targets q_0 .. q_{ell-extra-1}
int he_get_moddown_table_x(he_ctx *c, int ell, int extra, const BconvTable **out) {
    std::lock_guard<std::mutex> g(c->mu);
    const int key = ell * 16 + extra;
    auto it = c->moddown_tab.find(key);
    if (it == c->moddown_tab.end()) {
        std::vector<int> src, dst;
        for (int s = ell - extra; s < ell; s++) src.push_back(s);
        for (int k = 0; k < c->K; k++) src.push_back(c->L + k);
        for (int t = 0; t < ell - extra; t++) dst.push_back(t);
        BconvTable t;
        HE_TRY(make_table(c, src, dst, t));
        it = c->moddown_tab.emplace(key, t).first;
    }
    *out = &it->second;
    return HE_OK;
}

// ---------------------------------------------------------------- keys
const uint64_t *he_get_key(he_ctx *c, uint32_t g) {
    std::lock_guard<std::mutex> lk(c->mu);
    auto it = c->keys.find(g);
    return it == c->keys.end() ? nullptr : it->second;
}

extern "C" int he_gen_switch_key(he_ctx *c, uint32_t g, void *stream) {
    if (!c) return HE_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    // g = 0: relinearisation key (s^2); even g = 2, 4: power keys s^(g/2+2); odd g: galois
    if (g % 2 == 0 ? g > 4 : g >= 2u * (uint32_t)c->N) {
        he_set_error("key code %u: galois elements are odd and < 2N, power keys are 0, 2, 4", g);
        return HE_EINVAL;
    }
    if (he_get_key(c, g)) return HE_OK;  // idempotent (RotationKeySet.register)
    int N = c->N, L = c->L, K = c->K, M = L + K;
    size_t per = (size_t)M * N, tot = (size_t)c->dnum * per;
    uint64_t *key = nullptr, *err = nullptr, *sp = nullptr, *pm = nullptr;
    if (cudaMalloc(&key, tot * 2 * 8) != cudaSuccess) {
        he_set_error("cudaMalloc switch key (%zu MB) failed", tot * 16 >> 20);
        return HE_ENOMEM;
    }
    HE_TRY(he_scratch_alloc((void **)&err, tot * 8, s));
    HE_TRY(he_scratch_alloc((void **)&sp, (size_t)L * N * 8, s));
    HE_TRY(he_scratch_alloc((void **)&pm, (size_t)L * 8, s));
    HE_CHECK_CUDA(he_h2d(pm, c->h_pmodq.data(), L * 8, s));
    if (g % 2 == 0)
        k_sk_power<<<ceil_div((size_t)L * N, 256), 256, 0, s>>>(sp, c->d_sk, c->d_mc, N, L, g == 0 ? 2 : (int)g / 2 + 2);
    else
        k_automorph<<<ceil_div((size_t)L * N, 256), 256, 0, s>>>(sp, c->d_sk, L, c->logN, g);
    k_ksk_err<<<ceil_div(tot, 256), 256, 0, s>>>(err, c->d_mc, N, M, c->dnum, g, c->prm.seed);
    HE_CHECK_LAUNCH();
    HE_TRY(he_ntt_fwd(c, err, c->dnum * M, c->d_ident, M, s));
    k_ksk_final<<<ceil_div(tot, 256), 256, 0, s>>>(key, err, c->d_sk, sp, c->d_mc, pm, N, L, K, c->alpha, c->dnum, g,
                                                   c->prm.seed);
    HE_CHECK_LAUNCH();
    he_scratch_free(err, s);
    he_scratch_free(sp, s);
    he_scratch_free(pm, s);
    HE_CHECK_CUDA(cudaStreamSynchronize(s));
    std::lock_guard<std::mutex> lk(c->mu);
    c->keys[g] = key;
    return HE_OK;
}

// Hoisting key of Galois element g (oracle oc_hoist_key): the switch key with
// every polynomial moved by sigma_{g^-1}; stored under HE_HOIST_CODE | g.
extern "C" int he_gen_hoist_key(he_ctx *c, uint32_t g, void *stream) {
    if (!c || g % 2 == 0 || g >= 2u * (uint32_t)c->N) {
        he_set_error("he_gen_hoist_key: %u is not a galois element", g);
        return HE_EINVAL;
    }
    if (he_get_key(c, HE_HOIST_CODE | g)) return HE_OK;
    const uint64_t *key = he_get_key(c, g);
    if (!key) {
        he_set_error("no rotation key for galois element %u", g);
        return HE_ENOKEY;
    }
    const uint64_t twoN = 2 * (uint64_t)c->N;
    uint32_t gi = 1;
    while (((uint64_t)gi * g) % twoN != 1) gi += 2;
    const size_t np = (size_t)c->dnum * 2 * (c->L + c->K);
    uint64_t *hk = nullptr;
    if (cudaMalloc(&hk, np * c->N * 8) != cudaSuccess) {
        he_set_error("cudaMalloc hoisting key failed");
        return HE_ENOMEM;
    }
    cudaStream_t s = (cudaStream_t)stream;
    k_automorph<<<ceil_div(np * c->N, 256), 256, 0, s>>>(hk, key, np, c->logN, gi);
    HE_CHECK_LAUNCH();
    HE_CHECK_CUDA(cudaStreamSynchronize(s));
    std::lock_guard<std::mutex> lk(c->mu);
    c->keys[HE_HOIST_CODE | g] = hk;
    return HE_OK;
}

extern "C" int he_drop_switch_key(he_ctx *c, uint32_t g) {
    if (!c) return HE_EINVAL;
    std::lock_guard<std::mutex> lk(c->mu);
    for (uint32_t code : {g, HE_HOIST_CODE | g}) {  // the key and its hoisting key
        auto it = c->keys.find(code);
        if (it != c->keys.end()) {
            cudaDeviceSynchronize();
            cudaFree(it->second);
            c->keys.erase(it);
        }
    }
    return HE_OK;
}

extern "C" int he_has_switch_key(const he_ctx *c, uint32_t g) {
    return c && c->keys.count(g) ? 1 : 0;
}

extern "C" int he_export_secret_key(he_ctx *c, uint64_t *dev_out, void *stream) {
    if (!c || !dev_out) return HE_EINVAL;
    HE_CHECK_CUDA(cudaMemcpyAsync(dev_out, c->d_sk, (size_t)(c->L + c->K) * c->N * 8, cudaMemcpyDeviceToDevice,
                                  (cudaStream_t)stream));
    return HE_OK;
}

extern "C" int he_export_switch_key(he_ctx *c, uint32_t g, uint64_t *dev_out, void *stream) {
    if (!c || !dev_out) return HE_EINVAL;
    const uint64_t *k = he_get_key(c, g);
    if (!k) {
        he_set_error("no switch key for galois element %u", g);
        return HE_ENOKEY;
    }
    size_t tot = (size_t)c->dnum * 2 * (c->L + c->K) * c->N;
    k_from_mont<<<ceil_div(tot, 256), 256, 0, (cudaStream_t)stream>>>(dev_out, k, c->d_mc, c->N, c->L + c->K, tot);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// canonical residues -> Montgomery form (x 2^64 mod q = redc(x r2)); flags any residue >= q
__global__ void k_to_mont(uint64_t *out, const uint64_t *in, const ModConst *mc, int N, int M, size_t total,
                          int *bad) {
    size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (idx >= total) return;
    const ModConst &c = mc[(idx / N) % M];
    const uint64_t x = in[idx];
    if (x >= c.q) atomicOr(bad, 1);
    out[idx] = redc(mulhi(x, c.r2), x * c.r2, c.q, c.qinv);
}

// Install an evaluation key received over the wire (canonical residues, layout of
// he_export_switch_key).  The server side of the threat model
// holds evaluation keys but never the secret key.
extern "C" int he_import_switch_key(he_ctx *c, uint32_t g, const uint64_t *dev_in, void *stream) {
    if (!c || !dev_in) return HE_EINVAL;
    if (g % 2 == 0 ? g > 4 : g >= 2u * (uint32_t)c->N) {
        he_set_error("key code %u: galois elements are odd and < 2N, power keys are 0, 2, 4", g);
        return HE_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const size_t tot = (size_t)c->dnum * 2 * (c->L + c->K) * c->N;
    uint64_t *key = nullptr;
    int *bad = nullptr, hbad = 0;
    if (cudaMalloc(&key, tot * 8) != cudaSuccess) {
        (void)cudaGetLastError();
        he_set_error("cudaMalloc switch key (%zu MB) failed", tot * 8 >> 20);
        return HE_ENOMEM;
    }
    HE_TRY(he_scratch_alloc((void **)&bad, sizeof(int), s));
    HE_CHECK_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
    k_to_mont<<<ceil_div(tot, 256), 256, 0, s>>>(key, dev_in, c->d_mc, c->N, c->L + c->K, tot, bad);
    HE_CHECK_LAUNCH();
    HE_CHECK_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    he_scratch_free(bad, s);
    HE_CHECK_CUDA(cudaStreamSynchronize(s));
    if (hbad) {
        cudaFree(key);
        he_set_error("imported key %u holds residues outside [0, q)", g);
        return HE_EINVAL;
    }
    he_drop_switch_key(c, g);  // replaces an existing key (and its hoisting key)
    std::lock_guard<std::mutex> lk(c->mu);
    c->keys[g] = key;
    return HE_OK;
}

extern "C" int he_sync(void *stream) {
    HE_CHECK_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    return HE_OK;
}
