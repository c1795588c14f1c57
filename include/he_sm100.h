/*
 * he_sm100.h -- C-ABI of the B200 (sm_100a) RNS-CKKS engine, libhe_sm100.so.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `hebatch` (/root/reference/pkg/src/hebatch).  The reference's boundary is
 * the Python `VectorEngine` protocol (engine.py:164-177) whose only backend,
 * `SimulatorEngine` (engine.py:229-420), does float64 slot arithmetic with
 * numpy.  Each entry point below is what that protocol's operations bind to
 * in the B200 build; the Python host layer (paper_2604_16834_b200/engine.py,
 * `GpuEngine`) calls them through ctypes.  The reference interface each one
 * replaces is cited beside it.
 *
 * Conventions
 *   - Every function returns 0 on success or a negative HE_E* code; the
 *     message for the last failure on the calling thread is he_last_error().
 *     Validation happens before any device work is enqueued (the reference
 *     raises before touching counters: engine.py:280-283, :300-303).
 *   - A ciphertext is ONE device allocation laid out uint64 [n_comp][ell][N]
 *     (n_comp = 2, or 3 after a tensor product), NTT domain, bit-reversed
 *     evaluation order, every residue canonical in [0, q_i).  Limb i < ell
 *     is modulo Q-prime i.
 *   - Batched calls take HOST arrays of `count` device pointers (plain
 *     uint64_t addresses); work is enqueued on `stream` (a cudaStream_t, NULL
 *     = legacy default stream) and is asynchronous unless stated.
 *   - No torch types cross this boundary.
 */
#ifndef HE_SM100_H
#define HE_SM100_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HE_ABI_VERSION 2

enum {
    HE_OK = 0,
    HE_EINVAL = -1,         /* bad argument (ShapeMismatch / ValueError)       */
    HE_ECUDA = -2,          /* CUDA runtime failure                            */
    HE_ENOKEY = -3,         /* MissingRotationKey (errors.py:12-17)            */
    HE_ELEVEL = -4,         /* LevelExhausted (errors.py:24-25)                */
    HE_ENOMEM = -5,         /* device allocation failed                        */
    HE_ECONTEXT = -6,       /* ContextMismatch (errors.py:20-21)               */
    HE_ELENGTH = -7,        /* LengthExceedsSlots (errors.py:8-9)              */
};

/* Parameter set.  Replaces EngineContext (engine.py:36-63): the reference's
 * inert first_modulus_bits / rescale_bits / key_switch_digits become the
 * live q_bits[0] / q_bits[1..] / alpha.  Same layout as oracle/ckks_oracle.h. */
typedef struct {
    int32_t log_n;
    int32_t n_q;          /* L  = max_level + 1 Q-primes                  */
    int32_t n_p;          /* K  special primes                             */
    int32_t alpha;        /* limbs per key-switch digit, dnum=ceil(L/alpha) */
    int32_t q_bits[48];
    int32_t p_bits[16];
    uint64_t seed;        /* Philox4x32-10 key for every random stream     */
    double scale;         /* default encoding scale Delta                  */
    int32_t sk_hamming;   /* 0: dense ternary secret; h > 0: sparse secret  */
                          /* with expected Hamming weight h (bootstrapping) */
    int32_t reserved;
} he_params;

typedef struct he_ctx he_ctx;

const char *he_last_error(void);
int he_abi_version(void);

/* context: moduli, twiddle tables, BConv tables; secret key sampled from
 * params.seed and kept on the device.  Replaces SimulatorEngine.__init__
 * (engine.py:237-243). */
int he_ctx_create(const he_params *p, int device, he_ctx **out);
int he_ctx_destroy(he_ctx *ctx);
int he_ctx_moduli(const he_ctx *ctx, uint64_t *moduli /* L+K */, uint64_t *psi /* L+K */);

/* keys.  galois_elt 0 = relinearisation key (s^2); 2 and 4 = the power keys
 * s^3, s^4 of 5-component relinearisation (he_relin_rescale_n); odd values =
 * the key for X -> X^galois_elt.  Replaces register_rotation_keys / unload_rotation_keys
 * (engine.py:343-354; RotationKeySet engine.py:93-136). */
int he_gen_switch_key(he_ctx *ctx, uint32_t galois_elt, void *stream);
int he_drop_switch_key(he_ctx *ctx, uint32_t galois_elt);
int he_has_switch_key(const he_ctx *ctx, uint32_t galois_elt);
/* copies (canonical form) for parity tests: sk [L+K][N]; key [dnum][2][L+K][N] */
int he_export_secret_key(he_ctx *ctx, uint64_t *dev_out, void *stream);
int he_export_switch_key(he_ctx *ctx, uint32_t galois_elt, uint64_t *dev_out, void *stream);
/* install a key received over the wire (canonical residues, he_export_switch_key's
 * layout; residues >= q are rejected with HE_EINVAL).  The server side of the
 * client/server threat model evaluates with imported keys and
 * never holds the client's secret key.  Replaces an existing key of that code. */
int he_import_switch_key(he_ctx *ctx, uint32_t galois_elt, const uint64_t *dev_in, void *stream);

/* batched NTT / INTT over data [batch][ell][N]; limb i uses Q-prime i. */
int he_ntt(he_ctx *ctx, uint64_t *data, int batch, int ell, int inverse, void *stream);

/* encode + encrypt.  vals: device float64 [count][nvals] (zero-padded to
 * n = N/2 slots); ct k gets randomness index ct_index0 + k.  Output cts are
 * at the top level (ell = L).  Replaces encrypt (engine.py:257-264) and the
 * per-channel loop of pack_inputs (packing.py:119-123). */
int he_encrypt(he_ctx *ctx, const double *vals, int count, int nvals, double scale,
               uint32_t ct_index0, uint64_t *const *out, void *stream);
/* the same at ell <= L limbs (out: [2][ell][N] each): a ciphertext encrypted
 * directly at a lower level, equal limb for limb to the first ell limbs of the
 * top-level encryption (the randomness is drawn per limb).  Used when the
 * remaining circuit needs fewer limbs than the chain has. */
int he_encrypt_level(he_ctx *ctx, const double *vals, int count, int nvals, double scale,
                     uint32_t ct_index0, int ell, uint64_t *const *out, void *stream);
/* decrypt + decode to device float64 [count][N/2].  scales: host [count].
 * Replaces decrypt (engine.py:266-268) / unpack_outputs (packing.py:126-135). */
int he_decrypt(he_ctx *ctx, const uint64_t *const *cts, int count, int ell, const double *scales,
               double *slots_out, void *stream);
/* decrypt to integer coefficients (as float64 [count][N]) -- parity tests */
int he_decrypt_coeffs(he_ctx *ctx, const uint64_t *const *cts, int count, int ell, double *out,
                      void *stream);
/* encode a full-width plaintext at `scale` into NTT residues pt [ell][N]
 * (PlainVec encoding inside mult_plain / add_plain, engine.py:291-304). */
int he_encode_plain(he_ctx *ctx, const double *vals, int nvals, double scale, int ell,
                    uint64_t *pt_out, void *stream);
/* he_encode_plain for `count` vectors at once: vals [count][nvals] (device),
 * pt_out [count][ell][N] (contiguous); one FFT and one NTT launch sequence. */
int he_encode_plain_batch(he_ctx *ctx, const double *vals, int count, int nvals, double scale, int ell,
                          uint64_t *pt_out, void *stream);

/* element-wise.  add/sub: engine.py:285-289.  add_const: add_plain with a
 * constant over the occupied span (engine.py:291-295, conv.py:160-166);
 * residues host [count][ell].  mul_const: scalar plaintext product
 * (mult_plain before its rescale, engine.py:297-304); residues [count][ell]. */
/* he_encode_plain_batch for complex slot vectors: slot i = re[i] + j im[i]
 * (device arrays [count][nvals]).  Used for the CoeffToSlot / SlotToCoeff
 * diagonals of bootstrapping (engine.bootstrap; the reference's bootstrap,
 * /root/reference/pkg/src/hebatch/engine.py:315-327, is level accounting only). */
int he_encode_plain_batch_c(he_ctx *ctx, const double *re, const double *im, int count, int nvals, double scale,
                            int ell, uint64_t *pt_out, void *stream);
/* ModRaise: read each 2-component ciphertext of `in` (ell_in limbs) at level 0
 * (limb q_0) and lift it centred to ell_out limbs (INTT, lift, NTT): the result
 * decrypts to m + q_0 I(X).  First step of engine.bootstrap. */
int he_mod_raise(he_ctx *ctx, const uint64_t *const *in, int ell_in, uint64_t *const *out, int count, int ell_out,
                 void *stream);

int he_add(he_ctx *ctx, const uint64_t *const *a, const uint64_t *const *b, uint64_t *const *out,
           int count, int ell, int n_comp, void *stream);
int he_sub(he_ctx *ctx, const uint64_t *const *a, const uint64_t *const *b, uint64_t *const *out,
           int count, int ell, int n_comp, void *stream);
int he_add_const(he_ctx *ctx, const uint64_t *const *in, uint64_t *const *out, int count, int ell,
                 int n_comp, const uint64_t *residues, void *stream);
int he_mul_const(he_ctx *ctx, const uint64_t *const *in, uint64_t *const *out, int count, int ell,
                 int n_comp, const uint64_t *residues, void *stream);
int he_mul_plain(he_ctx *ctx, const uint64_t *const *in, const uint64_t *pt, uint64_t *const *out,
                 int count, int ell, int n_comp, void *stream);
/* keep the first ell_out limbs of each component (level drop, no rescale) */
int he_drop_limbs(he_ctx *ctx, const uint64_t *const *in, uint64_t *const *out, int count, int ell_in,
                  int ell_out, int n_comp, void *stream);

/* ct x ct pieces.  tensor: (a0b0, a0b1+a1b0, a1b1) -> out [3][ell][N].
 * relin: [3][ell][N] -> [2][ell][N] with the galois_elt-0 key.
 * keyswitch: d [ell][N] -> (o0, o1) with key galois_elt (parity tests).
 * rescale: [n_comp][ell][N] -> [n_comp][ell-1][N], divide-and-round by q_{ell-1}.
 * mult_ct = tensor + relin + rescale (mult_ct, engine.py:306-313). */
int he_tensor(he_ctx *ctx, const uint64_t *const *a, const uint64_t *const *b, uint64_t *const *out,
              int count, int ell, void *stream);
int he_relin(he_ctx *ctx, const uint64_t *const *d3, uint64_t *const *out, int count, int ell,
             void *stream);
/* relin + `extra` rescales as ONE ModDown over P u {q_{ell-extra}..q_{ell-1}}:
 * [3][ell][N] -> [2][ell-extra][N], result ~= relin(d3) / prod dropped q (fast BConv)
 * (the activation's mult_ct + the deferred conv rescale, engine.py:306-313;
 * N = 2^16 only, HE_EINVAL otherwise; extra in [0, min(ell-1, 8)]). */
int he_relin_rescale(he_ctx *ctx, const uint64_t *const *d3, uint64_t *const *out, int count, int ell,
                     int extra, void *stream);
/* nc-component form (nc = 3 or 5): component k >= 2 is key-switched with the
 * s^k key (codes 0, 2, 4; he_gen_switch_key) and the inner products are summed
 * before the one joint ModDown: [nc][ell][N] -> [2][ell-extra][N].  Lets a
 * degree-2 activation's 3-component output feed the next linear layer
 * unrelinearised; the squares of that layer (5 components) are relinearised
 * once after the global sum (featuremajor.run_cnn). */
int he_relin_rescale_n(he_ctx *ctx, const uint64_t *const *d, uint64_t *const *out, int count, int ell,
                       int extra, int nc, void *stream);
int he_keyswitch(he_ctx *ctx, uint32_t galois_elt, const uint64_t *const *d, uint64_t *const *out0,
                 uint64_t *const *out1, int count, int ell, void *stream);
int he_rescale(he_ctx *ctx, const uint64_t *const *in, uint64_t *const *out, int count, int ell,
               int n_comp, void *stream);
int he_mult_ct(he_ctx *ctx, const uint64_t *const *a, const uint64_t *const *b, uint64_t *const *out,
               int count, int ell, void *stream);

/* rotation: X -> X^galois_elt on both components, then key switch of the
 * permuted c1 (rotate, engine.py:276-283; galois_elt = 5^k mod 2N). */
int he_automorphism(he_ctx *ctx, uint32_t galois_elt, const uint64_t *const *in, uint64_t *const *out,
                    int count, int ell, int n_comp, void *stream);
int he_rotate(he_ctx *ctx, uint32_t galois_elt, const uint64_t *const *in, uint64_t *const *out,
              int count, int ell, void *stream);
/* Hoisted rotations of `count` ciphertexts by R Galois elements gs[0..R-1]
 * (oracle oc_rotate_hoisted): the key switch runs on the UNROTATED c1 with the
 * hoisting key sigma_g^-1(key_g), c0 is added, then sigma_g moves both
 * components; N = 2^16 shares ONE ModUp (INTT + basis extension + NTT pass 1)
 * of c1 among the R rotations.  out: host array [R][count] of [2][ell][N]
 * outputs.  Decrypts like he_rotate (np.roll, engine.py:276-283); limbs follow
 * the hoisted contract.  Keys must be registered (HE_ENOKEY otherwise); the
 * hoisting keys are derived on first use (he_gen_hoist_key). */
int he_rotate_hoisted(he_ctx *ctx, const uint32_t *galois_elts, int R, const uint64_t *const *in,
                      uint64_t *const *out, int count, int ell, void *stream);
/* derive the hoisting key of galois element g from its switch key */
int he_gen_hoist_key(he_ctx *ctx, uint32_t galois_elt, void *stream);

/* feature-major linear layer (the batched form of conv_forward's k=1 path,
 * conv.py:109-173, and of feature-major conv / pool):
 *   out[o] = sum_{t in [row_ptr[o], row_ptr[o+1])} w[t] * in[col[t]]   mod q_i
 * w: signed int64 (|w| < 2^62) shared by every limb; row_ptr/col/w are host
 * arrays.  Output is NOT rescaled (call he_rescale; bias via he_add_const). */
int he_lincomb(he_ctx *ctx, const uint64_t *const *in, int n_in, uint64_t *const *out, int n_out,
               const int32_t *row_ptr, const int32_t *col, const int64_t *w, int ell, int n_comp,
               void *stream);

/* the batched channel-by-channel conv fold (conv_forward k=3, conv.py:137-156):
 *   out[o] = sum_{j < n_in} in[j] (.) pts[o * n_in + j]      (element-wise, mod q_i)
 * in: n_in 2-component ciphertexts (the tap-aligned inputs); pts: n_out * n_in
 * encoded plaintexts [ell][N] (NTT domain); out: n_out 2-component ciphertexts.
 * Exact 128-bit accumulation, one reduction per value; NOT rescaled (call
 * he_rescale once per output).  n_in <= 1024; primes above 2^52 bound n_in by
 * n_in q^2 < 2^128. */
int he_lincomb_plain(he_ctx *ctx, const uint64_t *const *in, int n_in, const uint64_t *const *pts,
                     uint64_t *const *out, int n_out, int ell, void *stream);

/* grouped form of he_lincomb for feature-major convolutions: every group g
 * (an output pixel) shares one input gather and feeds M outputs:
 *   out[out_base[g] + m*out_stride] = sum_{t in group g} weights[m*T + tap[t]] * in[col[t]]
 * for m < M (M <= 32), mod q_i.  term_ptr [n_groups+1], col/tap [nnz],
 * out_base [n_groups], weights [M][T] signed int64; all host arrays.
 * residues: [M][ell] constant added to component 0 of channel m, or NULL.
 * Not rescaled.  Same semantics as expanding the groups into he_lincomb
 * (+ he_add_const). */
int he_lincomb_grouped(he_ctx *ctx, const uint64_t *const *in, int n_in, uint64_t *const *out, int n_out,
                       int n_groups, const int32_t *term_ptr, const int32_t *term_col, const int32_t *term_tap,
                       const int32_t *out_base, int out_stride, int M, int T, const int64_t *weights,
                       const uint64_t *residues, int ell, int n_comp, void *stream);

/* tensor-core form of he_lincomb_grouped for convolutions: every group has
 * exactly T tap slots, gcol [n_groups][T] = input index or -1 (zero tap):
 *   out[out_base[g] + m*out_stride] = sum_t weights[m][t] * in[gcol[g][t]] mod q_i
 * (+ residues[m][i] on component 0).  Exact int8 digit decomposition on
 * mma.sync u8 x s8 -> s32; needs |weights| < 2^31 and ceil(M*E/8) <= 12
 * (E = signed byte digits of the largest weight), else HE_EINVAL. */
int he_conv_mma(he_ctx *ctx, const uint64_t *const *in, int n_in, uint64_t *const *out, int n_out, int n_groups,
                const int32_t *gcol, const int32_t *out_base, int out_stride, int M, int T, const int64_t *weights,
                const uint64_t *residues, int ell, int n_comp, void *stream);

/* lazy degree-2 activation fused with a pooling / GAP sum (feature-major):
 *   out[o] = sum_{t in [row_ptr[o], row_ptr[o+1])} in[col[t]] (x) in[col[t]]  (+ residues[o] on c0)
 * (x) = tensor product without relinearisation: inputs [2][ell][N], outputs
 * [3][ell][N], no rescale.  residues: host [n_out][ell] or NULL.  Identical to
 * he_tensor + he_add_const per input followed by a unit-weight he_lincomb. */
int he_square_sum(he_ctx *ctx, const uint64_t *const *in, int n_in, uint64_t *const *out, int n_out,
                  const int32_t *row_ptr, const int32_t *col, const uint64_t *residues, int ell, void *stream);

/* conv -> lazy square -> window sum in ONE kernel (the conv map is never
 * written): 3x3 / pad-1 conv of p channels over H x W (inputs in[i*H*W +
 * y*W + x], [2][ell][N]) with weights [M][9p] (tap k = i*9 + (dy+1)*3 +
 * (dx+1)) and bias[m][i] on component 0, for conv output rows [y0, y1); then
 * per pixel the tensor square (y0^2, 2 y0 y1, y1^2); then
 *   pool = 1: out[m*nwin + (y/2 - y0/2)*(W/2) + x/2] = 2x2-window sums
 *   pool = 0: out[m] = sum over all pixels of the rows
 * plus cst[i] on component 0 of every output ([3][ell][N]).  Equals
 * he_conv_mma + he_square_sum bit for bit.  Bounds (else HE_EINVAL): 9p <= 160,
 * M <= 32, |weights| < 2^23, every prime >= 2^36.  bias / cst may be NULL. */
int he_conv_square_sum(he_ctx *ctx, const uint64_t *const *in, int p, int H, int W, uint64_t *const *out, int M,
                       int pool, int y0, int y1, const int64_t *weights, const uint64_t *bias,
                       const uint64_t *cst, int ell, void *stream);
/* the same with nci = 2 or 3 input components: 3-component inputs (the
 * unrelinearised squares of the previous block) give 5-component outputs
 * (y0^2, 2 y0 y1, 2 y0 y2 + y1^2, 2 y1 y2, y2^2) summed, relinearised later
 * by he_relin_rescale_n; needs even W (pixel pairs share a tensor-core tile). */
int he_conv_square_sum_n(he_ctx *ctx, const uint64_t *const *in, int nci, int p, int H, int W,
                         uint64_t *const *out, int M, int pool, int y0, int y1, const int64_t *weights,
                         const uint64_t *bias, const uint64_t *cst, int ell, void *stream);

/* block until all work on `stream` is done; returns HE_ECUDA on async error */
int he_sync(void *stream);
/* number of kernels this library has launched in the process (bench evidence) */
unsigned long long he_launch_count(void);
/* integer-pipe peak on `device`: ops_per_s[0] = 32-bit IMAD/s,
 * ops_per_s[1] = 64x64->128 multiply-accumulates/s (roofline denominators) */
int he_microbench_intpipe(int device, double *ops_per_s);
/* FP64 modular products per second (the a*w mod q form of the < 2^42 prime
 * datapath, ntt_core.cuh fmulmod): the key switch's second roofline peak. */
int he_microbench_fp64(int device, double *modmul_per_s);
/* int8 multiply-accumulates per second through mma.sync.m16n8k32.u8.s8 (the
 * fused conv's tensor-core instruction): the conv kernel's tensor roofline. */
int he_microbench_imma(int device, double *mac_per_s);
/* tcgen05.mma kind::i8 (u8 x s8 -> s32, M = 128, accumulators in TMEM): the
 * Blackwell tensor-core path of the fused conv kernels (csrc/convtc.cu).
 * he_tc5_selftest writes D = A B (128 x n int32, row-major) of a fixed
 * deterministic A (128 x 64 u8) and B (n x 64 s8) to the DEVICE buffer d_out;
 * layout 0/1 selects the shared-memory operand layout exercised.
 * he_microbench_tc5: rates[0] = int8 MAC/s over all SMs of back-to-back
 * M=128 x N=n x K=32 MMAs from shared memory, rates[1] = cycles per MMA. */
int he_tc5_selftest(int device, int n, int layout, int32_t *d_out);
int he_microbench_tc5(int device, int n, double *rates);
/* the same with the A operand's 8-row groups a_sbo bytes apart and its K chunks
 * a_lbo bytes apart (pixel-strided conv rings) */
int he_microbench_tc5_strided(int device, int n, int a_sbo, int a_lbo, double *rates);
/* the same with the MMAs rotating over ndst disjoint TMEM accumulators (independent chains) */
int he_microbench_tc5_indep(int device, int n, int ndst, double *rates);
/* TMEM read throughput: rates[0] = bytes per cycle per SM with `warps` warps loading
 * 32x32b.x{cols} (cols 4, 8, 16), rates[1] = cycles */
int he_microbench_tmem_ld(int device, int warps, int cols, double *rates);
/* The fused conv + square + pool / global-sum layer on the 5th-generation
 * tensor cores (tcgen05.mma kind::i8, TMEM accumulators, warp-specialised
 * producer / MMA / epilogue; csrc/convtc.cu).  Same arguments and results as
 * he_conv_square_sum_n; returns HE_EINVAL without enqueuing work when the
 * shape is not covered (primes outside [2^36, 2^40), W not a multiple of 16,
 * ...).  he_conv_square_sum_n routes every covered shape here unless
 * he_set_conv_tc(0) was called (returns the previous setting). */
int he_conv_square_sum_tc(he_ctx *ctx, const uint64_t *const *in, int nci, int p, int H, int W,
                          uint64_t *const *out, int M, int pool, int y0, int y1, const int64_t *weights,
                          const uint64_t *bias, const uint64_t *cst, int ell, void *stream);
int he_set_conv_tc(int on);
/* diagnostics: per-role cycle counters of the tcgen05 conv kernels.  on != 0
 * enables and zeroes them; on == 0 writes out[7] = summed cycles (producer
 * wait-empty, producer total, MMA wait-full, MMA wait-dempty, MMA total,
 * epilogue wait-dfull, epilogue total; one sampled thread per role per CTA). */
int he_convtc_profile(int on, double *out);
/* Planar carry between the two fused convs of the config-3 plan: C <= 16
 * channels x H x W of 3-component ciphertexts on ell limbs of < 2^40 primes,
 * laid out [limb][N/8 coefficient chunks][y][x][component][byte plane 0..4]
 * [8 coefficients][16 channels] (one byte per residue byte): the conv2 kernel's
 * shared-memory ring layout, so one image row is one contiguous bulk copy, and
 * 5 bytes per residue instead of 8.  he_conv_square_sum_pl = he_conv_square_sum_tc
 * with the inputs read from pl_in (conv2 shape: p = 16, W = 16, GAP) or the
 * pooled outputs written to pl_out (conv1 shape, M = 16) instead of the
 * pointer lists.  he_planar_pack / he_planar_unpack convert C*H*W ciphertexts
 * (channel-major) to / from the layout (pl holds ell * N/8 * H * W * 1920 bytes). */
int he_conv_square_sum_pl(he_ctx *ctx, const uint64_t *const *in, int nci, int p, int H, int W,
                          uint64_t *const *out, int M, int pool, int y0, int y1, const int64_t *weights,
                          const uint64_t *bias, const uint64_t *cst, int ell, const void *pl_in, void *pl_out,
                          void *stream);
int he_planar_pack(he_ctx *ctx, const uint64_t *const *in, int C, int H, int W, int ell, void *pl, void *stream);
int he_planar_unpack(he_ctx *ctx, const void *pl, int C, int H, int W, int ell, uint64_t *const *out,
                     void *stream);

#ifdef __cplusplus
}
#endif
#endif
