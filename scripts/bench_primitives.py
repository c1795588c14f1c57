"""Config-2 primitive microbenchmark (BASELINE.json configs[1]).

N = 2^16, 24 x 50-bit Q limbs, 4 x 50-bit special primes (dnum 6), 256
ciphertexts of uniform residues.  Times forward / inverse NTT, the
relinearisation key switch (d2 := c1), rotation by +1 and +1024 and rescale
24 -> 23, each over all 256 ciphertexts, with CUDA events (warm-up first);
checks one ciphertext of each op bit-exactly against the CPU oracle; prints
one JSON line with per-op time, algorithmic GB/s and fraction of the
measured HBM peak, plus the measured integer-pipe peak.

usage: python scripts/bench_primitives.py [--cts 256] [--reps 5] [--no-oracle]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import torch

from paper_2604_16834_b200 import _lib, configs
from paper_2604_16834_b200.engine import GpuEngine

ap = argparse.ArgumentParser()
ap.add_argument("--cts", type=int, default=256)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--no-oracle", action="store_true")
args = ap.parse_args()

eng = GpuEngine(configs.context(2, seed=7))
L, N, B = eng.context.n_q, eng.N, args.cts
K = len(eng.context.p_chain_bits)
dev = eng.device
x = torch.empty((B, 2, L, N), dtype=torch.int64, device=dev)
g = torch.Generator(device=dev)
g.manual_seed(1)
for i, q in enumerate(eng.moduli[:L]):
    x[:, :, i] = torch.randint(0, q, (B, 2, N), generator=g, device=dev, dtype=torch.int64)
out = torch.empty_like(x)
out2 = torch.empty((2 * B, 2, L, N), dtype=torch.int64, device=dev)  # hoisted pair [rotation][ct]
out_rs = torch.empty((B, 2, L - 1, N), dtype=torch.int64, device=dev)
Lb = eng._L
eng._ensure_relin()
g1, g1024 = pow(5, 1, 2 * N), pow(5, 1024, 2 * N)
for gg in (g1, g1024):
    _lib.check(Lb.he_gen_switch_key(eng._h, gg, None))
torch.cuda.synchronize()

ptr = lambda t: _lib.ptr_array([t.data_ptr() + i * t.stride(0) * 8 for i in range(t.shape[0])])
px, po, prs = ptr(x), ptr(out), ptr(out_rs)
po2 = ptr(out2)
gpair = np.array([g1, g1024], np.uint32)
pc1 = _lib.ptr_array([x.data_ptr() + i * x.stride(0) * 8 + L * N * 8 for i in range(B)])
po0 = po
po1 = _lib.ptr_array([out.data_ptr() + i * out.stride(0) * 8 + L * N * 8 for i in range(B)])
work = x.clone()
s = eng.stream
A = _lib.addr

ops = {
    "ntt_fwd": lambda: Lb.he_ntt(eng._h, work.data_ptr(), 2 * B, L, 0, s),
    "ntt_inv": lambda: Lb.he_ntt(eng._h, work.data_ptr(), 2 * B, L, 1, s),
    "keyswitch_relin": lambda: Lb.he_keyswitch(eng._h, 0, A(pc1), A(po0), A(po1), B, L, s),
    "rotate_1": lambda: Lb.he_rotate(eng._h, g1, A(px), A(po), B, L, s),
    "rotate_1024": lambda: Lb.he_rotate(eng._h, g1024, A(px), A(po), B, L, s),
    "rescale": lambda: Lb.he_rescale(eng._h, A(px), A(prs), B, L, 2, s),
    # both rotations of every ciphertext with ONE ModUp of c1 (he_rotate_hoisted)
    "rotate_1_and_1024_hoisted": lambda: Lb.he_rotate_hoisted(eng._h, A(gpair), 2, A(px), A(po2), B, L, s),
}
beta = -(-L // eng.context.alpha)
poly = L * N * 8
alg_bytes = {
    "ntt_fwd": 2 * B * L * 16 * N, "ntt_inv": 2 * B * L * 16 * N,
    # d in + (c0, c1) out per ct; the 176 MB key is read once per key pass of the batch
    "keyswitch_relin": B * (poly + 2 * poly) + 2 * beta * (L + K) * N * 8,
    "rotate_1": B * (2 * poly + 2 * poly) + 2 * beta * (L + K) * N * 8,
    "rotate_1024": B * (2 * poly + 2 * poly) + 2 * beta * (L + K) * N * 8,
    "rescale": B * (2 * poly + 2 * (L - 1) * N * 8),
    "rotate_1_and_1024_hoisted": B * (2 * poly + 2 * 2 * poly) + 2 * 2 * beta * (L + K) * N * 8,
}
digits = [min(eng.context.alpha, L - j * eng.context.alpha) for j in range(beta)]
bfly = (N // 2) * 16


def ks_modmuls(ell):  # NTT butterflies + BConv + inner-product MACs of one key switch
    ext = ell + K
    n_ntt = ell + sum(ext - a for a in digits) + 2 * K + 2 * ell
    return n_ntt * bfly + (sum(a * (ext - a) for a in digits) + 2 * K * ell + 2 * beta * ext) * N


modmuls = {
    "ntt_fwd": 2 * B * L * bfly, "ntt_inv": 2 * B * L * bfly,
    "keyswitch_relin": B * ks_modmuls(L), "rotate_1": B * ks_modmuls(L), "rotate_1024": B * ks_modmuls(L),
    "rescale": B * 2 * (1 + (L - 1)) * bfly,
    # algorithmic work of two independent rotations (the hoisted form does less)
    "rotate_1_and_1024_hoisted": 2 * B * ks_modmuls(L),
}
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
res = {}
for name, fn in ops.items():
    for _ in range(2):
        _lib.check(fn(), name)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        _lib.check(fn(), name)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.reps
    gbs = alg_bytes[name] / (ms * 1e6)
    res[name] = {"ms": round(ms, 3), "alg_GBps": round(gbs, 1), "hbm_frac": round(gbs / peaks["hbm_gbs"], 3)}
    if name.startswith("ntt"):
        bf = B * 2 * L * (N // 2) * 16
        res[name]["Gbutterfly_per_s"] = round(bf / (ms * 1e6), 1)
ip, fp = np.zeros(2), np.zeros(1)
_lib.check(Lb.he_microbench_intpipe(eng.context.device, A(ip)))
_lib.check(Lb.he_microbench_fp64(eng.context.device, A(fp)))
res["intpipe"] = {"imad32_per_s": ip[0], "mac128_per_s": ip[1], "fp64_modmul_per_s": fp[0]}
# modular-product roofline: algorithmic modular multiplications (butterflies, BConv,
# inner product) against the measured rate of the datapath they run on.  Every
# config-2 prime is below 2^50, so the NTTs and every key-switch pass multiply on
# the FP64 pipe (centred fmulmod_c); the BConv of the key switch stays integer.
# int_frac: vs the faster measured rate (FP64 fmulmod), frac_vs_mac128: vs the
# 64x64->128 multiply-accumulate rate (the integer datapath of round-1 v1).
peak_mm = max(ip[1], fp[0])
for name in ops:
    rate = modmuls[name] / (res[name]["ms"] * 1e-3)
    res[name]["Gmodmul_per_s"] = round(rate / 1e9, 1)
    res[name]["int_frac"] = round(rate / peak_mm, 3)
    res[name]["frac_vs_mac128"] = round(rate / ip[1], 3)

if not args.no_oracle:   # bit-exact spot check of ct 0 for every op
    import oracle as O

    orc = O.Oracle(16, [50] * 24, [50] * 4, 4, seed=7, scale=2.0 ** 50)
    xn = x[0].cpu().numpy().view(np.uint64)
    chk = {}
    w = torch.from_numpy(xn.copy().view(np.int64)).to(dev)
    _lib.check(Lb.he_ntt(eng._h, w.data_ptr(), 2, L, 0, s))
    ref = np.stack([np.stack([orc.ntt(xn[c, i], i) for i in range(L)]) for c in range(2)])
    chk["ntt_fwd"] = bool(np.array_equal(w.cpu().numpy().view(np.uint64), ref))
    _lib.check(Lb.he_ntt(eng._h, w.data_ptr(), 2, L, 1, s))
    chk["ntt_inv"] = bool(np.array_equal(w.cpu().numpy().view(np.uint64), xn))
    _lib.check(ops["rescale"]())
    chk["rescale"] = bool(np.array_equal(out_rs[0].cpu().numpy().view(np.uint64), orc.rescale(xn)))
    _lib.check(ops["rotate_1"]())
    chk["rotate_1"] = bool(np.array_equal(out[0].cpu().numpy().view(np.uint64), orc.rotate(xn, g1, orc.switch_key(g1))))
    _lib.check(ops["keyswitch_relin"]())
    k0, k1 = orc.keyswitch(xn[1].copy(), orc.switch_key(0))
    chk["keyswitch_relin"] = bool(np.array_equal(out[0].cpu().numpy().view(np.uint64), np.stack([k0, k1])))
    _lib.check(ops["rotate_1_and_1024_hoisted"]())
    chk["rotate_hoisted"] = all(
        bool(np.array_equal(out2[r * B].cpu().numpy().view(np.uint64),
                            orc.rotate_hoisted(xn, gg, orc.hoist_key(orc.switch_key(gg), gg))))
        for r, gg in enumerate((g1, g1024)))
    res["bit_exact_vs_oracle"] = chk
print(json.dumps({"config": "cfg2: N=2^16, 24x50 + 4x50 bits, dnum 6", "cts": B, "reps": args.reps,
                  "hbm_peak_GBps": peaks["hbm_gbs"], "ops": res}))
