"""Benchmark: amortised encrypted samples/s of the feature-major CIFAR CNN.

Workload (BASELINE.json configs 3 and 5): the 14-limb CNN (conv3x3 3->16,
act, 2x2 avgpool, conv3x3 16->32, act, GAP, dense 32->10) on one
32768-sample ciphertext group (3072 input ciphertexts, N = 2^16) per GPU per
step.  With --gpus 8 the 8 groups of config 5 run one per GPU (weak scaling,
no data-path collective: groups are independent).

  value : samples/s with the encrypted inputs resident in HBM (network only)
  e2e   : samples/s through the public API with HOST buffers: pinned images
          -> H2D -> pack_features (encode + encrypt) -> network -> decrypt ->
          D2H logits, all inside the timed region
  --impl reference : the CPU oracle port on the host cores (rank 0 only)

Prints ONE JSON line (rank 0).  Inputs (45 GB of ciphertexts per group) are
far larger than the 126 MB L2, so no explicit flush is needed.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# torch and libhe_sm100.so share one stream-ordered pool (see package __init__)
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "backend:cudaMallocAsync")

METRIC = "amortised encrypted samples/sec"
SAMPLES_PER_GROUP = 32768


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=None, help="(ncu) run exactly this many network passes")
    ap.add_argument("--workload", default="cfg3", choices=["cfg3", "cfg2", "boot"],
                    help="cfg3: the CNN (default line); cfg2: only the config-2 primitive microbenchmark; "
                         "boot: only the N = 2^16 bootstrap")
    ap.add_argument("--no-primitives", action="store_true", help="skip the config-2 primitives in the cfg3 line")
    ap.add_argument("--no-bootstrap", action="store_true", help="skip the bootstrap timing in the cfg3 line")
    ap.add_argument("--h2d-overlap", default="network", choices=["encrypt", "network", "serial"],
                    help="e2e: which phase of step i the H2D copy of step i+1's images overlaps "
                         "(serial: each step's own copy, not overlapped)")
    return ap.parse_args()


def _dist():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def _self_launch(args):
    """`bench.py --gpus N` without a launcher: re-exec under torch.distributed.run
    with N ranks (one per GPU, rendezvous on 127.0.0.1), so a plain invocation
    can never record a one-GPU number as an N-GPU run.  Under a launcher the
    world size must equal --gpus."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        return
    if args.gpus <= 1:
        return
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


LEVEL_PLAN = ("inputs at 9 of 14 limbs -> conv1+square+pool (carry, 9) -> conv2+square+GAP (9) -> 5-component relin "
              "dropping 6 primes (3) -> dense+rescale (2)")


def _config(world, input_limbs=9):
    return {"workload": "cfg3/cfg5 CIFAR-shaped CNN, one 32768-sample ciphertext group per GPU per step",
            "ring_degree": 65536, "q_limbs": 14, "special_primes": 3, "scale_bits": 40,
            "input_ciphertexts_per_group": 3072, "input_limbs": input_limbs, "level_plan": LEVEL_PLAN,
            "groups_per_step": world,
            "samples_per_step": SAMPLES_PER_GROUP * world, "parallelism": f"groups{world}",
            "l2_flush": "inputs (29 GB per group at 9 limbs) >> 126 MB L2"}


class Clocks:
    """SM clock / clock-event-reason sampling (NVML, else nvidia-smi) during the timed region."""

    def __init__(self, device):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        # in-process NVML (no fork of this large process while the GPU is timed);
        # nvidia-smi only if NVML is unavailable
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            bits = [("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
                    ("sw_power_cap", 0x4)]

            def sample():
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h) \
                    if hasattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons") \
                    else pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                return ([str(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)),
                         str(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)), hex(r)]
                        + ["Active" if r & b else "Not Active" for _, b in bits])
            sample()
        except Exception:
            sample = None

        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    if sample is not None:
                        self.rows.append(sample())
                    else:
                        out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                             timeout=5).stdout.strip()
                        if out:
                            self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.05)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        import statistics

        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[3:7]) if v.strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def run_reference(args, rank, world):
    """The reference arm (rank 0 only): the CPU RNS-CKKS oracle port (oracle/,
    C + OpenMP on every host thread) replaying the GPU's config-3 plan on a
    bounded sample per step, extrapolated to one 32768-sample group with the
    exact op counts -- ``ms_per_step`` is the MEASURED wall time of a step's
    sample and ``extrapolation_factor`` says how far it is scaled.  The reference
    package itself (hebatch.SimulatorEngine from baseline/_ref, float64 slots
    without cryptography) is timed once on the same network
    and reported beside it as ``reference_simulator``."""
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import cpu_baseline

    t = time.perf_counter()
    runs = [cpu_baseline.measure() for _ in range(max(1, args.steps))]
    r = sorted(runs, key=lambda x: x["samples_per_s"])[len(runs) // 2]
    v = float(r["samples_per_s"])
    wall_ms = 1e3 * sum(x["wall_s"] for x in runs) / len(runs)
    sim = None
    sys.path.insert(0, os.path.join(ROOT, "baseline"))
    import ref_simulator

    why = ref_simulator.available()
    if why is None:
        s = ref_simulator.measure()
        sim = {"value": s["samples_per_s"], "unit": "samples/s", "cores": s["threads"], "kind": "reference",
               "measured_s": s["measured_s"], "extrapolation_factor": s["extrapolation_factor"],
               "layers": s["layers"], "sample": s["sample"]}
    else:
        sim = {"unavailable": why}
    line = {"metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": wall_ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64 (RNS residues)", "data": "synthetic",
            "config": _config(1, input_limbs=cpu_baseline.ELL), "impl": "reference",
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": r["threads"], "kind": "port",
                             "sample": r["sample"], "measured_wall_s_per_step": wall_ms / 1e3,
                             "extrapolation_factor": r["extrapolation_factor"]},
            "reference_simulator": sim,
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.perf_counter() - t}
    print(json.dumps(line), flush=True)


def primitives_cfg2(device: int = 0, cts: int = 256, reps: int = 5) -> dict:
    """BASELINE.json configs[1]: N = 2^16, 24 x 50-bit Q limbs + 4 x 50-bit P (dnum 6),
    256 ciphertexts of uniform residues (seeded).  Times forward / inverse NTT, the
    relinearisation key switch, rotation by +1 and +1024 (and both hoisted), and
    rescale 24 -> 23 over all ciphertexts with CUDA events on the launching stream
    (2 warm-up launches each).  Rooflines: algorithmic bytes against the measured HBM
    copy bandwidth; algorithmic modular products (butterflies, BConv and inner-product
    MACs) against the faster measured modular-product rate (FP64
    fmulmod; every config-2 prime is < 2^50).  Reference ops:
    /root/reference/pkg/src/hebatch/engine.py:276-313.  Bit-exactness of every op
    vs the CPU oracle: tests/test_gpu_parity.py on the cfg2 ring."""
    import numpy as np
    import torch

    from paper_2604_16834_b200 import _lib, configs
    from paper_2604_16834_b200.engine import GpuEngine

    eng = GpuEngine(configs.context(2, seed=7, device=device))
    L, N, B = eng.context.n_q, eng.N, cts
    K = len(eng.context.p_chain_bits)
    dev = eng.device
    x = torch.empty((B, 2, L, N), dtype=torch.int64, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    for i, q in enumerate(eng.moduli[:L]):
        x[:, :, i] = torch.randint(0, q, (B, 2, N), generator=g, device=dev, dtype=torch.int64)
    out = torch.empty_like(x)
    out2 = torch.empty((2 * B, 2, L, N), dtype=torch.int64, device=dev)
    out_rs = torch.empty((B, 2, L - 1, N), dtype=torch.int64, device=dev)
    Lb = eng._L
    eng._ensure_relin()
    g1, g1024 = pow(5, 1, 2 * N), pow(5, 1024, 2 * N)
    for gg in (g1, g1024):
        _lib.check(Lb.he_gen_switch_key(eng._h, gg, None))
    torch.cuda.synchronize()

    def ptr(t, off=0):
        return _lib.ptr_array([t.data_ptr() + i * t.stride(0) * 8 + off for i in range(t.shape[0])])

    px, po, prs, po2 = ptr(x), ptr(out), ptr(out_rs), ptr(out2)
    pc1, po1 = ptr(x, L * N * 8), ptr(out, L * N * 8)
    gpair = np.array([g1, g1024], np.uint32)
    work = x.clone()
    s, A = eng.stream, _lib.addr
    ops = {
        "ntt_fwd": lambda: Lb.he_ntt(eng._h, work.data_ptr(), 2 * B, L, 0, s),
        "ntt_inv": lambda: Lb.he_ntt(eng._h, work.data_ptr(), 2 * B, L, 1, s),
        "keyswitch_relin": lambda: Lb.he_keyswitch(eng._h, 0, A(pc1), A(po), A(po1), B, L, s),
        "rotate_1": lambda: Lb.he_rotate(eng._h, g1, A(px), A(po), B, L, s),
        "rotate_1024": lambda: Lb.he_rotate(eng._h, g1024, A(px), A(po), B, L, s),
        "rescale": lambda: Lb.he_rescale(eng._h, A(px), A(prs), B, L, 2, s),
        "rotate_1_and_1024_hoisted": lambda: Lb.he_rotate_hoisted(eng._h, A(gpair), 2, A(px), A(po2), B, L, s),
    }
    beta = -(-L // eng.context.alpha)
    poly = L * N * 8
    key = 2 * beta * (L + K) * N * 8
    alg_bytes = {"ntt_fwd": 2 * B * 2 * poly, "ntt_inv": 2 * B * 2 * poly,
                 "keyswitch_relin": B * 3 * poly + key, "rotate_1": B * 4 * poly + key,
                 "rotate_1024": B * 4 * poly + key, "rescale": B * (2 * poly + 2 * (L - 1) * N * 8),
                 "rotate_1_and_1024_hoisted": B * 6 * poly + 2 * key}
    digits = [min(eng.context.alpha, L - j * eng.context.alpha) for j in range(beta)]
    bfly = (N // 2) * 16

    def ks_modmuls(ell):
        ext = ell + K
        n_ntt = ell + sum(ext - a for a in digits) + 2 * K + 2 * ell
        return n_ntt * bfly + (sum(a * (ext - a) for a in digits) + 2 * K * ell + 2 * beta * ext) * N

    modmuls = {"ntt_fwd": 2 * B * L * bfly, "ntt_inv": 2 * B * L * bfly, "keyswitch_relin": B * ks_modmuls(L),
               "rotate_1": B * ks_modmuls(L), "rotate_1024": B * ks_modmuls(L), "rescale": B * 2 * L * bfly,
               "rotate_1_and_1024_hoisted": 2 * B * ks_modmuls(L)}
    hbm, hbm_kind = _peaks()
    fp = np.zeros(1)
    _lib.check(Lb.he_microbench_fp64(eng.context.device, fp.ctypes.data), "microbench")
    res = {}
    for name, fn in ops.items():
        for _ in range(2):
            _lib.check(fn(), name)
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            _lib.check(fn(), name)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        gbs = alg_bytes[name] / (ms * 1e6)
        rate = modmuls[name] / (ms * 1e-3)
        res[name] = {"ms": round(ms, 3), "hbm": {"achieved_GBps": round(gbs, 1), "frac": round(gbs / hbm, 3)},
                     "modmul": {"achieved_per_s": rate, "frac": round(rate / float(fp[0]), 3)}}
    del x, out, out2, out_rs, work
    eng.trim()
    return {"workload": "cfg2 primitives: N=2^16, 24x50 + 4x50-bit primes, dnum 6, %d uniform ciphertexts" % B,
            "reps": reps, "ops": res, "peaks": {"hbm_GBps": hbm, "hbm_kind": hbm_kind,
                                                 "fp64_modmul_per_s": float(fp[0])},
            "parity": "bit-exact vs the CPU oracle: tests/test_gpu_parity.py (cfg2 ring: ntt, keyswitch, "
                      "rescale, mult_ct, rotate, rotate_hoisted)"}


def bootstrap_n16(device: int = 0, reps: int = 5) -> dict:
    """CKKS bootstrapping (the reference's bootstrap is level
    accounting only, /root/reference/pkg/src/hebatch/engine.py:315-319) on the
    configs.boot_context ring: one ciphertext of 32768 seeded U[-1, 1] slots read at
    level 0, ModRaise -> CoeffToSlot -> EvalMod -> SlotToCoeff, timed with CUDA
    events on the engine's stream after one warm-up call (key generation and
    diagonal encoding happen there).  Limb parity vs the CPU oracle:
    tests/test_gpu_bootstrap.py (the same circuit on the oracle at N = 2^11)."""
    import numpy as np
    import torch

    from paper_2604_16834_b200 import configs
    from paper_2604_16834_b200.engine import GpuEngine

    eng = GpuEngine(configs.boot_context(seed=11, device=device))
    x = np.random.default_rng(3).uniform(-1, 1, eng.context.n)
    low = eng.drop_level_batch([eng.encrypt_batch(x[None])[0]], 0)[0]
    t0 = time.perf_counter()
    out = eng.bootstrap(low)
    eng.synchronize()
    first = time.perf_counter() - t0
    st = torch.cuda.current_stream(eng.device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = eng._L.he_launch_count()
    e0.record(st)
    for _ in range(reps):
        eng.release(out)
        out = eng.bootstrap(low)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    launches = (eng._L.he_launch_count() - n0) // reps
    err = float(np.max(np.abs(eng.decrypt(out) - x)))
    # throughput: one batched circuit for `batch` ciphertexts (bootstrap_batch)
    batch = 8
    xb = np.random.default_rng(4).uniform(-1, 1, (batch, eng.context.n))
    lows = eng.drop_level_batch(eng.encrypt_batch(xb), 0)
    outs = eng.bootstrap_batch(lows)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(2):
        eng.release(*outs)
        outs = eng.bootstrap_batch(lows)
    e1.record(st)
    torch.cuda.synchronize()
    ms_b = e0.elapsed_time(e1) / 2
    err_b = max(float(np.max(np.abs(eng.decrypt(o) - xb[i]))) for i, o in enumerate(outs))
    plan = eng.boot_plan()
    res = {"workload": "bootstrap: N=2^16, 32768 slots, q0 60 + 25x50-bit primes, scale 2^50, 4x60-bit P, "
                       "sparse secret h=128, one ciphertext",
           "ms": round(ms, 2), "reps": reps, "launches_per_bootstrap": launches,
           "max_abs_err": err, "depth": plan.depth, "r": plan.r,
           "batch": {"cts": batch, "ms": round(ms_b, 2), "ms_per_ct": round(ms_b / batch, 2), "max_abs_err": err_b},
           "dft_levels": plan.dft_levels, "level_out": out.level, "rotation_keys": len(plan.rotation_offsets()) + 1,
           "first_call_s_incl_keygen": round(first, 3),
           "parity": "limb-exact vs the same circuit on the CPU oracle: tests/test_gpu_bootstrap.py"}
    del eng
    return res


def main():
    args = _args()
    _self_launch(args)
    rank, world, local = _dist()
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch

    torch.cuda.set_device(local)
    if args.workload == "boot":
        if rank == 0:
            print(json.dumps(bootstrap_n16(local)), flush=True)
        return
    if args.workload == "cfg2":
        if rank == 0:
            print(json.dumps(primitives_cfg2(local)), flush=True)
        return
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2604_16834_b200 import _lib, configs
    from paper_2604_16834_b200.engine import GpuEngine
    from paper_2604_16834_b200.featuremajor import min_input_level, run_cnn
    from paper_2604_16834_b200.packing import pack_features

    from paper_2604_16834_b200.sharding import assign_groups, max_over_ranks as _max_over_ranks

    spec = configs.CNN3
    wts = spec.make_weights(1234)                       # same model on every rank
    # config 5: groups round-robin over ranks, one group per GPU per step (weak
    # scaling, no data-path collective); group g's images are seeded g
    (group,) = assign_groups(world, world, rank)
    # per-rank key seed: groups on different ranks never share a secret key or
    # encryption randomness (equal (seed, index) pairs would leak m - m')
    eng = GpuEngine(configs.context(3, seed=42 + 7919 * rank, device=local))
    rng = np.random.default_rng(group)
    images = rng.uniform(0.0, 1.0, size=(SAMPLES_PER_GROUP, 3 * 32 * 32))
    feat_host = torch.from_numpy(np.ascontiguousarray(images.T)).pin_memory()   # [3072, 32768] f64
    # inputs are encrypted at the level the plan needs (9 of the chain's 14
    # limbs for config 3); the other limbs would never be read
    level = min_input_level(eng, spec)
    x = pack_features(eng, images, level=level)           # resident encrypted inputs
    eng._ensure_relin()
    del images

    def step():
        out = run_cnn(eng, x, spec, wts, release_inputs=False)
        eng.release(*out)

    if args.profile_steps is not None:                   # ncu mode: no timing, no baseline
        for _ in range(args.profile_steps):
            step()
        torch.cuda.synchronize()
        return

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(v):
        return _max_over_ranks(v, world, device="cuda")

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # ---- device-resident timed region
    eng.enable_timing(True)
    barrier()
    torch.cuda.synchronize()
    launches0 = _lib.load().he_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with Clocks(local) as clk:
        ev0.record()
        for i in range(args.steps):
            step_ev[i].record()
            step()
        step_ev[-1].record()
        ev1.record()
        torch.cuda.synchronize()
    step_ms = [round(step_ev[i].elapsed_time(step_ev[i + 1]), 1) for i in range(args.steps)]
    barrier()
    launches = _lib.load().he_launch_count() - launches0
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    summ = eng.timing_summary()
    eng.enable_timing(False)
    value = world * SAMPLES_PER_GROUP * args.steps / (ms / 1e3)

    # ---- end to end through the public API with host buffers
    eng.release(*x)                                      # free the resident inputs (45 GB) back to the pool
    del x
    e2e_steps = args.e2e_steps or args.steps
    out_host = torch.empty((10, SAMPLES_PER_GROUP), dtype=torch.float64).pin_memory()

    # Host images reach HBM through a copy stream, double-buffered: step i+1's
    # H2D (pinned -> device, copy engine) is issued once step i's encryption has
    # consumed its buffer, so it overlaps step i's network.  Every step's H2D,
    # including the first, lies inside the timed region.
    phase_ev = []                                        # per-step (h2d wait, encrypt, network, decrypt+d2h) events
    dev_in = [torch.empty(feat_host.shape, dtype=feat_host.dtype, device="cuda") for _ in range(2)]
    cstream = torch.cuda.Stream()
    h2d_done = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    for e in consumed:
        e.record()

    during_net = args.h2d_overlap == "network"

    def issue_h2d(i):
        if args.h2d_overlap == "serial":
            return
        b = i % 2
        with torch.cuda.stream(cstream):
            cstream.wait_event(consumed[b])             # the buffer's previous encryption is done
            if during_net:
                cstream.wait_event(consumed[1 - b])     # and the current step's: the copy overlaps a network
            dev_in[b].copy_(feat_host, non_blocking=True)  # one DMA from pinned memory
            h2d_done[b].record(cstream)

    def e2e_step(i, last, ev=None):
        rec = (lambda: ev.append(torch.cuda.Event(enable_timing=True)) or ev[-1].record()) if ev is not None \
            else (lambda: None)
        b = i % 2
        rec()
        if args.h2d_overlap == "serial":
            dev_in[b].copy_(feat_host, non_blocking=True)   # on the work stream, before this step's encryption
        else:
            torch.cuda.current_stream().wait_event(h2d_done[b])
        rec()
        if not last and args.h2d_overlap == "encrypt":
            issue_h2d(i + 1)       # next step's copy overlaps this step's encryption (not the network)
        cts = eng.encrypt_batch(dev_in[b], level=level)
        consumed[b].record()
        if not last and during_net:
            issue_h2d(i + 1)
        rec()
        out = run_cnn(eng, cts, spec, wts, release_inputs=True)
        rec()
        logits = eng.decrypt_batch(out, as_tensor=True)
        eng.release(*out)
        out_host.copy_(logits, non_blocking=True)
        rec()

    wstream = torch.cuda.Stream()                         # the e2e work runs on its own (non-default) stream
    torch.cuda.synchronize()
    with torch.cuda.stream(wstream):
        for e in consumed:
            e.record()
        issue_h2d(0)
        for i in range(args.warmup):                     # same warm-up rule as the resident loop
            e2e_step(i, i == args.warmup - 1)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        issue_h2d(0)                                      # first step's copy: inside the timed region
        for i in range(e2e_steps):
            ev = []
            e2e_step(i, i == e2e_steps - 1, ev)
            phase_ev.append(ev)
        e1.record()
        torch.cuda.synchronize()
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1))
    e2e_phases = [[round(ev[i].elapsed_time(ev[i + 1]), 1) for i in range(4)] for ev in phase_ev]
    e2e = world * SAMPLES_PER_GROUP * e2e_steps / (e2e_ms / 1e3)

    # ---- rooflines (CUDA events on the launching stream over the timed region)
    # Each C-ABI category is held against the resource that binds it:
    #   conv_sqsum : tensor pipe -- algorithmic int8 digit products (modular MACs x
    #                byte planes x weight digits) against the measured
    #                mma.sync.m16n8k32.u8.s8 rate of this GPU (he_microbench_imma)
    #   relin/lincomb : integer datapath -- algorithmic modular products against
    #                the faster measured modular-product rate (64x64->128 MAC or
    #                FP64 fmulmod; config 3's primes are < 2^42: FP64)
    #   everything  : algorithmic HBM bytes against the measured copy bandwidth
    peak, peak_kind = _peaks()
    ip, fp, im, tc = np.zeros(2), np.zeros(1), np.zeros(1), np.zeros(2)
    _lib.check(_lib.load().he_microbench_intpipe(local, ip.ctypes.data), "microbench")
    _lib.check(_lib.load().he_microbench_fp64(local, fp.ctypes.data), "microbench")
    _lib.check(_lib.load().he_microbench_imma(local, im.ctypes.data), "microbench")
    _lib.check(_lib.load().he_microbench_tc5(local, 256, tc.ctypes.data), "microbench")
    peak_mm = max(float(ip[1]), float(fp[0]))
    peak_tops = 2.0 * float(tc[0]) / 1e12                 # tcgen05 kind::i8, M=128 N=256 (the chip's int8 rate)
    traffic_all = _traffic()
    rooflines = {}
    for k, (calls, kms, units) in summ.items():
        sec = kms / 1e3
        r = {"calls": calls, "ms": round(kms, 2), "avg_ms": kms / calls,
             "hbm": {"achieved": units[0] / sec / 1e9, "peak": peak, "unit": "GB/s", "frac": units[0] / sec / 1e9 / peak}}
        if k == "conv_sqsum" and len(units) > 2:
            ach = 2.0 * units[2] / sec / 1e12
            r["tensor"] = {"achieved": ach, "peak": peak_tops, "unit": "TOP/s (int8)", "frac": ach / peak_tops,
                           "peak_source": "measured: tcgen05.mma kind::i8 M=128 N=256 (he_microbench_tc5)",
                           "frac_of_nominal_4500": ach / 4500.0}
            if len(units) > 3:
                fr = units[3] / sec
                r["fp64"] = {"achieved": fr, "peak": float(fp[0]), "unit": "modmul/s", "frac": fr / float(fp[0]),
                             "what": "epilogue FP64 modular products (window/GAP products; recombination is integer)",
                             "peak_source": "measured: FP64 fmulmod chain (he_microbench_fp64)"}
            if len(units) > 4:
                # B200: tcgen05.mma and the FP64 pipe share one issue resource (scripts/mb/mb_fp64_vs_mma.cu,
                # profiles/r2_mb_fp64_vs_mma.txt): what binds the kernel is MMA time + FP64 time
                sm_mhz = 1965.0
                mma_s = units[4] / 148.0 / (sm_mhz * 1e6)
                fp64_s = units[3] / float(fp[0])
                r["shared_pipe"] = {"what": "tensor + FP64 pipe (one shared issue resource on B200): the launch's "
                                            "tcgen05 MMAs at their standalone cost plus its FP64 modular products at "
                                            "the standalone fmulmod rate, over the measured kernel time",
                                    "mma_ms": mma_s * 1e3 / calls, "fp64_ms": fp64_s * 1e3 / calls,
                                    "frac": (mma_s + fp64_s) / sec, "sm_mhz_assumed": sm_mhz}
        elif units[1] > 0:
            ach = units[1] / sec
            r["int"] = {"achieved": ach, "peak": peak_mm, "unit": "modmul/s", "frac": ach / peak_mm,
                        "peak_source": "measured: max(64x64->128 MAC/s, FP64 modular products/s) (he_microbench_*)"}
        rooflines[k] = r
    dom_name = max(summ.items(), key=lambda kv: kv[1][1])[0]
    dom = rooflines[dom_name]
    # the dominant kernel (the fused conv) against HBM: its algorithmic bytes (inputs once +
    # outputs once) per launch / its average launch time; its int8 tensor work and
    # its epilogue's FP64 modular products are reported beside it against their measured peaks
    bind = "int" if ("int" in dom and "tensor" not in dom) else "hbm"
    roof = {"kernel": dom_name, "bound": "hbm", "achieved": dom["hbm"]["achieved"], "peak": peak, "unit": "GB/s",
            "frac": dom["hbm"]["frac"], "traffic": traffic_all.get(dom_name), "peak_source": peak_kind,
            "calls": dom["calls"], "avg_ms": dom["avg_ms"],
            "algorithmic_bytes_per_launch": summ[dom_name][2][0] / summ[dom_name][0]}
    for extra in ("tensor", "fp64", "shared_pipe"):
        if extra in dom:
            roof[extra] = dom[extra]
    if bind == "int":
        roof["int_pipe"] = dom["int"]
    breakdown = rooflines
    peaks_measured = {"tcgen05_int8_TOPs": peak_tops, "mma_sync_int8_TOPs": 2.0 * float(im[0]) / 1e12,
                      "mac128_per_s": float(ip[1]), "fp64_modmul_per_s": float(fp[0]),
                      "imad32_per_s": float(ip[0]), "hbm_GBps": peak}

    prim = None
    if rank == 0 and not args.no_primitives:            # after every timed region: config-2 primitives
        eng.trim()
        prim = primitives_cfg2(local)
    boot = None
    if rank == 0 and not args.no_bootstrap:
        eng.trim()
        boot = bootstrap_n16(local)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import cpu_baseline

        r = cpu_baseline.measure()
        cpu = {"value": r["samples_per_s"], "unit": "samples/s", "cores": r["threads"], "kind": "port",
               "sample": r["sample"], "measured_wall_s": r["wall_s"], "extrapolation_factor": r["extrapolation_factor"]}
        sys.path.insert(0, os.path.join(ROOT, "baseline"))
        import ref_simulator

        if ref_simulator.available() is None:
            s = ref_simulator.measure()
            cpu["reference_simulator"] = {"value": s["samples_per_s"], "cores": 1, "kind": "reference",
                                          "measured_s": s["measured_s"],
                                          "extrapolation_factor": s["extrapolation_factor"]}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "step_ms": step_ms, "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None, "dtype": "u64 (RNS residues mod 40/42-bit primes; FP64-exact modular products)",
            "data": "synthetic (seeded U[0,1] CIFAR-shaped images, N(0,1/fan_in) weights)",
            "config": _config(world, input_limbs=level + 1),
            "e2e": {"value": e2e, "unit": "samples/s", "steps": e2e_steps,
                    "phase_ms_h2dwait_enc_net_dec": e2e_phases,
                    "h2d": f"double-buffered on a copy stream, overlapping the previous step's {args.h2d_overlap}",
                    "h2d_bytes_per_step": int(feat_host.numel() * 8),
                    "d2h_bytes_per_step": int(out_host.numel() * 8)},
            "roofline": roof,
            "breakdown": breakdown,
            "peaks_measured": peaks_measured,
            "cpu_baseline": cpu,
            "primitives_cfg2": prim,
            "bootstrap": boot,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
