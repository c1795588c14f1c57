"""Phase timing of bench.py's end-to-end step (H2D, encrypt, network, decrypt, D2H).

Run on the GPU box:  python scripts/e2e_probe.py [steps]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "backend:cudaMallocAsync")

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_16834_b200 import configs  # noqa: E402
from paper_2604_16834_b200.engine import GpuEngine  # noqa: E402
from paper_2604_16834_b200.featuremajor import run_cnn  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    S = 32768
    spec = configs.CNN3
    wts = spec.make_weights(1234)
    eng = GpuEngine(configs.context(3, seed=42, device=0))
    eng._ensure_relin()
    rng = np.random.default_rng(0)
    images = rng.uniform(0.0, 1.0, size=(S, 3 * 32 * 32))
    feat_host = torch.from_numpy(np.ascontiguousarray(images.T)).pin_memory()
    out_host = torch.empty((10, S), dtype=torch.float64).pin_memory()
    if os.environ.get("PROBE_NOGC"):
        import gc

        gc.disable()
    if os.environ.get("PROBE_MODE") == "bench":   # bench.py's order: resident phase, release, e2e without syncs
        from paper_2604_16834_b200.packing import pack_features

        x = pack_features(eng, images)
        for _ in range(2):
            eng.release(*run_cnn(eng, x, spec, wts, release_inputs=False))
        torch.cuda.synchronize()
        eng.release(*x)
        del x
        torch.cuda.empty_cache()
        for it in range(steps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            w0 = time.perf_counter()
            e0.record()
            dev = feat_host.to("cuda", non_blocking=True)
            cts = eng.encrypt_batch(dev)
            del dev
            w1 = time.perf_counter()
            out = run_cnn(eng, cts, spec, wts, release_inputs=True)
            w2 = time.perf_counter()
            logits = eng.decrypt_batch(out, as_tensor=True)
            eng.release(*out)
            out_host.copy_(logits, non_blocking=True)
            e1.record()
            w3 = time.perf_counter()
            torch.cuda.synchronize()
            print(f"bench-mode step {it}: events={e0.elapsed_time(e1):.1f}ms host enqueue: enc={1e3 * (w1 - w0):.1f} "
                  f"net={1e3 * (w2 - w1):.1f} dec={1e3 * (w3 - w2):.1f} wall={1e3 * (time.perf_counter() - w0):.1f}",
                  flush=True)
        return
    for it in range(steps + 1):
        t = [time.perf_counter()]
        torch.cuda.synchronize()
        dev = feat_host.to("cuda", non_blocking=True)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        cts = eng.encrypt_batch(dev)
        del dev
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        out = run_cnn(eng, cts, spec, wts, release_inputs=True)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        logits = eng.decrypt_batch(out, as_tensor=True)
        eng.release(*out)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        out_host.copy_(logits, non_blocking=True)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        names = ["h2d", "encrypt", "network", "decrypt", "d2h"]
        print(f"step {it}: " + " ".join(f"{n}={1e3 * (b - a):.1f}ms" for n, a, b in zip(names, t, t[1:])),
              f"total={1e3 * (t[-1] - t[0]):.1f}ms", flush=True)


if __name__ == "__main__":
    main()
