"""Config 4 (deep CNN, 24 x 50-bit limbs, degree-3 activations) with output-channel
sharding over the ranks of one node (sharded_cnn.run_cnn_sharded over NCCL).

    python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
        --master-port 29511 scripts/run_cfg4.py [--hw 32] [--samples 32768]

Prints one JSON line on rank 0: samples/s (device time, max over ranks), the peak
HBM held by torch on rank 0, and the decrypt error of the first 64 samples against
the float64 forward pass.  The network is streamed over image rows, so the full
32x32 maps run on one GPU (inputs encrypted at sharded_cnn.plan_input_level: 15 of
the 24 limbs).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "backend:cudaMallocAsync")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--hw", type=int, default=32)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--tile-rows", type=int, default=2)
    ap.add_argument("--mem-trace", action="store_true", help="print HBM use at every tile")
    ap.add_argument("--max-outputs", type=int, default=512)
    ap.add_argument("--slab-cap-gb", type=float, default=None, help="GpuEngine.SLAB_FREE_CAP override")
    args = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    import numpy as np
    import torch

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2604_16834_b200 import configs
    from paper_2604_16834_b200.engine import GpuEngine
    from paper_2604_16834_b200.featuremajor import CnnSpec
    from paper_2604_16834_b200.packing import pack_features
    from paper_2604_16834_b200.sharded_cnn import TorchRing, plan_input_level, run_cnn_sharded
    from paper_2604_16834_b200.sharding import max_over_ranks

    base = configs.CNN4
    spec = CnnSpec(channels=base.channels, H=args.hw, W=args.hw, act=base.act, pool_after=base.pool_after)
    wts = spec.make_weights(1234)
    eng = GpuEngine(configs.context(4, seed=42, device=local))
    if args.slab_cap_gb is not None:
        eng.SLAB_FREE_CAP = int(args.slab_cap_gb * (1 << 30))
    n = eng.context.n
    rng = np.random.default_rng(args.seed)
    images = rng.uniform(0.0, 1.0, size=(n, 3 * args.hw * args.hw))
    level = plan_input_level(spec)
    x = pack_features(eng, images, level=level)        # replicated layer-0 input
    eng._ensure_relin()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.reset_peak_memory_stats()
    eng.enable_timing(True)
    e0.record()
    def mem_trace(stage, cts, info):
        free, total = torch.cuda.mem_get_info()
        print(f"{stage} blk {info.get('blk')} rows {info.get('rows')} ch {info.get('channels')}: torch alloc "
              f"{torch.cuda.memory_allocated() / 1e9:.1f} GB, device used {(total - free) / 1e9:.1f} GB, "
              f"slab {sum(t.numel() * 8 for v in eng._slab.values() for t in v) / 1e9:.1f} GB", flush=True)

    out = run_cnn_sharded(eng, x, spec, wts, rank, world, ring=TorchRing(rank, world), tile_rows=args.tile_rows,
                          trace=mem_trace if args.mem_trace else None, max_outputs=args.max_outputs)
    e1.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1), world, device="cuda")
    got = eng.decrypt_batch(out).T[:64]
    ref = spec.forward_plain(wts, images[:64].reshape(64, 3, args.hw, args.hw))
    if rank == 0:
        print(json.dumps({"config": f"cfg4 CNN {base.channels} on {args.hw}x{args.hw}", "n_gpus": world,
                          "samples": n, "ms": ms, "samples_per_s": n / (ms / 1e3),
                          "max_abs_err_64": float(np.max(np.abs(got - ref))), "input_limbs": level + 1,
                          "peak_hbm_gb_rank0": torch.cuda.max_memory_allocated() / 1e9,
                          "tile_rows": args.tile_rows, "pool_releases": eng.pool_releases,
                          "max_outputs": args.max_outputs, "slab_cap_gb": args.slab_cap_gb, "ms_by_category": {k: [v[0], round(v[1], 1)] for k, v in eng.timing_summary().items()},
                          "parallelism": f"output-channel shards x{world}, ring exchange"}), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
