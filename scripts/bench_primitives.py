"""Config-2 primitive microbenchmark (BASELINE.json configs[1]) on its own:
the same measurement bench.py puts in its line as "primitives_cfg2"
(`python bench.py --workload cfg2` prints it alone).

usage: python scripts/bench_primitives.py [--cts 256] [--reps 5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "backend:cudaMallocAsync")

import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cts", type=int, default=256)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
print(json.dumps(bench.primitives_cfg2(0, args.cts, args.reps)))
