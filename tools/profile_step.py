"""Run W eager layer steps of a workload (for ncu captures: the last step's kernels are the
ones to profile; every kernel of a step launches once per step)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from gen import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="mnist")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--set", nargs="*", default=[],
                help="config overrides key=int, e.g. M=16 T=4096 (a transformer-shaped slice: 64 rows/expert)")
a = ap.parse_args()
cfg = CONFIGS[a.config]
if a.set:
    cfg = cfg.with_(**{kv.split("=")[0]: int(kv.split("=")[1]) for kv in a.set})
lay, x, dy, alive, resp = bench.build_layer(cfg, 0, torch.device("cuda", 0), cfg.T)
for _ in range(a.steps):
    bench.run_calls(lay, x, dy, alive, resp)
torch.cuda.synchronize()
print("ok")
