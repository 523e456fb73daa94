"""Per-phase time of one expert-parallel (peer-memory) step on each rank: CUDA events between the
ABI calls of PeerEPDMoELayer.forward/backward (eager, after warm-up).

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/ep_phases.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from gen import CONFIGS  # noqa: E402
from paper_2002_04013_b200 import _lib as L  # noqa: E402

dist.init_process_group("nccl")
rank, world = dist.get_rank(), dist.get_world_size()
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "mnist"]
lay, x, dy, alive, resp = bench.build_ep_layer(cfg, 0, torch.device("cuda", local), cfg.T, rank, world)
for _ in range(5):
    lay.step(x, dy, alive, resp)
torch.cuda.synchronize()
dist.barrier()

marks = []


def mark(name):
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    marks.append((name, e))


# wrap the binding's calls used by the layer so that each is bracketed by events
names = ["dmoe_ep_begin", "dmoe_gate_topk", "dmoe_dispatch", "dmoe_ep_exchange_counts",
         "dmoe_ep_push_rows", "dmoe_expert_ffn_fwd", "dmoe_ep_return_rows", "dmoe_combine", "dmoe_combine_bwd",
         "dmoe_expert_ffn_bwd", "dmoe_gate_bwd"]
orig = {n: getattr(L, n) for n in names}
for n in names:
    def wrap(*a, _n=n, **k):
        r = orig[_n](*a, **k)
        mark(_n)
        return r
    setattr(L, n, wrap)
ar = dist.all_reduce


def ar_wrap(*a, **k):
    r = ar(*a, **k)
    mark("all_reduce")
    return r


dist.all_reduce = ar_wrap
mark("start")
lay.step(x, dy, alive, resp)
torch.cuda.synchronize()
rows = [f"rank {rank}: total {marks[0][1].elapsed_time(marks[-1][1]) * 1e3:.1f} us"]
for (_, a), (n, b) in zip(marks, marks[1:]):
    rows.append(f"  {n:26s} {a.elapsed_time(b) * 1e3:8.1f} us")
for r in range(world):
    dist.barrier()
    if r == rank:
        print("\n".join(rows), flush=True)
dist.barrier()
dist.destroy_process_group()
