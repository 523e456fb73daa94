"""Per-call timing of the routing calls at a BASELINE shape (CUDA events, L2 flushed before each
call, median of N): fused gate + SelectExperts vs gate scores and the standalone search."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from gen import CONFIGS  # noqa: E402
from paper_2002_04013_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="transformer")
ap.add_argument("--n", type=int, default=20)
a = ap.parse_args()
cfg = CONFIGS[a.config]
lay, x, dy, alive, resp = bench.build_layer(cfg, 0, torch.device("cuda", 0), cfg.T)
G = torch.empty(cfg.T, cfg.dM, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
T = cfg.T
calls = {
    "gate_topk(fused, no G)": lambda: L.dmoe_gate_topk(x, lay.Wg, lay.bg, lay.g, alive, None, lay.sel[:T], lay.sel_score[:T], lay.ws),
    "gate_topk(fused, +G)": lambda: L.dmoe_gate_topk(x, lay.Wg, lay.bg, lay.g, alive, G, lay.sel[:T], lay.sel_score[:T], lay.ws),
    "gate_scores": lambda: L.dmoe_gate_scores(x, lay.Wg, lay.bg, lay.g, G, lay.ws),
    "beam_topk(standalone)": lambda: L.dmoe_beam_topk(G, lay.g, alive, lay.sel[:T], lay.sel_score[:T], lay.ws),
}
for name, f in calls.items():
    ts = []
    for i in range(a.n + 3):
        flush.fill_(i & 0xFF)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        f()
        e.record()
        e.synchronize()
        if i >= 3:
            ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    print(f"{a.config} {name:28s} median {ts[len(ts) // 2]:8.1f} us  min {ts[0]:8.1f} us")
