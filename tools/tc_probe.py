"""Timeline of CTA 0 in the last tcgen05 GEMM of an ABI call (needs DMOE_TC_DEBUG=8)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["DMOE_TC_DEBUG"] = str(8 | int(os.environ.get("DBG", "0")))
import torch  # noqa: E402

import bench  # noqa: E402
from gen import CONFIGS  # noqa: E402
from paper_2002_04013_b200 import _lib as L  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "mnist"]
if len(sys.argv) > 2:  # overrides key=int, e.g. M=16 T=4096
    cfg = cfg.with_(**{kv.split("=")[0]: int(kv.split("=")[1]) for kv in sys.argv[2:]})
lay, x, dy, alive, resp = bench.build_layer(cfg, 0, torch.device("cuda", 0), cfg.T)
for _ in range(2):
    bench.run_calls(lay, x, dy, alive, resp)
torch.cuda.synchronize()
R = 9
buf = (ctypes.c_ulonglong * (8 * R * 32))()
f = L._L.dmoe_debug_tc_probe
names = ["prod0", "prodN", "mma0", "mmaC", "epi0", "epiD", "mmaW", "mmaL"]
order = [0, 1, 6, 2, 7, 3, 4, 5]
c0 = L.dmoe_launch_counters()[1]
bench.run_calls(lay, x, dy, alive, resp)
torch.cuda.synchronize()
c1 = L.dmoe_launch_counters()[1]
f(buf, 8 * R * 32)
want = os.environ.get("KERNEL")  # e.g. "128,1,4": BN, SEGK, EPI
for launch in range(c0, c1):
    slot = launch % 8
    t = [[buf[(slot * R + r) * 32 + i] for i in range(32)] for r in range(R)]
    kid, grid = t[8][0], t[8][1]
    bn, segk, epi = kid >> 8, (kid >> 4) & 15, kid & 15
    if want and want != f"{bn},{segk},{epi}":
        continue
    vals = [v for row in t[:8] for v in row if v] + [v for v in t[8][2:6] if v]
    if not vals:
        continue
    t0 = min(vals)
    print(f"== launch {launch - c0}: k_tc_gemm<BN={bn}, SEGK={segk}, EPI={epi}> grid {grid}; CTA 0, us since its first event")
    ent, setup, epi_end, ext = t[8][2], t[8][3], t[8][4], t[8][5]
    if ent:
        us = lambda v: f"{(v - t0) / 1e3:7.2f}" if v else "   -   "
        print(f"   entry(after PDL wait) {us(ent)}  setup done {us(setup)}  epilogue-warp-0 done {us(epi_end)}  exit {us(ext)}")
    for i in range(int(os.environ.get("NT", "12"))):
        if not any(t[r][i] for r in range(8)):
            continue
        print(f"tile {i:2d} " + " ".join(f"{names[r]}={(t[r][i] - t0) / 1e3:7.2f}" if t[r][i] else f"{names[r]}=    -  "
                                         for r in order))
