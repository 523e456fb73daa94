"""Timeline of CTA 0 in the last tcgen05 GEMM of an ABI call (needs DMOE_TC_DEBUG=8)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["DMOE_TC_DEBUG"] = "8"
import torch  # noqa: E402

import bench  # noqa: E402
from gen import CONFIGS  # noqa: E402
from paper_2002_04013_b200 import _lib as L  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "mnist"]
lay, x, dy, alive, resp = bench.build_layer(cfg, 0, torch.device("cuda", 0), cfg.T)
for _ in range(2):
    bench.run_calls(lay, x, dy, alive, resp)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 192)()
f = L._L.dmoe_debug_tc_probe
names = ["prod0", "prodN", "mma0", "mmaC", "epi0", "epiD"]
calls = [
    ("fwd (GEMM2: out)", lambda: L.dmoe_expert_ffn_fwd(lay.xd, lay.offsets, lay.W1, lay.b1, lay.W2, lay.b2, lay.h, lay.out, lay.ws)),
    ("bwd (GEMM6: dW1)", lambda: L.dmoe_expert_ffn_bwd(lay.xd, lay.h, lay.dout, lay.offsets, lay.W1, lay.W2, lay.dxd, lay.dW1, lay.db1, lay.dW2, lay.db2, lay.ws)),
]
for name, fn in calls:
    fn()
    torch.cuda.synchronize()
    f(buf, 192)
    t = [[buf[r * 32 + i] for i in range(32)] for r in range(6)]
    t0 = min(v for row in t for v in row if v)
    print("==", name, "us since first event of CTA 0")
    for i in range(16):
        print(f"tile {i:2d} " + " ".join(f"{names[r]}={(t[r][i] - t0) / 1e3:7.2f}" if t[r][i] else f"{names[r]}=    -  " for r in range(6)))
