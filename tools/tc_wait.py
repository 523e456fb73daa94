"""Where the tcgen05 GEMMs' pipeline roles spend their cycles (DMOE_TC_DEBUG=64 | 8): per launch of
one layer step, cycles summed over all CTAs, as a share of each role's loop time.

  python tools/tc_wait.py mnist           (DBG=<extra flags>, e.g. DBG=7 to strip the pipeline)
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["DMOE_TC_DEBUG"] = str(8 | 64 | int(os.environ.get("DBG", "0")))
import torch  # noqa: E402

import bench  # noqa: E402
from gen import CONFIGS  # noqa: E402
from paper_2002_04013_b200 import _lib as L  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "mnist"]
if len(sys.argv) > 2:  # overrides key=int, e.g. M=16 T=4096 (a transformer-shaped slice)
    cfg = cfg.with_(**{kv.split("=")[0]: int(kv.split("=")[1]) for kv in sys.argv[2:]})
lay, x, dy, alive, resp = bench.build_layer(cfg, 0, torch.device("cuda", 0), cfg.T)
for _ in range(2):
    bench.run_calls(lay, x, dy, alive, resp)
w = (ctypes.c_ulonglong * (8 * 20))()
L._L.dmoe_debug_tc_wait(w, 1)
c0 = L.dmoe_launch_counters()[1]
bench.run_calls(lay, x, dy, alive, resp)
c1 = L.dmoe_launch_counters()[1]
L._L.dmoe_debug_tc_wait(w, 0)
R = 9
pb = (ctypes.c_ulonglong * (8 * R * 32))()
L._L.dmoe_debug_tc_probe(pb, 8 * R * 32)
for launch in range(c0, c1):
    s = launch % 8
    v = [w[s * 20 + i] for i in range(20)]
    kid = pb[(s * R + 8) * 32]
    bn, segk, epi = kid >> 8, (kid >> 4) & 15, kid & 15
    ctas, tiles = max(v[11], 1), max(v[10], 1)
    f = lambda a, b: f"{100 * a / max(b, 1):5.1f}%"
    print(f"launch {launch - c0} k_tc_gemm<BN={bn}, SEGK={segk}, EPI={epi}>: {ctas} CTAs, {tiles} MMA tiles, "
          f"loop {v[6] / ctas / 1965:.1f} us/CTA @1965MHz, {v[6] / tiles:.0f} cyc/tile")
    print(f"   producer: empty-wait {f(v[0], v[1])}")
    print(f"   mma     : tempty-wait {f(v[2], v[6])} full-wait {f(v[3], v[6])} zeroing {f(v[4], v[6])} "
          f"issue+commit {f(v[5], v[6])}  (per tile: tempty {v[2] / tiles:.0f} full {v[3] / tiles:.0f} "
          f"zero {v[4] / tiles:.0f} issue {v[5] / tiles:.0f} (mma only {v[12] / tiles:.0f}) cyc)")
    if v[14]:
        print(f"   fix-up  : full-wait {f(v[13], v[14])} colsum {f(v[15], v[14])}")
    print(f"   epilogue: tfull-wait {f(v[7], v[9])} store-read-wait {f(v[8], v[9])} tmem-load {f(v[16], v[9])} "
          f"pack+stage {f(v[17], v[9])} store-issue {f(v[18], v[9])}  (per tile: {v[9] / tiles:.0f} cyc)")
