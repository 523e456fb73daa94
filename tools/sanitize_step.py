"""One small layer step of each path for compute-sanitizer (SURVEY.md §5 policy: memcheck,
racecheck, synccheck, initcheck on config 1): tiny fp32 (SIMT path), an MNIST-shaped bf16 step
(tcgen05 GEMMs, fused gate + top-k, dispatch, combine, gate backward) and its fused-SGD
backward with recomputed h."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from harness import CONFIGS, gpu_layer, make_inputs  # noqa: E402

for name, T in (("tiny", 32), ("mnist", 256)):
    cfg = CONFIGS[name]
    inp = make_inputs(cfg, seed=3, T=T)
    lay = gpu_layer(cfg, inp)
    if name == "mnist":
        x, dy, alive, resp = lay._inputs
        lay.forward(x, alive, resp)
        lay.backward(dy, sgd_lr=1e-3, recompute=True)
    torch.cuda.synchronize()
    print(name, "ok", flush=True)
