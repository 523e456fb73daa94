"""NEXT-1: the runtime's Backward request with the parameter update fused into the
weight-gradient GEMMs (dmoe_expert_ffn_bwd_sgd) and gradient checkpointing
(h recomputed in the backward), against the oracle's gradient step."""
import numpy as np
import pytest
import torch

from harness import CONFIGS, TOL, gpu_layer, make_inputs, np64, oracle_step, rel_err
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _snap(lay):
    return {n: getattr(lay, n).clone() for n in ("W1", "b1", "W2", "b2")}


@pytest.mark.parametrize("recompute", [False, True])
@pytest.mark.parametrize("name,T", [("mnist", 700), ("mnist", 1), ("stress_tied", 96)])
def test_fused_sgd_step(name, T, recompute):
    cfg = CONFIGS["stress"].with_(pool=8) if name == "stress_tied" else CONFIGS[name]
    inp = make_inputs(cfg, seed=40 + T, T=T)
    lay = gpu_layer(cfg, inp)            # one plain step: dW buffers, dxd
    dxd_ref = lay.dxd.clone()
    ref = oracle_step(cfg, inp, sel_override=np64(lay.sel[:T]))
    scale = max(np.abs(ref["dW1"]).max(), np.abs(ref["dW2"]).max())
    lr = 0.5 / scale if scale > 0 else 1.0   # the update is comparable to the weights themselves
    before = _snap(lay)
    x, dy, alive, resp = lay._inputs
    lay.forward(x, alive, resp)
    lay.backward(dy, sgd_lr=lr, recompute=recompute)
    torch.cuda.synchronize()
    R = int(lay.offsets[cfg.E].item())
    # dxd is computed with the weights before the update: the plain call's bits exactly
    assert torch.equal(lay.dxd[:R], dxd_ref[:R])
    for n, g in (("W1", "dW1"), ("b1", "db1"), ("W2", "dW2"), ("b2", "db2")):
        want = O.sgd_update(np64(before[n]), ref[g], lr)
        got = np64(getattr(lay, n))
        e = rel_err(got - np64(before[n]), want - np64(before[n]))
        # bf16 weights: one rounding of W - lr dW (reading X21): half an ulp of |W| on top of the
        # tolerance of dW itself
        ulp = np.abs(want).max() * 2.0 ** -8 if n in ("W1", "W2") else 0.0
        bound = TOL["bf16"] + ulp / max(np.abs(want - np64(before[n])).max(), 1e-30)
        assert e <= bound, (n, e, bound)
    # slots without rows keep their parameters bit for bit
    seg = np64(lay.seg)
    idle = np.nonzero(np.diff(seg) == 0)[0]
    for i in idle[:4]:
        assert torch.equal(lay.W1[int(i)], before["W1"][int(i)]) and torch.equal(lay.W2[int(i)], before["W2"][int(i)])


def test_recompute_equals_saved_h():
    """Gradient checkpointing changes nothing: recomputing h gives the saved-h update bit for bit."""
    cfg = CONFIGS["mnist"]
    inp = make_inputs(cfg, seed=45, T=1000)
    a, b = gpu_layer(cfg, inp), gpu_layer(cfg, inp)
    for lay, rc in ((a, False), (b, True)):
        x, dy, alive, resp = lay._inputs
        lay.forward(x, alive, resp)
        lay.backward(dy, sgd_lr=1e-2, recompute=rc)
    torch.cuda.synchronize()
    for n in ("W1", "b1", "W2", "b2", "dxd", "dx", "dWg"):
        assert torch.equal(getattr(a, n), getattr(b, n)), n
