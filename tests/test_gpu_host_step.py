"""dmoe_layer_step_host (include/dmoe.h): one whole layer step from host buffers through the C ABI
equals the per-call path (the layer's Python sequencing of the same entry points) bit for bit —
the calls, their order and their inputs are the same, and every kernel is deterministic — and the
per-call path itself is what the oracle parity tests check."""
import pytest
import torch

from harness import CONFIGS, gpu_layer, make_inputs

pytestmark = pytest.mark.gpu

OUT = ("y", "dx", "dW1", "db1", "dW2", "db2", "dWg", "dbg", "sel", "w", "offsets")


@pytest.mark.parametrize("name,T,T_run", [("mnist", 700, 700), ("mnist", 700, 333), ("mnist_pool8", 700, 700),
                                          ("tiny", 32, 32)])
def test_host_step_equals_per_call_path(name, T, T_run):
    cfg = {"mnist_pool8": CONFIGS["mnist"].with_(pool=8)}.get(name, CONFIGS.get(name))
    inp = make_inputs(cfg, seed=70 + T_run, T=T)
    lay = gpu_layer(cfg, inp)
    x, dy, alive, resp = lay._inputs
    x, dy = x[:T_run], dy[:T_run]
    lay.step(x, dy, alive, resp)             # the per-call path at T_run
    torch.cuda.synchronize()
    ref = {n: getattr(lay, n).clone() for n in OUT}
    for n in ("y", "dx", "dWg", "dW1"):      # make sure the host step really writes them
        getattr(lay, n).fill_(float("nan") if getattr(lay, n).is_floating_point() else 0)
    hx = x.cpu().pin_memory()
    hdy = dy.cpu().pin_memory()
    hy = torch.empty_like(hx).pin_memory()
    hdx = torch.empty_like(hx).pin_memory()
    desc = lay.host_desc(alive, resp)
    lay.step_host_c(desc, hx, hdy, hy, hdx)
    torch.cuda.synchronize()
    assert torch.equal(hy, ref["y"][:T_run].cpu())
    assert torch.equal(hdx, ref["dx"][:T_run].cpu())
    for n in OUT:
        got, want = getattr(lay, n), ref[n]
        if n in ("y", "dx"):
            got, want = got[:T_run], want[:T_run]
        assert torch.equal(got, want), n


def test_check_finite_switch():
    """dmoe_set_check_finite(1): a NaN reaching an output is reported as DMOE_ERR_NONFINITE (the
    gate scores of a token with a NaN input); finite steps pass; off by default."""
    from paper_2002_04013_b200 import _lib as L
    cfg = CONFIGS["mnist"]
    inp = make_inputs(cfg, seed=77, T=300)
    lay = gpu_layer(cfg, inp)
    x, dy, alive, resp = lay._inputs
    L.dmoe_set_check_finite(True)
    try:
        lay.step(x, dy, alive, resp)          # finite: every checked output passes
        bad = x.clone()
        bad[5, 3] = float("nan")
        with pytest.raises(L.DMoEError) as ei:
            lay.forward(bad, alive, resp)
        assert ei.value.status == -5 and "non-finite" in str(ei.value)
    finally:
        L.dmoe_set_check_finite(False)
    lay.forward(bad, alive, resp)             # switch off: no check, no error
    torch.cuda.synchronize()
