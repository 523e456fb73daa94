"""Shared test helpers: seeded inputs (gen/), the CUDA path through the C ABI, the oracle.

Inputs come from the counter-based generator only; expected values only from oracle/.
"""
import numpy as np

import gen
from gen import CONFIGS  # noqa: F401
from gen.inputs import make_inputs  # noqa: F401

TOL = {"bf16": 2e-2, "f32": 1e-4}   # north_star: max-abs error relative to max |oracle|
GAP = 1e-3                          # north_star: routing compared where the oracle gap > 1e-3


def to_torch(arr, dtype, shape=None):
    import torch
    arr = np.ascontiguousarray(arr)
    if dtype == "bf16":
        t = torch.from_numpy(arr.view(np.int16)).view(torch.bfloat16)
    else:
        t = torch.from_numpy(arr)
    t = t.cuda()
    return t.reshape(shape) if shape is not None else t


def gpu_layer(cfg, inp, T=None):
    """Run one forward+backward through the C ABI; returns the DMoELayer (buffers hold everything)."""
    import torch
    from paper_2002_04013_b200 import DMoELayer
    T = inp["X"].shape[0] if T is None else T
    dt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    lay = DMoELayer(cfg.d, cfg.M, cfg.k, cfg.D, cfg.H, dtype=dt, beam=cfg.beam, T_max=max(T, 1), pool=cfg.pool,
                    keep_G=True)
    E, D, H, dM = cfg.P, cfg.D, cfg.H, cfg.dM   # parameter slots
    lay.Wg.copy_(to_torch(inp["dev_Wg"], cfg.dtype, (D, dM)))
    lay.bg.copy_(torch.from_numpy(inp["dev_bg"]).cuda())
    lay.W1.copy_(to_torch(inp["dev_W1"], cfg.dtype, (E, H, D)))
    lay.b1.copy_(torch.from_numpy(inp["dev_b1"]).cuda().reshape(E, H))
    lay.W2.copy_(to_torch(inp["dev_W2"], cfg.dtype, (E, D, H)))
    lay.b2.copy_(torch.from_numpy(inp["dev_b2"]).cuda().reshape(E, D))
    x = to_torch(inp["dev_X"], cfg.dtype, (T, D))
    dy = to_torch(inp["dev_dY"], cfg.dtype, (T, D))
    alive = torch.from_numpy(inp["alive_bits"].view(np.int32)).cuda()
    resp = torch.from_numpy(inp["responded_bits"].view(np.int32)).cuda()
    lay._inputs = (x, dy, alive, resp)
    lay.step(x, dy, alive, resp)
    torch.cuda.synchronize()
    return lay


def np64(t):
    import torch
    return t.detach().to(torch.float64).cpu().numpy() if t.dtype != torch.int32 else t.cpu().numpy()


def rel_err(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    den = np.abs(want).max() if want.size else 0.0
    num = np.abs(got - want).max() if want.size else 0.0
    return num / den if den > 0 else num


def oracle_step(cfg, inp, sel_override=None):
    from oracle import oracle as O
    return O.layer_step(inp["X"], inp["Wg"], inp["bg"], inp["W1"], inp["b1"], inp["W2"], inp["b2"],
                        inp["dY"], inp["alive"], inp["responded"], cfg.d, cfg.M, cfg.k, cfg.B,
                        sel_override=sel_override, tie=cfg.tie)


def check_routing(cfg, gsel, ref, exact, alive):
    """sel must equal the oracle's on every token (exact-grid) or where gap > GAP (continuous);
    elsewhere the GPU's choice must be a valid alternative: alive experts whose oracle Eq. 2
    scores are within GAP of the oracle's slot scores.  Returns the #tokens compared."""
    from oracle import oracle as O
    osel, gap = ref["sel"], ref["gap"]
    mask = np.ones(len(gap), bool) if exact else gap > GAP
    bad = np.nonzero((gsel != osel).any(1) & mask)[0]
    assert len(bad) == 0, f"routing mismatch on tokens {bad[:10]}: gpu {gsel[bad[:3]]} oracle {osel[bad[:3]]}"
    rest = np.nonzero(~mask & (gsel != osel).any(1))[0]
    if len(rest):
        s_gpu = O._scores_of(ref["G"][rest], gsel[rest], cfg.d, cfg.M)
        assert np.all(np.abs(np.where(gsel[rest] >= 0, s_gpu, 0) - np.where(osel[rest] >= 0, ref["sel_score"][rest], 0)) <= 2 * GAP)
        chosen = gsel[rest][gsel[rest] >= 0]
        assert np.all(alive[chosen] == 1)
        assert ((gsel[rest] >= 0).sum(1) == (osel[rest] >= 0).sum(1)).all()
    return int(mask.sum())
