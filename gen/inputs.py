"""Host-side synthetic inputs of one layer step (the recipe of gen/configs.py).

Generator output only: every element comes from gen/counter_gen.h; the float64 arrays are
exact upcasts of what the device sees (bf16 bits or fp32).  No method arithmetic.
"""
import numpy as np

import gen


def make_inputs(cfg, seed=0, T=None, experts=None):
    """Host arrays for one step of `cfg`.  Returns dict: for every tensor both the device form
    (`dev_*`: uint16 bf16 bits or float32) and the exact float64 upcast the oracle sees."""
    T = cfg.T if T is None else T
    E, D, H, dM = cfg.E, cfg.D, cfg.H, cfg.dM
    bf = cfg.dtype == "bf16"
    out = {}

    def param(name, tid, n, idx0=0, force_f32=False):
        dist, scale = cfg.dist(tid)
        if bf and not force_f32:
            bits = gen.host_bf16_bits(seed, tid, dist, scale, n, idx0)
            out["dev_" + name] = bits
            return gen.bf16_bits_to_f64(bits)
        v = gen.host_f32(seed, tid, dist, scale, n, idx0)
        out["dev_" + name] = v
        return v.astype(np.float64)

    out["X"] = param("X", gen.X, T * D).reshape(T, D)
    out["Wg"] = param("Wg", gen.WG, D * dM).reshape(D, dM)
    out["bg"] = param("bg", gen.BG, dM, force_f32=True)
    ex = range(cfg.P) if experts is None else experts   # parameter slots (== experts unless tied)
    W1, b1, W2, b2 = [], [], [], []
    dev = {k: [] for k in ("W1", "b1", "W2", "b2")}
    for e in ex:
        W1.append(param("_w1", gen.W1, H * D, e * H * D).reshape(H, D)); dev["W1"].append(out.pop("dev__w1"))
        b1.append(param("_b1", gen.B1, H, e * H, force_f32=True)); dev["b1"].append(out.pop("dev__b1"))
        W2.append(param("_w2", gen.W2, D * H, e * D * H).reshape(D, H)); dev["W2"].append(out.pop("dev__w2"))
        b2.append(param("_b2", gen.B2, D, e * D, force_f32=True)); dev["b2"].append(out.pop("dev__b2"))
    if len(W1):
        out["W1"], out["b1"], out["W2"], out["b2"] = (np.stack(v) for v in (W1, b1, W2, b2))
        for k_, v in dev.items():
            out["dev_" + k_] = np.concatenate(v)
    out["dY"] = param("dY", gen.DY, T * D).reshape(T, D)
    out["alive_bits"] = gen.host_mask(seed, gen.ALIVE, cfg.dead_frac, E)
    out["responded_bits"] = gen.host_mask(seed, gen.RESPONDED, cfg.fail_frac, E)
    out["alive"] = gen.unpack_mask(out["alive_bits"], E)
    out["responded"] = gen.unpack_mask(out["responded_bits"], E)
    return out
