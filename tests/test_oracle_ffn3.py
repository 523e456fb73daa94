"""Pins for the oracle of the paper's expert block (NEXT-2: Linear -> LayerNorm ->
ReLU -> Linear -> LayerNorm -> ReLU -> Linear; reading X23): central finite differences of a
scalar loss against every gradient, LayerNorm closed forms, and the whole layer against FD."""
import numpy as np
import pytest

from oracle import oracle as O


def _params(rng, S, D, H, gscale=1.0):
    return {"W1": rng.standard_normal((S, H, D)) / np.sqrt(D), "b1": 0.1 * rng.standard_normal((S, H)),
            "g1": gscale * (1 + 0.3 * rng.standard_normal((S, H))), "be1": 0.2 * rng.standard_normal((S, H)),
            "W2": rng.standard_normal((S, H, H)) / np.sqrt(H), "b2": 0.1 * rng.standard_normal((S, H)),
            "g2": gscale * (1 + 0.3 * rng.standard_normal((S, H))), "be2": 0.2 * rng.standard_normal((S, H)),
            "W3": rng.standard_normal((S, D, H)) / np.sqrt(H), "b3": 0.1 * rng.standard_normal((S, D))}


def test_ffn3_gradients_match_central_differences():
    rng = np.random.default_rng(1)
    S, D, H = 2, 5, 9
    P = _params(rng, S, D, H)
    x = rng.standard_normal((5, D))
    seg = np.array([0, 3, 5], np.int32)
    gy = rng.standard_normal((5, D))
    loss = lambda P_, x_: float((O.ffn3_fwd(x_, seg, P_)[4] * gy).sum())
    z1, a1, z2, a2, out = O.ffn3_fwd(x, seg, P)
    dx, G = O.ffn3_bwd(x, z1, a1, z2, a2, gy, seg, P)
    h = 1e-6
    # ReLU kinks: skip entries whose pre-activation sits within the FD step of 0 (none expected)
    worst = 0.0
    for name in P:
        g = G["d" + name]
        idx = [tuple(rng.integers(0, s) for s in P[name].shape) for _ in range(12)]
        for ix in idx:
            Pp = {k: v.copy() for k, v in P.items()}
            Pm = {k: v.copy() for k, v in P.items()}
            Pp[name][ix] += h
            Pm[name][ix] -= h
            fd = (loss(Pp, x) - loss(Pm, x)) / (2 * h)
            worst = max(worst, abs(fd - g[ix]) / max(1e-3, abs(fd)))
    for ix in [(r, c) for r in range(5) for c in range(D)]:
        xp, xm = x.copy(), x.copy()
        xp[ix] += h
        xm[ix] -= h
        fd = (loss(P, xp) - loss(P, xm)) / (2 * h)
        worst = max(worst, abs(fd - dx[ix]) / max(1e-3, abs(fd)))
    assert worst <= 1e-6, worst


def test_ffn3_layernorm_closed_forms():
    """Constant pre-LN rows (W2 = 0, b2 = c): var = 0, xhat = 0, so a2 = relu(be2) and the block
    output is W3 relu(be2) + b3 whatever x is; LN rows of the first stage are standardised:
    with g1 = 1, be1 = 0 and (here) no ReLU cut, a1 = relu(xhat) where xhat has mean 0 and
    variance var / (var + eps)."""
    rng = np.random.default_rng(2)
    S, D, H = 1, 6, 8
    P = _params(rng, S, D, H)
    P["W2"][:] = 0.0
    P["b2"][:] = 0.7
    x = rng.standard_normal((4, D))
    seg = np.array([0, 4], np.int32)
    z1, a1, z2, a2, out = O.ffn3_fwd(x, seg, P)
    want = P["W3"][0] @ np.maximum(P["be2"][0], 0.0) + P["b3"][0]
    np.testing.assert_allclose(out, np.tile(want, (4, 1)), rtol=0, atol=1e-12)
    P = _params(rng, S, D, H)
    P["g1"][:] = 1.0
    P["be1"][:] = 0.0
    z1, a1, *_ = O.ffn3_fwd(x, seg, P)
    mu, var = z1.mean(1, keepdims=True), z1.var(1, keepdims=True)
    xhat = (z1 - mu) / np.sqrt(var + O.LN_EPS)
    np.testing.assert_allclose(a1, np.maximum(xhat, 0.0), rtol=0, atol=1e-12)
    np.testing.assert_allclose(xhat.mean(1), 0.0, atol=1e-12)
    np.testing.assert_allclose(xhat.var(1), (var / (var + O.LN_EPS)).ravel(), rtol=1e-12)


def test_layer_step_ffn3_end_to_end_fd():
    """The whole DMoE layer with the §4.1 block: d/dX and d/dW_g of sum(y * dY) by central FD with
    routing held fixed (SPEC.md:304 style), 2x3 grid, k = 2."""
    rng = np.random.default_rng(3)
    d, M, k, D, H, T = 2, 3, 2, 5, 7, 6
    E = M ** d
    X = rng.standard_normal((T, D))
    Wg = rng.standard_normal((D, d * M))
    bg = 0.1 * rng.standard_normal(d * M)
    P = _params(rng, E, D, H)
    dY = rng.standard_normal((T, D))
    alive = np.ones(E, np.uint8)
    resp = np.ones(E, np.uint8)
    ref = O.layer_step_ffn3(X, Wg, bg, P, dY, alive, resp, d, M, k, k)
    sel = ref["sel"]

    def loss(X_, Wg_):
        r = O.layer_step_ffn3(X_, Wg_, bg, P, dY, alive, resp, d, M, k, k, sel_override=sel)
        return float((r["y"] * dY).sum())
    h = 1e-6
    worst = 0.0
    for ix in [(t, c) for t in range(T) for c in range(D)]:
        Xp, Xm = X.copy(), X.copy()
        Xp[ix] += h
        Xm[ix] -= h
        fd = (loss(Xp, Wg) - loss(Xm, Wg)) / (2 * h)
        worst = max(worst, abs(fd - ref["dX"][ix]) / max(1e-3, abs(fd)))
    for ix in [(c, j) for c in range(D) for j in range(d * M)]:
        Wp, Wm = Wg.copy(), Wg.copy()
        Wp[ix] += h
        Wm[ix] -= h
        fd = (loss(X, Wp) - loss(X, Wm)) / (2 * h)
        worst = max(worst, abs(fd - ref["dWg"][ix]) / max(1e-3, abs(fd)))
    assert worst <= 1e-5, worst
