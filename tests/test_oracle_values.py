"""Pins for the oracle's value half: Eq. 3 weights (S4), dispatch (S5), expert FFN (S6/S9),
combine (S7/S8), gate backward (S10) and the whole layer against central finite differences.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


# ------------------------------------------------------------------ S4 weights
def test_weights_ln7_ln3_and_failure():
    g = GOLD["aggregate_ln7_ln3"]
    sel = np.array([[0, 1]], np.int32)
    sc = np.array([g["scores"]])
    w, ok, valid, nd = O.weights(sel, sc, np.ones(2, np.uint8))
    np.testing.assert_allclose(w[0], g["w"], rtol=1e-14)
    w, ok, valid, nd = O.weights(sel, sc, np.array([1, 0], np.uint8))   # second expert failed
    assert w[0].tolist() == g["w_second_failed"] and ok[0].tolist() == [1, 0] and valid[0] == 1


def test_weights_equal_and_saturation():
    g = GOLD["aggregate_equal"]
    w, *_ = O.weights(np.array([[0, 1, 2]], np.int32), np.array([g["scores"]]), np.ones(3, np.uint8))
    np.testing.assert_allclose(w[0], g["w"], rtol=1e-15)
    g = GOLD["aggregate_saturation"]
    w, *_ = O.weights(np.array([[0, 1]], np.int32), np.array([g["scores"]]), np.ones(2, np.uint8))
    assert w[0, 1] >= g["min_w_second"] and np.isfinite(w).all()


def test_weights_sum_to_one_and_shift_invariant():
    rng = np.random.default_rng(3)
    T, k, E = 200, 5, 40
    sel = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    sc = rng.integers(-64, 64, (T, k)) / 8.0         # multiples of 1/8: shifts are exact
    resp = (rng.random(E) < 0.7).astype(np.uint8)
    w, ok, valid, nd = O.weights(sel, sc, resp)
    s = w.sum(1)
    assert np.all(np.abs(s[valid == 1] - 1) <= 1e-12)
    assert np.all(w[ok == 0] == 0) and np.all(s[valid == 0] == 0)
    assert nd == int((valid == 0).sum())
    w2, *_ = O.weights(sel, sc + 37.0, resp)
    assert np.array_equal(w, w2)                         # SPEC.md:310, bit for bit


def test_drop_equals_renormalise_without_it():
    """North star / SPEC.md:309: a non-responding expert == Eq. 3 recomputed over the survivors."""
    rng = np.random.default_rng(4)
    T, k, E = 100, 4, 30
    sel = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    sc = rng.standard_normal((T, k))
    resp = np.ones(E, np.uint8)
    dead = 7
    resp_d = resp.copy()
    resp_d[dead] = 0
    w_fail, *_ = O.weights(sel, sc, resp_d)
    # same tokens, with the dead expert's slot simply removed from the selection (-1 pad)
    sel_rm = np.where(sel == dead, -1, sel).astype(np.int32)
    w_rm, *_ = O.weights(sel_rm, sc, resp)
    assert np.array_equal(w_fail, w_rm)


def test_all_crashed_drops_token():
    sel = np.array([[3, 4], [1, 2]], np.int32)
    w, ok, valid, nd = O.weights(sel, np.zeros((2, 2)), np.array([1, 1, 1, 0, 0], np.uint8))
    assert valid.tolist() == [0, 1] and nd == 1 and (w[0] == 0).all()


# ------------------------------------------------------------------ S5 dispatch
def test_dispatch_is_stable_sort():
    rng = np.random.default_rng(5)
    for T, k, E in [(1, 1, 1), (50, 4, 16), (300, 3, 7), (64, 8, 100)]:
        sel = np.stack([rng.permutation(E)[:k] if E >= k else rng.integers(0, E, k) for _ in range(T)]).astype(np.int32)
        ok = (rng.random((T, k)) < 0.8).astype(np.uint8)
        counts, offsets, ros, tor = O.dispatch(sel, ok, E)
        q = np.nonzero(ok.ravel())[0]                       # ok pairs in increasing pair index t*k+s
        order = q[np.argsort(sel.ravel()[q], kind="stable")]  # library stable sort by expert
        assert counts.tolist() == np.bincount(sel.ravel()[q], minlength=E).tolist()
        assert offsets[0] == 0 and np.array_equal(np.diff(offsets), counts)
        assert tor.tolist() == (order // k).tolist()
        want_ros = -np.ones(T * k, np.int64)
        want_ros[order] = np.arange(len(order))
        assert ros.ravel().tolist() == want_ros.tolist()


# ----------------------------------------------------------------- S6 / S9 FFN
def _ffn_params(rng, S, D, H, scale=1.0):
    return (rng.standard_normal((S, H, D)) * scale, rng.standard_normal((S, H)) * scale,
            rng.standard_normal((S, D, H)) * scale, rng.standard_normal((S, D)) * scale)


def test_ffn_zero_and_identity():
    rng = np.random.default_rng(6)
    x = rng.standard_normal((5, 4))
    seg = np.array([0, 2, 5], np.int32)
    z = np.zeros
    a, out = O.ffn_fwd(x, seg, z((2, 6, 4)), z((2, 6)), z((2, 4, 6)), z((2, 4)))
    assert (out == 0).all() and (a == 0).all()
    I = np.stack([np.eye(3)] * 2)
    xp = np.abs(rng.standard_normal((4, 3))) + 0.1
    a, out = O.ffn_fwd(xp, np.array([0, 1, 4], np.int32), I, z((2, 3)), I, z((2, 3)))
    assert np.array_equal(out, xp)                        # SPEC.md:42 identity case


def test_ffn_backward_zero_cotangent_and_linear_case():
    rng = np.random.default_rng(7)
    S, D, H, R = 2, 4, 6, 5
    W1, b1, W2, b2 = _ffn_params(rng, S, D, H)
    seg = np.array([0, 3, 5], np.int32)
    x = rng.standard_normal((R, D))
    a, out = O.ffn_fwd(x, seg, W1, b1, W2, b2)
    dx, dW1, db1, dW2, db2 = O.ffn_bwd(x, a, np.zeros((R, D)), seg, W1, W2)
    assert all((v == 0).all() for v in (dx, dW1, db1, dW2, db2))
    # linear regime (all pre-activations > 0): dx = W1^T W2^T g
    b1p = np.full((S, H), 1e3)
    a, out = O.ffn_fwd(x, seg, W1, b1p, W2, b2)
    assert (a > 0).all()
    g = rng.standard_normal((R, D))
    dx, *_ = O.ffn_bwd(x, a, g, seg, W1, W2)
    for r in range(R):
        s = 0 if r < 3 else 1
        np.testing.assert_allclose(dx[r], W1[s].T @ (W2[s].T @ g[r]), rtol=1e-12, atol=1e-12)


def test_ffn_backward_finite_differences():
    rng = np.random.default_rng(8)
    S, D, H, R = 2, 3, 5, 4
    W1, b1, W2, b2 = _ffn_params(rng, S, D, H)
    seg = np.array([0, 1, 4], np.int32)
    x = rng.standard_normal((R, D))
    g = rng.standard_normal((R, D))
    a, _ = O.ffn_fwd(x, seg, W1, b1, W2, b2)
    dx, dW1, db1, dW2, db2 = O.ffn_bwd(x, a, g, seg, W1, W2)
    L = lambda *p: float((O.ffn_fwd(p[0], seg, *p[1:])[1] * g).sum())
    params = [x, W1, b1, W2, b2]
    grads = [dx, dW1, db1, dW2, db2]
    h = 1e-5
    for pi, (P, dP) in enumerate(zip(params, grads)):
        for idx in np.ndindex(P.shape):
            Pp, Pm = P.copy(), P.copy()
            Pp[idx] += h
            Pm[idx] -= h
            ap = [Pp if j == pi else params[j] for j in range(5)]
            am = [Pm if j == pi else params[j] for j in range(5)]
            fd = (L(*ap) - L(*am)) / (2 * h)
            assert abs(fd - dP[idx]) <= 1e-6 * max(1.0, abs(fd)), (pi, idx, fd, dP[idx])


# ------------------------------------------------------------- whole layer
def _tiny_layer(seed, T=12, D=5, H=7, M=3, d=2, k=3, fail=()):
    rng = np.random.default_rng(seed)
    E = M ** d
    X = rng.standard_normal((T, D))
    Wg = rng.standard_normal((D, d * M))
    bg = rng.standard_normal(d * M) * 0.1
    W1, b1, W2, b2 = _ffn_params(rng, E, D, H, 0.5)
    dY = rng.standard_normal((T, D))
    alive = np.ones(E, np.uint8)
    resp = np.ones(E, np.uint8)
    resp[list(fail)] = 0
    return dict(X=X, Wg=Wg, bg=bg, W1=W1, b1=b1, W2=W2, b2=b2, dY=dY, alive=alive,
                responded=resp, d=d, M=M, k=k, B=k)


def test_layer_all_experts_identical():
    """Identical experts: y = f(x) for every valid token (weights sum to 1), dscore = 0."""
    p = _tiny_layer(9, fail=(1, 4))
    for n in ("W1", "b1", "W2", "b2"):
        p[n] = np.broadcast_to(p[n][:1], p[n].shape).copy()
    r = O.layer_step(**p)
    _, f = O.ffn_fwd(p["X"], np.array([0, len(p["X"])], np.int32), p["W1"][:1], p["b1"][:1], p["W2"][:1], p["b2"][:1])
    v = r["valid"] == 1
    np.testing.assert_allclose(r["y"][v], f[v], rtol=1e-12, atol=1e-12)
    assert np.abs(r["dscore"]).max() < 1e-12
    # dG row sums vanish -> db_g sums to 0 within each grid dimension
    M, d = p["M"], p["d"]
    assert np.abs(r["dbg"].reshape(d, M).sum(1)).max() < 1e-12


def test_layer_single_ok_slot_has_no_gate_gradient():
    p = _tiny_layer(10, k=1)
    r = O.layer_step(**p)
    assert (r["dscore"] == 0).all() and (r["dbg"] == 0).all() and (r["dWg"] == 0).all()
    # k=1 with a healthy expert: y == f(x) exactly
    for t in range(len(p["X"])):
        e = r["sel"][t, 0]
        _, f = O.ffn_fwd(p["X"][t:t + 1], np.array([0, 1], np.int32), p["W1"][e:e + 1], p["b1"][e:e + 1],
                         p["W2"][e:e + 1], p["b2"][e:e + 1])
        assert np.array_equal(r["y"][t], f[0])


def test_layer_dG_rows_sum_to_zero():
    p = _tiny_layer(11, fail=(2,))
    r = O.layer_step(**p)
    d, M = p["d"], p["M"]
    assert np.abs(r["dscore"].sum(1)).max() < 1e-12
    assert np.abs(r["dbg"].reshape(d, M).sum(1)).max() < 1e-12


@pytest.mark.parametrize("seed,fail", [(12, ()), (13, (0, 5))])
def test_layer_backward_finite_differences(seed, fail):
    """End-to-end central FD in float64 with routing held fixed: rel err <= 1e-5."""
    p = _tiny_layer(seed, fail=fail)
    r = O.layer_step(**p)
    sel0 = r["sel"]
    dY = p["dY"]

    def loss(q):
        rr = O.layer_step(**q, sel_override=sel0)
        return float((rr["y"] * dY).sum())

    h = 1e-6
    checked = 0
    for name, gname in [("X", "dX"), ("Wg", "dWg"), ("bg", "dbg"), ("W1", "dW1"), ("b1", "db1"),
                        ("W2", "dW2"), ("b2", "db2")]:
        P = p[name]
        G = r[gname]
        for idx in list(np.ndindex(P.shape))[:: max(1, P.size // 40)]:
            qp, qm = dict(p), dict(p)
            qp[name] = P.copy(); qp[name][idx] += h
            qm[name] = P.copy(); qm[name][idx] -= h
            # skip entries whose perturbation would change the routing or cross a ReLU kink
            if not (np.array_equal(O.layer_step(**qp)["sel"], sel0) and np.array_equal(O.layer_step(**qm)["sel"], sel0)):
                continue
            ap = O.layer_step(**qp, sel_override=sel0)["a"]
            am = O.layer_step(**qm, sel_override=sel0)["a"]
            if not np.array_equal(ap > 0, am > 0):
                continue
            fd = (loss(qp) - loss(qm)) / (2 * h)
            assert abs(fd - G[idx]) <= 1e-5 * max(1.0, abs(fd)), (name, idx, fd, G[idx])
            checked += 1
    assert checked > 100
