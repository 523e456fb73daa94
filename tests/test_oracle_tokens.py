"""Pins for the two oracle entry points the large workloads use instead of the plain
`layer_step` over every expert:

* `layer_step_tokens` (token subsample, weights of the touched experts fetched on demand): on a
  workload small enough for `layer_step`, it must give every token's routing, weights, y, dscore
  and dX exactly as `layer_step` does, and the weight gradients of every touched expert.
* `layer_step(tie=t)`, the declared tied-weight pool (reading X20: expert e computes with slot
  e // t): it must equal the untied layer whose per-expert weights are copies of their slot's,
  with each slot's gradient the sum of its experts' gradients (the gradient of tied parameters).

Neither pin re-runs the function under test: each compares against `layer_step` over a
differently shaped input (all experts materialised, or the pool expanded to one copy per expert).
"""
import numpy as np
import pytest

from gen import CONFIGS
from gen.inputs import make_inputs
from oracle import oracle as O


def _full(cfg, inp, **kw):
    return O.layer_step(inp["X"], inp["Wg"], inp["bg"], inp["W1"], inp["b1"], inp["W2"], inp["b2"], inp["dY"],
                        inp["alive"], inp["responded"], cfg.d, cfg.M, cfg.k, cfg.B, **kw)


@pytest.mark.parametrize("name,seed,T", [("tiny", 0, 32), ("mnist", 1, 96), ("mnist", 2, 1)])
def test_layer_step_tokens_equals_layer_step(name, seed, T):
    cfg = CONFIGS[name].with_(D=64, H=128) if name == "mnist" else CONFIGS[name]
    inp = make_inputs(cfg, seed=seed, T=T)
    full = _full(cfg, inp)
    fetched = []

    def experts(ids):
        fetched.append(np.array(ids))
        return inp["W1"][ids], inp["b1"][ids], inp["W2"][ids], inp["b2"][ids]

    r = O.layer_step_tokens(inp["X"], inp["dY"], inp["Wg"], inp["bg"], experts, inp["alive"], inp["responded"],
                            cfg.d, cfg.M, cfg.k, cfg.B)
    for key in ("sel", "valid"):
        assert np.array_equal(r[key], full[key]), key
    assert r["n_dropped"] == full["n_dropped"]
    for key in ("sel_score", "w", "y", "dscore", "dX", "dWg", "dbg"):
        np.testing.assert_allclose(r[key], full[key], rtol=0, atol=1e-12 * max(1.0, np.abs(full[key]).max()),
                                   err_msg=key)
    used = r["experts"]
    # the touched experts are exactly those with dispatched rows, fetched once in slot order
    assert np.array_equal(used, np.nonzero(full["counts"] > 0)[0])
    assert len(fetched) == 1 and np.array_equal(fetched[0], used)
    for key in ("dW1", "db1", "dW2", "db2"):
        np.testing.assert_allclose(r[key], full[key][used], rtol=0, atol=1e-12 * np.abs(full[key]).max(), err_msg=key)
    # experts nobody selected have zero gradient in the full layer (nothing is lost by skipping them)
    idle = np.setdiff1d(np.arange(cfg.E), used)
    assert not full["dW1"][idle].any() and not full["dW2"][idle].any()


@pytest.mark.parametrize("tie,k,fail", [(4, 4, 0.0), (16, 8, 0.3), (1, 2, 0.1)])
def test_tied_pool_equals_expanded_weights(tie, k, fail):
    cfg = CONFIGS["mnist"].with_(D=32, H=64, k=k, fail_frac=fail, pool=256 // tie)
    inp = make_inputs(cfg, seed=3 + tie, T=80)
    assert inp["W1"].shape[0] == cfg.P == cfg.E // tie
    tied = _full(cfg, inp, tie=tie)
    exp = {k_: np.repeat(inp[k_], tie, axis=0) for k_ in ("W1", "b1", "W2", "b2")}   # slot e // tie per expert
    full = O.layer_step(inp["X"], inp["Wg"], inp["bg"], exp["W1"], exp["b1"], exp["W2"], exp["b2"], inp["dY"],
                        inp["alive"], inp["responded"], cfg.d, cfg.M, cfg.k, cfg.B)
    for key in ("sel", "row_of_slot", "token_of_row", "offsets"):
        assert np.array_equal(tied[key], full[key]), key
    for key in ("y", "dscore", "dX", "dWg", "dbg", "out", "a"):
        np.testing.assert_array_equal(tied[key], full[key], err_msg=key)   # same rows, same weights: same bits
    for key in ("dW1", "db1", "dW2", "db2"):
        summed = full[key].reshape(cfg.P, tie, *full[key].shape[1:]).sum(1)
        np.testing.assert_allclose(tied[key], summed, rtol=0, atol=1e-12 * max(1.0, np.abs(summed).max()), err_msg=key)


def test_sgd_update_closed_form():
    """Gradient descent on L(W) = |W - W*|^2 / 2 (gradient W - W*): lr = 1 lands on W* in one step,
    lr = 1/2 halves the distance, lr = 0 keeps W ("update ... by gradient descent")."""
    rng = np.random.default_rng(0)
    W, Ws = rng.standard_normal((3, 5, 7)), rng.standard_normal((3, 5, 7))
    np.testing.assert_allclose(O.sgd_update(W, W - Ws, 1.0), Ws, rtol=0, atol=1e-15)
    np.testing.assert_allclose(O.sgd_update(W, W - Ws, 0.5) - Ws, (W - Ws) / 2, rtol=0, atol=1e-15)
    assert np.array_equal(O.sgd_update(W, W - Ws, 0.0), W)


def test_backward_only_failures():
    """Reading X22 (SPEC.md:300/305 for PAPER.md:287): an expert lost in the backward only is
    omitted from dx without renormalisation.  Pinned against the full step with that expert's
    input-gradient rows subtracted afterwards, an independent formulation; the gating gradient
    and the forward are unchanged; the lost experts get no parameter gradient."""
    cfg = CONFIGS["mnist"].with_(D=32, H=64, fail_frac=0.1)
    inp = make_inputs(cfg, seed=9, T=120)
    full = _full(cfg, inp)
    rng = np.random.default_rng(2)
    rb = (rng.random(cfg.E) > 0.3).astype(np.uint8)
    part = _full(cfg, inp, responded_bwd=rb)
    for key in ("y", "dscore", "dWg", "dbg", "w", "sel"):
        assert np.array_equal(part[key], full[key]), key
    lost_rows = np.nonzero(rb[np.repeat(np.arange(cfg.E), full["counts"])] == 0)[0]
    assert len(lost_rows) > 0
    want = full["dX"].copy()
    for r in lost_rows:
        want[full["token_of_row"][r]] -= full["dx_rows"][r]
    np.testing.assert_allclose(part["dX"], want, rtol=0, atol=1e-12 * np.abs(full["dX"]).max())
    lost = np.nonzero(rb == 0)[0]
    kept = np.nonzero(rb == 1)[0]
    assert not part["dW1"][lost].any() and not part["dW2"][lost].any() and not part["db1"][lost].any()
    for key in ("dW1", "dW2", "db1", "db2"):
        assert np.array_equal(part[key][kept], full[key][kept]), key
