"""Pins for the oracle's routing half: gate scores (S1), FilterAlive (S2), Alg. 1 (S3).

Each pin checks the oracle against something other than itself: a hand sum or worked
example (tests/golden, cited), an independent library routine (numpy matmul), brute
force over all M^d experts, or a closed-form property.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


def _alive(E, dead):
    a = np.ones(E, np.uint8)
    a[list(dead)] = 0
    return a


def brute_topk(Grow, d, M, k, alive):
    """Exhaustive top-k over all alive experts; score summed in Alg. 1's order (0 + g_0 + ...)."""
    items = []
    for uid in itertools.product(range(M), repeat=d):
        e = 0
        for u in uid:
            e = e * M + u
        if not alive[e]:
            continue
        s = 0.0
        for i, u in enumerate(uid):
            s = s + Grow[i * M + u]
        items.append((-s, e, s))
    items.sort()
    return [e for _, e, _ in items[:k]], [s for _, _, s in items[:k]]


# ---------------------------------------------------------------- S1 gate scores
def test_gate_hand_sum():
    g = GOLD["gate_hand_sum"]
    # linear gate with D=1, x=[1], W_g = the g vector, b_g = 0 -> G = g (Eq. 2)
    G = O.gate_scores(np.ones((1, 1)), np.array([g["g"]]), np.zeros(4))
    assert G.tolist() == [g["g"]]
    u0, u1 = g["uid"]
    assert G[0, 0 * 2 + u0] + G[0, 1 * 2 + u1] == g["score"]


def test_gate_vs_numpy_matmul():
    rng = np.random.default_rng(0)
    for T, D, dM in [(1, 1, 2), (7, 13, 8), (33, 64, 48), (5, 300, 32)]:
        X = rng.standard_normal((T, D))
        Wg = rng.standard_normal((D, dM))
        bg = rng.standard_normal(dM)
        G = O.gate_scores(X, Wg, bg)
        np.testing.assert_allclose(G, X @ Wg + bg, rtol=1e-12, atol=1e-12)


def test_gate_zero_params_all_tie():
    G = O.gate_scores(np.random.default_rng(1).standard_normal((3, 5)), np.zeros((5, 6)), np.zeros(6))
    assert (G == 0).all()
    # every expert ties -> the total order (reading X4) returns the lowest flat indices
    sel, sc, gap = O.select_experts(G, 2, 3, 4, 4, np.ones(9, np.uint8))
    assert sel.tolist() == [[0, 1, 2, 3]] * 3
    assert (sc == 0).all() and (gap == 0).all()


# ------------------------------------------------------------- S2 FilterAlive
def test_prefix_alive_definition():
    rng = np.random.default_rng(2)
    for d, M in [(1, 5), (2, 3), (3, 4)]:
        E = M ** d
        alive = (rng.random(E) < 0.4).astype(np.uint8)
        PA = O.prefix_alive(alive, d, M)
        for i in range(d):
            for p in range(M ** (i + 1)):
                # brute force: any alive uid whose first i+1 coordinates spell p
                want = any(alive[e] and (e // M ** (d - 1 - i)) == p for e in range(E))
                assert PA[i][p] == want
        assert (PA[d - 1] == alive).all()


# ------------------------------------------------------------------- S3 Alg. 1
@pytest.mark.parametrize("case", ["beam_all_alive_k1", "beam_masked_B2", "beam_masked_B1_derived"])
def test_beam_worked_examples(case):
    g = GOLD[case]
    E = g["M"] ** g["d"]
    sel, sc, _ = O.select_experts(np.array([g["g"]]), g["d"], g["M"], g["k"], g["B"], _alive(E, g["dead"]))
    assert sel[0].tolist() == g["sel"]
    assert sc[0].tolist() == g["score"]


@pytest.mark.parametrize("d,M", [(1, 8), (2, 2), (2, 5), (2, 8), (3, 3), (3, 4)])
@pytest.mark.parametrize("tied", [False, True])
def test_beam_equals_bruteforce_all_alive(d, M, tied):
    """All alive: Alg. 1 with any B >= k is exact top-k (closed argument)."""
    rng = np.random.default_rng(d * 100 + M + 7 * tied)
    T = 60
    G = rng.integers(-2, 3, (T, d * M)).astype(np.float64) if tied else rng.standard_normal((T, d * M))
    E = M ** d
    alive = np.ones(E, np.uint8)
    for k in sorted({1, 2, min(4, E), min(7, E)}):
        for B in sorted({k, k + 1, 2 * k}):
            sel, sc, _ = O.select_experts(G, d, M, k, B, alive)
            for t in range(T):
                be, bs = brute_topk(G[t], d, M, k, alive)
                assert sel[t].tolist() == be, (k, B, t)
                assert sc[t].tolist() == bs


@pytest.mark.parametrize("d,M", [(2, 3), (2, 5), (3, 3), (3, 4)])
def test_beam_wide_equals_bruteforce_masked(d, M):
    """With B >= #alive prefixes at every level, Alg. 1 = brute force over alive."""
    rng = np.random.default_rng(11 * d + M)
    E = M ** d
    for trial in range(25):
        alive = (rng.random(E) < rng.uniform(0.1, 0.9)).astype(np.uint8)
        G = rng.standard_normal((4, d * M))
        k = int(rng.integers(1, 5))
        sel, sc, _ = O.select_experts(G, d, M, k, max(E, k), alive)
        for t in range(4):
            be, bs = brute_topk(G[t], d, M, k, alive)
            assert sel[t, :len(be)].tolist() == be
            assert (sel[t, len(be):] == -1).all() and np.isneginf(sc[t, len(be):]).all()
            assert len(be) == min(k, int(alive.sum()))


def test_beam_final_size_is_min_k_alive():
    """Reading X6: the beam never shrinks below min(k, #alive) (DESIGN.md proof)."""
    rng = np.random.default_rng(5)
    for trial in range(200):
        d, M = int(rng.integers(1, 4)), int(rng.integers(2, 5))
        E = M ** d
        alive = (rng.random(E) < rng.uniform(0.0, 0.6)).astype(np.uint8)
        k = int(rng.integers(1, 6))
        sel, sc, _ = O.select_experts(rng.standard_normal((1, d * M)), d, M, k, k, alive)
        n = int((sel[0] >= 0).sum())
        assert n == min(k, int(alive.sum()))
        assert all(alive[e] for e in sel[0] if e >= 0)                 # only alive experts
        assert len(set(sel[0][sel[0] >= 0].tolist())) == n             # distinct
        assert (np.diff(sc[0][:n]) <= 0).all()                          # scores non-increasing


def test_beam_k1_B1_separable_argmax():
    """all alive, k = B = 1 -> per-dimension argmax (greedy is exact for additive scores)."""
    rng = np.random.default_rng(6)
    d, M = 3, 6
    G = rng.standard_normal((50, d * M))
    sel, sc, _ = O.select_experts(G, d, M, 1, 1, np.ones(M ** d, np.uint8))
    for t in range(50):
        e = 0
        for i in range(d):
            e = e * M + int(np.argmax(G[t, i * M:(i + 1) * M]))
        assert sel[t, 0] == e


def test_beam_score_is_eq2_sum():
    rng = np.random.default_rng(8)
    d, M, k = 3, 5, 4
    G = rng.standard_normal((20, d * M))
    sel, sc, _ = O.select_experts(G, d, M, k, k, np.ones(M ** d, np.uint8))
    for t in range(20):
        for s in range(k):
            e = sel[t, s]
            uid = [(e // M ** (d - 1 - i)) % M for i in range(d)]
            assert math.isclose(sc[t, s], sum(G[t, i * M + u] for i, u in enumerate(uid)), rel_tol=0, abs_tol=1e-14)


def test_beam_monotone_in_width():
    """SPEC.md:246 property: a wider beam never lowers the best returned score."""
    rng = np.random.default_rng(9)
    for trial in range(100):
        d, M = 3, 4
        alive = (rng.random(M ** d) < 0.3).astype(np.uint8)
        if not alive.any():
            continue
        G = rng.standard_normal((1, d * M))
        best = [O.select_experts(G, d, M, 1, B, alive)[1][0, 0] for B in (1, 2, 4, 8, 64)]
        assert all(b2 >= b1 for b1, b2 in zip(best, best[1:]))


def test_gap_definition():
    # sorted last-level candidates 3.0, 2.5, 2.5, ... -> adjacent tie among the top k -> gap 0
    G = np.array([[0.0, 0.0, 3.0, 2.5, 2.5, 1.0]])  # d=2, M=3
    sel, sc, gap = O.select_experts(G, 2, 3, 2, 3, np.ones(9, np.uint8))
    assert gap[0] == 0.0
    assert sel[0].tolist() == [2 * 3 + 0, 2 * 3 + 1]  # tie 5.5/5.5 broken by lower flat index
    G2 = np.array([[0.0, -5.0, 3.0, 2.0, 0.5]])  # d=1, M=5
    _, _, gap2 = O.select_experts(G2, 1, 5, 2, 2, np.ones(5, np.uint8))
    assert gap2[0] == 1.0  # min(3-2, 2-0.5)


@pytest.mark.parametrize("d,M,k,dead,seed", [(2, 4, 3, 0.4, 0), (3, 3, 4, 0.5, 1), (2, 6, 5, 0.2, 2), (1, 9, 4, 0.3, 3)])
def test_topk_exact_equals_wide_beam(d, M, k, dead, seed):
    """The exact alive top-k (the plain definition) equals Alg. 1 run with a beam at least as wide
    as the number of prefixes at every level (reading X3: then no alive prefix is ever cut), with
    integer-valued scores full of exact ties (X4 order), and on every all-dead / fully-alive case."""
    rng = np.random.default_rng(seed)
    E = M ** d
    T = 300
    G = rng.integers(-3, 4, (T, d * M)).astype(np.float64)
    for alive in [(rng.random(E) >= dead).astype(np.uint8), np.ones(E, np.uint8), np.zeros(E, np.uint8)]:
        sel_x, sc_x = O.topk_exact(G, d, M, k, alive)
        B = max(k, M ** max(d - 1, 1))
        sel_b, sc_b, _ = O.select_experts(G, d, M, k, B, alive)
        assert np.array_equal(sel_x, sel_b)
        np.testing.assert_array_equal(sc_x, sc_b)
