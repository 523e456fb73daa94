"""ctypes front end of the float64 DMoE oracle (oracle/dmoe_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg may import this module.  It shares nothing
with the CUDA path (paper_2002_04013_b200/) and never imports it.

Every function takes/returns float64 numpy arrays (bf16 inputs are upcast exactly by
the caller) and follows the step of the same name in dmoe_oracle.c, which cites the
paper passage it implements.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None

_d = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i32 = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u8 = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_I64, _I32 = ctypes.c_int64, ctypes.c_int32


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make` (or __graft_entry__.build())")
        L = ctypes.CDLL(path)
        L.oracle_gate_scores.argtypes = [_d, _I64, _I32, _d, _d, _I32, _d]
        L.oracle_prefix_alive.argtypes = [_u8, _I32, _I32, _u8]
        L.oracle_select_experts.argtypes = [_d, _I64, _I32, _I32, _I32, _I32, _u8, _i32, _d,
                                            ctypes.c_void_p]
        L.oracle_weights.argtypes = [_i32, _d, _I64, _I32, _u8, _d, _u8, _u8]
        L.oracle_weights.restype = ctypes.c_int64
        L.oracle_dispatch.argtypes = [_i32, _u8, _I64, _I32, _I64, _i32, _i32, _i32, _i32]
        L.oracle_dispatch.restype = ctypes.c_int64
        L.oracle_ffn_fwd.argtypes = [_d, _i32, _I32, _I32, _I32, _d, _d, _d, _d, _d, _d]
        L.oracle_combine.argtypes = [_d, _i32, _d, _I64, _I32, _I32, _d]
        L.oracle_combine_bwd.argtypes = [_d, _d, _i32, _d, _I64, _I32, _I32, _d, _d]
        L.oracle_ffn_bwd.argtypes = [_d, _d, _d, _i32, _I32, _I32, _I32, _d, _d,
                                     _d, _d, _d, _d, _d]
        L.oracle_ffn3_fwd.argtypes = [_d, _i32, _I32, _I32, _I32] + [_d] * 10 + [ctypes.c_double] + [_d] * 5 + [
            ctypes.c_void_p] * 2
        L.oracle_ffn3_bwd.argtypes = ([_d] * 6 + [_i32, _I32, _I32, _I32] + [_d] * 7 + [ctypes.c_double]
                                      + [_d] * 11 + [ctypes.c_void_p] * 2)
        L.oracle_gate_bwd.argtypes = [_d, _d, _i32, _d, _d, _i32, _I64, _I32, _I32, _I32, _I32,
                                      _d, _d, _d]
        _lib = L
    return _lib


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def gate_scores(X, Wg, bg):
    """S1, Eq. 2: G = X Wg + bg, [T, d*M]."""
    X, Wg, bg = _c(X, np.float64), _c(Wg, np.float64), _c(bg, np.float64)
    T, D = X.shape
    dM = Wg.shape[1]
    G = np.empty((T, dM), np.float64)
    lib().oracle_gate_scores(X, T, D, Wg, bg, dM, G)
    return G


def prefix_alive(alive, d, M):
    """S2, FilterAlive prefixes. Returns list of d uint8 arrays, level i has M^(i+1)."""
    alive = _c(alive, np.uint8)
    n = sum(M ** (i + 1) for i in range(d))
    PA = np.empty(n, np.uint8)
    lib().oracle_prefix_alive(alive, d, M, PA)
    out, off = [], 0
    for i in range(d):
        out.append(PA[off:off + M ** (i + 1)])
        off += M ** (i + 1)
    return out


def select_experts(G, d, M, k, B, alive):
    """S3, Algorithm 1 with FilterAlive from `alive` (E uint8).

    Returns sel int32 [T,k] (-1 pad), sel_score float64 [T,k] (-inf pad), gap float64 [T].
    """
    G = _c(G, np.float64)
    T = G.shape[0]
    PA = np.concatenate(prefix_alive(alive, d, M))
    sel = np.empty((T, k), np.int32)
    sc = np.empty((T, k), np.float64)
    gap = np.empty(T, np.float64)
    lib().oracle_select_experts(G, T, d, M, k, B, PA, sel, sc, gap.ctypes.data)
    return sel, sc, gap


def weights(sel, sel_score, responded):
    """S4, Eq. 3 renormalised over responders. Returns w, ok, valid, n_dropped."""
    sel, sc = _c(sel, np.int32), _c(sel_score, np.float64)
    T, k = sel.shape
    w = np.empty((T, k), np.float64)
    ok = np.empty((T, k), np.uint8)
    valid = np.empty(T, np.uint8)
    nd = lib().oracle_weights(sel, sc, T, k, _c(responded, np.uint8), w, ok, valid)
    return w, ok, valid, int(nd)


def dispatch(sel, ok, E):
    """S5, stable counting sort of ok pairs by expert."""
    sel, ok = _c(sel, np.int32), _c(ok, np.uint8)
    T, k = sel.shape
    counts = np.empty(E, np.int32)
    offsets = np.empty(E + 1, np.int32)
    row_of_slot = np.empty((T, k), np.int32)
    token_of_row = np.full(T * k, -1, np.int32)
    R = lib().oracle_dispatch(sel, ok, T, k, E, counts, offsets, row_of_slot, token_of_row)
    return counts, offsets, row_of_slot, token_of_row[:R].copy()


def ffn_fwd(x_rows, seg, W1, b1, W2, b2):
    """S6, expert Forward: returns a = relu(W1 x + b1) [R,H], out [R,D]."""
    x_rows = _c(x_rows, np.float64)
    R, D = x_rows.shape
    S, H, _ = W1.shape
    a = np.empty((R, H), np.float64)
    out = np.empty((R, D), np.float64)
    lib().oracle_ffn_fwd(x_rows, _c(seg, np.int32), S, D, H, _c(W1, np.float64), _c(b1, np.float64),
                         _c(W2, np.float64), _c(b2, np.float64), a, out)
    return a, out


def combine(out, row_of_slot, w):
    """S7, Eq. 3 weighted average."""
    out = _c(out, np.float64)
    T, k = row_of_slot.shape
    D = out.shape[1] if out.ndim == 2 and out.shape[0] else 0
    y = np.empty((T, D), np.float64)
    lib().oracle_combine(out if out.size else np.zeros((1, D)), _c(row_of_slot, np.int32),
                         _c(w, np.float64), T, D, k, y)
    return y


def combine_bwd(dy, out, row_of_slot, w):
    """S8: returns g_rows (= w dY per row) [R,D] and dscore [T,k]."""
    dy, out = _c(dy, np.float64), _c(out, np.float64)
    T, D = dy.shape
    k = row_of_slot.shape[1]
    R = out.shape[0]
    g = np.zeros((max(R, 1), D), np.float64)
    dscore = np.empty((T, k), np.float64)
    lib().oracle_combine_bwd(dy, out if R else np.zeros((1, D)), _c(row_of_slot, np.int32),
                             _c(w, np.float64), T, D, k, g, dscore)
    return g[:R], dscore


def ffn_bwd(x_rows, a_rows, g_rows, seg, W1, W2):
    """S9, expert Backward: dx rows, dW1, db1, dW2, db2."""
    x_rows, a_rows, g_rows = (_c(v, np.float64) for v in (x_rows, a_rows, g_rows))
    R, D = x_rows.shape
    S, H, _ = W1.shape
    dx = np.zeros((max(R, 1), D))
    dW1 = np.empty((S, H, D))
    db1 = np.empty((S, H))
    dW2 = np.empty((S, D, H))
    db2 = np.empty((S, D))
    z = lambda v, c: v if R else np.zeros((1, c))
    lib().oracle_ffn_bwd(z(x_rows, D), z(a_rows, H), z(g_rows, D), _c(seg, np.int32), S, D, H,
                         _c(W1, np.float64), _c(W2, np.float64), dx, dW1, db1, dW2, db2)
    return dx[:R], dW1, db1, dW2, db2


def gate_bwd(X, Wg, sel, dscore, dx_rows, row_of_slot, d, M):
    """S10: dX [T,D], dWg [D,dM], dbg [dM]."""
    X = _c(X, np.float64)
    T, D = X.shape
    k = sel.shape[1]
    dM = d * M
    dX = np.empty((T, D))
    dWg = np.empty((D, dM))
    dbg = np.empty(dM)
    dxr = _c(dx_rows, np.float64)
    lib().oracle_gate_bwd(X, _c(Wg, np.float64), _c(sel, np.int32), _c(dscore, np.float64),
                          dxr if dxr.size else np.zeros((1, D)), _c(row_of_slot, np.int32),
                          T, D, d, M, k, dX, dWg, dbg)
    return dX, dWg, dbg


def layer_step(X, Wg, bg, W1, b1, W2, b2, dY, alive, responded, d, M, k, B, sel_override=None, tie=1,
               responded_bwd=None):
    """One DMoE layer step, forward + backward, composed from S1..S10 in the paper's order.

    W1/b1/W2/b2 cover all E experts, or E / tie parameter slots when `tie` > 1: the declared
    tied-weight pool of the stress workload (reading X20), where expert e computes with
    slot e // tie.  Rows are dispatched per expert exactly as without tying (S5); the FFN then runs
    each slot over the rows of its tied experts, which are contiguous in the expert-major order,
    so the slot segments are offsets[::tie] and dW of a slot is the gradient of the tied weights
    (the sum over its experts' rows).  `responded_bwd` (optional E uint8): experts whose Backward
    request succeeds (reading X22; the others get a zero cotangent, no renormalisation).  `sel_override` (optional [T,k] int32) replaces the
    oracle's own routing downstream of S3 (stage-wise parity with forced routing).
    Returns a dict of every intermediate and gradient.
    """
    E = M ** d
    assert E % tie == 0 and W1.shape[0] == E // tie
    G = gate_scores(X, Wg, bg)
    sel, sc, gap = select_experts(G, d, M, k, B, alive)
    if sel_override is not None:
        sel = np.ascontiguousarray(sel_override, np.int32)
        sc = np.where(sel >= 0, _scores_of(G, sel, d, M), -np.inf)
    w, ok, valid, nd = weights(sel, sc, responded)
    counts, offsets, ros, tor = dispatch(sel, ok, E)
    seg = np.ascontiguousarray(offsets[::tie])
    x_rows = np.asarray(X, np.float64)[tor]
    a, out = ffn_fwd(x_rows, seg, W1, b1, W2, b2)
    y = combine(out, ros, w)
    g, dscore = combine_bwd(dY, out, ros, w)
    if responded_bwd is not None:
        # backward-only failures (reading X22): the lost Backward requests are omitted
        # from the gradient without renormalisation: their experts' cotangent rows are zero
        # (dscore, formed from the forward's record, is unchanged)
        e_of_row = np.repeat(np.arange(E), np.diff(offsets))
        g = np.where(np.asarray(responded_bwd)[e_of_row][:, None] == 1, g, 0.0)
    dx_rows, dW1, db1, dW2, db2 = ffn_bwd(x_rows, a, g, seg, W1, W2)
    dX, dWg, dbg = gate_bwd(X, Wg, sel, dscore, dx_rows, ros, d, M)
    return dict(G=G, sel=sel, sel_score=sc, gap=gap, w=w, ok=ok, valid=valid, n_dropped=nd,
                counts=counts, offsets=offsets, row_of_slot=ros, token_of_row=tor, a=a, out=out,
                y=y, g_rows=g, dscore=dscore, dx_rows=dx_rows, dW1=dW1, db1=db1, dW2=dW2, db2=db2,
                dX=dX, dWg=dWg, dbg=dbg)


def _scores_of(G, sel, d, M):
    """Eq. 2 score of a given full uid: sum_i G[t, i*M + u_i] (u_i per reading X1)."""
    T, k = sel.shape
    s = np.zeros((T, k))
    e = np.where(sel >= 0, sel, 0).astype(np.int64)
    for i in range(d):
        u = (e // (M ** (d - 1 - i))) % M
        s += np.take_along_axis(G, i * M + u, axis=1)
    return s


def layer_step_tokens(X, dY, Wg, bg, experts, alive, responded, d, M, k, B, sel_override=None):
    """The layer step restricted to a subset of tokens (rows of X / dY), for workloads whose full
    expert set cannot be materialised in float64: S1-S4 on the given tokens, the experts they
    select fetched through `experts(ids) -> (W1, b1, W2, b2)` (stacked in `ids` order), S5-S10
    over those tokens' rows only.  y, w, dscore and dX of each token are exactly the full layer's
    (a token's outputs depend only on its own routing and the experts' weights); expert
    gradients cover only the sampled rows.  `sel_override` forces the routing (forced-routing
    parity).  Returns a dict like layer_step plus `experts` (ids in slot order)."""
    G = gate_scores(X, Wg, bg)
    sel, sc, gap = select_experts(G, d, M, k, B, alive)
    if sel_override is not None:
        sel = np.ascontiguousarray(sel_override, np.int32)
        sc = np.where(sel >= 0, _scores_of(G, sel, d, M), -np.inf)
    w, ok, valid, nd = weights(sel, sc, responded)
    used = np.unique(sel[ok == 1]).astype(np.int64)
    slot = -np.ones(M ** d, np.int64)
    slot[used] = np.arange(len(used))
    local = np.where(ok == 1, slot[np.where(sel >= 0, sel, 0)], -1).astype(np.int32)
    # dispatch over the local expert slots (same stable definition as S5)
    counts, offsets, ros, tor = dispatch(local, ok, max(len(used), 1))
    W1, b1, W2, b2 = experts(used) if len(used) else (np.zeros((1, 1, 1)),) * 4
    x_rows = np.asarray(X, np.float64)[tor]
    a, out = ffn_fwd(x_rows, offsets, W1, b1, W2, b2)
    y = combine(out, ros, w)
    g, dscore = combine_bwd(dY, out, ros, w)
    dx_rows, dW1, db1, dW2, db2 = ffn_bwd(x_rows, a, g, offsets, W1, W2)
    dX, dWg, dbg = gate_bwd(X, Wg, sel, dscore, dx_rows, ros, d, M)
    return dict(G=G, sel=sel, sel_score=sc, gap=gap, w=w, ok=ok, valid=valid, n_dropped=nd, experts=used,
                y=y, dscore=dscore, dX=dX, a=a, out=out, dW1=dW1, db1=db1, dW2=dW2, db2=db2, dWg=dWg, dbg=dbg)


def sgd_update(param, grad, lr):
    """The runtime's parameter update after a Backward request: "update expert parameters by
    gradient descent" (§3.3), plain SGD: param - lr * grad (float64)."""
    return np.asarray(param, np.float64) - float(lr) * np.asarray(grad, np.float64)


# ---------------------------------------------------------------- NEXT-2: the paper's expert block
LN_EPS = 1e-5   # reading X23 (PyTorch LayerNorm default)


def ffn3_fwd(x_rows, seg, P, eps=LN_EPS, pre_relu=False):
    """The §4.1 block: Linear -> LayerNorm -> ReLU -> Linear -> LayerNorm -> ReLU ->
    Linear, per slot segment (dmoe_oracle_ffn3.c).  P: dict W1 [S,H,D], b1, g1, be1 [S,H], W2
    [S,H,H], b2, g2, be2 [S,H], W3 [S,D,H], b3 [S,D].  Returns z1, a1, z2, a2 [R,H], out [R,D]
    (+ the pre-ReLU LayerNorm outputs y1, y2 when pre_relu)."""
    x_rows = _c(x_rows, np.float64)
    R, D = x_rows.shape
    S, H, _ = P["W1"].shape
    z1, a1, z2, a2 = (np.empty((max(R, 1), H)) for _ in range(4))
    out = np.empty((max(R, 1), D))
    args = [_c(P[n], np.float64) for n in ("W1", "b1", "g1", "be1", "W2", "b2", "g2", "be2", "W3", "b3")]
    y1, y2 = np.empty((max(R, 1), H)), np.empty((max(R, 1), H))
    lib().oracle_ffn3_fwd(x_rows if R else np.zeros((1, D)), _c(seg, np.int32), S, D, H, *args, float(eps),
                          z1, a1, z2, a2, out, y1.ctypes.data, y2.ctypes.data)
    if pre_relu:
        return z1[:R], a1[:R], z2[:R], a2[:R], out[:R], y1[:R], y2[:R]
    return z1[:R], a1[:R], z2[:R], a2[:R], out[:R]


def ffn3_bwd(x_rows, z1, a1, z2, a2, g_rows, seg, P, eps=LN_EPS, masks=None):
    """Backward of ffn3_fwd with row cotangents g_rows [R,D]: dx rows and every parameter gradient
    (dict with keys dW1, db1, dg1, dbe1, dW2, db2, dg2, dbe2, dW3, db3).  masks: optional (m1, m2)
    uint8 [R,H] ReLU decisions to take instead of 1[y > 0] (forced-decision parity, X23b)."""
    x_rows = _c(x_rows, np.float64)
    R, D = x_rows.shape
    S, H, _ = P["W1"].shape
    z = lambda v, c: _c(v, np.float64) if R else np.zeros((1, c))
    dx = np.zeros((max(R, 1), D))
    G = {"dW1": np.empty((S, H, D)), "db1": np.empty((S, H)), "dg1": np.empty((S, H)), "dbe1": np.empty((S, H)),
         "dW2": np.empty((S, H, H)), "db2": np.empty((S, H)), "dg2": np.empty((S, H)), "dbe2": np.empty((S, H)),
         "dW3": np.empty((S, D, H)), "db3": np.empty((S, D))}
    lib().oracle_ffn3_bwd(z(x_rows, D), z(z1, H), z(a1, H), z(z2, H), z(a2, H), z(g_rows, D), _c(seg, np.int32),
                          S, D, H, *[_c(P[n], np.float64) for n in ("W1", "g1", "be1", "W2", "g2", "be2", "W3")],
                          float(eps), dx, *[G[n] for n in ("dW1", "db1", "dg1", "dbe1", "dW2", "db2", "dg2", "dbe2",
                                                             "dW3", "db3")],
                          *((None, None) if masks is None or not R else
                            (_c(masks[0], np.uint8).ctypes.data, _c(masks[1], np.uint8).ctypes.data)))
    return dx[:R], G


def layer_step_ffn3(X, Wg, bg, P, dY, alive, responded, d, M, k, B, sel_override=None, eps=LN_EPS,
                    relu_override=None):
    """layer_step with the paper's §4.1 expert block (ffn3_fwd / ffn3_bwd) in place of the
    2-linear FFN; routing, weights, dispatch, combine and the gate gradient are the same steps.
    relu_override(y1, y2) -> (m1, m2): the ReLU decisions the backward takes (X23b)."""
    E = M ** d
    G = gate_scores(X, Wg, bg)
    sel, sc, gap = select_experts(G, d, M, k, B, alive)
    if sel_override is not None:
        sel = np.ascontiguousarray(sel_override, np.int32)
        sc = np.where(sel >= 0, _scores_of(G, sel, d, M), -np.inf)
    w, ok, valid, nd = weights(sel, sc, responded)
    counts, offsets, ros, tor = dispatch(sel, ok, E)
    x_rows = np.asarray(X, np.float64)[tor]
    z1, a1, z2, a2, out, y1, y2 = ffn3_fwd(x_rows, offsets, P, eps, pre_relu=True)
    y = combine(out, ros, w)
    g, dscore = combine_bwd(dY, out, ros, w)
    masks = relu_override(y1, y2) if relu_override is not None else None
    dx_rows, grads = ffn3_bwd(x_rows, z1, a1, z2, a2, g, offsets, P, eps, masks=masks)
    dX, dWg, dbg = gate_bwd(X, Wg, sel, dscore, dx_rows, ros, d, M)
    return dict(G=G, sel=sel, sel_score=sc, gap=gap, w=w, ok=ok, valid=valid, n_dropped=nd, counts=counts,
                offsets=offsets, row_of_slot=ros, token_of_row=tor, z1=z1, a1=a1, z2=z2, a2=a2, y1=y1, y2=y2,
                out=out, y=y,
                g_rows=g, dscore=dscore, dx_rows=dx_rows, dX=dX, dWg=dWg, dbg=dbg, **grads)


def topk_exact(G, d, M, k, alive):
    """Exact top-k over the ALIVE experts by the Eq. 2 score (the north star's "exact top-k ...
    restricted to a liveness mask"; NEXT-3): the plain definition, every expert scored with the
    level-order sum of reading X1, ordered by (score desc, flat index asc) (reading X4), the first
    k alive kept, -1 / -inf pad (X6).  Returns sel [T,k] int32 and sel_score [T,k]."""
    G = np.asarray(G, np.float64)
    T = G.shape[0]
    E = M ** d
    e = np.arange(E)
    s = np.zeros((T, E))
    for i in range(d):
        s = s + G[:, i * M + (e // M ** (d - 1 - i)) % M]
    live = np.nonzero(np.asarray(alive) == 1)[0]
    sel = -np.ones((T, k), np.int32)
    sc = np.full((T, k), -np.inf)
    for t in range(T):
        order = live[np.lexsort((live, -s[t, live]))][:k]
        sel[t, :len(order)] = order
        sc[t, :len(order)] = s[t, order]
    return sel, sc
