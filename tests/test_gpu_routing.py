"""S1-S3 through the C ABI: the standalone SelectExperts kernel (dmoe_beam_topk, thread per
token) and the fused gate + SelectExperts call (dmoe_gate_topk, Alg. 1 in the gate GEMM's
epilogue) against the oracle's Alg. 1, over grids, beam widths and masks
beyond the BASELINE configs (wide beams, 3-D grids, dead experts, forced ties)."""
import numpy as np
import pytest
import torch

from harness import GAP, np64, to_torch
from oracle import oracle as O
import paper_2002_04013_b200 as P
from paper_2002_04013_b200 import _lib as L

pytestmark = pytest.mark.gpu


def _alive_bits(alive):
    E = len(alive)
    words = np.zeros((E + 31) // 32, np.uint32)
    for e in np.nonzero(alive)[0]:
        words[e >> 5] |= np.uint32(1) << np.uint32(e & 31)
    return torch.from_numpy(words.view(np.int32)).cuda()


def _ws(T, D, d, M, k, B):
    g = L.grid(d, M, k, B)
    return g, torch.empty(L.dmoe_workspace_bytes(T, D, 64, g, M ** d, T * k), dtype=torch.uint8, device="cuda")


def _check(G, sel, sc, d, M, k, B, alive, exact):
    osel, osc, gap = O.select_experts(G, d, M, k, B, alive)
    mask = np.ones(len(gap), bool) if exact else gap > GAP
    bad = np.nonzero((sel != osel).any(1) & mask)[0]
    assert len(bad) == 0, (bad[:5], sel[bad[:3]], osel[bad[:3]])
    # the reported scores are the Eq. 2 sums of the reported experts (fp32 of the kernel vs fp64)
    m = sel >= 0
    assert np.allclose(sc[m], O._scores_of(G, np.where(m, sel, 0), d, M)[m], atol=1e-4)
    assert np.all(np.isneginf(sc[~m]))
    return int(mask.sum())


@pytest.mark.parametrize("d,M,k,B,dead,exact,T", [
    (2, 64, 4, 4, 0.0, False, 3000),    # transformer grid
    (3, 16, 4, 4, 0.0, False, 2500),    # 3-D grid
    (2, 64, 8, 8, 0.0, False, 1000),    # stress k
    (2, 64, 4, 12, 0.0, False, 700),    # B > 8: standalone kernel only
    (2, 16, 5, 6, 0.3, True, 2000),     # dead experts, exact-grid ties
    (3, 8, 2, 5, 0.5, True, 2000),      # masked 3-D, heavy ties
    (2, 128, 4, 4, 0.0, False, 600),    # d*M = 256 > 128: unfused gate
    (4, 4, 3, 3, 0.2, True, 800),       # 4-D grid
    (2, 64, 16, 32, 0.0, False, 300),   # widest envelope
])
def test_beam_topk_vs_oracle(d, M, k, B, dead, exact, T):
    rng = np.random.default_rng(d * 1000 + M + k + B)
    E, dM = M ** d, d * M
    if exact:
        G = rng.integers(-8, 9, (T, dM)).astype(np.float32) / 8   # many exact ties
    else:
        G = rng.standard_normal((T, dM)).astype(np.float32)
    alive = (rng.random(E) >= dead).astype(np.uint8)
    g, ws = _ws(T, 64, d, M, k, B)
    Gt = torch.from_numpy(G).cuda()
    sel = torch.empty(T, k, dtype=torch.int32, device="cuda")
    sc = torch.empty(T, k, dtype=torch.float32, device="cuda")
    L.dmoe_beam_topk(Gt, g, _alive_bits(alive), sel, sc, ws)
    torch.cuda.synchronize()
    _check(G.astype(np.float64), np64(sel), np64(sc), d, M, k, B, alive, exact)


@pytest.mark.parametrize("d,M,k,B,D,dead,T", [
    (2, 64, 4, 4, 1024, 0.0, 1500), (3, 16, 4, 4, 1024, 0.0, 1300), (2, 16, 4, 4, 256, 0.1, 777),
    (2, 64, 8, 8, 2048, 0.0, 500), (2, 16, 5, 6, 256, 0.3, 999), (2, 128, 4, 4, 256, 0.0, 300)])
def test_gate_topk_equals_gate_then_beam(d, M, k, B, D, dead, T):
    """The fused call gives exactly (bit for bit) what the two separate calls give, with and
    without writing G, on the tensor-core path (bf16) and the fallback (d*M > 128)."""
    rng = np.random.default_rng(T + D)
    E, dM = M ** d, d * M
    x = torch.from_numpy(rng.standard_normal((T, D)).astype(np.float32)).to(torch.bfloat16).cuda()
    Wg = torch.from_numpy((rng.standard_normal((D, dM)) / np.sqrt(D)).astype(np.float32)).to(torch.bfloat16).cuda()
    bg = torch.from_numpy((0.1 * rng.standard_normal(dM)).astype(np.float32)).cuda()
    alive = _alive_bits((rng.random(E) >= dead).astype(np.uint8))
    g, ws = _ws(T, D, d, M, k, B)
    G1 = torch.empty(T, dM, device="cuda")
    s1 = torch.empty(T, k, dtype=torch.int32, device="cuda")
    c1 = torch.empty(T, k, device="cuda")
    L.dmoe_gate_scores(x, Wg, bg, g, G1, ws)
    L.dmoe_beam_topk(G1, g, alive, s1, c1, ws)
    for keep in (True, False):
        G2 = torch.full((T, dM), float("nan"), device="cuda") if keep else None
        s2 = torch.full((T, k), -7, dtype=torch.int32, device="cuda")
        c2 = torch.empty(T, k, device="cuda")
        L.dmoe_gate_topk(x, Wg, bg, g, alive, G2, s2, c2, ws)
        torch.cuda.synchronize()
        assert torch.equal(s1, s2) and torch.equal(c1.view(torch.int32), c2.view(torch.int32))
        if keep:
            assert torch.equal(G1.view(torch.int32), G2.view(torch.int32))


@pytest.mark.parametrize("d,M,k,dead,T", [(2, 64, 4, 0.3, 2000), (3, 16, 4, 0.1, 1500), (2, 16, 8, 0.5, 999),
                                          (2, 64, 4, 0.0, 700)])
def test_topk_exact_vs_oracle(d, M, k, dead, T):
    """dmoe_topk_exact against the plain definition (oracle.topk_exact) on exact-grid scores
    (every fp32 sum exact, ties everywhere): bit-exact on every token; with every expert alive it
    also equals Alg. 1 (dmoe_beam_topk) bit for bit."""
    rng = np.random.default_rng(T + d)
    E = M ** d
    G = (rng.integers(-8, 9, (T, d * M)) / 8).astype(np.float32)
    alive = (rng.random(E) >= dead).astype(np.uint8)
    g = L.grid(d, M, k, k)
    Gt = torch.from_numpy(G).cuda()
    sel = torch.empty(T, k, dtype=torch.int32, device="cuda")
    sc = torch.empty(T, k, dtype=torch.float32, device="cuda")
    L.dmoe_topk_exact(Gt, g, _alive_bits(alive), sel, sc)
    torch.cuda.synchronize()
    osel, osc = O.topk_exact(G.astype(np.float64), d, M, k, alive)
    assert np.array_equal(np64(sel), osel)
    assert np.array_equal(np64(sc), osc.astype(np.float32).astype(np.float64))
    if dead == 0.0:
        _, ws = _ws(T, 64, d, M, k, k)
        s2 = torch.empty_like(sel)
        c2 = torch.empty_like(sc)
        L.dmoe_beam_topk(Gt, g, _alive_bits(alive), s2, c2, ws)
        torch.cuda.synchronize()
        assert torch.equal(sel, s2) and torch.equal(sc.view(torch.int32), c2.view(torch.int32))
