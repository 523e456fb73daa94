"""Stage-level parity of the grouped expert GEMMs (S6, S9) on ragged segments: empty experts,
single rows, exact 128-row tiles, multi-tile segments, and capacity rows past R."""
import numpy as np
import pytest
import torch

import gen
from harness import TOL, np64, rel_err
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _run(counts, D, H, dtype, seed=0, cap_extra=37):
    import paper_2002_04013_b200 as P
    counts = np.asarray(counts, np.int32)
    E = len(counts)
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    R = int(offsets[-1])
    Rc = R + cap_extra
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32

    def t(tid, n, scale, shape, dist=gen.UNIFORM):
        if dtype == "bf16":
            bits = gen.host_bf16_bits(seed, tid, dist, scale, n)
            return torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).reshape(shape).cuda(), gen.bf16_bits_to_f64(bits).reshape(shape)
        v = gen.host_f32(seed, tid, dist, scale, n)
        return torch.from_numpy(v).reshape(shape).cuda(), v.astype(np.float64).reshape(shape)

    xd, xd64 = t(gen.X, Rc * D, 1.0, (Rc, D), gen.NORMAL)
    W1, W164 = t(gen.W1, E * H * D, D ** -0.5, (E, H, D))
    W2, W264 = t(gen.W2, E * D * H, H ** -0.5, (E, D, H))
    b1 = torch.from_numpy(gen.host_f32(seed, gen.B1, gen.UNIFORM, D ** -0.5, E * H)).reshape(E, H).cuda()
    b2 = torch.from_numpy(gen.host_f32(seed, gen.B2, gen.UNIFORM, H ** -0.5, E * D)).reshape(E, D).cuda()
    dout, dout64 = t(gen.DY, Rc * D, 1.0, (Rc, D), gen.NORMAL)
    # poison the capacity rows past R with NaN: they must never leak into any result
    if Rc > R:
        xd[R:] = float("nan"); dout[R:] = float("nan")
    off = torch.from_numpy(offsets).cuda()
    h = torch.full((Rc, H), float("nan"), dtype=tdt, device="cuda")
    out = torch.empty(Rc, D, dtype=tdt, device="cuda")
    g = P.grid(1, E, 1)
    ws = torch.empty(P.dmoe_workspace_bytes(1, D, H, g, E, Rc), dtype=torch.uint8, device="cuda")
    c0 = P.dmoe_launch_counters()
    P.dmoe_expert_ffn_fwd(xd, off, W1, b1, W2, b2, h, out, ws)
    dxd = torch.empty_like(xd)
    dW1, dW2 = torch.empty_like(W1), torch.empty_like(W2)
    db1, db2 = torch.empty_like(b1), torch.empty_like(b2)
    P.dmoe_expert_ffn_bwd(xd, h, dout, off, W1, W2, dxd, dW1, db1, dW2, db2, ws)
    torch.cuda.synchronize()
    c1 = P.dmoe_launch_counters()
    if dtype == "bf16":   # the bf16 path must run on the tensor cores (h, out, dh, dxd and the two
        # weight-gradient GEMMs: 6 tcgen05 launches, 5 when dW2 and dW1 share one), no SIMT GEMM
        assert c1[1] - c0[1] in (5, 6) and c1[2] == c0[2], (c0, c1)
    a_ref, out_ref = O.ffn_fwd(xd64[:R], offsets, W164, np64(b1), W264, np64(b2))
    dx_ref, dW1_ref, db1_ref, dW2_ref, db2_ref = O.ffn_bwd(xd64[:R], a_ref, dout64[:R], offsets, W164, W264)
    tol = TOL[dtype]
    errs = dict(h=rel_err(np64(h[:R]), a_ref), out=rel_err(np64(out[:R]), out_ref),
                dxd=rel_err(np64(dxd[:R]), dx_ref), dW1=rel_err(np64(dW1), dW1_ref),
                db1=rel_err(np64(db1), db1_ref), dW2=rel_err(np64(dW2), dW2_ref), db2=rel_err(np64(db2), db2_ref))
    assert all(v <= tol for v in errs.values()), errs
    # the packed ReLU record (forward -> backward) reproduces the h-read masks bit for bit
    hm = torch.full(((H + 31) // 32, Rc), -1, dtype=torch.int32, device="cuda")
    h2, out2 = torch.empty_like(h), torch.empty_like(out)
    P.dmoe_expert_ffn_fwd(xd, off, W1, b1, W2, b2, h2, out2, ws, hmask=hm)
    dxd2, dW12, dW22 = torch.empty_like(dxd), torch.empty_like(dW1), torch.empty_like(dW2)
    db12, db22 = torch.empty_like(db1), torch.empty_like(db2)
    P.dmoe_expert_ffn_bwd(xd, h2, dout, off, W1, W2, dxd2, dW12, db12, dW22, db22, ws, hmask=hm)
    torch.cuda.synchronize()
    for a, b in [(h[:R], h2[:R]), (out[:R], out2[:R]), (dxd[:R], dxd2[:R]), (dW1, dW12), (dW2, dW22), (db1, db12),
                 (db2, db22)]:
        assert torch.equal(a, b)
    for i in np.nonzero(counts == 0)[0]:
        assert (np64(dW1[i]) == 0).all() and (np64(dW2[i]) == 0).all() and (np64(db1[i]) == 0).all()
    return errs


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_ragged_segments(dtype):
    _run([0, 1, 127, 128, 129, 0, 300, 64, 5, 256], D=128, H=256, dtype=dtype)


def test_bf16_wide_tiles():
    # N = 1024 / 256 -> BN = 256 tiles on both GEMMs
    _run([58, 70, 0, 131, 1, 64], D=256, H=1024, dtype="bf16", seed=3)


def test_bf16_single_expert_many_tiles():
    _run([1000], D=128, H=384, dtype="bf16", seed=4)


def test_bf16_cta_pair_row_gemms():
    """Experts averaging >= 256 rows of capacity run the row GEMMs on CTA pairs (cta_group::2,
    M = 256; each CTA loads half of the weight tile): segments shorter than one CTA's 128 rows
    (the peer's rows fall past the segment), exact 256-row pair tiles, odd tails, an empty expert."""
    _run([300, 257, 0, 512, 1, 700, 256, 255], D=256, H=1024, dtype="bf16", seed=5)


def test_bf16_cta_pair_many_experts():
    rng = np.random.default_rng(6)
    _run(list(rng.poisson(300, 24)), D=512, H=1024, dtype="bf16", seed=6)
