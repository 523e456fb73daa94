"""Multi-process (world_size 2, gloo, CPU) test of the expert-parallel exchange logic: the
G-rank layer equals the 1-rank layer on the same global batch (SURVEY.md §4 "G-GPU == 1-GPU
invariant").  The ABI is replaced by tests/ep_fake.py (oracle-backed, float64), so this checks
split sizes, all-to-all ordering, the expert-major receive layout and the inverse permutation."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen  # noqa: F401
from gen import CONFIGS
from gen.inputs import make_inputs

CFG = CONFIGS["tiny"].with_(M=4, d=2, D=8, H=12, k=3, T=24, fail_frac=0.2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _layer(rank_tokens, inp, G, rank):
    import paper_2002_04013_b200.expert_parallel as EP
    from ep_fake import FakeLib
    EP.L = FakeLib
    cfg = CFG
    lay = EP.EPDMoELayer(cfg.d, cfg.M, cfg.k, cfg.D, cfg.H, dtype=torch.float64, T_max=len(rank_tokens),
                         device="cpu")
    El = cfg.E // G
    lay.Wg.copy_(torch.from_numpy(inp["Wg"]))
    lay.bg.copy_(torch.from_numpy(inp["bg"]).float())
    sl = slice(rank * El, (rank + 1) * El)
    lay.W1.copy_(torch.from_numpy(inp["W1"][sl]))
    lay.b1.copy_(torch.from_numpy(inp["b1"][sl]).float())
    lay.W2.copy_(torch.from_numpy(inp["W2"][sl]))
    lay.b2.copy_(torch.from_numpy(inp["b2"][sl]).float())
    x = torch.from_numpy(inp["X"][rank_tokens]).contiguous()
    dy = torch.from_numpy(inp["dY"][rank_tokens]).contiguous()
    alive = torch.from_numpy(inp["alive_bits"].view(np.int32))
    resp = torch.from_numpy(inp["responded_bits"].view(np.int32))
    y = lay.forward(x, alive, resp).clone()
    dx = lay.backward(dy).clone()
    return dict(y=y.numpy(), dx=dx.numpy(), dW1=lay.dW1.numpy().copy(), dW2=lay.dW2.numpy().copy(),
                db1=lay.db1.numpy().copy(), db2=lay.db2.numpy().copy(), dWg=lay.dWg.numpy().copy(),
                dbg=lay.dbg.numpy().copy(), sent=lay.send_splits, recv=lay.recv_splits)


def _worker(rank, G, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=G)
    inp = make_inputs(CFG, seed=3)
    T = CFG.T // G
    out = _layer(np.arange(rank * T, (rank + 1) * T), inp, G, rank)
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def _run(G):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, G, port, q)) for r in range(G)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(G))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_two_ranks_equal_one_rank():
    one = _run(1)[0]
    two = _run(2)
    T = CFG.T // 2
    El = CFG.E // 2
    for r in range(2):
        assert np.array_equal(two[r]["y"], one["y"][r * T:(r + 1) * T])
        assert np.array_equal(two[r]["dx"], one["dx"][r * T:(r + 1) * T])
        for n in ("dW1", "dW2", "db1", "db2"):
            assert np.array_equal(two[r][n], one[n][r * El:(r + 1) * El]), n
        np.testing.assert_allclose(two[r]["dWg"], one["dWg"], rtol=1e-5, atol=1e-6)  # fp32 storage, 2-term sum
        np.testing.assert_allclose(two[r]["dbg"], one["dbg"], rtol=1e-5, atol=1e-6)
    # every row a rank sends is received by its owner
    assert two[0]["sent"][1] == two[1]["recv"][0] and two[1]["sent"][0] == two[0]["recv"][1]
