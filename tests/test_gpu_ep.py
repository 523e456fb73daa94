"""Expert parallelism on real GPUs over NCCL (needs >= 2 GPUs; skipped otherwise): the
G-GPU layer equals the 1-GPU layer bit for bit on y, dX and expert dW."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from harness import CONFIGS, gpu_layer, make_inputs, np64

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")]

CFG = CONFIGS["mnist"].with_(T=1024)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, G, port, q, kind="nccl", graph=False):
    import torch.distributed as dist
    from harness import to_torch
    from paper_2002_04013_b200.expert_parallel import EPDMoELayer
    from paper_2002_04013_b200.peer_ep import PeerEPDMoELayer
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=G, device_id=torch.device("cuda", rank))
    cfg = CFG
    inp = make_inputs(cfg, seed=21)
    T = cfg.T // G
    El = cfg.E // G
    Cls = PeerEPDMoELayer if kind == "peer" else EPDMoELayer
    kw = dict(timeout_s=2.0) if kind == "peer" else {}
    lay = Cls(cfg.d, cfg.M, cfg.k, cfg.D, cfg.H, dtype=torch.bfloat16, T_max=T, **kw)
    D, H, dM = cfg.D, cfg.H, cfg.dM
    lay.Wg.copy_(to_torch(inp["dev_Wg"], "bf16", (D, dM)))
    lay.bg.copy_(torch.from_numpy(inp["dev_bg"]).cuda())
    W1 = inp["dev_W1"].reshape(cfg.E, H, D)[rank * El:(rank + 1) * El]
    W2 = inp["dev_W2"].reshape(cfg.E, D, H)[rank * El:(rank + 1) * El]
    lay.W1.copy_(to_torch(W1, "bf16"))
    lay.W2.copy_(to_torch(W2, "bf16"))
    lay.b1.copy_(torch.from_numpy(inp["dev_b1"].reshape(cfg.E, H)[rank * El:(rank + 1) * El]).cuda())
    lay.b2.copy_(torch.from_numpy(inp["dev_b2"].reshape(cfg.E, D)[rank * El:(rank + 1) * El]).cuda())
    x = to_torch(inp["dev_X"], "bf16", (cfg.T, D))[rank * T:(rank + 1) * T].contiguous()
    dy = to_torch(inp["dev_dY"], "bf16", (cfg.T, D))[rank * T:(rank + 1) * T].contiguous()
    alive = torch.from_numpy(inp["alive_bits"].view(np.int32)).cuda()
    resp = torch.from_numpy(inp["responded_bits"].view(np.int32)).cuda()
    if graph == "pipe":
        # the host-buffer pipeline (per-slot CUDA graphs, overlapped copies), three steps
        from paper_2002_04013_b200.host_pipeline import HostPipeline
        hx, hdy = x.cpu().pin_memory(), dy.cpu().pin_memory()
        hy, hdx = torch.empty_like(hx).pin_memory(), torch.empty_like(hx).pin_memory()
        pipe = HostPipeline(lay, T, alive, resp)
        for _ in range(3):
            pipe.submit(hx, hdy, hy, hdx)
        pipe.synchronize()
        y, dx = hy.cuda(), hdx.cuda()
        del pipe
    elif graph:
        # capture one step in a CUDA graph (peer exchange needs no host sync), replay it twice
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            lay.step(x, dy, alive, resp)                 # warm-up (NCCL communicator init etc.)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            lay.step(x, dy, alive, resp)
        for _ in range(2):
            gr.replay()
        torch.cuda.synchronize()
        y, dx = lay.y[:T].clone(), lay.dx[:T].clone()
        del gr   # release graph-captured NCCL work before the communicator is torn down
    else:
        y = lay.forward(x, alive, resp)
        dx = lay.backward(dy)
    torch.cuda.synchronize()
    err = int(lay.err.item()) if kind == "peer" else 0
    out = {n: np64(t) for n, t in dict(y=y, dx=dx, dW1=lay.dW1, dW2=lay.dW2, db1=lay.db1, db2=lay.db2,
                                       dWg=lay.dWg, dbg=lay.dbg).items()}
    out["err"] = err
    if kind == "peer":
        out["epoch"] = int(lay.epoch.item())
        out["flags"] = lay.flags.cpu().tolist()
    q.put((rank, out))
    dist.barrier()
    if kind == "peer":
        lay.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("G,kind,graph", [(2, "nccl", False), (2, "peer", False), (2, "peer", True),
                                          (2, "peer", "pipe")])
def test_ep_equals_single_gpu(G, kind, graph):
    if torch.cuda.device_count() < G:
        pytest.skip(f"needs {G} GPUs")
    cfg = CFG
    ref = gpu_layer(cfg, make_inputs(cfg, seed=21))
    one = {n: np64(getattr(ref, n)) for n in ("y", "dx", "dW1", "dW2", "db1", "db2", "dWg", "dbg")}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, G, port, q, kind, graph)) for r in range(G)]
    for p in ps:
        p.start()
    res = {}
    import queue
    while len(res) < G:
        try:
            r, out = q.get(timeout=5)
            res[r] = out
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in ps):
                for p in ps:
                    p.kill()
                pytest.fail("a rank died")
    for p in ps:
        p.join(timeout=60)
        if p.exitcode is None:
            p.kill()
    T, El = cfg.T // G, cfg.E // G
    for r in range(G):
        assert res[r]["err"] == 0, {k: res[k].get(n) for k in res for n in ("err", "epoch", "flags")}
        assert np.array_equal(res[r]["y"], one["y"][r * T:(r + 1) * T])
        assert np.array_equal(res[r]["dx"], one["dx"][r * T:(r + 1) * T])
        for n in ("dW1", "dW2", "db1", "db2"):
            assert np.array_equal(res[r][n], one[n][r * El:(r + 1) * El]), n
        np.testing.assert_allclose(res[r]["dWg"], one["dWg"], rtol=1e-5, atol=1e-5)
        np.testing.assert_allclose(res[r]["dbg"], one["dbg"], rtol=1e-5, atol=1e-5)
    assert all(p.exitcode == 0 for p in ps), [p.exitcode for p in ps]
