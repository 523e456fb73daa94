"""Test double of the libdmoe ABI on CPU tensors (float64), for the multi-process gloo tests of
the expert-parallel orchestration (paper_2002_04013_b200/expert_parallel.py).  Each call does
what include/dmoe.h specifies, computed by the float64 oracle — TEST-ONLY: the product path
never imports this module; it checks the host-side exchange logic without a GPU."""
from types import SimpleNamespace

import numpy as np
import torch

from oracle import oracle as O


def _bits(t, n):
    return np.unpackbits(t.numpy().view(np.uint8), bitorder="little")[:n].astype(np.uint8)


class FakeLib:
    @staticmethod
    def grid(d, M, k, beam=0):
        return SimpleNamespace(d=d, M=M, k=k, beam=beam or k)

    @staticmethod
    def dmoe_workspace_bytes(*a):
        return 8

    @staticmethod
    def dmoe_gate_scores(x, Wg, bg, g, G, ws):
        G[:] = torch.from_numpy(O.gate_scores(x.numpy(), Wg.numpy(), bg.numpy()))

    @staticmethod
    def dmoe_gate_topk(x, Wg, bg, g, alive_bits, G, sel, sel_score, ws):
        Gv = O.gate_scores(x.numpy(), Wg.numpy(), bg.numpy())
        if G is not None:
            G[:] = torch.from_numpy(Gv)
        s, sc, _ = O.select_experts(Gv, g.d, g.M, g.k, g.beam, _bits(alive_bits, g.M ** g.d))
        sel[:] = torch.from_numpy(s)
        sel_score[:] = torch.from_numpy(sc)

    @staticmethod
    def dmoe_beam_topk(G, g, alive_bits, sel, sel_score, ws):
        s, sc, _ = O.select_experts(G.numpy(), g.d, g.M, g.k, g.beam, _bits(alive_bits, g.M ** g.d))
        sel[:] = torch.from_numpy(s)
        sel_score[:] = torch.from_numpy(sc)

    @staticmethod
    def dmoe_dispatch(x, g, sel, sel_score, resp_bits, w, valid, n_dropped, counts, offsets, ros, tor, xd, ws):
        E = g.M ** g.d
        w_, ok, v_, nd = O.weights(sel.numpy(), sel_score.numpy(), _bits(resp_bits, E))
        c, off, r, t = O.dispatch(sel.numpy(), ok, E)
        w[:] = torch.from_numpy(w_)
        valid[:] = torch.from_numpy(v_)
        n_dropped[0] = nd
        counts[:] = torch.from_numpy(c)
        offsets[:] = torch.from_numpy(off)
        ros[:] = torch.from_numpy(r)
        tor[: len(t)] = torch.from_numpy(t)
        xd[: len(t)] = x[torch.from_numpy(t).long()]

    @staticmethod
    def dmoe_expert_ffn_fwd(xd, offsets, W1, b1, W2, b2, h, out, ws, hmask=None):
        off = offsets.numpy()
        R = int(off[-1])
        a, o = O.ffn_fwd(xd[:R].numpy(), off, W1.numpy(), b1.numpy(), W2.numpy(), b2.numpy())
        h[:R] = torch.from_numpy(a)
        out[:R] = torch.from_numpy(o)

    @staticmethod
    def dmoe_combine(out, ros, w, valid, y):
        y[:] = torch.from_numpy(O.combine(out.numpy(), ros.numpy(), w.numpy()))

    @staticmethod
    def dmoe_combine_bwd(dy, out, ros, w, dout, dscore):
        R = int(ros.numpy().max()) + 1 if (ros.numpy() >= 0).any() else 0
        gr, ds = O.combine_bwd(dy.numpy(), out[:R].numpy(), ros.numpy(), w.numpy())
        dout[:R] = torch.from_numpy(gr)
        dscore[:] = torch.from_numpy(ds)

    @staticmethod
    def dmoe_expert_ffn_bwd(xd, h, dout, offsets, W1, W2, dxd, dW1, db1, dW2, db2, ws, hmask=None):
        off = offsets.numpy()
        R = int(off[-1])
        dx, a, b, c, d = O.ffn_bwd(xd[:R].numpy(), h[:R].numpy(), dout[:R].numpy(), off, W1.numpy(), W2.numpy())
        dxd[:R] = torch.from_numpy(dx)
        dW1[:], db1[:], dW2[:], db2[:] = (torch.from_numpy(v) for v in (a, b, c, d))

    @staticmethod
    def dmoe_gate_bwd(x, Wg, sel, dscore, dxd, ros, g, dx, dWg, dbg, ws):
        R = int(ros.numpy().max()) + 1 if (ros.numpy() >= 0).any() else 0
        a, b, c = O.gate_bwd(x.numpy(), Wg.numpy(), sel.numpy(), dscore.numpy(), dxd[:R].numpy(), ros.numpy(),
                             g.d, g.M)
        dx[:], dWg[:], dbg[:] = torch.from_numpy(a), torch.from_numpy(b), torch.from_numpy(c)

    @staticmethod
    def dmoe_exchange_layout(recv_counts, G, El, offsets, src_of_dst, ws):
        c = recv_counts.numpy().reshape(G, El)
        src_off = np.concatenate([[0], np.cumsum(c.ravel())])[:-1].reshape(G, El)
        r = 0
        offsets[0] = 0
        for e in range(El):
            for s in range(G):
                n = int(c[s, e])
                src_of_dst[r:r + n] = torch.arange(int(src_off[s, e]), int(src_off[s, e]) + n, dtype=torch.int32)
                r += n
            offsets[e + 1] = r

    @staticmethod
    def dmoe_permute_rows(src, idx, n, inverse, dst):
        R = int(n[0])
        i = idx[:R].long()
        if inverse:
            dst[i] = src[:R]
        else:
            dst[:R] = src[i]
