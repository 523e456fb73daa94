"""Expert-parallel DMoE layer with the exchange done over NVLink peer memory (S11 fused form).

Same math and sharding as expert_parallel.EPDMoELayer (rank r owns experts
[r*E/G, (r+1)*E/G) and the token block [r*T, (r+1)*T)), but the paper's "send inputs to those
workers and collect outputs" is done by the library's kernels writing straight
into peer GPUs' buffers (dmoe_ep_* in include/dmoe.h): the dispatch gather stores x rows
directly into each owner's expert-major receive buffer, the owners store expert outputs directly
back into the sources' dispatch-order buffers, and per-source epoch flags replace the host-side
split sizes.  No host sync, so the whole step (including the NCCL all-reduce of the
replicated gate gradient) can be captured in one CUDA graph.

Setup plumbing only: one zeroed cudaMalloc arena per rank holds every peer-written buffer at the
same offset on all ranks; IPC handles are exchanged once with all_gather_object.
"""
import ctypes

import torch
import torch.distributed as dist

from . import _lib as L


class _CAI:
    """Minimal __cuda_array_interface__ wrapper to view raw device memory as a torch tensor."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 2}


def _view(ptr, shape, dtype, device):
    typestr = {torch.bfloat16: "<i2", torch.float32: "<f4", torch.int32: "<i4", torch.int64: "<i8"}[dtype]
    t = torch.as_tensor(_CAI(ptr, shape, typestr), device=device)
    return t.view(torch.bfloat16) if dtype == torch.bfloat16 else t


class PeerEPDMoELayer:
    def __init__(self, d, M, k, D, H, dtype=torch.bfloat16, beam=0, T_max=4096, device="cuda", group=None,
                 recv_slack=2.0, timeout_s=10.0):
        self.group = group
        self.G = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.d, self.M, self.k, self.D, self.H = d, M, k, D, H
        self.E = M ** d
        if self.E % self.G:
            raise ValueError(f"E={self.E} experts do not shard over {self.G} ranks")
        self.El = self.E // self.G
        self.beam = beam or k
        self.dtype = dtype
        self.T_max = T_max
        self.dev = torch.device(device)
        if self.dev.index is None:
            self.dev = torch.device("cuda", torch.cuda.current_device())
        self.g = L.grid(d, M, k, self.beam)
        f32, i32 = torch.float32, torch.int32
        e = lambda *s, dt=dtype: torch.empty(*s, dtype=dt, device=self.dev)
        G, E, El, dM = self.G, self.E, self.El, d * M
        T, R = T_max, T_max * k
        self.rout_cap = max(R, 1)
        self.rin_cap = max(int(recv_slack * R), 1)
        # parameters / gradients (experts: the local slice)
        self.Wg, self.bg = e(D, dM), e(dM, dt=f32)
        self.W1, self.b1 = e(El, H, D), e(El, H, dt=f32)
        self.W2, self.b2 = e(El, D, H), e(El, D, dt=f32)
        # dW_g and db_g share one buffer: one all-reduce per step (C6)
        self._dgate = e(D * dM + dM, dt=f32)
        self.dWg, self.dbg = self._dgate[: D * dM].view(D, dM), self._dgate[D * dM:]
        self.dW1, self.db1 = e(El, H, D), e(El, H, dt=f32)
        self.dW2, self.db2 = e(El, D, H), e(El, D, dt=f32)
        # local (not peer-written) buffers
        self.sel, self.sel_score = e(T, k, dt=i32), e(T, k, dt=f32)
        self.w, self.valid, self.n_dropped = e(T, k, dt=f32), e(T, dt=torch.uint8), e(1, dt=i32)
        self.counts, self.offsets = e(E, dt=i32), e(E + 1, dt=i32)
        self.row_of_slot, self.token_of_row = e(T, k, dt=i32), e(self.rout_cap, dt=i32)
        self.dout = e(self.rout_cap, D)
        self.y, self.dx, self.dscore = e(T, D), e(T, D), e(T, k, dt=f32)
        self.h_loc, self.out_loc, self.dxd_loc = e(self.rin_cap, H), e(self.rin_cap, D), e(self.rin_cap, D)
        self.hmask = e((H + 31) // 32, self.rin_cap, dt=i32)  # packed ReLU record (forward -> backward)
        self.epoch = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self.err = torch.zeros(1, dtype=i32, device=self.dev)
        self.base, self.off_loc = e(E, dt=i32), e(El + 1, dt=i32)
        self.src_off, self.dst_off = e(G, El, dt=i32), e(G, El, dt=i32)
        self.ws = torch.empty(L.dmoe_workspace_bytes(T, D, H, self.g, El, self.rin_cap), dtype=torch.uint8,
                              device=self.dev)
        # symmetric arena: flags [G] u64 | cnt [G][E] i32 | xin, din [rin_cap, D] | ret, dret [rout_cap, D]
        es = torch.tensor([], dtype=dtype).element_size()
        al = lambda n: (n + 255) // 256 * 256
        self._lay = {}
        off = 0
        for name, nbytes in (("flags", G * 8), ("cnt", G * E * 4), ("xin", self.rin_cap * D * es),
                             ("din", self.rin_cap * D * es), ("ret", self.rout_cap * D * es),
                             ("dret", self.rout_cap * D * es)):
            self._lay[name] = off
            off += al(nbytes)
        with torch.cuda.device(self.dev):
            self.arena, handle = L.dmoe_ipc_alloc(off)
        handles = [None] * G
        dist.all_gather_object(handles, handle, group=group)
        self.peer_base = []
        for j in range(G):
            self.peer_base.append(self.arena if j == self.rank else L.dmoe_ipc_open(handles[j]))
        ptrs = lambda name: torch.tensor([b + self._lay[name] for b in self.peer_base], dtype=torch.int64,
                                         device=self.dev)
        self.peer = {n: ptrs(n) for n in self._lay}
        loc = lambda name: self.arena + self._lay[name]
        self.flags = _view(loc("flags"), (G,), torch.int64, self.dev)
        self.cnt = _view(loc("cnt"), (G, E), i32, self.dev)
        self.xin = _view(loc("xin"), (self.rin_cap, D), dtype, self.dev)
        self.din = _view(loc("din"), (self.rin_cap, D), dtype, self.dev)
        self.ret = _view(loc("ret"), (self.rout_cap, D), dtype, self.dev)
        self.dret = _view(loc("dret"), (self.rout_cap, D), dtype, self.dev)
        self.ep = L.dmoe_ep(G, self.rank, E, El, self.rin_cap, int(timeout_s * 1e9),
                            self.epoch.data_ptr(), self.flags.data_ptr(), self.peer["flags"].data_ptr(),
                            self.cnt.data_ptr(), self.peer["cnt"].data_ptr(), self.err.data_ptr(),
                            self.base.data_ptr(), self.off_loc.data_ptr(), self.src_off.data_ptr(),
                            self.dst_off.data_ptr())
        dist.barrier(group=group)

    def close(self):
        torch.cuda.synchronize(self.dev)
        dist.barrier(group=self.group)
        for j, b in enumerate(self.peer_base):
            if j != self.rank:
                L.dmoe_ipc_close(b)
        dist.barrier(group=self.group)
        L.dmoe_ipc_free(self.arena)

    # ------------------------------------------------------------------ forward
    def forward(self, x, alive_bits, responded_bits):
        T = x.shape[0]
        self._x = x
        ep = self.ep
        L.dmoe_ep_begin(ep)
        L.dmoe_gate_topk(x, self.Wg, self.bg, self.g, alive_bits, None, self.sel[:T], self.sel_score[:T], self.ws)
        L.dmoe_dispatch(x, self.g, self.sel[:T], self.sel_score[:T], responded_bits, self.w[:T], self.valid[:T],
                        self.n_dropped, self.counts, self.offsets, self.row_of_slot[:T], self.token_of_row,
                        None, self.ws)
        L.dmoe_ep_exchange_counts(ep, self.counts)                                  # C1
        L.dmoe_ep_push_rows(ep, x, self.token_of_row, self.offsets, self.peer["xin"], 1)   # C2 (gather+send)
        L.dmoe_expert_ffn_fwd(self.xin, self.off_loc, self.W1, self.b1, self.W2, self.b2, self.h_loc,
                              self.out_loc, self.ws, hmask=self.hmask)
        L.dmoe_ep_return_rows(ep, self.out_loc, self.peer["ret"], 2)                   # C3
        L.dmoe_combine(self.ret, self.row_of_slot[:T], self.w[:T], self.valid[:T], self.y[:T])
        return self.y[:T]

    # ----------------------------------------------------------------- backward
    def backward(self, dy):
        x = self._x
        T = x.shape[0]
        ep = self.ep
        L.dmoe_combine_bwd(dy, self.ret, self.row_of_slot[:T], self.w[:T], self.dout, self.dscore[:T])
        L.dmoe_ep_push_rows(ep, self.dout, None, self.offsets, self.peer["din"], 3)   # C4
        L.dmoe_expert_ffn_bwd(self.xin, self.h_loc, self.din, self.off_loc, self.W1, self.W2, self.dxd_loc,
                              self.dW1, self.db1, self.dW2, self.db2, self.ws, hmask=self.hmask)
        L.dmoe_ep_return_rows(ep, self.dxd_loc, self.peer["dret"], 4)                  # C5
        L.dmoe_gate_bwd(x, self.Wg, self.sel[:T], self.dscore[:T], self.dret, self.row_of_slot[:T], self.g,
                        self.dx[:T], self.dWg, self.dbg, self.ws)
        dist.all_reduce(self._dgate, group=self.group)                                 # C6 (dW_g, db_g)
        return self.dx[:T]

    def step(self, x, dy, alive_bits, responded_bits):
        self.forward(x, alive_bits, responded_bits)
        return self.backward(dy)

    def step_host(self, hx, hdy, hy, hdx, alive_bits, responded_bits):
        """Pinned-host step with the dy upload / y download overlapped (see layer.host_step)."""
        from .layer import host_step
        return host_step(self, hx, hdy, hy, hdx, alive_bits, responded_bits)

    def check(self):
        """Raise if a wait timed out (err & 1) or a receive buffer would have overflowed (err & 2)
        since the last check.  The error word is sticky inside the kernels (once set, every later
        push / return of this rank skips its row writes, so a broken step cannot scribble over
        peers' buffers); reading it here clears it, so the next step runs normally.  Callers must
        check at their sync points: HostPipeline.synchronize() does."""
        v = int(self.err.item())
        if v:
            self.err.zero_()
            raise RuntimeError(f"peer exchange error word {v} (1 = wait timeout, 2 = receive overflow)")
