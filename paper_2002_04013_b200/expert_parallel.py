"""Expert-parallel DMoE layer: one process per GPU, experts sharded over the group.

The paper's DMoE procedure sends each input to the workers owning its k experts and collects
their outputs (§3.1); the runtime batches requests per expert
and serves Forward and Backward requests.  On one B200 box the workers are
the G GPUs: rank r owns experts [r*E/G, (r+1)*E/G) (contiguous flat indices, so each owner's
rows are one contiguous block of the dispatch buffer) and the "send / collect" steps are NCCL
all-to-alls over NVLink:

  forward : gate -> beam -> dispatch (all E)  | counts a2a | rows a2a | layout + permute ->
            expert FFN (local experts) -> inverse permute | rows a2a back | combine
  backward: combine_bwd | rows a2a | permute -> expert FFN bwd -> inverse permute |
            rows a2a back | gate_bwd | all-reduce(dW_g, db_g)

Gate parameters are replicated; expert gradients stay on their owner (no collective).  Rank r
holds the global token block [r*T, (r+1)*T), so every expert segment receives rows in global
token order and the result equals the single-GPU layer (bitwise for y, dX and expert dW;
dW_g/db_g up to the fp32 all-reduce order).  Host work here is bookkeeping only: split sizes
come from one device->host copy of the counts per step (the only host sync).
"""
import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L


class EPDMoELayer:
    def __init__(self, d, M, k, D, H, dtype=torch.bfloat16, beam=0, T_max=4096, device="cuda", group=None,
                 recv_slack=2.0):
        self.group = group
        self.G = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.d, self.M, self.k, self.D, self.H = d, M, k, D, H
        self.E = M ** d
        if self.E % self.G:
            raise ValueError(f"E={self.E} experts do not shard over {self.G} ranks")
        self.El = self.E // self.G
        self.e0 = self.rank * self.El
        self.beam = beam or k
        self.dtype = dtype
        self.T_max = T_max
        self.dev = torch.device(device)
        self.g = L.grid(d, M, k, self.beam)
        f32, i32 = torch.float32, torch.int32
        e = lambda *s, dt=dtype: torch.empty(*s, dtype=dt, device=self.dev)
        dM, El, E = d * M, self.El, self.E
        self.Wg, self.bg = e(D, dM), e(dM, dt=f32)
        self.W1, self.b1 = e(El, H, D), e(El, H, dt=f32)
        self.W2, self.b2 = e(El, D, H), e(El, D, dt=f32)
        self.dWg, self.dbg = e(D, dM, dt=f32), e(dM, dt=f32)
        self.dW1, self.db1 = e(El, H, D), e(El, H, dt=f32)
        self.dW2, self.db2 = e(El, D, H), e(El, D, dt=f32)
        T = T_max
        R = T * k                                     # rows this rank sends at most
        self.sel, self.sel_score = e(T, k, dt=i32), e(T, k, dt=f32)
        self.w, self.valid, self.n_dropped = e(T, k, dt=f32), e(T, dt=torch.uint8), e(1, dt=i32)
        self.counts, self.offsets = e(E, dt=i32), e(E + 1, dt=i32)
        self.row_of_slot, self.token_of_row = e(T, k, dt=i32), e(max(R, 1), dt=i32)
        self.xd, self.out, self.dout, self.dxd = (e(max(R, 1), D) for _ in range(4))
        self.y, self.dx, self.dscore = e(T, D), e(T, D), e(T, k, dt=f32)
        self.recv_counts = e(self.G, El, dt=i32)
        self.off_loc = e(El + 1, dt=i32)
        self.ws = torch.empty(L.dmoe_workspace_bytes(T, D, H, self.g, E, R), dtype=torch.uint8, device=self.dev)
        self._rcap = 0
        self._ensure_recv(int(recv_slack * R))

    # receive-side buffers grow on demand (the exact size is known on the host before the a2a)
    def _ensure_recv(self, rows):
        if rows <= self._rcap:
            return
        rows = max(rows, 1)
        e = lambda *s, dt=self.dtype: torch.empty(*s, dtype=dt, device=self.dev)
        self.xd_recv, self.xd_loc = e(rows, self.D), e(rows, self.D)
        self.h_loc, self.out_loc, self.out_recv = e(rows, self.H), e(rows, self.D), e(rows, self.D)
        self.dout_recv, self.dout_loc = e(rows, self.D), e(rows, self.D)
        self.dxd_loc, self.dxd_recv = e(rows, self.D), e(rows, self.D)
        self.src_of_dst = e(rows, dt=torch.int32)
        ws = L.dmoe_workspace_bytes(self.T_max, self.D, self.H, self.g, self.El, rows)
        if ws > self.ws.numel():
            self.ws = torch.empty(ws, dtype=torch.uint8, device=self.dev)
        self._rcap = rows

    def _a2a(self, out, inp, out_splits, in_splits):
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)

    # ------------------------------------------------------------------ forward
    def forward(self, x, alive_bits, responded_bits):
        T = x.shape[0]
        self._x = x
        L.dmoe_gate_topk(x, self.Wg, self.bg, self.g, alive_bits, None, self.sel[:T], self.sel_score[:T], self.ws)
        L.dmoe_dispatch(x, self.g, self.sel[:T], self.sel_score[:T], responded_bits, self.w[:T], self.valid[:T],
                        self.n_dropped, self.counts, self.offsets, self.row_of_slot[:T], self.token_of_row,
                        self.xd, self.ws)
        # C1: per-expert counts to the owners (equal splits), then the split sizes on the host
        self._a2a(self.recv_counts.view(-1), self.counts, None, None)
        host = torch.cat([self.offsets[:: self.El], self.recv_counts.view(-1)]).cpu().numpy()
        bounds = host[: self.G + 1].astype(np.int64)
        self.send_splits = [int(v) for v in np.diff(bounds)]
        rc = host[self.G + 1:].reshape(self.G, self.El)
        self.recv_splits = [int(v) for v in rc.sum(1)]
        self.R_out, self.R_in = int(bounds[-1]), int(rc.sum())
        self._ensure_recv(self.R_in)
        # C2: rows to the expert owners; expert-major layout of what arrived
        self._a2a(self.xd_recv[: self.R_in], self.xd[: self.R_out], self.recv_splits, self.send_splits)
        L.dmoe_exchange_layout(self.recv_counts, self.G, self.El, self.off_loc, self.src_of_dst[: self._rcap],
                               self.ws)
        n = self.off_loc[self.El:]
        L.dmoe_permute_rows(self.xd_recv, self.src_of_dst, n, 0, self.xd_loc)
        L.dmoe_expert_ffn_fwd(self.xd_loc, self.off_loc, self.W1, self.b1, self.W2, self.b2, self.h_loc,
                              self.out_loc, self.ws)
        L.dmoe_permute_rows(self.out_loc, self.src_of_dst, n, 1, self.out_recv)
        # C3: outputs back to the token owners, in their dispatch order
        self._a2a(self.out[: self.R_out], self.out_recv[: self.R_in], self.send_splits, self.recv_splits)
        L.dmoe_combine(self.out, self.row_of_slot[:T], self.w[:T], self.valid[:T], self.y[:T])
        return self.y[:T]

    # ----------------------------------------------------------------- backward
    def backward(self, dy):
        x = self._x
        T = x.shape[0]
        n = self.off_loc[self.El:]
        L.dmoe_combine_bwd(dy, self.out, self.row_of_slot[:T], self.w[:T], self.dout, self.dscore[:T])
        # C4: output gradients to the expert owners (the Backward request)
        self._a2a(self.dout_recv[: self.R_in], self.dout[: self.R_out], self.recv_splits, self.send_splits)
        L.dmoe_permute_rows(self.dout_recv, self.src_of_dst, n, 0, self.dout_loc)
        L.dmoe_expert_ffn_bwd(self.xd_loc, self.h_loc, self.dout_loc, self.off_loc, self.W1, self.W2,
                              self.dxd_loc, self.dW1, self.db1, self.dW2, self.db2, self.ws)
        L.dmoe_permute_rows(self.dxd_loc, self.src_of_dst, n, 1, self.dxd_recv)
        # C5: input gradients back to the token owners
        self._a2a(self.dxd[: self.R_out], self.dxd_recv[: self.R_in], self.send_splits, self.recv_splits)
        L.dmoe_gate_bwd(x, self.Wg, self.sel[:T], self.dscore[:T], self.dxd, self.row_of_slot[:T], self.g,
                        self.dx[:T], self.dWg, self.dbg, self.ws)
        # C6: replicated gate parameters
        dist.all_reduce(self.dWg, group=self.group)
        dist.all_reduce(self.dbg, group=self.group)
        return self.dx[:T]

    def step(self, x, dy, alive_bits, responded_bits):
        self.forward(x, alive_bits, responded_bits)
        return self.backward(dy)

    def step_host(self, hx, hdy, hy, hdx, alive_bits, responded_bits):
        """Pinned-host step with the dy upload / y download overlapped (see layer.host_step)."""
        from .layer import host_step
        return host_step(self, hx, hdy, hy, hdx, alive_bits, responded_bits)
