"""DMoELayer: one Decentralized Mixture-of-Experts layer on one B200, driven through the C ABI.

The forward pass is the paper's DMoE inference procedure (§3.1) with the
structured gate of §3.2: gate scores (Eq. 2) -> SelectExperts (Alg. 1) -> renormalised Eq. 3
weights + dispatch -> expert Forward (runtime, §3.3) -> weighted average (Eq. 3).  The
backward pass is the runtime's Backward request plus the gating gradient.

All buffers are allocated once for T_max tokens, so a step allocates nothing and can be
captured in a CUDA graph.  Python only marshals arguments; every step runs in libdmoe.so.
"""
import torch

from . import _lib as L


class DMoELayer:
    def __init__(self, d, M, k, D, H, dtype=torch.bfloat16, beam=0, T_max=4096, device="cuda",
                 E_local=None, R_cap=None, pool=0, keep_G=False, grads=True, expert="ffn2", ln_eps=1e-5):
        self.d, self.M, self.k, self.D, self.H = d, M, k, D, H
        self.keep_G = keep_G  # also write the gate scores G (tests); the fused path otherwise never stores them
        self.sgd_lr = None    # default of backward(): a learning rate here makes every step an SGD step
        self.beam = beam or k
        self.E = M ** d
        self.E_local = E_local or self.E
        self.dtype = dtype
        self.T_max = T_max
        self.R_cap = R_cap if R_cap is not None else T_max * k
        self.g = L.grid(d, M, k, self.beam)
        dev = torch.device(device)
        f32 = torch.float32
        dM = d * M
        E = self.E
        # tied-weight pool (reading X20): `pool` parameter slots, expert e -> slot e // tie
        self.P = pool or self.E_local
        assert self.E_local % self.P == 0
        self.tie = self.E_local // self.P
        El = self.P
        e = lambda *s, dt=dtype: torch.empty(*s, dtype=dt, device=dev)
        # parameters (filled by the caller / generator)
        self.expert, self.ln_eps = expert, ln_eps
        self.Wg, self.bg = e(D, dM), e(dM, dt=f32)
        if expert == "ffn3":  # the paper's block: D -> H -> H -> D with LayerNorm + ReLU
            self.P3 = {"W1": e(El, H, D), "b1": e(El, H, dt=f32), "g1": e(El, H, dt=f32), "be1": e(El, H, dt=f32),
                      "W2": e(El, H, H), "b2": e(El, H, dt=f32), "g2": e(El, H, dt=f32), "be2": e(El, H, dt=f32),
                      "W3": e(El, D, H), "b3": e(El, D, dt=f32)}
            self.Gr = {"d" + n: torch.empty_like(v) for n, v in self.P3.items()}
            R0 = max(self.R_cap, 1)
            self.z1, self.a1, self.z2, self.a2 = e(R0, H), e(R0, H), e(R0, H), e(R0, H)
            self.stats = e(2, R0, 2, dt=f32)
            self.W1, self.b1, self.W2, self.b2 = self.P3["W1"], self.P3["b1"], self.P3["W2"], self.P3["b2"]
        else:
            self.W1, self.b1 = e(El, H, D), e(El, H, dt=f32)
            self.W2, self.b2 = e(El, D, H), e(El, D, dt=f32)
        # gradients
        self.dWg, self.dbg = e(D, dM, dt=f32), e(dM, dt=f32)
        # grads=False: the layer is only stepped with the fused SGD backward (no dW buffers)
        gE = El if (grads and expert == "ffn2") else 1   # the 2-linear expert's gradient buffers
        self.dW1, self.db1 = e(gE, H, D), e(gE, H, dt=f32)
        self.dW2, self.db2 = e(gE, D, H), e(gE, D, dt=f32)
        # activations / routing records (forward) and backward buffers
        T, R = T_max, self.R_cap
        self.G = e(T if keep_G else 1, dM, dt=f32)
        self.sel = e(T, k, dt=torch.int32)
        self.sel_score = e(T, k, dt=f32)
        self.w = e(T, k, dt=f32)
        self.valid = e(T, dt=torch.uint8)
        self.n_dropped = e(1, dt=torch.int32)
        self.counts = e(E, dt=torch.int32)
        self.offsets = e(E + 1, dt=torch.int32)
        # FFN segments: the slot segments offsets[::tie] when tied, else offsets itself
        self.seg = e(El + 1, dt=torch.int32) if self.tie > 1 else self.offsets
        self.row_of_slot = e(T, k, dt=torch.int32)
        self.token_of_row = e(max(T * k, 1), dt=torch.int32)
        self.xd = e(max(R, 1), D)
        R2 = max(R, 1) if expert == "ffn2" else 1
        self.h = e(R2, H)
        # packed ReLU record [H/32, R_cap] (forward -> backward): 1/16 of h's bytes for dh's mask
        self.hmask = e((H + 31) // 32, R2, dt=torch.int32)
        self.out = e(max(R, 1), D)
        self.y = e(T, D)
        self.dout = e(max(R, 1), D)
        self.dscore = e(T, k, dt=f32)
        self.dxd = e(max(R, 1), D)
        self.dx = e(T, D)
        ws = L.dmoe_workspace_bytes(T, D, H, self.g, El, R)
        self.ws = torch.empty(ws, dtype=torch.uint8, device=dev)

    # ------------------------------------------------------------------ forward
    def forward(self, x, alive_bits, responded_bits):
        T = x.shape[0]
        assert T <= self.T_max and x.dtype == self.dtype and x.shape[1] == self.D
        self._x = x
        L.dmoe_gate_topk(x, self.Wg, self.bg, self.g, alive_bits, self.G[:T] if self.keep_G else None,
                         self.sel[:T], self.sel_score[:T], self.ws)
        L.dmoe_dispatch(x, self.g, self.sel[:T], self.sel_score[:T], responded_bits, self.w[:T], self.valid[:T],
                        self.n_dropped, self.counts, self.offsets, self.row_of_slot[:T], self.token_of_row,
                        self.xd, self.ws)
        if self.tie > 1:
            L.dmoe_segment_offsets(self.offsets, self.tie, self.seg)
        if self.expert == "ffn3":
            L.dmoe_expert_ffn3_fwd(self.xd, self.seg, self.P3, self.ln_eps, self.z1, self.a1, self.z2, self.a2,
                                   self.stats, self.out, self.ws)
        else:
            L.dmoe_expert_ffn_fwd(self.xd, self.seg, self.W1, self.b1, self.W2, self.b2, self.h, self.out,
                                  self.ws, hmask=self.hmask)
        L.dmoe_combine(self.out, self.row_of_slot[:T], self.w[:T], self.valid[:T], self.y[:T])
        return self.y[:T]

    # ----------------------------------------------------------------- backward
    def backward(self, dy, sgd_lr=None, recompute=False, responded_bwd=None):
        """Gradients of the layer.  sgd_lr: the runtime's Backward request semantics:
        the expert parameters are updated in place, W -= lr * dW, inside the weight-gradient GEMMs
        (dW1 / dW2 / db1 / db2 are then not written).  recompute: h is recomputed from xd in the
        backward (gradient checkpointing) instead of read from the forward's
        buffer (SGD form only).  responded_bwd: bit mask of experts whose Backward request
        succeeds; the others are omitted from the gradient without renormalisation (reading X22)."""
        x = self._x
        T = x.shape[0]
        if sgd_lr is None:
            sgd_lr = self.sgd_lr
        if responded_bwd is not None:  # backward-only failures (reading X22)
            L.dmoe_combine_bwd_failures(dy, self.out, self.row_of_slot[:T], self.w[:T], self.sel[:T], responded_bwd,
                                        self.dout, self.dscore[:T])
        else:
            L.dmoe_combine_bwd(dy, self.out, self.row_of_slot[:T], self.w[:T], self.dout, self.dscore[:T])
        if self.expert == "ffn3":
            assert sgd_lr is None, "fused SGD is implemented for the 2-linear expert"
            L.dmoe_expert_ffn3_bwd(self.xd, self.z1, self.a1, self.z2, self.a2, self.stats, self.dout, self.seg,
                                   self.P3, self.dxd, self.Gr, self.ws)
        elif sgd_lr is not None:
            L.dmoe_expert_ffn_bwd_sgd(self.xd, None if recompute else self.h, self.dout, self.seg, self.W1, self.b1,
                                      self.W2, self.b2, sgd_lr, self.dxd, self.ws,
                                      hmask=None if recompute else self.hmask)
        else:
            L.dmoe_expert_ffn_bwd(self.xd, self.h, self.dout, self.seg, self.W1, self.W2, self.dxd,
                                  self.dW1, self.db1, self.dW2, self.db2, self.ws, hmask=self.hmask)
        L.dmoe_gate_bwd(x, self.Wg, self.sel[:T], self.dscore[:T], self.dxd, self.row_of_slot[:T], self.g,
                        self.dx[:T], self.dWg, self.dbg, self.ws)
        return self.dx[:T]

    def step(self, x, dy, alive_bits, responded_bits):
        """One layer step: forward + backward (the unit bench.py times)."""
        self.forward(x, alive_bits, responded_bits)
        return self.backward(dy)

    def host_desc(self, alive_bits, responded_bits):
        """The include/dmoe.h dmoe_layer of this layer (device pointers; 2-linear experts, one GPU)
        for dmoe_layer_step_host, with its own [T_max, D] device staging for x and dy."""
        assert self.expert == "ffn2" and self.E_local == self.E and self.dW1.shape[0] == self.P
        if not hasattr(self, "_stage_x"):
            self._stage_x = torch.empty(self.T_max, self.D, dtype=self.dtype, device=self.y.device)
            self._stage_dy = torch.empty_like(self._stage_x)
        p = L._p
        return L.dmoe_layer(
            self.g, self.D, self.H, self.tie, L._dt(self.y), self.T_max, self.R_cap,
            p(self.Wg), p(self.bg), p(self.W1), p(self.b1), p(self.W2), p(self.b2), p(alive_bits),
            p(responded_bits), p(self._stage_x), p(self._stage_dy), p(self.G) if self.keep_G else None,
            p(self.sel), p(self.sel_score), p(self.w), p(self.valid), p(self.n_dropped), p(self.counts),
            p(self.offsets), p(self.seg), p(self.row_of_slot), p(self.token_of_row), p(self.xd), p(self.h),
            p(self.hmask), p(self.out), p(self.y), p(self.dout), p(self.dscore), p(self.dxd), p(self.dW1),
            p(self.db1), p(self.dW2), p(self.db2), p(self.dx), p(self.dWg), p(self.dbg), p(self.ws),
            self.ws.numel())

    def step_host_c(self, desc, hx, hdy, hy, hdx):
        """One step through the C ABI's host-buffer entry point (dmoe_layer_step_host): x, dy in
        and y, dX out as pinned host tensors, copies inside the call."""
        L.dmoe_layer_step_host(desc, hx.shape[0], hx, hdy, hy, hdx)
        return hdx

    def step_host(self, hx, hdy, hy, hdx, alive_bits, responded_bits):
        """One step from pinned host buffers: x in, y and dX out.  The dy upload overlaps the
        forward pass and the y download overlaps the backward pass (copy stream + events);
        only x-in and dX-out are on the critical path."""
        return host_step(self, hx, hdy, hy, hdx, alive_bits, responded_bits)


def host_step(lay, hx, hdy, hy, hdx, alive_bits, responded_bits):
    """Host-buffer step for any layer with forward/backward/y (DMoELayer, PeerEPDMoELayer, ...)."""
    T = hx.shape[0]
    cur = torch.cuda.current_stream()
    if not hasattr(lay, "_copy_stream"):
        lay._copy_stream = torch.cuda.Stream(device=lay.y.device)
        lay._xin = torch.empty(lay.T_max, lay.D, dtype=lay.dtype, device=lay.y.device)
        lay._dyin = torch.empty(lay.T_max, lay.D, dtype=lay.dtype, device=lay.y.device)
        lay._ev = [torch.cuda.Event() for _ in range(3)]
    side = lay._copy_stream
    x, dy = lay._xin[:T], lay._dyin[:T]
    side.wait_stream(cur)                       # buffers free (previous step done with them)
    x.copy_(hx, non_blocking=True)
    with torch.cuda.stream(side):
        dy.copy_(hdy, non_blocking=True)
        lay._ev[0].record(side)
    lay.forward(x, alive_bits, responded_bits)
    lay._ev[1].record(cur)
    with torch.cuda.stream(side):
        side.wait_event(lay._ev[1])
        hy.copy_(lay.y[:T], non_blocking=True)
        lay._ev[2].record(side)
    cur.wait_event(lay._ev[0])
    dx = lay.backward(dy)
    hdx.copy_(dx, non_blocking=True)
    cur.wait_event(lay._ev[2])
    return dx
