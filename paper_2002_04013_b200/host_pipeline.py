"""HostPipeline: training steps streamed from pinned host memory through one DMoE layer.

A training loop feeds each layer step from host memory: x in, dy in (the upstream gradient),
y out, dX out.  Done one step at a time (DMoELayer.step_host), the x upload and the dX
download sit on the critical path of every step.  This pipeline overlaps them with the
neighbouring steps' compute:

  H2D stream : x_i+1, dy_i+1 upload          (into staging slot (i+1) % 2)
  compute    : forward_i, backward_i         (one CUDA-graph launch each, captured per slot)
  D2H stream : y_i (after forward_i), dX_i (after backward_i) download (from slot i % 2)

Staging buffers are double-buffered by step parity and guarded by events, so step i+1's upload
never overwrites inputs step i is still reading and step i+2's forward never overwrites outputs
step i's download is still reading.  Every step still moves its own inputs host->device and its
own results device->host; only the ordering between steps changes.  Python marshals the
launches; every step of the layer runs in libdmoe.so.
"""
import torch


class HostPipeline:
    def __init__(self, lay, T, alive_bits, responded_bits, use_graphs=True):
        self.lay, self.T = lay, T
        self.alive, self.resp = alive_bits, responded_bits
        dev = lay.y.device
        e = lambda: torch.empty(T, lay.D, dtype=lay.dtype, device=dev)
        self.xin, self.dyin = [e(), e()], [e(), e()]
        self.yout, self.dxout = [e(), e()], [e(), e()]
        self.compute = torch.cuda.Stream(device=dev)
        self.h2d = torch.cuda.Stream(device=dev)
        self.d2h = torch.cuda.Stream(device=dev)
        mk = lambda: [torch.cuda.Event(), torch.cuda.Event()]
        self.ev_up, self.ev_fwd, self.ev_bwd, self.ev_down = mk(), mk(), mk(), mk()
        self.n = 0
        self.graphs = None
        self.use_graphs = use_graphs

    # one half-step body per slot: the layer pass plus the copy into the slot's output staging
    def _fwd(self, s):
        y = self.lay.forward(self.xin[s], self.alive, self.resp)
        self.yout[s].copy_(y)

    def _bwd(self, s):
        dx = self.lay.backward(self.dyin[s])
        self.dxout[s].copy_(dx)

    def _capture(self, hx, hdy):
        # warm-up and capture on the first batch's data (routing on uninitialised staging could
        # send every token to a few experts, beyond an expert-parallel receive capacity)
        for s in (0, 1):
            self.xin[s].copy_(hx)
            self.dyin[s].copy_(hdy)
        torch.cuda.synchronize(self.xin[0].device)
        with torch.cuda.stream(self.compute):
            for s in (0, 1):  # warm-up through the eager path (also builds library side streams)
                self._fwd(s)
                self._bwd(s)
        self.compute.synchronize()
        self.graphs = []
        for s in (0, 1):
            gf, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(gf, stream=self.compute):
                self._fwd(s)
            with torch.cuda.graph(gb, stream=self.compute):
                self._bwd(s)
            self.graphs.append((gf, gb))
        self.compute.synchronize()

    def submit(self, hx, hdy, hy, hdx):
        """Enqueue one step: pinned host x, dy in; y, dX out (valid after synchronize())."""
        if self.use_graphs and self.graphs is None:
            self._capture(hx, hdy)
        i, s = self.n, self.n % 2
        cur = self.compute
        with torch.cuda.stream(self.h2d):
            if i >= 2:
                self.h2d.wait_event(self.ev_bwd[s])  # step i-2 is done reading this slot's inputs
            self.xin[s].copy_(hx, non_blocking=True)
            self.dyin[s].copy_(hdy, non_blocking=True)
            self.ev_up[s].record(self.h2d)
        cur.wait_event(self.ev_up[s])
        if i >= 2:
            cur.wait_event(self.ev_down[s])  # step i-2's downloads are done with this slot's outputs
        with torch.cuda.stream(cur):
            if self.graphs:
                self.graphs[s][0].replay()
            else:
                self._fwd(s)
            self.ev_fwd[s].record(cur)
            if self.graphs:
                self.graphs[s][1].replay()
            else:
                self._bwd(s)
            self.ev_bwd[s].record(cur)
        with torch.cuda.stream(self.d2h):
            self.d2h.wait_event(self.ev_fwd[s])
            hy.copy_(self.yout[s], non_blocking=True)
            self.d2h.wait_event(self.ev_bwd[s])
            hdx.copy_(self.dxout[s], non_blocking=True)
            self.ev_down[s].record(self.d2h)
        self.n += 1

    def synchronize(self):
        """Wait for every submitted step; raises if the layer's exchange reported an error."""
        self.d2h.synchronize()
        self.compute.synchronize()
        self.h2d.synchronize()
        if hasattr(self.lay, "check"):
            self.lay.check()
