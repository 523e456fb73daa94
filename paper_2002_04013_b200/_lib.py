"""Thin ctypes binding of libdmoe.so (include/dmoe.h).

Argument marshalling only: every function takes torch CUDA tensors, reads shapes and
data pointers, passes torch's current stream, and raises on a non-OK status.  No compute
happens here and there is no fallback: importing fails loudly if the library is missing.
"""
import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdmoe.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `make` or __graft_entry__.build() (no CPU fallback exists)")

_L = ctypes.CDLL(LIB_PATH)

DMOE_F32, DMOE_BF16 = 0, 1
_STATUS = {0: "DMOE_OK", -1: "DMOE_ERR_ARG", -2: "DMOE_ERR_SHAPE", -3: "DMOE_ERR_UNSUPPORTED", -4: "DMOE_ERR_CUDA",
           -5: "DMOE_ERR_NONFINITE"}


class dmoe_grid(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int32), ("M", ctypes.c_int32), ("k", ctypes.c_int32), ("beam", ctypes.c_int32)]


class dmoe_ep(ctypes.Structure):
    _fields_ = [("G", ctypes.c_int32), ("rank", ctypes.c_int32), ("E", ctypes.c_int32), ("E_local", ctypes.c_int32),
                ("rin_cap", ctypes.c_int64), ("timeout_ns", ctypes.c_uint64)] + [
        (n, ctypes.c_void_p) for n in ("epoch", "flags", "peer_flags", "cnt", "peer_cnt", "err", "base", "off_loc",
                                       "src_off", "dst_off")]


class dmoe_layer(ctypes.Structure):
    """include/dmoe.h dmoe_layer: device pointers of one layer for dmoe_layer_step_host."""
    _fields_ = [("g", dmoe_grid), ("D", ctypes.c_int32), ("H", ctypes.c_int32), ("tie", ctypes.c_int32),
                ("dt", ctypes.c_int32), ("T_max", ctypes.c_int64), ("R_cap", ctypes.c_int64)] + [
        (n, ctypes.c_void_p) for n in (
            "Wg", "bg", "W1", "b1", "W2", "b2", "alive_bits", "responded_bits", "x", "dy", "G",
            "sel", "sel_score", "w", "valid", "n_dropped", "counts", "offsets", "seg", "row_of_slot",
            "token_of_row", "xd", "h", "hmask", "out", "y", "dout", "dscore", "dxd", "dW1", "db1", "dW2",
            "db2", "dx", "dWg", "dbg", "ws")] + [("ws_bytes", ctypes.c_size_t)]


class DMoEError(RuntimeError):
    def __init__(self, fn, status):
        msg = _L.dmoe_last_error().decode()
        super().__init__(f"{fn}: {_STATUS.get(status, status)}: {msg}")
        self.status = status


_P, _I64, _I32, _SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t
_SIGS = {
    "dmoe_last_error": ([], ctypes.c_char_p),
    "dmoe_version": ([], ctypes.c_int32),
    "dmoe_launch_counters": ([_P, _I32], ctypes.c_int32),
    "dmoe_workspace_bytes": ([_I64, _I32, _I32, dmoe_grid, _I32, _I64], ctypes.c_size_t),
    "dmoe_gate_scores": ([_P, _I32, _I64, _I32, _P, _P, dmoe_grid, _P, _P, _SZ, _P], ctypes.c_int),
    "dmoe_topk_exact": ([_P, _I64, dmoe_grid, _P, _P, _P, _P], ctypes.c_int),
    "dmoe_gate_topk": ([_P, _I32, _I64, _I32, _P, _P, dmoe_grid, _P, _P, _P, _P, _P, _SZ, _P], ctypes.c_int),
    "dmoe_beam_topk": ([_P, _I64, dmoe_grid, _P, _P, _P, _P, _SZ, _P], ctypes.c_int),
    "dmoe_dispatch": ([_P, _I32, _I64, _I32, dmoe_grid, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                       _SZ, _P], ctypes.c_int),
    "dmoe_expert_ffn_fwd": ([_P, _P, _I32, _I64, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P],
                            ctypes.c_int),
    "dmoe_combine": ([_P, _P, _P, _P, _I64, _I32, _I32, _I32, _P, _P], ctypes.c_int),
    "dmoe_combine_bwd": ([_P, _P, _P, _P, _I64, _I32, _I32, _I32, _P, _P, _P], ctypes.c_int),
    "dmoe_combine_bwd_failures": ([_P, _P, _P, _P, _P, _P, _I64, _I32, _I32, _I32, _P, _P, _P], ctypes.c_int),
    "dmoe_expert_ffn_bwd": ([_P, _P, _P, _P, _P, _I32, _I64, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P,
                             _SZ, _P], ctypes.c_int),
    "dmoe_expert_ffn_bwd_sgd": ([_P, _P, _P, _P, _P, _I32, _I64, _I32, _I32, _I32, _P, _P, _P, _P, ctypes.c_float,
                                 _P, _P, _SZ, _P], ctypes.c_int),
    "dmoe_expert_ffn3_fwd": ([_P, _P, _I32, _I64, _I32, _I32, _I32] + [_P] * 10 + [ctypes.c_float] + [_P] * 6
                             + [_P, _SZ, _P], ctypes.c_int),
    "dmoe_expert_ffn3_bwd": ([_P] * 8 + [_I32, _I64, _I32, _I32, _I32] + [_P] * 19 + [_SZ, _P], ctypes.c_int),
    "dmoe_gate_bwd": ([_P, _P, _P, _P, _P, _P, _I64, _I32, dmoe_grid, _I32, _P, _P, _P, _P, _SZ, _P],
                      ctypes.c_int),
    "dmoe_segment_offsets": ([_P, _I32, _I32, _P, _P], ctypes.c_int),
    "dmoe_exchange_layout": ([_P, _I32, _I32, _I64, _P, _P, _P, _SZ, _P], ctypes.c_int),
    "dmoe_ep_begin": ([_P, _P], ctypes.c_int),
    "dmoe_ep_exchange_counts": ([_P, _P, _P], ctypes.c_int),
    "dmoe_ep_push_rows": ([_P, _P, _I32, _P, _P, _I32, _P, _I32, _P], ctypes.c_int),
    "dmoe_ep_return_rows": ([_P, _P, _I32, _I32, _P, _I32, _P], ctypes.c_int),
    "dmoe_ipc_alloc": ([_SZ, _P, _P], ctypes.c_int),
    "dmoe_ipc_open": ([_P, _P], ctypes.c_int),
    "dmoe_ipc_close": ([_P], ctypes.c_int),
    "dmoe_ipc_free": ([_P], ctypes.c_int),
    "dmoe_permute_rows": ([_P, _I32, _P, _P, _I32, _I32, _P, _P], ctypes.c_int),
    "dmoe_layer_step_host": ([_P, _I64, _P, _P, _P, _P, _P], ctypes.c_int),
    "dmoe_set_check_finite": ([ctypes.c_int], None),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(_L, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_SIGS)
__all__ = [n for n in _SIGS if n != "dmoe_last_error"] + ["grid", "DMoEError", "dmoe_ep", "dmoe_grid", "dmoe_layer"]


def _check(fn, st):
    if st != 0:
        raise DMoEError(fn, st)


def _p(t):
    return None if t is None else t.data_ptr()


def _dt(t):
    if t.dtype == torch.bfloat16:
        return DMOE_BF16
    if t.dtype == torch.float32:
        return DMOE_F32
    raise TypeError(f"unsupported dtype {t.dtype}")


def _stream():
    return torch.cuda.current_stream().cuda_stream


def grid(d, M, k, beam=0):
    return dmoe_grid(d, M, k, beam)


def dmoe_version():
    return _L.dmoe_version()


def dmoe_launch_counters():
    """(all launches, tcgen05 GEMM launches, SIMT GEMM launches) issued by this process."""
    buf = (ctypes.c_int64 * 4)()
    _L.dmoe_launch_counters(buf, 4)
    return tuple(buf[:3])


def dmoe_workspace_bytes(T, D, H, g, E_local, R_cap):
    return int(_L.dmoe_workspace_bytes(T, D, H, g, E_local, R_cap))


def dmoe_gate_scores(x, Wg, bg, g, G, ws):
    T, D = x.shape
    _check("dmoe_gate_scores", _L.dmoe_gate_scores(_p(x), _dt(x), T, D, _p(Wg), _p(bg), g, _p(G), _p(ws),
                                                   ws.numel() * ws.element_size(), _stream()))


def dmoe_gate_topk(x, Wg, bg, g, alive_bits, G, sel, sel_score, ws):
    """G may be None (not written)."""
    T, D = x.shape
    _check("dmoe_gate_topk", _L.dmoe_gate_topk(_p(x), _dt(x), T, D, _p(Wg), _p(bg), g, _p(alive_bits), _p(G),
                                               _p(sel), _p(sel_score), _p(ws), ws.numel() * ws.element_size(),
                                               _stream()))


def dmoe_topk_exact(G, g, alive_bits, sel, sel_score):
    _check("dmoe_topk_exact", _L.dmoe_topk_exact(_p(G), G.shape[0], g, _p(alive_bits), _p(sel), _p(sel_score),
                                                 _stream()))


def dmoe_beam_topk(G, g, alive_bits, sel, sel_score, ws):
    _check("dmoe_beam_topk", _L.dmoe_beam_topk(_p(G), G.shape[0], g, _p(alive_bits), _p(sel), _p(sel_score),
                                               _p(ws), ws.numel() * ws.element_size(), _stream()))


def dmoe_dispatch(x, g, sel, sel_score, responded_bits, w, valid, n_dropped, counts, offsets,
                  row_of_slot, token_of_row, xd, ws):
    T, D = x.shape
    _check("dmoe_dispatch", _L.dmoe_dispatch(
        _p(x), _dt(x), T, D, g, _p(sel), _p(sel_score), _p(responded_bits), _p(w), _p(valid), _p(n_dropped),
        _p(counts), _p(offsets), _p(row_of_slot), _p(token_of_row), _p(xd), _p(ws),
        ws.numel() * ws.element_size(), _stream()))


def dmoe_expert_ffn_fwd(xd, offsets, W1, b1, W2, b2, h, out, ws, hmask=None):
    E_local, H, D = W1.shape
    _check("dmoe_expert_ffn_fwd", _L.dmoe_expert_ffn_fwd(
        _p(xd), _p(offsets), E_local, xd.shape[0], D, H, _dt(xd), _p(W1), _p(b1), _p(W2), _p(b2), _p(h),
        _p(hmask) if hmask is not None else None, _p(out), _p(ws), ws.numel() * ws.element_size(), _stream()))


def dmoe_combine(out, row_of_slot, w, valid, y):
    T, D = y.shape
    _check("dmoe_combine", _L.dmoe_combine(_p(out), _p(row_of_slot), _p(w), _p(valid), T, D,
                                           row_of_slot.shape[1], _dt(y), _p(y), _stream()))


def dmoe_combine_bwd(dy, out, row_of_slot, w, dout, dscore):
    T, D = dy.shape
    _check("dmoe_combine_bwd", _L.dmoe_combine_bwd(_p(dy), _p(out), _p(row_of_slot), _p(w), T, D,
                                                   row_of_slot.shape[1], _dt(dy), _p(dout), _p(dscore),
                                                   _stream()))


def dmoe_combine_bwd_failures(dy, out, row_of_slot, w, sel, responded_bwd_bits, dout, dscore):
    T, D = dy.shape
    _check("dmoe_combine_bwd_failures", _L.dmoe_combine_bwd_failures(
        _p(dy), _p(out), _p(row_of_slot), _p(w), _p(sel), _p(responded_bwd_bits), T, D, row_of_slot.shape[1],
        _dt(dy), _p(dout), _p(dscore), _stream()))


def dmoe_expert_ffn_bwd(xd, h, dout, offsets, W1, W2, dxd, dW1, db1, dW2, db2, ws, hmask=None):
    E_local, H, D = W1.shape
    _check("dmoe_expert_ffn_bwd", _L.dmoe_expert_ffn_bwd(
        _p(xd), _p(h), _p(hmask) if hmask is not None else None, _p(dout), _p(offsets), E_local, xd.shape[0], D, H, _dt(xd), _p(W1), _p(W2), _p(dxd),
        _p(dW1), _p(db1), _p(dW2), _p(db2), _p(ws), ws.numel() * ws.element_size(), _stream()))


def dmoe_expert_ffn_bwd_sgd(xd, h, dout, offsets, W1, b1, W2, b2, lr, dxd, ws, hmask=None):
    """h may be None (recomputed in the call: gradient checkpointing)."""
    E_local, H, D = W1.shape
    _check("dmoe_expert_ffn_bwd_sgd", _L.dmoe_expert_ffn_bwd_sgd(
        _p(xd), _p(h), _p(hmask), _p(dout), _p(offsets), E_local, xd.shape[0], D, H, _dt(xd), _p(W1), _p(b1),
        _p(W2), _p(b2), float(lr), _p(dxd), _p(ws), ws.numel() * ws.element_size(), _stream()))


def dmoe_expert_ffn3_fwd(xd, offsets, P, eps, z1, a1, z2, a2, stats, out, ws):
    """P: dict of the block's parameters W1, b1, g1, be1, W2, b2, g2, be2, W3, b3 (layer.py)."""
    E_local, H, D = P["W1"].shape
    _check("dmoe_expert_ffn3_fwd", _L.dmoe_expert_ffn3_fwd(
        _p(xd), _p(offsets), E_local, xd.shape[0], D, H, _dt(xd),
        *[_p(P[n]) for n in ("W1", "b1", "g1", "be1", "W2", "b2", "g2", "be2", "W3", "b3")], float(eps),
        _p(z1), _p(a1), _p(z2), _p(a2), _p(stats), _p(out), _p(ws), ws.numel() * ws.element_size(), _stream()))


def dmoe_expert_ffn3_bwd(xd, z1, a1, z2, a2, stats, dout, offsets, P, dxd, Gr, ws):
    """Gr: dict of gradient buffers dW1, db1, dg1, dbe1, dW2, db2, dg2, dbe2, dW3, db3."""
    E_local, H, D = P["W1"].shape
    _check("dmoe_expert_ffn3_bwd", _L.dmoe_expert_ffn3_bwd(
        _p(xd), _p(z1), _p(a1), _p(z2), _p(a2), _p(stats), _p(dout), _p(offsets), E_local, xd.shape[0], D, H,
        _dt(xd), *[_p(P[n]) for n in ("W1", "g1", "be1", "W2", "g2", "be2", "W3")], _p(dxd),
        *[_p(Gr[n]) for n in ("dW1", "db1", "dg1", "dbe1", "dW2", "db2", "dg2", "dbe2", "dW3", "db3")],
        _p(ws), ws.numel() * ws.element_size(), _stream()))


def dmoe_gate_bwd(x, Wg, sel, dscore, dxd, row_of_slot, g, dx, dWg, dbg, ws):
    T, D = x.shape
    _check("dmoe_gate_bwd", _L.dmoe_gate_bwd(
        _p(x), _p(Wg), _p(sel), _p(dscore), _p(dxd), _p(row_of_slot), T, D, g, _dt(x), _p(dx), _p(dWg),
        _p(dbg), _p(ws), ws.numel() * ws.element_size(), _stream()))


def dmoe_segment_offsets(offsets, group, seg):
    E = offsets.shape[0] - 1
    _check("dmoe_segment_offsets", _L.dmoe_segment_offsets(_p(offsets), E, group, _p(seg), _stream()))


def dmoe_exchange_layout(recv_counts, G, E_local, offsets, src_of_dst, ws):
    _check("dmoe_exchange_layout", _L.dmoe_exchange_layout(
        _p(recv_counts), G, E_local, src_of_dst.shape[0], _p(offsets), _p(src_of_dst), _p(ws),
        ws.numel() * ws.element_size(), _stream()))


def dmoe_permute_rows(src, idx, n_rows, inverse, dst):
    _check("dmoe_permute_rows", _L.dmoe_permute_rows(_p(src), _dt(src), _p(idx), _p(n_rows), src.shape[1],
                                                     int(inverse), _p(dst), _stream()))


# ---------------------------------------------------------------- peer-memory exchange
def dmoe_ep_begin(ep):
    _check("dmoe_ep_begin", _L.dmoe_ep_begin(ctypes.byref(ep), _stream()))


def dmoe_ep_exchange_counts(ep, counts):
    _check("dmoe_ep_exchange_counts", _L.dmoe_ep_exchange_counts(ctypes.byref(ep), _p(counts), _stream()))


def dmoe_ep_push_rows(ep, src, gather_idx, offsets, peer_dst, phase):
    _check("dmoe_ep_push_rows", _L.dmoe_ep_push_rows(ctypes.byref(ep), _p(src), _dt(src), _p(gather_idx), _p(offsets),
                                                     src.shape[1], _p(peer_dst), phase, _stream()))


def dmoe_ep_return_rows(ep, src, peer_dst, phase):
    _check("dmoe_ep_return_rows", _L.dmoe_ep_return_rows(ctypes.byref(ep), _p(src), _dt(src), src.shape[1],
                                                         _p(peer_dst), phase, _stream()))


def dmoe_ipc_alloc(nbytes):
    ptr = ctypes.c_void_p()
    handle = (ctypes.c_char * 64)()
    _check("dmoe_ipc_alloc", _L.dmoe_ipc_alloc(nbytes, ctypes.byref(ptr), handle))
    return ptr.value, bytes(handle)


def dmoe_ipc_open(handle):
    ptr = ctypes.c_void_p()
    buf = (ctypes.c_char * 64).from_buffer_copy(handle)
    _check("dmoe_ipc_open", _L.dmoe_ipc_open(buf, ctypes.byref(ptr)))
    return ptr.value


def dmoe_ipc_close(ptr):
    _check("dmoe_ipc_close", _L.dmoe_ipc_close(ptr))


def dmoe_ipc_free(ptr):
    _check("dmoe_ipc_free", _L.dmoe_ipc_free(ptr))


def dmoe_layer_step_host(layer, T, x_host, dy_host, y_host, dx_host):
    """One layer step from host buffers (pinned torch CPU tensors [T, D]); layer: dmoe_layer."""
    for t in (x_host, dy_host, y_host, dx_host):
        assert not t.is_cuda and t.is_contiguous()
    _check("dmoe_layer_step_host", _L.dmoe_layer_step_host(ctypes.byref(layer), T, _p(x_host), _p(dy_host),
                                                           _p(y_host), _p(dx_host), _stream()))


def dmoe_set_check_finite(on):
    """Debug switch: calls scan their outputs, synchronise and raise DMOE_ERR_NONFINITE on NaN / Inf."""
    _L.dmoe_set_check_finite(1 if on else 0)
