"""Counter-based synthetic input generator (shared by the oracle side and the GPU side).

Holds none of the DMoE method's arithmetic: it maps (seed, tensor_id, index) to a value
(see gen/counter_gen.h).  Host arrays come from libgen_host.so, device buffers from
libgen_device.so; both compile the same header, so they agree bit for bit
(tests/test_gen.py, tests/test_gpu_gen.py).
"""
import ctypes
import os

import numpy as np

from .configs import CONFIGS, Config  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))

X, WG, BG, W1, B1, W2, B2, DY, ALIVE, RESPONDED = range(1, 11)
# the §4.1 expert block (NEXT-2): middle linear W2 [E,H,H] / b2 reuse W2 / B2's ids; these are new
W3, B3, LN1G, LN1B, LN2G, LN2B = range(11, 17)
NORMAL, UNIFORM, GRID8, ZERO = range(4)

_host = None
_dev = None


def _load_host():
    global _host
    if _host is None:
        path = os.path.join(_HERE, "libgen_host.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make` (or __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        lib.gen_fill_f32.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_float,
                                     ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p]
        lib.gen_fill_bf16.argtypes = lib.gen_fill_f32.argtypes
        lib.gen_fill_mask.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                      ctypes.c_int64, ctypes.c_void_p]
        _host = lib
    return _host


def _load_dev():
    global _dev
    if _dev is None:
        path = os.path.join(_HERE, "libgen_device.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make` (or __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        lib.gen_dev_fill_f32.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_float,
                                         ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        lib.gen_dev_fill_bf16.argtypes = lib.gen_dev_fill_f32.argtypes
        lib.gen_dev_fill_mask.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                          ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        for f in (lib.gen_dev_fill_f32, lib.gen_dev_fill_bf16, lib.gen_dev_fill_mask):
            f.restype = ctypes.c_int
        _dev = lib
    return _dev


# ---------------------------------------------------------------- host side
def host_f32(seed, tid, dist, scale, n, idx0=0):
    out = np.empty(n, dtype=np.float32)
    _load_host().gen_fill_f32(seed, tid, dist, float(np.float32(scale)), idx0, n, out.ctypes.data)
    return out


def host_bf16_bits(seed, tid, dist, scale, n, idx0=0):
    out = np.empty(n, dtype=np.uint16)
    _load_host().gen_fill_bf16(seed, tid, dist, float(np.float32(scale)), idx0, n, out.ctypes.data)
    return out


def bf16_bits_to_f64(bits):
    """Exact upcast of bf16 bit patterns (uint16) to float64."""
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def host_mask(seed, tid, fail_frac, nbits):
    out = np.empty((nbits + 31) // 32, dtype=np.uint32)
    _load_host().gen_fill_mask(seed, tid, mask_threshold(fail_frac), nbits, out.ctypes.data)
    return out


def mask_threshold(fail_frac):
    return int(round(float(fail_frac) * (1 << 24)))


def unpack_mask(words, nbits):
    b = np.unpackbits(words.view(np.uint8), bitorder="little")[:nbits]
    return b.astype(np.uint8)


# -------------------------------------------------------------- device side
def dev_fill(tensor, seed, tid, dist, scale, idx0=0, stream=None):
    """Fill a CUDA tensor (float32 or bfloat16) in place with elements [idx0, idx0+numel)."""
    import torch
    lib = _load_dev()
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    n = tensor.numel()
    if tensor.dtype == torch.float32:
        rc = lib.gen_dev_fill_f32(seed, tid, dist, float(np.float32(scale)), idx0, n, tensor.data_ptr(), s)
    elif tensor.dtype == torch.bfloat16:
        rc = lib.gen_dev_fill_bf16(seed, tid, dist, float(np.float32(scale)), idx0, n, tensor.data_ptr(), s)
    else:
        raise TypeError(tensor.dtype)
    if rc != 0:
        raise RuntimeError(f"gen_dev_fill failed: cuda error {rc}")
    return tensor


def dev_mask(tensor_u32, seed, tid, fail_frac, nbits, stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    rc = _load_dev().gen_dev_fill_mask(seed, tid, mask_threshold(fail_frac), nbits, tensor_u32.data_ptr(), s)
    if rc != 0:
        raise RuntimeError(f"gen_dev_fill_mask failed: cuda error {rc}")
    return tensor_u32
