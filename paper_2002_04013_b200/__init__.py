"""B200-native DMoE layer hot path (Learning@home, arXiv 2002.04013).

The product is libdmoe.so (C ABI, include/dmoe.h); this package is its thin binding
(same names as the C functions) plus the layer sequencers DMoELayer (one GPU),
EPDMoELayer (experts sharded, NCCL exchange) and PeerEPDMoELayer (experts sharded,
NVLink peer-memory exchange, graph-capturable), and HostPipeline (steps streamed from
pinned host memory with neighbouring steps' copies overlapped).
"""
from ._lib import *  # noqa: F401,F403
from ._lib import DMoEError, EXPORTED, LIB_PATH, grid  # noqa: F401
from .host_pipeline import HostPipeline  # noqa: F401
from .layer import DMoELayer  # noqa: F401
