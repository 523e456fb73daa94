"""B200-native DMoE layer hot path (Learning@home, arXiv 2002.04013).

The product is libdmoe.so (C ABI, include/dmoe.h); this package is its thin binding.
"""
from ._lib import (  # noqa: F401
    DMoEError, EXPORTED, LIB_PATH, dmoe_beam_topk, dmoe_combine, dmoe_combine_bwd, dmoe_dispatch,
    dmoe_expert_ffn_bwd, dmoe_expert_ffn_fwd, dmoe_gate_bwd, dmoe_gate_scores, dmoe_launch_counters, dmoe_version,
    dmoe_workspace_bytes, dmoe_exchange_layout, dmoe_permute_rows, grid,
)
from .layer import DMoELayer  # noqa: F401
