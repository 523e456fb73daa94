"""The five BASELINE.json workloads and the synthetic-input recipe.

No method arithmetic here: shapes, distributions and scales only.  Recipe:
continuous mode X ~ N(0,1), W_g ~ N(0, 1/D) so each per-dimension logit ~ N(0,1), b_g = 0,
W1,b1 ~ U(+-1/sqrt(D)), W2,b2 ~ U(+-1/sqrt(H)) (SPEC.md:79 init), dY ~ N(0,1);
exact-grid mode: X, W_g, b_g in {-7..7}/8 (exact in bf16, every fp32 partial sum exact).
`alive` all-true unless `dead_frac` > 0; `responded` ~ Bernoulli(1 - fail_frac) per expert.
"""
from dataclasses import dataclass, replace
import math

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    M: int          # grid size per dimension
    d: int          # grid dimensions
    D: int          # d_model
    H: int          # expert FFN hidden
    k: int          # experts per token
    T: int          # tokens per step
    dtype: str      # "f32" or "bf16"
    fail_frac: float = 0.0   # P(expert does not respond) -> `responded`
    dead_frac: float = 0.0   # P(expert dead before selection) -> `alive`
    beam: int = 0            # beam width B (0 -> k, the paper's Alg. 1)
    exact_grid: bool = False
    pool: int = 0            # parameter slots of the tied-weight pool (0 -> E, no tying; X20)
    expert: str = "ffn2"     # "ffn2": D -> H -> D (X14); "ffn3": the paper's §4.1 block (X23)
    chunk: int = 0           # bench: tokens per layer call when the step does not fit one call
                             # (each chunk is a Backward request with the fused SGD update)

    @property
    def E(self):
        return self.M ** self.d

    @property
    def dM(self):
        return self.d * self.M

    @property
    def P(self):
        """Expert parameter slots: expert e computes with slot e // tie (reading X20)."""
        return self.pool if self.pool else self.E

    @property
    def tie(self):
        return self.E // self.P

    @property
    def B(self):
        return self.beam if self.beam else self.k

    def with_(self, **kw):
        return replace(self, **kw)

    # ---- recipe: (distribution, scale) per tensor id
    def dist(self, tid):
        from . import X, WG, BG, W1, B1, W2, B2, DY, NORMAL, UNIFORM, GRID8, ZERO
        f32 = lambda v: float(np.float32(v))
        if self.exact_grid and tid in (X, WG, BG):
            return GRID8, 1.0
        return {
            X: (NORMAL, 1.0),
            WG: (NORMAL, f32(1.0 / math.sqrt(self.D))),
            BG: (ZERO, 0.0),
            W1: (UNIFORM, f32(1.0 / math.sqrt(self.D))),
            B1: (UNIFORM, f32(1.0 / math.sqrt(self.D))),
            W2: (UNIFORM, f32(1.0 / math.sqrt(self.H))),
            B2: (UNIFORM, f32(1.0 / math.sqrt(self.H))),
            DY: (NORMAL, 1.0),
        }[tid]


CONFIGS = {
    # BASELINE.json configs[0..4]
    "tiny": Config("tiny", M=4, d=2, D=64, H=256, k=4, T=32, dtype="f32"),
    "mnist": Config("mnist", M=16, d=2, D=256, H=1024, k=4, T=4096, dtype="bf16", fail_frac=0.10),
    "transformer": Config("transformer", M=64, d=2, D=1024, H=4096, k=4, T=65536, dtype="bf16"),
    "grid3d": Config("grid3d", M=16, d=3, D=1024, H=4096, k=4, T=262144, dtype="bf16"),
    # the paper's own expert block (§4.1: D -> H -> H -> D with LayerNorm + ReLU;
    # NEXT-2) on the MNIST-style layer, and on the Transformer layer with a 1024-slot tied pool
    # (4096 distinct blocks would need 206 GB of weights alone)
    "mnist_block": Config("mnist_block", M=16, d=2, D=256, H=1024, k=4, T=4096, dtype="bf16", fail_frac=0.10,
                          expert="ffn3"),
    "transformer_block": Config("transformer_block", M=64, d=2, D=1024, H=4096, k=4, T=65536, dtype="bf16",
                                expert="ffn3", pool=1024),
    # 1M tokens per GPU: 8 calls of 131,072 tokens, each a full fwd + bwd with the runtime's SGD
    # update; 512 parameter slots (the tied pool SURVEY §8(d) declares for G <= 2)
    "stress": Config("stress", M=64, d=2, D=2048, H=8192, k=8, T=1048576, dtype="bf16", fail_frac=0.30,
                     pool=512, chunk=131072),
}
