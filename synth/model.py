"""Seeded random GRU-RNNLM parameters (stand-in for trained weights).

Shapes follow the paper's model: a single GRU hidden layer with "six weight
matrices and three bias vectors", an NCE output matrix of size
H x V plus bias (stored row-per-word, V x H) and a hashed MaxEnt
table.  E (embedding width) and M (MaxEnt table size) are not
stated by the paper; E = H (SURVEY 8(c) reading 14) and M = 2^m per
BASELINE.json's configs.

Distribution: every entry i.i.d.
U(-a, a) with a = 0.1 * sqrt(256 / H), then rounded to the nearest bf16
value (round-to-nearest-even).  The bf16 grid makes the tensor-core path's
operand conversion lossless; the 1/sqrt(H) scale keeps the recurrent
spectral radius below one so that histories with a common recent past
converge, which is what the paper's lossy history keys rely on.
"""
from __future__ import annotations

import dataclasses

import numpy as np

# BASELINE.json "configs", made concrete.
CONFIGS = {
    "tiny": dict(V=1000, E=64, H=64, maxent_log2=16, N=3, S=1, B_s=32, frames=100),
    "moderate": dict(V=100_000, E=256, H=256, maxent_log2=22, N=4, S=1, B_s=256, frames=400),
    "large": dict(V=200_000, E=1024, H=1024, maxent_log2=27, N=4, S=1, B_s=2048, frames=400),
    "multi": dict(V=200_000, E=1024, H=1024, maxent_log2=27, N=4, S=64, B_s=2048, frames=400),
}

PARAM_ORDER = ("emb", "Wz", "Uz", "bz", "Wr", "Ur", "br", "Wh", "Uh", "bh",
               "nce_w", "nce_b", "maxent")


@dataclasses.dataclass(frozen=True)
class ModelDims:
    V: int
    E: int
    H: int
    maxent_log2: int
    N: int

    @property
    def M(self) -> int:
        return 1 << self.maxent_log2

    def shapes(self) -> dict:
        V, E, H, M = self.V, self.E, self.H, self.M
        return {"emb": (V, E), "Wz": (H, E), "Uz": (H, H), "bz": (H,),
                "Wr": (H, E), "Ur": (H, H), "br": (H,),
                "Wh": (H, E), "Uh": (H, H), "bh": (H,),
                "nce_w": (V, H), "nce_b": (V,), "maxent": (M,)}


def model_dims(name: str) -> ModelDims:
    c = CONFIGS[name]
    return ModelDims(V=c["V"], E=c["E"], H=c["H"], maxent_log2=c["maxent_log2"], N=c["N"])


def round_to_bf16_grid(x: np.ndarray) -> np.ndarray:
    """Nearest bf16 value (ties to even), returned as float32."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    lsb = (u >> np.uint32(16)) & np.uint32(1)
    r = (u + np.uint32(0x7FFF) + lsb) & np.uint32(0xFFFF0000)
    return r.view(np.float32)


def generate_model(dims: ModelDims, seed: int = 1234, scale: float | None = None,
                   bf16_grid: bool = True) -> dict:
    """Return {name: float32 C-contiguous array} for every parameter.

    Each tensor has its own child seed (SeedSequence.spawn), so a tensor's
    values do not depend on which other tensors were drawn.
    """
    a = 0.1 * np.sqrt(256.0 / dims.H) if scale is None else float(scale)
    shapes = dims.shapes()
    children = np.random.SeedSequence(seed).spawn(len(PARAM_ORDER))
    out = {}
    for name, ss in zip(PARAM_ORDER, children):
        rng = np.random.Generator(np.random.PCG64(ss))
        n = int(np.prod(shapes[name]))
        v = rng.random(n, dtype=np.float32)
        v *= np.float32(2.0 * a)
        v -= np.float32(a)
        if bf16_grid:
            v = round_to_bf16_grid(v)
        out[name] = v.reshape(shapes[name])
    return out


def zero_model(dims: ModelDims) -> dict:
    return {k: np.zeros(s, dtype=np.float32) for k, s in dims.shapes().items()}
