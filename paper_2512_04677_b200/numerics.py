"""Host-side numerics: counter-based RNG and rotary tables.

``Prng`` keeps the reference's seeding contract (numerics.py:118-143):
Philox keyed by (seed, stream), standard normal float32 -- so weights,
noise and conditioning generated here are the reference's numbers.  Rotary
angles are computed in fp64 and rounded to fp32 tables (numerics.py:104-109)
that the device kernels consume.
"""

from __future__ import annotations

import numpy as np

F32 = np.float32


class Prng:
    """Philox(key=[seed, stream]) standard-normal source (numerics.py:118-143)."""

    def __init__(self, seed: int, stream: int = 0):
        if seed < 0 or stream < 0:
            raise ValueError("seed and stream must be non-negative")
        self.seed = seed
        self.stream = stream
        self._gen = np.random.Generator(np.random.Philox(key=np.array([seed, stream], dtype=np.uint64)))

    def gaussian(self, dim: int) -> np.ndarray:
        if dim < 1:
            raise ValueError("dim must be >= 1")
        return self._gen.standard_normal(dim, dtype=F32)

    def normal(self, shape) -> np.ndarray:
        return self._gen.standard_normal(shape, dtype=F32)


def gaussian(prng: Prng, dim: int) -> np.ndarray:
    return prng.gaussian(dim)


def rope_frequencies(dim: int, base: float) -> np.ndarray:
    """base^(-2k/dim), fp64 (numerics.py:81-86)."""
    if dim % 2 != 0:
        raise ValueError(f"RoPE needs an even dim, got {dim}")
    return base ** (-2.0 * np.arange(dim // 2, dtype=np.float64) / dim)


def rope_table(pos, dim: int, base: float):
    """fp64 angles pos * theta_k, cos/sin rounded to fp32."""
    ang = np.multiply.outer(np.asarray(pos, dtype=np.float64), rope_frequencies(dim, base))
    return np.cos(ang).astype(F32), np.sin(ang).astype(F32)


def spatial_tables(grid_h: int, grid_w: int, dh: int, dw: int, base: float):
    """Per-token (h, w) rotary tables for a patch grid: (S, dh/2 + dw/2)."""
    s = grid_h * grid_w
    idx = np.arange(s)
    parts_c, parts_s = [], []
    if dh:
        c, sn = rope_table(idx // grid_w, dh, base)
        parts_c.append(c)
        parts_s.append(sn)
    if dw:
        c, sn = rope_table(idx % grid_w, dw, base)
        parts_c.append(c)
        parts_s.append(sn)
    if not parts_c:
        return np.zeros((s, 0), F32), np.zeros((s, 0), F32)
    return np.ascontiguousarray(np.concatenate(parts_c, 1)), np.ascontiguousarray(np.concatenate(parts_s, 1))
