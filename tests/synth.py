"""Deterministic synthetic FLUX-like activation trajectories.

x0[i,j] = a_i * c_j * z_ij with a ~ LogNormal(0, 0.25) per token, c ~ LogNormal(0, 1)
per channel (outlier channels), z ~ N(0, 1); drift x_t = bf16(x_{t-1} + 0.1 a_i c_j xi_t).
Every value is bf16-representable, so the f32 upcast seen by the oracle is exact.
numpy PCG64 streams are reproducible for a fixed numpy version (2.3.5 in this image
and on the GPU box), which is what lets golden fixtures store digests instead of inputs.
"""

from __future__ import annotations

import hashlib

import numpy as np


def bf16_round(x):
    """Round f32 -> bf16 (round-to-nearest-even), returned as f32."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def flux_like(rows, cols, steps, seed, drift=0.1):
    rng = np.random.Generator(np.random.PCG64(seed))
    a = rng.lognormal(0.0, 0.25, rows)
    c = rng.lognormal(0.0, 1.0, cols)
    scale = np.outer(a, c)
    x = bf16_round((scale * rng.standard_normal((rows, cols))).astype(np.float32))
    out = [x]
    for _ in range(1, steps):
        x = bf16_round((x + drift * scale * rng.standard_normal((rows, cols))).astype(np.float32))
        out.append(x)
    return out


def gaussian(rows, cols, seed, std=1.0):
    rng = np.random.Generator(np.random.PCG64(seed))
    return (rng.standard_normal((rows, cols)) * std).astype(np.float32)


def digest(a):
    if isinstance(a, (bytes, bytearray, memoryview)):
        return hashlib.sha256(bytes(a)).hexdigest()
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
