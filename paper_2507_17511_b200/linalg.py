"""Host-side pieces of the reference's linalg substrate (la = linalg.py) that the
device path still needs: the error class and the seeded PCG64 streams that the
low-rank codec draws its initial Gaussian block from (la:20-27, la:67-74)."""

from __future__ import annotations

import numpy as np

DEGENERATE_COL_TOL = 1e-12  # la:13


class ShapeError(ValueError):
    """Same role as compactcomm.linalg.ShapeError (la:16)."""


def make_rng(seed):
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(seed)))  # la:20-22


def spawn_rng(seed, *key):
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(entropy=seed, spawn_key=tuple(key))))


def gaussian_matrix(rng, rows, cols, stddev=1.0):
    """Host draw identical to la.gaussian_matrix (f64 normals -> f32)."""
    if rows < 1 or cols < 1:
        raise ShapeError("gaussian_matrix needs rows, cols >= 1")
    if stddev <= 0:
        raise ValueError("stddev must be positive")
    return (rng.standard_normal((rows, cols), dtype=np.float64) * stddev).astype(np.float32)
