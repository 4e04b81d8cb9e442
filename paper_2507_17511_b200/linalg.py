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


def assembled_entropy(seed, key):
    """SeedSequence's assembled entropy words (numpy bit_generator.pyx
    get_assembled_entropy): the entropy's little-endian uint32 words, zero-padded to
    the 4-word pool when a spawn key follows, then the spawn key's words."""
    def words(v):
        v = int(v)
        if v < 0:
            raise ValueError("entropy and spawn keys must be non-negative")
        out = [] if v else [0]
        while v:
            out.append(v & 0xFFFFFFFF)
            v >>= 32
        return out

    run = words(seed)
    spawn = [w for k in key for w in words(k)]
    if spawn and len(run) < 4:
        run += [0] * (4 - len(run))
    return run + spawn


class DeviceKey:
    """`spawn_rng(seed, *key)` drawn on the GPU (cc_gaussian_keyed): the low-rank
    start block comes out bit-identical to `gaussian_matrix(spawn_rng(seed, *key),
    ...)` (la:25-27, la:67-74) without a host draw.  With `advance=True` the LAST
    key element is a step counter held in device memory and incremented by every
    draw, so a captured step draws the next step's block on each replay (the keys
    of pl:190 `(seed, 5, t)` and mesh:193 `(seed, 6, device, t)`)."""

    def __init__(self, seed, *key, advance=False, device=None):
        import torch

        words = assembled_entropy(seed, key)
        if len(words) > 16:
            raise ValueError("key too long for the device generator (16 words)")
        if advance and (not key or int(key[-1]) >= 2**32 - 1024):
            raise ValueError("an advancing key needs a last element < 2^32 (the step counter)")
        self.seed, self.key, self.advance = seed, tuple(key), bool(advance)
        self.nwords = len(words)
        self.step_word = self.nwords - 1 if advance else -1
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.words = torch.tensor(words, dtype=torch.int64).to(torch.int32).to(dev)

    def host_generator(self):
        """The numpy stream this key stands for at its current step (test helper; syncs)."""
        words = [int(w) & 0xFFFFFFFF for w in self.words.cpu().tolist()]
        key = list(self.key)
        if self.advance:
            key[-1] = words[self.step_word]
        return spawn_rng(self.seed, *key)
