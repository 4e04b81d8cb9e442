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

    def start_block(self, rows, cols):
        """This step's start block [rows, cols] f32 on the device, drawn one step AHEAD.

        An advancing key's next block depends only on the key, so every call also queues
        the NEXT step's draw on a side stream (forked from the caller's stream, joined at
        the start of the next call): the draw overlaps the rest of the step instead of
        leading it.  The block is handed over by a stream-ordered copy (next -> current),
        so a captured step stays correct however its graph is replayed.  The first call
        draws its own block in line; non-advancing keys always draw in line.  Returns a
        device tensor valid until the next call."""
        import torch

        from . import _lib

        lib = _lib.load()
        cur = torch.cuda.current_stream()
        shape = (int(rows), int(cols))
        if getattr(self, "_shape", None) != shape:  # (re)initialise the buffers
            self._shape = shape
            self._cur = torch.empty(shape, dtype=torch.float32, device=self.words.device)
            self._next = torch.empty_like(self._cur)
            self._ws = [torch.empty(_lib.check(lib.cc_gaussian_workspace_bytes(*shape)), dtype=torch.uint8,
                                    device=self.words.device) for _ in range(2)]
            self._side = torch.cuda.Stream(self.words.device)
            self._ready = False

        def draw(buf, ws):
            _lib.check(lib.cc_gaussian_keyed(shape[0], shape[1], _lib.ptr(self.words), self.nwords, self.step_word,
                                             _lib.ptr(buf), _lib.ptr(ws), ws.numel(), _lib.stream_ptr()),
                       "gaussian_keyed")

        if not self.advance:
            draw(self._cur, self._ws[0])
            return self._cur
        if self._ready:  # the block drawn ahead by the previous call (joined by its join())
            self._cur.copy_(self._next)
        else:
            draw(self._cur, self._ws[0])
        self._side.wait_stream(cur)  # `next` is free (copied above) and the key word is current
        with torch.cuda.stream(self._side):
            draw(self._next, self._ws[1])  # the next step's block (the key advances)
        self._ready = True
        return self._cur

    def join(self):
        """Join the draw-ahead side stream back into the caller's stream.  Called right
        after the step's launches are queued: the draw (tens of us) finishes long before
        the step (hundreds), so nothing waits, and a capture never ends with unjoined work."""
        import torch

        if getattr(self, "_ready", False) and self.advance:
            torch.cuda.current_stream().wait_stream(self._side)

    def host_generator(self):
        """The numpy stream this key stands for at its current step (test helper; syncs)."""
        import torch

        torch.cuda.synchronize()
        words = [int(w) & 0xFFFFFFFF for w in self.words.cpu().tolist()]
        key = list(self.key)
        if self.advance:  # a block drawn ahead has already advanced the device word
            key[-1] = words[self.step_word] - (1 if getattr(self, "_ready", False) else 0)
        return spawn_rng(self.seed, *key)
