"""TEST INFRASTRUCTURE (oracle): pure-Python restatement of the random stream the
reference draws its low-rank start block from, so the device generator
(csrc/rng.cu) can be checked step by step.  Only tests/ may import this.

Reference call chain: compressors.py:407 `linalg.gaussian_matrix(rng, cols, r)`
(linalg.py:67-74: `rng.standard_normal((rows, cols), dtype=float64) * stddev`
-> float32), with rng = `linalg.spawn_rng(seed, *key)` (linalg.py:25-27:
`Generator(PCG64(SeedSequence(entropy=seed, spawn_key=key)))`), keys from
pipeline.py:190 (seed, 5, t) and mesh.py:193 (seed, 6, device, t).

The algorithms are numpy's (the reference's only dependency; numpy 2.3.5 here,
pkg/pyproject.toml:10 pins numpy>=1.24): SeedSequence entropy mixing
(numpy/random/bit_generator.pyx), PCG64 = 128-bit LCG with the XSL-RR output
(numpy/random/src/pcg64), and random_standard_normal's 256-level ziggurat
(numpy/random/src/distributions).  The ziggurat tables come from
oracle/ziggurat_tables.npz (scripts/gen_ziggurat.py); tests/test_np_random.py
pins this restatement to numpy's own draws.
"""

from __future__ import annotations

import math
import os

import numpy as np

M32 = 0xFFFFFFFF
M64 = (1 << 64) - 1
M128 = (1 << 128) - 1
INIT_A, MULT_A = 0x43B0D7E5, 0x931E8875
INIT_B, MULT_B = 0x8B51F9DD, 0x58F38DED
MIX_MULT_L, MIX_MULT_R = 0xCA01F9DD, 0x4973F715
XSHIFT = 16
POOL = 4
PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645

_T = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "ziggurat_tables.npz"))
KI = [int(v) for v in _T["ki"]]
WI = [float(v) for v in _T["wi"]]
FI = [float(v) for v in _T["fi"]]
NOR_R = float(_T["nor_r"])
NOR_INV_R = float(_T["nor_inv_r"])


def uint32_words(v):
    """_int_to_uint32_array: little-endian 32-bit words of a non-negative int (0 -> [0])."""
    if v < 0:
        raise ValueError("negative entropy")
    if v == 0:
        return [0]
    out = []
    while v:
        out.append(v & M32)
        v >>= 32
    return out


def assembled_entropy(seed, key):
    """SeedSequence.get_assembled_entropy: run entropy zero-padded to the pool size
    when a spawn key follows, then the spawn key's words."""
    run = uint32_words(seed)
    spawn = [w for k in key for w in uint32_words(k)]
    if spawn and len(run) < POOL:
        run = run + [0] * (POOL - len(run))
    return run + spawn


def _hashmix(value, hc):
    value ^= hc[0]
    hc[0] = (hc[0] * MULT_A) & M32
    value = (value * hc[0]) & M32
    value ^= value >> XSHIFT
    return value


def _mix(x, y):
    r = (MIX_MULT_L * x - MIX_MULT_R * y) & M32
    r ^= r >> XSHIFT
    return r


def seed_pool(words):
    """SeedSequence.mix_entropy over the assembled entropy words -> pool[4]."""
    hc = [INIT_A]
    pool = [0] * POOL
    for i in range(POOL):
        pool[i] = _hashmix(words[i] if i < len(words) else 0, hc)
    for s in range(POOL):
        for d in range(POOL):
            if s != d:
                pool[d] = _mix(pool[d], _hashmix(pool[s], hc))
    for s in range(POOL, len(words)):
        for d in range(POOL):
            pool[d] = _mix(pool[d], _hashmix(words[s], hc))
    return pool


def generate_state(pool, n_words):
    """SeedSequence.generate_state(n_words, uint32)."""
    hc = INIT_B
    out = []
    for i in range(n_words):
        v = pool[i % POOL]
        v ^= hc
        hc = (hc * MULT_B) & M32
        v = (v * hc) & M32
        v ^= v >> XSHIFT
        out.append(v)
    return out


def pcg64_seed(seed, key):
    """PCG64(SeedSequence(seed, spawn_key=key)) -> (state, inc) 128-bit ints
    (generate_state(4, uint64); pcg64_set_seed: srandom(initstate, initseq))."""
    w = generate_state(seed_pool(assembled_entropy(seed, key)), 8)
    v = [w[2 * i] | (w[2 * i + 1] << 32) for i in range(4)]
    initstate = (v[0] << 64) | v[1]
    initseq = (v[2] << 64) | v[3]
    inc = ((initseq << 1) | 1) & M128
    state = (0 * PCG_MULT + inc) & M128
    state = (state + initstate) & M128
    state = (state * PCG_MULT + inc) & M128
    return state, inc


class PCG64:
    def __init__(self, state, inc):
        self.state, self.inc = state, inc

    def next64(self):
        self.state = (self.state * PCG_MULT + self.inc) & M128
        hi, lo = self.state >> 64, self.state & M64
        rot = hi >> 58
        x = hi ^ lo
        return ((x >> rot) | (x << ((64 - rot) & 63))) & M64

    def next_double(self):
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)


PATHS = {"fast": 0, "wedge": 0, "tail": 0}  # slow-path visits (tests check coverage)


def standard_normal(g):
    """random_standard_normal (one f64 draw)."""
    while True:
        r = g.next64()
        idx = r & 0xFF
        r >>= 8
        sign = r & 1
        rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
        x = rabs * WI[idx]
        if sign:
            x = -x
        if rabs < KI[idx]:
            PATHS["fast"] += 1
            return x
        if idx == 0:
            PATHS["tail"] += 1
            while True:
                xx = -NOR_INV_R * math.log1p(-g.next_double())
                yy = -math.log1p(-g.next_double())
                if yy + yy > xx * xx:
                    return -(NOR_R + xx) if (rabs >> 8) & 1 else NOR_R + xx
        elif (FI[idx - 1] - FI[idx]) * g.next_double() + FI[idx] < math.exp(-0.5 * x * x):
            PATHS["wedge"] += 1
            return x
        else:
            PATHS["wedge"] += 1


def gaussian_matrix(seed, key, rows, cols):
    """linalg.gaussian_matrix(spawn_rng(seed, *key), rows, cols): f32 [rows, cols]."""
    g = PCG64(*pcg64_seed(seed, key))
    out = np.empty(rows * cols, np.float64)
    for i in range(rows * cols):
        out[i] = standard_normal(g)
    return out.reshape(rows, cols).astype(np.float32)
