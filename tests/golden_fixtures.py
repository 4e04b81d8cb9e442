"""Loader for the committed golden fixtures (produced by tests/golden/make_golden.py
from the reference implementation itself)."""

from __future__ import annotations

import functools
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

TAG = {"raw": 0, "sign1bit": 1, "quant2bit": 2, "lowrank": 3, "lowrank4": 4, "nmblock": 5, "topk": 6}


@functools.lru_cache(maxsize=None)
def manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        return json.load(f)


@functools.lru_cache(maxsize=None)
def codec_arrays():
    return dict(np.load(os.path.join(GOLDEN, "codec_cases.npz")))


@functools.lru_cache(maxsize=None)
def traj_arrays():
    return dict(np.load(os.path.join(GOLDEN, "traj_small.npz")))


@functools.lru_cache(maxsize=None)
def traj_nm_arrays():
    return dict(np.load(os.path.join(GOLDEN, "traj_nm.npz")))


def oracle_codec(spec):
    """Map a reference spec dict to an oracle Codec."""
    from oracle import cc_oracle as O

    kind = spec["kind"]
    if kind == "sign1bit":
        return O.Codec(O.SIGN1)
    if kind == "quant2bit":
        return O.Codec(O.QUANT2)
    if kind == "topk":
        return O.Codec(O.TOPK, keep_fraction=spec["keep_fraction"])
    if kind == "lowrank":
        return O.Codec(O.LOWRANK4 if spec["int4_factors"] else O.LOWRANK, rank=spec["rank"],
                       iters=spec["iterations"])
    if kind == "nm_block":
        return O.Codec(O.NMBLOCK, nm=(spec["n"], spec["m"]))
    if kind == "identity":
        return O.Codec(O.RAW)
    raise ValueError(kind)
