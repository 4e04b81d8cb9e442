"""CPU-side checks of the C ABI: the in-tree library loads (no GPU needed to
dlopen it), exports every symbol include/compactcomm.h declares, and its pure
host functions (sizes, top-k count) agree with the oracle / reference formulas."""

import ctypes
import re

import pytest

from oracle import cc_oracle as O
from paper_2507_17511_b200 import _lib


def test_library_loads_and_exports_every_header_symbol():
    lib = _lib.load()
    syms = _lib.header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), f"missing export {s}"
    assert set(syms) <= set(_lib.SIGNATURES), "binding table out of date"
    dbg = _lib.header_symbols(_lib.DEBUG_HEADER)
    assert dbg and not set(dbg) & set(syms), "debug knobs belong to the private header only"
    assert set(syms) | set(dbg) == set(_lib.SIGNATURES)
    for s in dbg:
        assert hasattr(lib, s), f"missing export {s}"


def test_header_constants_match_binding():
    txt = open(_lib.HEADER).read()
    consts = dict(re.findall(r"#define (CC_\w+) \(?(-?\d+)\)?", txt))
    for name, val in consts.items():
        if hasattr(_lib, name):
            assert getattr(_lib, name) == int(val), name


@pytest.mark.parametrize("shape", [(1, 1), (3, 5), (4096, 3072), (512, 384), (7, 1000), (1024, 3072)])
def test_body_bytes_match_reference_bit_size(shape):
    lib = _lib.load()
    n, c = shape
    for tag in (O.RAW, O.SIGN1, O.QUANT2):
        assert lib.cc_body_bytes(tag, n, c, 0) == O.body_bytes(tag, n, c)
    for r in (1, 4, 16, 32):
        if r <= min(n, c):
            assert lib.cc_body_bytes(O.LOWRANK, n, c, r) == O.body_bytes(O.LOWRANK, n, c, rank=r)
            assert lib.cc_body_bytes(O.LOWRANK4, n, c, r) == O.body_bytes(O.LOWRANK4, n, c, rank=r)
    for f in (0.01, 0.02, 0.05, 0.1, 0.3, 1.0):
        k = lib.cc_topk_count(n, c, f)
        assert k == O.topk_count(n, c, f)
        assert lib.cc_body_bytes(O.TOPK, n, c, k) == O.body_bytes(O.TOPK, n, c, k=k)


def test_bad_arguments_rejected_without_gpu():
    lib = _lib.load()
    assert lib.cc_body_bytes(O.QUANT2, 0, 5, 0) == _lib.CC_ERR_SHAPE
    assert lib.cc_body_bytes(99, 3, 5, 0) == _lib.CC_ERR_ARG
    assert lib.cc_topk_count(3, 5, 0.0) == _lib.CC_ERR_ARG
    assert lib.cc_topk_count(3, 5, 1.5) == _lib.CC_ERR_ARG
    assert lib.cc_lowrank_workspace_bytes(4, 4, 5) == _lib.CC_ERR_SHAPE
    # encode with an empty shape fails before touching the device
    st = lib.cc_encode_step(O.QUANT2, 2, 0, 0, 8, None, 0, None, None, None, None, 0, None, None)
    assert st == _lib.CC_ERR_SHAPE
    assert b"empty" in lib.cc_last_error()
    st = lib.cc_encode_step(O.QUANT2, 7, 0, 4, 8, ctypes.c_void_p(16), 0, ctypes.c_void_p(16), ctypes.c_void_p(16),
                            ctypes.c_void_p(16), None, 0, ctypes.c_void_p(16), None)
    assert st == _lib.CC_ERR_ARG


def test_status_codes_map_to_reference_exceptions():
    from paper_2507_17511_b200 import compressors as cx
    from paper_2507_17511_b200 import linalg
    from paper_2507_17511_b200 import pipeline as pl

    with pytest.raises(linalg.ShapeError):
        _lib.check(_lib.CC_ERR_SHAPE)
    with pytest.raises(cx.PayloadError):
        _lib.check(_lib.CC_ERR_PAYLOAD)
    with pytest.raises(pl.ProtocolError):
        _lib.check(_lib.CC_ERR_PROTOCOL)
    with pytest.raises(ValueError):
        _lib.check(_lib.CC_ERR_ARG)
