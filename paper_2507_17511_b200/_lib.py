"""ctypes binding of the sm_100a C ABI (include/compactcomm.h).

There is no CPU fallback: if the in-tree library is missing, importing any
compute entry point raises.  Status codes map to the reference package's
exception classes (compressors.PayloadError, linalg.ShapeError,
pipeline.ProtocolError, ValueError).
"""

from __future__ import annotations

import ctypes
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libcompactcomm_b200.so")
# experiments only: load an alternative build (A/B of kernel variants in one process)
LIB_PATH = os.environ.get("CC_LIB_OVERRIDE", LIB_PATH)
HEADER = os.path.join(os.path.dirname(HERE), "include", "compactcomm.h")

# constants mirrored from include/compactcomm.h (checked by tests/test_abi.py)
CC_OK, CC_ERR_ARG, CC_ERR_SHAPE, CC_ERR_PAYLOAD, CC_ERR_PROTOCOL, CC_ERR_CUDA, CC_ERR_UNSUPPORTED = 0, -1, -2, -3, -4, -5, -6
CC_ERR_NCCL = -7
CC_RAW, CC_SIGN1, CC_QUANT2, CC_LOWRANK, CC_LOWRANK4, CC_NMBLOCK, CC_TOPK, CC_QUANT4 = 0, 1, 2, 3, 4, 5, 6, 16
CC_NAIVE, CC_NO_FEEDBACK, CC_WITH_FEEDBACK = 0, 1, 2
CC_F32, CC_BF16 = 0, 1
CC_SCALE_RANK1, CC_SCALE_PER_TOKEN, CC_SCALE_PER_CHANNEL = 0, 1, 2


class CodecSpec(ctypes.Structure):
    """cc_codec_spec of include/compactcomm.h."""

    _fields_ = [("codec", ctypes.c_int), ("scale_mode", ctypes.c_int), ("keep_fraction", ctypes.c_double),
                ("nm_n", ctypes.c_int), ("nm_m", ctypes.c_int)]


def nm_param(n, m):
    """CC_NM_PARAM(n, m) of include/compactcomm.h."""
    return (int(n) << 16) | int(m)

_i64, _i32, _p, _d = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_double

SIGNATURES = {
    "cc_body_bytes": (_i64, [_i32, _i64, _i64, _i64]),
    "cc_workspace_bytes": (_i64, [_i32, _i64, _i64, _i64]),
    "cc_encode_step": (_i32, [_i32, _i32, _i32, _i64, _i64, _p, _i32, _p, _p, _p, _p, _i64, _p, _p]),
    "cc_encode_step_segmented": (_i32, [_i32, _i32, _i32, _i64, _i64, _i32, _p, _i32, _p, _p, _p, _i64, _p, _i64,
                                        _p, _p]),
    "cc_warmup_step": (_i32, [_i32, _i64, _i64, _p, _i32, _p, _p, _p, _i32, _p, _p]),
    "cc_decode_step": (_i32, [_i32, _i32, _i64, _i64, _i64, _p, _i32, _p, _p]),
    "cc_decode_batched": (_i32, [_i32, _i32, _i32, ctypes.POINTER(_i64), _i64, _i64, ctypes.POINTER(_p), _i32,
                                 ctypes.POINTER(_p), _p]),
    "cc_residual_target": (_i32, [_i32, _i64, _i64, _p, _i32, _p, _p, _p, _p]),
    "cc_apply_decoded": (_i32, [_i32, _i64, _i64, _p, _i32, _p, _p, _p, _p, _p, _p, _i64, _p]),
    "cc_encode": (_i32, [_i32, _i32, _i64, _i64, _i64, _p, _p, _p, _p, _i64, _p]),
    "cc_topk_count": (_i64, [_i64, _i64, _d]),
    "cc_topk_encode": (_i32, [_i64, _i64, _i64, _p, _p, _p, _p, _i64, _p]),
    "cc_topk_encode_step": (_i32, [_i32, _i64, _i64, _i64, _p, _i32, _p, _p, _p, _p, _i64, _p, _p]),
    "cc_nm_encode": (_i32, [_i64, _i64, _i32, _i32, _p, _p, _p, _p, _i64, _p]),
    "cc_nm_encode_step": (_i32, [_i32, _i64, _i64, _i32, _i32, _p, _i32, _p, _p, _p, _p, _i64, _p, _p]),
    "cc_lowrank_encode": (_i32, [_i32, _i64, _i64, _i64, _i32, _p, _p, _p, _p, _p, _i64, _p]),
    "cc_lowrank_workspace_bytes": (_i64, [_i64, _i64, _i64]),
    "cc_gaussian_workspace_bytes": (_i64, [_i64, _i64]),
    "cc_lowrank_step_workspace_bytes": (_i64, [_i64, _i64, _i64]),
    "cc_lowrank_encode_step": (_i32, [_i32, _i64, _i64, _i64, _i32, _i32, _p, _i32, _p, _p, _p, _p, _i32, _i32, _p,
                                      _p, _i64, _p, _p]),
    "cc_gaussian_keyed": (_i32, [_i64, _i64, _p, _i32, _i32, _p, _p, _i64, _p]),
    "cc_comm_get_unique_id": (_i32, [_p]),
    "cc_comm_init_rank": (_i32, [_p, _i32, _i32, ctypes.POINTER(_p)]),
    "cc_comm_wrap": (_i32, [_p, ctypes.POINTER(_p)]),
    "cc_comm_rank": (_i32, [_p]),
    "cc_comm_size": (_i32, [_p]),
    "cc_comm_destroy": (_i32, [_p]),
    "cc_allgather_create": (_i32, [_p, _p, _i32, _i64, _i64, _i32, _i32, ctypes.POINTER(_p)]),
    "cc_allgather_step": (_i32, [_p, _p, _p]),
    "cc_allgather_reconstruction": (_p, [_p]),
    "cc_allgather_sender_base": (_p, [_p]),
    "cc_allgather_sender_aux": (_p, [_p]),
    "cc_allgather_body": (_p, [_p, ctypes.POINTER(_i64)]),
    "cc_allgather_record": (_p, [_p]),
    "cc_allgather_shard": (_i32, [_p, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "cc_allgather_destroy": (_i32, [_p]),
    "cc_alltoall_create": (_i32, [_p, _p, _i32, _i64, _i64, _i32, _i32, ctypes.POINTER(_p)]),
    "cc_alltoall_step": (_i32, [_p, _p, _p]),
    "cc_alltoall_output": (_p, [_p]),
    "cc_alltoall_sender_base": (_p, [_p]),
    "cc_alltoall_destroy": (_i32, [_p]),
    "cc_last_error": (ctypes.c_char_p, []),
    "cc_version": (_i32, []),
    "cc_launch_count": (_i64, []),
    "cc_set_quant_path": (None, [_i32]),
    "cc_debug_fused_stop": (None, [_i32]),
    "cc_debug_fused_timer": (None, [_p]),
    "cc_debug_fused_policy": (None, [_i32]),
    "cc_debug_fused_rings": (None, [_i32, _i32]),
    "cc_debug_fused_tail": (None, [_i32, _i32]),
    "cc_debug_lowrank_tma": (None, [_i32, _i32]),
    "cc_set_pdl": (None, [_i32]),
    "cc_debug_fused_phase_a": (None, [_i32, _i32]),
    "cc_set_lowrank_backend": (None, [_i32]),
    "cc_debug_k1_resident": (None, [_i32]),
    "cc_debug_k1_resident_count": (_i64, []),
    "cc_debug_k1_resident_nq": (None, [_i32]),
    "cc_debug_topk_resident": (None, [_i32]),
    "cc_debug_topk_resident_count": (_i64, []),
    "cc_debug_topk_timer": (None, [_p]),
    "cc_debug_orth_stamps": (None, [_p]),
    "cc_debug_orth_cluster": (None, [_i32]),
    "cc_debug_gauss_stamps": (None, [_p]),
    "cc_debug_lowrank_fused": (None, [_i32]),
    "cc_debug_lowrank_fused_count": (_i64, []),
    "cc_debug_lowrank_fused_stamps": (None, [_p]),
}
# private test / profiling knobs (csrc/cc_debug.h), not part of the public ABI
DEBUG_HEADER = os.path.join(HERE, "csrc", "cc_debug.h")

_LIB = None


def header_symbols(path=None):
    """Every CC_API function declared in include/compactcomm.h (or `path`)."""
    with open(path or HEADER) as f:
        txt = f.read()
    return sorted(set(re.findall(r"CC_API\s+[\w\s\*]+?\b(cc_\w+)\s*\(", txt)))


def load():
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


class CudaError(RuntimeError):
    pass


def check(status, what=""):
    if status >= 0:
        return status
    msg = (load().cc_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    from . import compressors, linalg, pipeline

    if status == CC_ERR_SHAPE:
        raise linalg.ShapeError(text)
    if status == CC_ERR_PAYLOAD:
        raise compressors.PayloadError(text)
    if status == CC_ERR_PROTOCOL:
        raise pipeline.ProtocolError(text)
    if status == CC_ERR_ARG:
        raise ValueError(text)
    if status == CC_ERR_UNSUPPORTED:
        raise NotImplementedError(text)
    if status == CC_ERR_NCCL:
        from . import comm

        raise comm.TransportError(text)
    raise CudaError(text)


def stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)
