"""Step-wise residual protocol with error feedback, on device.

Mirror of /root/reference/pkg/src/compactcomm/pipeline.py (cited pl:<line>):
PipelineMode, LayerState, StepRecord, encode_step, decode_step and the message
envelope (pack_message / unpack_message / message_for).  The difference is where
state lives: LayerState holds CUDA tensors (base f32, feedback f32, ref f32) that
the sm_100a kernels update IN PLACE, instead of rebinding fresh frozen numpy
arrays (pl:96-112).  All validation (shape, step counter, warmup flag) happens on
the host before any launch, so a rejected message leaves the state untouched
(pl:146-151).

StepRecord floats are computed on device and read lazily, so encode_step never
synchronizes the stream unless the caller looks at compression_error/delta_hat.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass
from enum import Enum

import torch

from . import _lib
from . import compressors as cx
from .linalg import ShapeError

_ENVELOPE = struct.Struct("<IB")  # pl:33


class ProtocolError(RuntimeError):
    pass


class PipelineMode(str, Enum):
    NAIVE = "naive"
    RESIDUAL_NO_FEEDBACK = "residual_no_feedback"
    RESIDUAL_WITH_FEEDBACK = "residual_with_feedback"


_MODE_CODE = {PipelineMode.NAIVE: _lib.CC_NAIVE, PipelineMode.RESIDUAL_NO_FEEDBACK: _lib.CC_NO_FEEDBACK,
              PipelineMode.RESIDUAL_WITH_FEEDBACK: _lib.CC_WITH_FEEDBACK}


class StepRecord:
    """pl:46-52.  compression_error / delta_hat resolve from a 2-double device
    record {||d - t||^2, ||t||^2} on first access."""

    __slots__ = ("step", "bits", "total_error", "_dev", "_host")

    def __init__(self, step, bits, dev_record, total_error=float("nan")):
        self.step = step
        self.bits = bits
        self.total_error = total_error
        self._dev = dev_record
        self._host = None

    def _resolve(self):
        if self._host is None:
            self._host = [float(v) for v in self._dev.cpu().tolist()]
        return self._host

    @property
    def compression_error(self):
        return self._resolve()[0]

    @property
    def target_sqnorm(self):
        """||target||^2 (f64).  Not a reference field; 0.0 on warmup / identity steps,
        whose record is {0, 0} (cc_warmup_step) since delta_hat is 1 there anyway."""
        return self._resolve()[1]

    @property
    def delta_hat(self):
        err, tot = self._resolve()
        if tot == 0.0 or err == 0.0:  # pl:76-81 (err == 0 -> 1.0 whatever tot is)
            return 1.0 if err == 0.0 else -math.inf
        return 1.0 - err / tot

    def __repr__(self):
        return f"StepRecord(step={self.step}, bits={self.bits})"


class LayerState:
    """Per-(layer, peer) state (pl:55-73), device resident, single owner.

    `base` is copied at construction (the caller's tensor is never mutated).
    `feedback` is kept for RESIDUAL_WITH_FEEDBACK (zeros otherwise); `ref` (the
    previous input) is only materialized for RESIDUAL_NO_FEEDBACK, the one mode
    that reads it.
    """

    def __init__(self, mode, warmup_steps, base, feedback=None, ref=None, step=0):
        self.mode = PipelineMode(mode)
        if warmup_steps < 1:
            raise ValueError("warmup_steps must be >= 1")
        self.warmup_steps = int(warmup_steps)
        self.base = cx.as_device_matrix(base, torch.float32).clone()
        self.feedback = (torch.zeros_like(self.base) if feedback is None
                         else cx.as_device_matrix(feedback, torch.float32).clone())
        self.ref = None
        if self.mode == PipelineMode.RESIDUAL_NO_FEEDBACK:
            self.ref = self.base.clone() if ref is None else cx.as_device_matrix(ref, torch.float32).clone()
        self.step = int(step)
        self._rec = None

    @property
    def shape(self):
        return tuple(self.base.shape)

    def _aux(self):
        if self.mode == PipelineMode.RESIDUAL_WITH_FEEDBACK:
            return self.feedback
        if self.mode == PipelineMode.RESIDUAL_NO_FEEDBACK:
            return self.ref
        return None


def _body_slice(body_out, nbytes):
    """The caller's body buffer cut to this step's body, or a fresh one.  A buffer
    shorter than the body is refused before any launch (the kernels write
    `nbytes` unconditionally)."""
    if body_out is None:
        return cx._empty_body(nbytes)
    if body_out.numel() < nbytes:
        raise ValueError(f"body buffer holds {body_out.numel()} bytes, this step's body needs {nbytes}")
    return body_out[:nbytes]


def _record_buffer():
    # every encode path writes both doubles, so no fill kernel is needed
    return torch.empty(2, dtype=torch.float64, device=cx._device())


def encode_step(state, a_star, codec, rng=None, body_out=None):
    """Advance the sender one step (pl:84-121); returns (payload, StepRecord).

    a_star: [rows, cols] CUDA tensor (bf16 or f32) or host array.  body_out:
    optional preallocated uint8 CUDA buffer (>= body size) the payload body is
    written into (used by the collective layer to write straight into the
    all-gather send buffer).
    """
    x = cx.as_device_matrix(a_star)
    if tuple(x.shape) != state.shape:
        raise ShapeError(f"input shape {tuple(x.shape)} != state shape {state.shape}")
    lib = _lib.load()
    rows, cols = state.shape
    t = state.step + 1
    mode = _MODE_CODE[state.mode]
    aux = state._aux()
    rec = _record_buffer()
    stream = _lib.stream_ptr()
    kind = cx.CompressorKind(codec.kind)

    if t <= state.warmup_steps or kind == cx.CompressorKind.IDENTITY:
        # warmup / identity: raw tensor, base <- a*, fb <- 0 (pl:89-97)
        wire = torch.bfloat16 if x.dtype == torch.bfloat16 else torch.float32
        nbytes = rows * cols * (2 if wire == torch.bfloat16 else 4)
        body = _body_slice(body_out, nbytes)
        _lib.check(lib.cc_warmup_step(mode, rows, cols, _lib.ptr(x), cx.dtype_code(x), _lib.ptr(state.base),
                                      _lib.ptr(aux), _lib.ptr(body), cx.dtype_code(x), _lib.ptr(rec), stream),
                   "warmup")
        payload = cx.RawPayload(rows, cols, body, wire_dtype=wire)
    else:
        tag = cx._spec_tag(codec)
        if kind == cx.CompressorKind.TOPK:
            k = cx.topk_count(rows, cols, codec.keep_fraction)
            nbytes = 6 * k
            body = _body_slice(body_out, nbytes)
            ws = cx.workspace(_lib.check(lib.cc_workspace_bytes(_lib.CC_TOPK, rows, cols, k)), "topk")
            _lib.check(lib.cc_topk_encode_step(mode, rows, cols, k, _lib.ptr(x), cx.dtype_code(x),
                                               _lib.ptr(state.base), _lib.ptr(aux), _lib.ptr(body), _lib.ptr(ws),
                                               ws.numel(), _lib.ptr(rec), stream), "topk encode_step")
            payload = cx.TopKPayload(rows, cols, body, k)
        elif kind == cx.CompressorKind.NM_BLOCK:
            n, m = codec.n, codec.m
            nbytes = cx.nm_body_bytes(rows, cols, n, m)
            body = _body_slice(body_out, nbytes)
            ws = cx.workspace(_lib.check(lib.cc_workspace_bytes(_lib.CC_NMBLOCK, rows, cols, _lib.nm_param(n, m))),
                              "nm")
            _lib.check(lib.cc_nm_encode_step(mode, rows, cols, n, m, _lib.ptr(x), cx.dtype_code(x),
                                             _lib.ptr(state.base), _lib.ptr(aux), _lib.ptr(body), _lib.ptr(ws),
                                             ws.numel(), _lib.ptr(rec), stream), "nm encode_step")
            payload = cx.NMBlockPayload(rows, cols, body, n, m)
        elif kind == cx.CompressorKind.LOWRANK:
            payload = _encode_step_lowrank(state, x, codec, rng, mode, aux, rec, body_out)
        elif tag is not None:
            nbytes = lib.cc_body_bytes(tag, rows, cols, 0)
            body = _body_slice(body_out, nbytes)
            ws = cx.workspace(_lib.check(lib.cc_workspace_bytes(tag, rows, cols, 0)))
            _lib.check(lib.cc_encode_step(tag, mode, cx._SCALE_MODES[codec.scale_mode], rows, cols, _lib.ptr(x),
                                          cx.dtype_code(x), _lib.ptr(state.base), _lib.ptr(aux), _lib.ptr(body),
                                          _lib.ptr(ws), ws.numel(), _lib.ptr(rec), stream), "encode_step")
            payload = cx._payload_for(tag, rows, cols, body)
        else:
            payload = _encode_step_generic(state, x, codec, rng, mode, aux, rec, body_out)
    state.step = t
    return payload, StepRecord(t, payload.nominal_bits, rec)


def _encode_step_lowrank(state, x, codec, rng, mode, aux, rec, body_out):
    """One fused low-rank encode_step (cc_lowrank_encode_step): target, Q0, subspace
    iteration (cx:394-426), body, and the state update with the decode fused in.  Q0
    comes from the caller's numpy Generator (host draw, cx:407) or, for a
    linalg.DeviceKey, is drawn on the device (no host work: graph-capturable)."""
    from .linalg import DeviceKey

    if rng is None:
        raise ValueError("lowrank encoding needs an rng")
    lib = _lib.load()
    rows, cols = state.shape
    r = codec.rank
    if not (1 <= r <= min(rows, cols)):
        raise ShapeError(f"rank {r} out of range for shape {(rows, cols)}")
    tag = _lib.CC_LOWRANK4 if codec.int4_factors else _lib.CC_LOWRANK
    body = _body_slice(body_out, lib.cc_body_bytes(tag, rows, cols, r))
    ws = cx.workspace(_lib.check(lib.cc_lowrank_step_workspace_bytes(rows, cols, r)), "lowrank_step")
    if isinstance(rng, DeviceKey):  # drawn on the device, one step ahead (DeviceKey.start_block)
        q0, key, nwords, step_word = rng.start_block(cols, r), None, 0, -1
    else:
        q0 = cx.subspace_init(rng, cols, r)
        q0 = cx._stage_h2d(q0, x.device)
        key, nwords, step_word = None, 0, -1
    _lib.check(lib.cc_lowrank_encode_step(mode, rows, cols, r, codec.iterations, int(codec.int4_factors),
                                          _lib.ptr(x), cx.dtype_code(x), _lib.ptr(state.base), _lib.ptr(aux),
                                          _lib.ptr(q0), _lib.ptr(key), nwords, step_word, _lib.ptr(body),
                                          _lib.ptr(ws), ws.numel(), _lib.ptr(rec), _lib.stream_ptr()),
               "lowrank encode_step")
    if isinstance(rng, DeviceKey):
        rng.join()
    return cx.LowRankPayload(rows, cols, body, r, codec.int4_factors)


def _encode_step_generic(state, x, codec, rng, mode, aux, rec, body_out):
    """Codecs that need the materialized target (top-k, low-rank)."""
    lib = _lib.load()
    rows, cols = state.shape
    stream = _lib.stream_ptr()
    tbuf = torch.empty((rows, cols), dtype=torch.float32, device=x.device)
    dec = torch.empty_like(tbuf)
    _lib.check(lib.cc_residual_target(mode, rows, cols, _lib.ptr(x), cx.dtype_code(x), _lib.ptr(state.base),
                                      _lib.ptr(aux), _lib.ptr(tbuf), stream), "residual_target")
    kind = cx.CompressorKind(codec.kind)
    if kind == cx.CompressorKind.TOPK:
        payload = cx.encode_topk(tbuf, codec.keep_fraction, decoded=dec)
    elif kind == cx.CompressorKind.LOWRANK:
        if rng is None:
            raise ValueError("lowrank encoding needs an rng")
        payload = cx.encode_lowrank(tbuf, codec, rng, decoded=dec)
    else:
        raise NotImplementedError(f"codec {kind} not on the device path")
    if body_out is not None:
        _body_slice(body_out, payload.body.numel())
        body_out[: payload.body.numel()].copy_(payload.body)
        payload.body = body_out[: payload.body.numel()]
    ws = cx.workspace(1 << 16, "apply")
    _lib.check(lib.cc_apply_decoded(mode, rows, cols, _lib.ptr(x), cx.dtype_code(x), _lib.ptr(tbuf), _lib.ptr(dec),
                                    _lib.ptr(state.base), _lib.ptr(aux), _lib.ptr(rec), _lib.ptr(ws), ws.numel(),
                                    stream), "apply_decoded")
    return payload


# ---------------------------------------------------------------------------
# envelope (pl:124-143) — host framing
# ---------------------------------------------------------------------------

def pack_message(step, payload):
    return _ENVELOPE.pack(step, 0) + cx.to_bytes(payload)


def pack_warmup_message(step, payload):
    return _ENVELOPE.pack(step, 1) + cx.to_bytes(payload)


def unpack_message(buf):
    if len(buf) < _ENVELOPE.size:
        raise cx.PayloadError("message shorter than envelope")
    step, warm = _ENVELOPE.unpack_from(buf, 0)
    return step, bool(warm), cx.from_bytes(bytes(buf[_ENVELOPE.size:]))


def message_for(state_step, warmup_steps, payload):
    if state_step <= warmup_steps:
        return pack_warmup_message(state_step, payload)
    return pack_message(state_step, payload)


@dataclass
class DeviceMessage:
    """Envelope whose payload body stays in HBM (what the collectives carry)."""

    step: int
    warmup: bool
    payload: object


def device_message(state_step, warmup_steps, payload):
    return DeviceMessage(state_step, state_step <= warmup_steps, payload)


def decode_step(state, message):
    """Advance the receiver one step (pl:146-165); returns state.base.

    `message` is either the reference byte envelope or a DeviceMessage.
    """
    if isinstance(message, DeviceMessage):
        step, is_warmup, payload = message.step, message.warmup, message.payload
    else:
        step, is_warmup, payload = unpack_message(message)
    if step != state.step + 1:
        raise ProtocolError(f"step desynchronization: got {step}, expected {state.step + 1}")
    if (step <= state.warmup_steps) != is_warmup:
        raise ProtocolError(f"warmup flag mismatch at step {step}")
    if (payload.rows, payload.cols) != state.shape:
        raise ProtocolError(f"payload shape {(payload.rows, payload.cols)} != state shape {state.shape}")
    replace = is_warmup or payload.tag == cx.TAG_RAW or state.mode == PipelineMode.NAIVE
    acc = 0 if replace else 1
    if payload.tag == cx.TAG_TOPK and acc:
        acc = 2  # dense `base + decoded` semantics for the sparse codec (-0.0 -> +0.0)
    lib = _lib.load()
    _lib.check(lib.cc_decode_step(payload.tag, acc, payload.rows, payload.cols, payload._param(),
                                  _lib.ptr(payload.body), payload._body_dtype(), _lib.ptr(state.base),
                                  _lib.stream_ptr()), "decode_step")
    state.step = step
    return state.base
