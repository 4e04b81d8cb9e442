"""Device codec family: the reference `compactcomm.compressors` API over CUDA tensors.

Same names, fields, tags, bit accounting and wire bytes as
/root/reference/pkg/src/compactcomm/compressors.py (cited as cx:<line>), but every
payload keeps its body in HBM (a torch.uint8 CUDA tensor holding exactly the
reference's codec body) and every encode/decode runs in the sm_100a kernels of
libcompactcomm_b200.so.  Host bytes only appear in to_bytes/from_bytes (frame
header parsing and validation, cx:580-720), which is host-side framing.

Extensions beyond the reference (north_star; parity unpinned, no reference code):
  * CompressorKind.QUANT4BIT: 4-bit element quantizer, 16 levels (k-7.5)/2 of u v^T
  * CompressorSpec.scale_mode: "rank1" (reference) | "per_token" | "per_channel"
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _lib
from .linalg import ShapeError

U_FLOOR = 1e-30  # cx:52
QUANT2_LEVELS = np.array([-2.0, -0.5, 0.5, 2.0], dtype=np.float64)  # cx:54

TAG_RAW = 0
TAG_SIGN1BIT = 1
TAG_QUANT2BIT = 2
TAG_LOWRANK = 3
TAG_LOWRANK_INT4 = 4
TAG_NMBLOCK = 5
TAG_TOPK = 6
TAG_QUANT4BIT = 16  # extension

_HEADER = struct.Struct("<BII")  # cx:64
_SCALE_MODES = {"rank1": _lib.CC_SCALE_RANK1, "per_token": _lib.CC_SCALE_PER_TOKEN,
                "per_channel": _lib.CC_SCALE_PER_CHANNEL}


class PayloadError(ValueError):
    """Malformed serialized payload; names the codec (cx:67)."""


class CompressorKind(str, Enum):
    IDENTITY = "identity"
    SIGN1BIT = "sign1bit"
    QUANT2BIT = "quant2bit"
    LOWRANK = "lowrank"
    NM_BLOCK = "nm_block"
    TOPK = "topk"
    QUANT4BIT = "quant4bit"  # extension


@dataclass(frozen=True)
class CompressorSpec:
    """cx:80-123, plus `scale_mode` for the 1/2/4-bit quantizers (extension)."""

    kind: CompressorKind
    rank: int = 0
    iterations: int = 1
    int4_factors: bool = False
    n: int = 0
    m: int = 0
    keep_fraction: float = 0.0
    scale_mode: str = "rank1"

    def __post_init__(self):
        k = CompressorKind(self.kind)
        if k == CompressorKind.LOWRANK:
            if self.rank < 1 or self.iterations < 1:
                raise ValueError("lowrank needs rank >= 1 and iterations >= 1")
        elif k == CompressorKind.NM_BLOCK:
            if not (1 <= self.n <= self.m):
                raise ValueError("nm_block needs 1 <= n <= m")
        elif k == CompressorKind.TOPK:
            if not (0.0 < self.keep_fraction <= 1.0):
                raise ValueError("topk needs keep_fraction in (0, 1]")
        if self.scale_mode not in _SCALE_MODES:
            raise ValueError(f"scale_mode must be one of {sorted(_SCALE_MODES)}")

    def label(self):
        k = self.kind
        if k == CompressorKind.LOWRANK:
            return f"lowrank-r{self.rank}-{'int4' if self.int4_factors else 'f16'}"
        if k == CompressorKind.NM_BLOCK:
            return f"nm{self.n}:{self.m}"
        if k == CompressorKind.TOPK:
            return f"topk{self.keep_fraction:g}"
        if self.scale_mode != "rank1":
            return f"{k.value}-{self.scale_mode}"
        return k.value

    @staticmethod
    def from_dict(d):
        return CompressorSpec(
            kind=CompressorKind(d["kind"]),
            rank=int(d.get("rank", 0)),
            iterations=int(d.get("iterations", 1)),
            int4_factors=bool(d.get("int4_factors", False)),
            n=int(d.get("n", 0)),
            m=int(d.get("m", 0)),
            keep_fraction=float(d.get("keep_fraction", 0.0)),
            scale_mode=str(d.get("scale_mode", "rank1")),
        )


@dataclass(frozen=True)
class ScalePair:
    u: torch.Tensor  # f32 [rows], strictly positive (rank1)
    v: torch.Tensor  # f32 [cols], nonnegative

    def outer(self):
        return torch.outer(self.u.double(), self.v.double())  # cx:131-132


# ---------------------------------------------------------------------------
# device tensors in / out
# ---------------------------------------------------------------------------

def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2507_17511_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def as_device_matrix(x, dtype=None):
    """Accept a CUDA tensor (f32/bf16) or host array; return a contiguous 2-D CUDA tensor."""
    if isinstance(x, torch.Tensor):
        t = x
        if not t.is_cuda:
            t = t.to(_device())
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float32))).to(_device())
    if t.dim() != 2 or t.shape[0] < 1 or t.shape[1] < 1:
        raise ShapeError(f"expected a non-empty 2-D matrix, got shape {tuple(t.shape)}")
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    if t.dtype not in (torch.float32, torch.bfloat16):
        t = t.float()
    return t.contiguous()


def dtype_code(t):
    return _lib.CC_BF16 if t.dtype == torch.bfloat16 else _lib.CC_F32


def _empty_body(nbytes):
    # +16 slack keeps vector stores of the last code word in bounds
    return torch.empty(int(nbytes), dtype=torch.uint8, device=_device())


_WS_CACHE: dict = {}


def workspace(nbytes, key="default"):
    """Per-device, per-stream scratch reused across calls (stream-ordered)."""
    dev = torch.cuda.current_device()
    sid = torch.cuda.current_stream().cuda_stream
    k = (dev, sid, key)
    buf = _WS_CACHE.get(k)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 1 << 16), dtype=torch.uint8, device=_device())
        _WS_CACHE[k] = buf
    return buf


_PIN_RING: dict = {}
_PIN_SLOTS = 8


def _stage_h2d(arr, device):
    """Asynchronous H2D copy of a small host array through a per-(device, stream, size)
    ring of pinned slots; a slot is rewritten only after its previous copy completed
    (its event), so a fresh pinned allocation per call (which can stall the host on
    cudaHostAlloc) is never needed."""
    arr = np.ascontiguousarray(arr)
    src = torch.from_numpy(arr)
    if torch.cuda.is_current_stream_capturing():  # no host event waits inside a capture
        return src.pin_memory().to(device, non_blocking=True)
    stream = torch.cuda.current_stream(device)
    k = (device.index, stream.cuda_stream, src.dtype, src.numel())
    ring = _PIN_RING.get(k)
    if ring is None:
        ring = _PIN_RING[k] = {"i": 0, "slots": [(torch.empty(src.numel(), dtype=src.dtype).pin_memory(),
                                                  torch.cuda.Event()) for _ in range(_PIN_SLOTS)]}
    buf, ev = ring["slots"][ring["i"]]
    ring["i"] = (ring["i"] + 1) % _PIN_SLOTS
    ev.synchronize()
    buf.copy_(src.reshape(-1))
    out = torch.empty(src.shape, dtype=src.dtype, device=device)
    out.copy_(buf.view(src.shape), non_blocking=True)
    ev.record(stream)
    return out


# ---------------------------------------------------------------------------
# payloads (cx:157-361): bodies live on the device
# ---------------------------------------------------------------------------

class _Payload:
    tag = -1
    kind_label = ""

    def __init__(self, rows, cols, body):
        self.rows = int(rows)
        self.cols = int(cols)
        self.body = body  # torch.uint8 CUDA tensor: the codec body bytes

    @property
    def payload_only_bits(self):
        raise NotImplementedError

    @property
    def nominal_bits(self):
        return self.bit_size

    def _param(self):
        return 0

    def body_bytes(self):
        """Reference wire body (host bytes)."""
        return self.body.cpu().numpy().tobytes()

    def decode(self, out=None):
        """Deterministic reconstruction into a fresh (or given) f32 CUDA tensor."""
        if out is None:
            out = torch.empty((self.rows, self.cols), dtype=torch.float32, device=self.body.device)
        _lib.check(_lib.load().cc_decode_step(self.tag if self.tag != TAG_QUANT4BIT else _lib.CC_QUANT4, 0,
                                              self.rows, self.cols, self._param(), _lib.ptr(self.body),
                                              self._body_dtype(), _lib.ptr(out), _lib.stream_ptr()),
                   f"decode {self.kind_label}")
        return out

    def _body_dtype(self):
        return _lib.CC_F32


class RawPayload(_Payload):
    """Raw f32 (cx:157-180).  `wire_dtype` bf16 keeps bf16 inputs bf16 on the
    wire (lossless); to_bytes always emits the reference's f32 body."""

    tag = TAG_RAW
    kind_label = "raw"

    def __init__(self, rows, cols, body, wire_dtype=torch.float32):
        super().__init__(rows, cols, body)
        self.wire_dtype = wire_dtype

    @property
    def bit_size(self):
        return 32 * self.rows * self.cols

    @property
    def nominal_bits(self):
        return 16 * self.rows * self.cols  # cx:170-173

    @property
    def payload_only_bits(self):
        return 16 * self.rows * self.cols

    def _body_dtype(self):
        return _lib.CC_BF16 if self.wire_dtype == torch.bfloat16 else _lib.CC_F32

    def body_bytes(self):
        if self.wire_dtype == torch.bfloat16:
            return self.body.view(torch.bfloat16).float().cpu().numpy().astype("<f4").tobytes()
        return self.body.cpu().numpy().tobytes()

    @property
    def data(self):
        return self.decode()


class _ScaledPayload(_Payload):
    bits_per_elem = 0

    @property
    def code_bytes(self):
        return -(-self.bits_per_elem * self.rows * self.cols // 8)

    @property
    def bit_size(self):
        return self.bits_per_elem * self.rows * self.cols + 32 * (self.rows + self.cols)

    @property
    def payload_only_bits(self):
        return self.bits_per_elem * self.rows * self.cols

    @property
    def u(self):
        o = self.code_bytes
        return self.body[o:o + 4 * self.rows].clone().view(torch.float32)

    @property
    def v(self):
        o = self.code_bytes + 4 * self.rows
        return self.body[o:o + 4 * self.cols].clone().view(torch.float32)

    @property
    def codes(self):
        return self.body[: self.code_bytes]


class SignPayload(_ScaledPayload):
    tag = TAG_SIGN1BIT
    kind_label = "sign1bit"
    bits_per_elem = 1

    @property
    def neg_bits(self):
        return self.codes


class Quant2Payload(_ScaledPayload):
    tag = TAG_QUANT2BIT
    kind_label = "quant2bit"
    bits_per_elem = 2


class Quant4Payload(_ScaledPayload):
    tag = TAG_QUANT4BIT
    kind_label = "quant4bit"
    bits_per_elem = 4


class TopKPayload(_Payload):
    tag = TAG_TOPK
    kind_label = "topk"

    def __init__(self, rows, cols, body, k):
        super().__init__(rows, cols, body)
        self.k = int(k)

    @property
    def kept(self):
        return self.k

    @property
    def bit_size(self):
        return 48 * self.k  # cx:347-348

    @property
    def payload_only_bits(self):
        return 16 * self.k

    def _param(self):
        return self.k

    @property
    def indices(self):
        return self.body[: 4 * self.k].clone().view(torch.int32)

    @property
    def values(self):
        return self.body[4 * self.k: 6 * self.k].clone().view(torch.float16)


class NMBlockPayload(_Payload):
    """N:M block payload (cx:291-329): body = packed keep-mask + f16 values."""

    tag = TAG_NMBLOCK
    kind_label = "nmblock"

    def __init__(self, rows, cols, body, n, m):
        super().__init__(rows, cols, body)
        self.n = int(n)
        self.m = int(m)

    @property
    def padded_cols(self):
        return -(-self.cols // self.m) * self.m

    @property
    def block_count(self):
        return self.rows * (self.padded_cols // self.m)

    @property
    def mask_bytes(self):
        return -(-self.block_count * self.m // 8)

    @property
    def bit_size(self):
        return self.block_count * (self.m + 16 * self.n)  # cx:318-319

    @property
    def payload_only_bits(self):
        return self.block_count * 16 * self.n

    def _param(self):
        return _lib.nm_param(self.n, self.m)

    @property
    def masks(self):
        return self.body[: self.mask_bytes]

    @property
    def values(self):
        return self.body[self.mask_bytes:].clone().view(torch.float16)


class LowRankPayload(_Payload):
    kind_label = "lowrank"

    def __init__(self, rows, cols, body, rank, int4):
        super().__init__(rows, cols, body)
        self.rank = int(rank)
        self.int4 = bool(int4)

    @property
    def tag(self):
        return TAG_LOWRANK_INT4 if self.int4 else TAG_LOWRANK

    @property
    def bit_size(self):
        per = 4 if self.int4 else 16
        return per * self.rank * (self.rows + self.cols) + (64 * self.rank if self.int4 else 0)  # cx:264-267

    @property
    def payload_only_bits(self):
        return (4 if self.int4 else 16) * self.rank * (self.rows + self.cols)

    def _param(self):
        return self.rank


# ---------------------------------------------------------------------------
# encoders (cx:369-476)
# ---------------------------------------------------------------------------

def _spec_tag(spec):
    k = CompressorKind(spec.kind)
    return {CompressorKind.SIGN1BIT: _lib.CC_SIGN1, CompressorKind.QUANT2BIT: _lib.CC_QUANT2,
            CompressorKind.QUANT4BIT: _lib.CC_QUANT4}.get(k)


def _payload_for(tag, rows, cols, body):
    cls = {_lib.CC_SIGN1: SignPayload, _lib.CC_QUANT2: Quant2Payload, _lib.CC_QUANT4: Quant4Payload}[tag]
    return cls(rows, cols, body)


def encode_raw(x):
    x = as_device_matrix(x)
    return RawPayload(x.shape[0], x.shape[1], x.contiguous().view(torch.uint8).reshape(-1).clone(),
                      wire_dtype=x.dtype)


def _encode_quant(x, tag, scale_mode="rank1", decoded=None):
    t = as_device_matrix(x, torch.float32)
    rows, cols = t.shape
    lib = _lib.load()
    body = _empty_body(lib.cc_body_bytes(tag, rows, cols, 0))
    dec = decoded if decoded is not None else torch.empty_like(t)
    wsb = _lib.check(lib.cc_workspace_bytes(tag, rows, cols, 0))
    ws = workspace(wsb)
    _lib.check(lib.cc_encode(tag, _SCALE_MODES[scale_mode], rows, cols, 0, _lib.ptr(t), _lib.ptr(body),
                             _lib.ptr(dec), _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "encode")
    return _payload_for(tag, rows, cols, body), dec


def encode_sign1bit(x, scale_mode="rank1"):
    return _encode_quant(x, _lib.CC_SIGN1, scale_mode)[0]


def encode_quant2bit(x, scale_mode="rank1"):
    return _encode_quant(x, _lib.CC_QUANT2, scale_mode)[0]


def encode_quant4bit(x, scale_mode="rank1"):
    return _encode_quant(x, _lib.CC_QUANT4, scale_mode)[0]


def scale_estimate(x):
    """u, v of the rank-1 magnitude model (cx:135-149), computed on device."""
    p = encode_sign1bit(x)
    return ScalePair(p.u, p.v)


def topk_count(rows, cols, keep_fraction):
    return _lib.check(_lib.load().cc_topk_count(rows, cols, float(keep_fraction)))


def encode_topk(x, keep_fraction, decoded=None):
    if not (0.0 < keep_fraction <= 1.0):
        raise ValueError("keep_fraction must be in (0, 1]")
    t = as_device_matrix(x, torch.float32)
    rows, cols = t.shape
    lib = _lib.load()
    k = topk_count(rows, cols, keep_fraction)
    body = _empty_body(max(6 * k, 1))
    ws = workspace(_lib.check(lib.cc_workspace_bytes(_lib.CC_TOPK, rows, cols, k)), "topk")
    _lib.check(lib.cc_topk_encode(rows, cols, k, _lib.ptr(t), _lib.ptr(body), _lib.ptr(decoded), _lib.ptr(ws),
                                  ws.numel(), _lib.stream_ptr()), "encode_topk")
    return TopKPayload(rows, cols, body[: 6 * k], k)


def nm_body_bytes(rows, cols, n, m):
    return _lib.check(_lib.load().cc_body_bytes(_lib.CC_NMBLOCK, rows, cols, _lib.nm_param(n, m)))


def encode_nm_block(x, n, m, decoded=None):
    """Keep the n largest-|value| entries of every 1 x m column block (cx:429-443)."""
    if not (1 <= n <= m):
        raise ValueError("need 1 <= n <= m")
    if m > 65535:
        raise ValueError("m must fit the u16 frame meta (cx:596)")
    t = as_device_matrix(x, torch.float32)
    rows, cols = t.shape
    lib = _lib.load()
    body = _empty_body(nm_body_bytes(rows, cols, n, m))
    ws = workspace(_lib.check(lib.cc_workspace_bytes(_lib.CC_NMBLOCK, rows, cols, _lib.nm_param(n, m))), "nm")
    _lib.check(lib.cc_nm_encode(rows, cols, n, m, _lib.ptr(t), _lib.ptr(body), _lib.ptr(decoded), _lib.ptr(ws),
                                ws.numel(), _lib.stream_ptr()), "encode_nm_block")
    return NMBlockPayload(rows, cols, body, n, m)


def subspace_init(rng, cols, rank):
    """Host draw of the initial block Q0 ~ N(0,1)[cols, r] (cx:407 / la:67-74)."""
    from .linalg import gaussian_matrix

    return gaussian_matrix(rng, cols, rank)


def encode_lowrank(a, spec, rng, decoded=None):
    if spec.kind != CompressorKind.LOWRANK:
        raise ValueError("spec.kind must be lowrank")
    t = as_device_matrix(a, torch.float32)
    rows, cols = t.shape
    r = spec.rank
    if not (1 <= r <= min(rows, cols)):
        raise ShapeError(f"rank {r} out of range for shape {(rows, cols)}")
    lib = _lib.load()
    from .linalg import DeviceKey

    if isinstance(rng, DeviceKey):
        # Q0 drawn on the device from the key's PCG64 stream, bit-identical to the host
        # draw (cc_gaussian_keyed); no host work, so the step can be graph-captured
        q0 = workspace(4 * cols * r, "lowrank_q0").view(torch.float32)[: cols * r]
        gws = workspace(_lib.check(lib.cc_gaussian_workspace_bytes(cols, r)), "gauss")
        _lib.check(lib.cc_gaussian_keyed(cols, r, _lib.ptr(rng.words), rng.nwords, rng.step_word, _lib.ptr(q0),
                                         _lib.ptr(gws), gws.numel(), _lib.stream_ptr()), "gaussian_keyed")
    else:
        # Q0 drawn on the host from the caller's numpy Generator (cx:407) and uploaded
        # through a reused pinned staging ring (asynchronous H2D, no per-step host alloc)
        q0 = subspace_init(rng, cols, r)
        q0 = _stage_h2d(q0, t.device) if t.is_cuda else torch.from_numpy(q0).to(t.device)
    tag = _lib.CC_LOWRANK4 if spec.int4_factors else _lib.CC_LOWRANK
    body = _empty_body(lib.cc_body_bytes(tag, rows, cols, r))
    ws = workspace(_lib.check(lib.cc_lowrank_workspace_bytes(rows, cols, r)), "lowrank")
    _lib.check(lib.cc_lowrank_encode(int(spec.int4_factors), rows, cols, r, spec.iterations, _lib.ptr(t),
                                     _lib.ptr(q0), _lib.ptr(body), _lib.ptr(decoded), _lib.ptr(ws), ws.numel(),
                                     _lib.stream_ptr()), "encode_lowrank")
    return LowRankPayload(rows, cols, body, r, spec.int4_factors)


def encode(x, spec, rng=None):
    """Encode with any CompressorSpec (cx:459-476); lowrank requires an rng."""
    k = CompressorKind(spec.kind)
    if k == CompressorKind.IDENTITY:
        return encode_raw(x)
    tag = _spec_tag(spec)
    if tag is not None:
        return _encode_quant(x, tag, spec.scale_mode)[0]
    if k == CompressorKind.LOWRANK:
        if rng is None:
            raise ValueError("lowrank encoding needs an rng")
        return encode_lowrank(x, spec, rng)
    if k == CompressorKind.TOPK:
        return encode_topk(x, spec.keep_fraction)
    if k == CompressorKind.NM_BLOCK:
        return encode_nm_block(x, spec.n, spec.m)
    raise ValueError(f"unknown codec kind {k}")


def decode(payload):
    return payload.decode()


def frob_norm_sq(t):
    d = t.double().reshape(-1)
    return float(torch.dot(d, d))


def empirical_delta(x, payload):
    """delta-hat = 1 - ||decode - X||^2 / ||X||^2 (cx:484-492)."""
    xm = as_device_matrix(x, torch.float32)
    err = frob_norm_sq(decode(payload).double() - xm.double())
    total = frob_norm_sq(xm)
    if total == 0.0:
        if err == 0.0:
            return 1.0
        raise ValueError("empirical delta undefined: zero input, nonzero error")
    return 1.0 - err / total


def baseline_bits(rows, cols):
    return 16 * rows * cols  # cx:500-502


def payload_only_ratio(p):
    return baseline_bits(p.rows, p.cols) / p.payload_only_bits


def overhead_ratio(p):
    return baseline_bits(p.rows, p.cols) / p.nominal_bits


def nominal_wire_bytes(p):
    return -(-p.nominal_bits // 8)  # cx:513-515


# ---------------------------------------------------------------------------
# wire format: host-side framing around the device body (cx:580-720)
# ---------------------------------------------------------------------------

def to_bytes(p):
    head = _HEADER.pack(p.tag, p.rows, p.cols)
    if p.tag in (TAG_LOWRANK, TAG_LOWRANK_INT4):
        head += struct.pack("<I", p.rank)
    elif p.tag == TAG_TOPK:
        head += struct.pack("<I", p.kept)
    elif p.tag == TAG_NMBLOCK:
        head += struct.pack("<HH", p.n, p.m)  # cx:596-597
    return head + p.body_bytes()


def _check_scales(body, off, rows, cols, codec, nonneg_u=False):
    u = np.frombuffer(body, "<f4", rows, off)
    v = np.frombuffer(body, "<f4", cols, off + 4 * rows)
    if not (np.all(np.isfinite(u)) and np.all(np.isfinite(v))):
        raise PayloadError(f"{codec}: non-finite scales")
    if (np.any(u < 0) if nonneg_u else np.any(u <= 0)) or np.any(v < 0):
        raise PayloadError(f"{codec}: invalid scale signs")


def from_bytes(buf):
    """Parse + validate a frame on the host, then stage its body in HBM."""
    buf = bytes(buf)
    if len(buf) < _HEADER.size:
        raise PayloadError("frame shorter than header")
    tag, rows, cols = _HEADER.unpack_from(buf, 0)
    body = buf[_HEADER.size:]

    def dev(b):
        return torch.frombuffer(bytearray(b), dtype=torch.uint8).to(_device()) if b else _empty_body(0)

    try:
        if tag == TAG_RAW:
            if len(body) != 4 * rows * cols:
                raise PayloadError("raw: body length mismatch")
            if not np.all(np.isfinite(np.frombuffer(body, "<f4"))):
                raise PayloadError("raw: non-finite entries")
            return RawPayload(rows, cols, dev(body))
        if tag in (TAG_SIGN1BIT, TAG_QUANT2BIT, TAG_QUANT4BIT):
            bits = {TAG_SIGN1BIT: 1, TAG_QUANT2BIT: 2, TAG_QUANT4BIT: 4}[tag]
            name = {TAG_SIGN1BIT: "sign1bit", TAG_QUANT2BIT: "quant2bit", TAG_QUANT4BIT: "quant4bit"}[tag]
            nb = -(-bits * rows * cols // 8)
            if len(body) < nb:
                raise PayloadError(f"{name}: truncated code map")
            if len(body) != nb + 4 * (rows + cols):
                raise PayloadError(f"{name}: body length mismatch")
            _check_scales(body, nb, rows, cols, name, nonneg_u=(tag == TAG_QUANT4BIT))
            cls = {TAG_SIGN1BIT: SignPayload, TAG_QUANT2BIT: Quant2Payload, TAG_QUANT4BIT: Quant4Payload}[tag]
            return cls(rows, cols, dev(body))
        if tag in (TAG_LOWRANK, TAG_LOWRANK_INT4):
            if len(body) < 4:
                raise PayloadError("lowrank: missing rank")
            (r,) = struct.unpack_from("<I", body, 0)
            if not (1 <= r <= min(rows, cols)):
                raise PayloadError(f"lowrank: rank {r} out of range for {rows}x{cols}")
            rest = body[4:]
            if tag == TAG_LOWRANK:
                if len(rest) != 2 * r * (rows + cols):
                    raise PayloadError("lowrank: body length mismatch")
            else:
                if len(rest) < 8 * r:
                    raise PayloadError("lowrank: body length mismatch")
                rg = np.frombuffer(rest, "<f4", 2 * r, 0)
                if not np.all(np.isfinite(rg)):
                    raise PayloadError("lowrank: non-finite ranges")
                if len(rest) - 8 * r != -(-r * (rows + cols) // 2):
                    raise PayloadError("lowrank: nibble stream length mismatch")
            return LowRankPayload(rows, cols, dev(rest), r, tag == TAG_LOWRANK_INT4)
        if tag == TAG_TOPK:
            if len(body) < 4:
                raise PayloadError("topk: missing count")
            (k,) = struct.unpack_from("<I", body, 0)
            rest = body[4:]
            if len(rest) != 6 * k:
                raise PayloadError("topk: truncated body")
            idx = np.frombuffer(rest, "<u4", k, 0)
            if k and int(idx.max()) >= rows * cols:
                raise PayloadError("topk: index out of range")
            return TopKPayload(rows, cols, dev(rest), k)
        if tag == TAG_NMBLOCK:  # cx:658-674
            if len(body) < 4:
                raise PayloadError("nmblock: missing n:m meta")
            n, m = struct.unpack_from("<HH", body, 0)
            if not (1 <= n <= m):
                raise PayloadError("nmblock: bad n:m")
            rest = body[4:]
            blocks = rows * (-(-cols // m))
            mask_bytes = -(-blocks * m // 8)
            if len(rest) < mask_bytes or (len(rest) - mask_bytes) % 2 or (len(rest) - mask_bytes) // 2 != blocks * n:
                raise PayloadError("nmblock: truncated body")
            masks = np.frombuffer(rest, np.uint8, mask_bytes, 0)
            # every 1 x m block keeps exactly n entries: the device decoders place a block's
            # values at block * n + local rank, so an uneven mask (which the reference would
            # fill in global flat order, cx:672) must not reach them
            bits = np.unpackbits(masks, count=blocks * m, bitorder="little")
            if blocks and not np.all(bits.reshape(blocks, m).sum(axis=1) == n):
                raise PayloadError("nmblock: mask popcount mismatch")
            return NMBlockPayload(rows, cols, dev(rest), n, m)
    except PayloadError:
        raise
    except Exception as exc:  # struct errors, bad slices
        raise PayloadError(f"tag {tag}: {exc}") from exc
    raise PayloadError(f"unknown codec tag {tag}")


__all__ = [n for n in dir() if not n.startswith("_")] + ["_lib"]
_ = ctypes  # keep import (ctypes pointers built in _lib)
