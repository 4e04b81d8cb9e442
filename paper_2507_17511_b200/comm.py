"""Compressed exchanges for patch parallelism (all-gather) and Ulysses (all-to-all).

Reference behaviour (mesh.py, cited mesh:<line>): every device owns a contiguous
row shard (last one takes the remainder, mesh:125-135), encodes it once per step
through its sender LayerState, ships the same body to every peer, decodes every
peer's body through a per-(sender, receiver) state, and reassembles the full
tensor with ITS OWN shard taken from sender.base (mesh:188-236).  Devices must
agree bit-for-bit (digest check, mesh:237, 320-324).

B200 design:
  * one process per GPU; the NCCL communicator comes from torch.distributed
    (plumbing only) — `all_gather_into_tensor` / `all_to_all_single` move the
    fixed-size packed bodies (sizes are a pure function of shape and codec);
  * the reconstruction lives in ONE [rows, cols] f32 tensor per layer: the
    sender base of this rank and every receiver base are row-views of it, so the
    vstack of mesh:232-236 costs nothing;
  * K1 writes its body straight into the per-layer send buffer; the collective
    runs on a dedicated comm stream and K2 (batched over all peers, one launch)
    on a decode stream, so layer l's exchange overlaps layer l+1's compression;
  * warmup steps move the raw activation in its own dtype (bf16 stays bf16 on
    the wire: lossless, half the bytes of the reference's f32 raw frame).

The per-step codec work is done by an *engine*.  The product engine is
`CudaEngine` (sm_100a kernels through the C ABI).  The exchange logic itself
(sharding, fixed-size framing, step counters, reassembly, digests) is
engine-agnostic so the multi-process tests can run it on CPU with the gloo
backend and a test-only engine (tests/oracle_engine.py).

Without a process group (world size 1) the exchange runs a loopback receiver on
the same GPU: BASELINE config 1 (sender + receiver LayerState, pl:182-192).
"""

from __future__ import annotations

import ctypes
import hashlib

import torch

from . import _lib
from . import compressors as cx
from . import pipeline as pl


class TransportError(RuntimeError):
    """A collective failed (the reference's transport.TransportError, tr:22)."""


def shard_bounds(rows, devices):
    """Contiguous row shards; the last device takes the remainder (mesh:125-135)."""
    q = rows // devices
    if q == 0:
        raise ValueError(f"cannot shard {rows} rows across {devices} devices")
    return [(d * q, rows if d == devices - 1 else (d + 1) * q) for d in range(devices)]


def codec_tag(spec):
    k = cx.CompressorKind(spec.kind)
    tag = cx._spec_tag(spec)
    if tag is not None:
        return tag
    if k == cx.CompressorKind.TOPK:
        return _lib.CC_TOPK
    if k == cx.CompressorKind.NM_BLOCK:
        return _lib.CC_NMBLOCK
    if k == cx.CompressorKind.LOWRANK:
        return _lib.CC_LOWRANK4 if spec.int4_factors else _lib.CC_LOWRANK
    if k == cx.CompressorKind.IDENTITY:
        return _lib.CC_RAW
    raise NotImplementedError(k)


def codec_param(spec, rows, cols):
    tag = codec_tag(spec)
    if tag == _lib.CC_TOPK:
        return cx.topk_count(rows, cols, spec.keep_fraction)
    if tag in (_lib.CC_LOWRANK, _lib.CC_LOWRANK4):
        return spec.rank
    if tag == _lib.CC_NMBLOCK:
        return _lib.nm_param(spec.n, spec.m)
    return 0


def body_bytes_for(spec, rows, cols):
    """Exact body bytes of one compressed (non-warmup) transmission (cx:195-348)."""
    tag = codec_tag(spec)
    if tag == _lib.CC_RAW:
        return 4 * rows * cols
    if tag == _lib.CC_TOPK:
        return 6 * cx.topk_count(rows, cols, spec.keep_fraction)
    s = rows * cols
    if tag == _lib.CC_SIGN1:
        return (s + 7) // 8 + 4 * (rows + cols)
    if tag == _lib.CC_QUANT2:
        return (2 * s + 7) // 8 + 4 * (rows + cols)
    if tag == _lib.CC_QUANT4:
        return (4 * s + 7) // 8 + 4 * (rows + cols)
    if tag == _lib.CC_NMBLOCK:
        blocks = rows * (-(-cols // spec.m))
        return -(-blocks * spec.m // 8) + 2 * blocks * spec.n
    if tag == _lib.CC_LOWRANK:
        return 2 * spec.rank * (rows + cols)
    if tag == _lib.CC_LOWRANK4:
        return (4 * spec.rank * (rows + cols) + 7) // 8 + 8 * spec.rank
    raise NotImplementedError(tag)


# ---------------------------------------------------------------------------
# engines
# ---------------------------------------------------------------------------

class CudaEngine:
    """The product engine: every encode / decode is a sm_100a kernel launch."""

    device_type = "cuda"

    def encode(self, sender, x, codec, body_out, rng=None):
        payload, rec = pl.encode_step(sender, x, codec, rng=rng, body_out=body_out)
        wire16 = isinstance(payload, cx.RawPayload) and payload.wire_dtype == torch.bfloat16
        return payload.body.numel(), wire16, rec

    def decode(self, codec, warm, wire16, accumulate, rows, cols, bodies, bases):
        """One batched K2 launch over all peers (mesh:234-235)."""
        lib = _lib.load()
        n = len(bodies)
        if n == 0:
            return
        if warm:
            tag, acc, dt, param = _lib.CC_RAW, 0, (_lib.CC_BF16 if wire16 else _lib.CC_F32), 0
        else:
            tag, acc, dt = codec_tag(codec), accumulate, _lib.CC_F32
            param = codec_param(codec, rows[0], cols)
        if tag in (_lib.CC_TOPK, _lib.CC_LOWRANK, _lib.CC_LOWRANK4) and len(set(rows)) > 1:
            for r, b, base in zip(rows, bodies, bases):
                _lib.check(lib.cc_decode_step(tag, acc, r, cols, codec_param(codec, r, cols), _lib.ptr(b), dt,
                                              _lib.ptr(base), _lib.stream_ptr()), "decode peer")
            return
        rows_arr = (ctypes.c_int64 * n)(*rows)
        b_arr = (ctypes.c_void_p * n)(*[b.data_ptr() for b in bodies])
        base_arr = (ctypes.c_void_p * n)(*[b.data_ptr() for b in bases])
        _lib.check(lib.cc_decode_batched(tag, acc, n, rows_arr, cols, param, b_arr, dt, base_arr,
                                         _lib.stream_ptr()), "decode peers")


class _Streams:
    """compute = the caller's current stream at step time (so a CUDA-graph
    capture stream is honoured); comm / decode are side streams joined back
    through events."""

    def __init__(self, device, overlap):
        self.device = device
        self.overlap = overlap
        if device.type != "cuda":
            self._comm = self._decode = None
            return
        if overlap:
            self._comm = torch.cuda.Stream(device)
            self._decode = torch.cuda.Stream(device)

    @property
    def compute(self):
        return torch.cuda.current_stream(self.device) if self.device.type == "cuda" else None

    @property
    def comm(self):
        return self._comm if self.overlap else self.compute

    @property
    def decode(self):
        return self._decode if self.overlap else self.compute


class _NullCtx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def _on(stream):
    return torch.cuda.stream(stream) if stream is not None else _NullCtx()


class _Event:
    """CUDA event on GPU, no-op on CPU (collectives there are synchronous)."""

    def __init__(self, cuda):
        self.ev = torch.cuda.Event() if cuda else None

    def record(self, stream):
        if self.ev is not None:
            self.ev.record(stream)

    def wait(self, stream):
        if self.ev is not None:
            stream.wait_event(self.ev)


def _segmented_ok(codec, n, cols, P):
    """cc_encode_step_segmented's shape rules (k1_fused.cu fused_segments_supported)."""
    kind = cx.CompressorKind(codec.kind)
    if kind not in (cx.CompressorKind.SIGN1BIT, cx.CompressorKind.QUANT2BIT, cx.CompressorKind.QUANT4BIT):
        return False
    if cols % 128 or cols > 3072 or cols % P or P > 16:
        return False
    cw = cols // P
    groups = 1 if cols // 4 > 384 else 384 // (cols // 4)
    return cw % 128 == 0 and 2 * groups * P <= 32


def _dist():
    import torch.distributed as dist

    return dist


def _backend(group):
    dist = _dist()
    try:
        return dist.get_backend(group)
    except Exception:
        return None


def all_gather_flat(out, inp, group=None):
    """all_gather_into_tensor of equal-size byte slots.  NCCL moves device memory
    directly; a gloo group (multi-process tests that share one GPU, or CPU runs)
    carries CUDA tensors through host staging on the current stream."""
    dist = _dist()
    if inp.is_cuda and _backend(group) == "gloo":
        o = torch.empty(out.shape, dtype=out.dtype)
        dist.all_gather_into_tensor(o, inp.cpu(), group=group)
        out.copy_(o)
        return
    dist.all_gather_into_tensor(out, inp, group=group)


def all_to_all_flat(out, inp, group=None):
    """all_to_all_single with equal splits (see all_gather_flat for gloo)."""
    dist = _dist()
    if inp.is_cuda and _backend(group) == "gloo":
        o = torch.empty(out.shape, dtype=out.dtype)
        dist.all_to_all_single(o, inp.cpu(), group=group)
        out.copy_(o)
        return
    dist.all_to_all_single(out, inp, group=group)


def sendrecv(send, dst, recv, src, group=None):
    """One ring hop: send `send` to dst while receiving `recv` from src."""
    dist = _dist()
    if send.is_cuda and _backend(group) == "gloo":
        hs, hr = send.cpu(), torch.empty(recv.shape, dtype=recv.dtype)
        ops = [dist.P2POp(dist.isend, hs, dst, group=group), dist.P2POp(dist.irecv, hr, src, group=group)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        recv.copy_(hr)
        return
    ops = [dist.P2POp(dist.isend, send, dst, group=group), dist.P2POp(dist.irecv, recv, src, group=group)]
    for w in dist.batch_isend_irecv(ops):
        w.wait()


def _check_dtype(x, in_dtype):
    """Send buffers are sized for raw (warmup) bodies of `in_dtype`; a wider input
    would overrun them."""
    if x.dtype != in_dtype:
        raise ValueError(f"input dtype {x.dtype} != the exchange's in_dtype {in_dtype}")


def _receiver_accumulate(codec, mode, canon_pending):
    if mode == pl.PipelineMode.NAIVE:
        return 0
    if codec_tag(codec) == _lib.CC_TOPK and canon_pending:
        return 2  # first sparse add after a dense replace: reference's dense `base + 0.0`
    return 1


class PatchParallelExchange:
    """Per-layer compressed all-gather of row shards (mesh:188-237).

    step(x_shard) encodes this rank's rows, all-gathers the packed bodies and
    reconstructs every peer's rows into `self.full` ([rows, cols] f32).  With no
    process group it is the world-size-1 loopback (sender + receiver).
    """

    def __init__(self, rows, cols, codec, mode="residual_with_feedback", warmup=1, group=None,
                 in_dtype=torch.bfloat16, overlap=True, streams=None, engine=None, device=None, sim_world=None):
        dist = _dist()
        self.rows, self.cols, self.codec = int(rows), int(cols), codec
        self.mode = pl.PipelineMode(mode)
        self.warmup = int(warmup)
        self.group = group
        # sim_world = (P, rank): single-GPU stand-in for one rank of a P-rank job (benchmarks
        # only): the collective is replaced by device copies of this rank's own body into
        # every peer slot, so K1 / K2 / the copies run at the real per-rank shapes
        self.sim = sim_world is not None
        if self.sim:
            self.P, self.rank = int(sim_world[0]), int(sim_world[1])
        elif dist.is_available() and dist.is_initialized():
            self.P, self.rank = dist.get_world_size(group), dist.get_rank(group)
        else:
            self.P, self.rank = 1, 0
        self.engine = engine or CudaEngine()
        self.device = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        self.cuda = self.device.type == "cuda"
        self.bounds = shard_bounds(self.rows, self.P) if self.P > 1 else [(0, self.rows)]
        self.lo, self.hi = self.bounds[self.rank]
        self.in_dtype = in_dtype
        self.streams = streams or _Streams(self.device, overlap)

        f32 = dict(dtype=torch.float32, device=self.device)
        self.full = torch.zeros(self.rows, self.cols, **f32)
        # sender state: base is a view of the full reconstruction (own shard = sender.base, mesh:233)
        self.sender = pl.LayerState.__new__(pl.LayerState)
        self.sender.mode, self.sender.warmup_steps, self.sender.step = self.mode, self.warmup, 0
        self.sender.base = self.full[self.lo:self.hi]
        self.sender.feedback = torch.zeros(self.hi - self.lo, self.cols, **f32)
        self.sender.ref = torch.zeros(self.hi - self.lo, self.cols, **f32) \
            if self.mode == pl.PipelineMode.RESIDUAL_NO_FEEDBACK else None
        self.sender._rec = None
        # receivers: bases are views of `full`; host keeps step counters (pl:153-156)
        self.peers = [p for p in range(self.P) if p != self.rank]
        self.peer_step = {p: 0 for p in self.peers}
        self.loop_base = torch.zeros(self.rows, self.cols, **f32) if self.P == 1 else None
        self.loop_step = 0
        self._canon_pending = True
        esz = 2 if in_dtype == torch.bfloat16 else 4
        shard_rows = [b[1] - b[0] for b in self.bounds]
        self.body_max = max(max(body_bytes_for(codec, r, self.cols) for r in shard_rows),
                            max(r * self.cols * esz for r in shard_rows))
        self.body_max = (self.body_max + 255) // 256 * 256
        self.sendbuf = torch.zeros(self.body_max, dtype=torch.uint8, device=self.device)
        # all-gather lands directly here: P contiguous slots of the step's wire size
        self.recvflat = torch.zeros(self.P * self.body_max, dtype=torch.uint8, device=self.device)
        self._per = self.body_max
        self.ev_encoded, self.ev_gathered, self.ev_decoded = (_Event(self.cuda) for _ in range(3))
        self.last_record = None
        self.last_nbytes = 0
        self.comm_bytes = 0

    def after_capture(self):
        """Events recorded inside a CUDA-graph capture cannot be waited on eagerly:
        start fresh ones (the captured graph keeps its own copies)."""
        self.ev_encoded, self.ev_gathered, self.ev_decoded = (_Event(self.cuda) for _ in range(3))

    def wire_bytes(self, warm, wire16):
        """Equal-size collective: every rank sends the largest shard's body, padded to
        16 bytes so every receive slot (rank p at p * wire_bytes) stays aligned for the
        vectorised decoders (top-k bodies are 6k bytes)."""
        if warm:
            per = max(b[1] - b[0] for b in self.bounds) * self.cols * (2 if wire16 else 4)
        else:
            per = max(body_bytes_for(self.codec, b[1] - b[0], self.cols) for b in self.bounds)
        return (per + 15) // 16 * 16

    # -- one step ---------------------------------------------------------------
    def step(self, x_shard, rng=None, skip_comm=False, k1_events=None, k2_events=None):
        """Returns the reconstruction tensor (on GPU: valid on the decode stream).
        k1_events / k2_events: optional (start, end) CUDA events recorded around the
        encode (K1, compute stream) / the peer decode (K2, decode stream), for
        per-kernel timing (also inside a CUDA-graph capture, with external events)."""
        S = self.streams
        _check_dtype(x_shard, self.in_dtype)
        t = self.sender.step + 1
        warm = t <= self.warmup or cx.CompressorKind(self.codec.kind) == cx.CompressorKind.IDENTITY
        with _on(S.compute):
            # the previous decode must not race this K1 on `full` (inside a CUDA-graph
            # capture that order is implied by the ordering of graph launches)
            if S.compute is not None and not torch.cuda.is_current_stream_capturing():
                self.ev_decoded.wait(S.compute)
            if k1_events is not None:
                k1_events[0].record()
            nbytes, wire16, rec = self.engine.encode(self.sender, x_shard, self.codec, self.sendbuf, rng)
            if k1_events is not None:
                k1_events[1].record()
            self.last_record, self.last_nbytes = rec, nbytes
            self.ev_encoded.record(S.compute)
        per = self.wire_bytes(warm, wire16)
        with _on(S.comm):
            if S.comm is not None:
                self.ev_encoded.wait(S.comm)
            if self.P > 1:
                self._per = per
                if skip_comm:
                    pass
                elif self.sim:  # the body into every peer slot (stands in for the all-gather)
                    # one broadcast copy in 8-byte words (per is a multiple of 16): a uint8
                    # element-wise copy is ~8x slower than the NCCL landing it stands for
                    w = per // 8
                    slots = self.recvflat[:self.P * per].view(torch.int64).view(self.P, w)
                    src = self.sendbuf[:per].view(torch.int64)
                    if self.peers == list(range(1, self.P)):
                        slots[1:].copy_(src.expand(self.P - 1, w))
                    else:
                        for p in self.peers:
                            slots[p].copy_(src)
                else:
                    all_gather_flat(self.recvflat[:self.P * per], self.sendbuf[:per], group=self.group)
                self.comm_bytes = per * (self.P - 1)
            self.ev_gathered.record(S.comm)
        with _on(S.decode):
            if S.decode is not None:
                self.ev_gathered.wait(S.decode)
            if k2_events is not None:
                k2_events[0].record(S.decode)
            if self.P == 1:
                self._loopback_decode(t, warm, wire16, nbytes)
            else:
                self._decode_peers(t, warm, wire16)
            if k2_events is not None:
                k2_events[1].record(S.decode)
            self.ev_decoded.record(S.decode)
        return self.full if self.P > 1 else self.loop_base

    def _decode_peers(self, t, warm, wire16):
        for p in self.peers:
            if self.peer_step[p] + 1 != t:
                raise pl.ProtocolError(f"peer {p}: step desynchronization")
        rows = [self.bounds[p][1] - self.bounds[p][0] for p in self.peers]
        acc = _receiver_accumulate(self.codec, self.mode, self._canon_pending)
        bases = [self.full[self.bounds[p][0]:self.bounds[p][1]] for p in self.peers]
        self.engine.decode(self.codec, warm, wire16, acc, rows, self.cols, [self.slot(p) for p in self.peers],
                           bases)
        self._canon_pending = warm or (self._canon_pending and acc == 0)
        for p in self.peers:
            self.peer_step[p] = t

    def slot(self, p):
        """Received body of rank p in the current step's layout."""
        return self.recvflat[p * self._per:(p + 1) * self._per]

    def _loopback_decode(self, t, warm, wire16, nbytes):
        if self.loop_step + 1 != t:
            raise pl.ProtocolError("loopback step desynchronization")
        acc = _receiver_accumulate(self.codec, self.mode, self._canon_pending)
        self.engine.decode(self.codec, warm, wire16, acc, [self.rows], self.cols, [self.sendbuf[:max(nbytes, 1)]],
                           [self.loop_base])
        self._canon_pending = warm or (self._canon_pending and acc == 0)
        self.loop_step = t

    def synchronize(self):
        if self.cuda:
            self.ev_decoded.wait(torch.cuda.current_stream(self.device))

    def reconstruction(self):
        self.synchronize()
        return self.full if self.P > 1 else self.loop_base

    def digest(self):
        """blake2b of the full reconstruction (mesh:237)."""
        return hashlib.blake2b(self.reconstruction().cpu().numpy().tobytes(), digest_size=16).digest()


class RingExchange(PatchParallelExchange):
    """Ring-attention style compressed exchange (mesh:214-229).

    The shard is encoded once at its origin; in each of the P-1 hops every rank
    forwards the body it received in the previous hop verbatim to (rank+1) % P
    while receiving from (rank-1) % P over NCCL point-to-point.  The body
    received in hop r originates at (rank - r) % P (the reference's
    `ring_origin` = (device - rnd + 1) % P is off by one, mesh:138-140, SURVEY
    §8f).  Hop r's body is decoded on the decode stream while hop r+1 is in
    flight, and the reconstruction is identical to the all-gather exchange.
    """

    def __init__(self, *args, **kw):
        super().__init__(*args, **kw)
        self.ev_hop = [_Event(self.cuda) for _ in range(max(self.P - 1, 1))]

    def after_capture(self):
        super().after_capture()
        self.ev_hop = [_Event(self.cuda) for _ in range(max(self.P - 1, 1))]

    @staticmethod
    def origin(rank, rnd, P):
        return (rank - rnd) % P

    def step(self, x_shard, rng=None, skip_comm=False, k1_events=None, k2_events=None):
        if self.P == 1 or self.sim:
            return super().step(x_shard, rng=rng, skip_comm=skip_comm, k1_events=k1_events, k2_events=k2_events)
        S = self.streams
        _check_dtype(x_shard, self.in_dtype)
        t = self.sender.step + 1
        warm = t <= self.warmup or cx.CompressorKind(self.codec.kind) == cx.CompressorKind.IDENTITY
        with _on(S.compute):
            if S.compute is not None and not torch.cuda.is_current_stream_capturing():
                self.ev_decoded.wait(S.compute)
            if k1_events is not None:
                k1_events[0].record()
            nbytes, wire16, rec = self.engine.encode(self.sender, x_shard, self.codec, self.sendbuf, rng)
            if k1_events is not None:
                k1_events[1].record()
            self.last_record, self.last_nbytes = rec, nbytes
            self.ev_encoded.record(S.compute)
        per = self.wire_bytes(warm, wire16)
        self._per = per
        for p in self.peers:
            if self.peer_step[p] + 1 != t:
                raise pl.ProtocolError(f"peer {p}: step desynchronization")
        acc = _receiver_accumulate(self.codec, self.mode, self._canon_pending)
        nxt, prv = (self.rank + 1) % self.P, (self.rank - 1) % self.P
        carried = self.sendbuf[:per]
        for rnd in range(1, self.P):
            o = self.origin(self.rank, rnd, self.P)
            recv = self.slot(o)
            with _on(S.comm):
                if rnd == 1 and S.comm is not None:
                    self.ev_encoded.wait(S.comm)
                if not skip_comm:
                    sendrecv(carried, nxt, recv, prv, group=self.group)
                self.ev_hop[rnd - 1].record(S.comm)
            with _on(S.decode):
                if S.decode is not None:
                    self.ev_hop[rnd - 1].wait(S.decode)
                lo, hi = self.bounds[o]
                self.engine.decode(self.codec, warm, wire16, acc, [hi - lo], self.cols, [recv],
                                   [self.full[lo:hi]])
            carried = recv
        self.comm_bytes = per * (self.P - 1)
        with _on(S.decode):
            self.ev_decoded.record(S.decode)
        self._canon_pending = warm or (self._canon_pending and acc == 0)
        for p in self.peers:
            self.peer_step[p] = t
        return self.full


class UlyssesAllToAll:
    """Ulysses sequence-parallel exchange of compressed residuals.

    Channel rule: every directed (src, dst) chunk is an independent
    LayerState pair.  Rank r holds its sequence shard x[n_local, C] for all heads;
    the all-to-all sends column chunk d (the heads of rank d, width C/P) to rank
    d, which ends up with the full sequence for its heads: out[P * n_local, C/P].
    Bodies are fixed-size, so `all_to_all_single` with equal splits suffices.
    With world size 1 the exchange is a loopback of one chunk.
    """

    def __init__(self, n_local, cols, codec, mode="residual_with_feedback", warmup=1, group=None,
                 in_dtype=torch.bfloat16, overlap=True, engine=None, device=None, sim_world=None):
        dist = _dist()
        self.group = group
        self.sim = sim_world is not None  # (P, rank): single-GPU stand-in (see PatchParallelExchange)
        if self.sim:
            self.P, self.rank = int(sim_world[0]), int(sim_world[1])
        elif dist.is_available() and dist.is_initialized():
            self.P, self.rank = dist.get_world_size(group), dist.get_rank(group)
        else:
            self.P, self.rank = 1, 0
        if cols % self.P:
            raise ValueError("cols must divide by world size (heads split evenly)")
        self.n, self.C, self.cw = int(n_local), int(cols), int(cols) // self.P
        self.codec, self.warmup = codec, int(warmup)
        self.mode = pl.PipelineMode(mode)
        self.engine = engine or CudaEngine()
        self.device = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        self.cuda = self.device.type == "cuda"
        self.in_dtype = in_dtype
        f32 = dict(dtype=torch.float32, device=self.device)
        # Segmented path: all P sender channels in ONE persistent K1 launch over the
        # full-width rows (cc_encode_step_segmented): the channel states are column
        # slices of [n, C] arrays and no chunk copies are made.  Otherwise one
        # encode_step per chunk on contiguous per-chunk states.
        self.segmented = self.cuda and self.P > 1 and _segmented_ok(codec, self.n, self.C, self.P)
        nofb = self.mode == pl.PipelineMode.RESIDUAL_NO_FEEDBACK
        if self.segmented:
            self.base_full = torch.zeros(self.n, self.C, **f32)
            self.aux_full = torch.zeros(self.n, self.C, **f32)  # feedback, or ref (no-feedback mode)
            self.rec_seg = torch.zeros(2 * self.P, dtype=torch.float64, device=self.device)
        self.senders = []
        for d in range(self.P):
            st = pl.LayerState.__new__(pl.LayerState)
            st.mode, st.warmup_steps, st.step, st._rec = self.mode, self.warmup, 0, None
            if self.segmented:
                sl = slice(d * self.cw, (d + 1) * self.cw)
                st.base = self.base_full[:, sl]
                st.feedback = None if nofb else self.aux_full[:, sl]
                st.ref = self.aux_full[:, sl] if nofb else None
            else:
                st.base = torch.zeros(self.n, self.cw, **f32)
                st.feedback = torch.zeros(self.n, self.cw, **f32)
                st.ref = torch.zeros(self.n, self.cw, **f32) if nofb else None
            self.senders.append(st)
        # out[src] block: rows of rank src for our heads; receiver bases are views
        self.out = torch.zeros(self.P * self.n, self.cw, **f32)
        self.recv_step = [0] * self.P
        self._canon_pending = True
        esz = 2 if in_dtype == torch.bfloat16 else 4
        self.body = max(body_bytes_for(codec, self.n, self.cw), self.n * self.cw * esz)
        self.body = (self.body + 255) // 256 * 256
        self.sendbuf = torch.zeros(self.P, self.body, dtype=torch.uint8, device=self.device)
        self.recvbuf = torch.zeros(self.P, self.body, dtype=torch.uint8, device=self.device)
        # packed wire staging (bodies shorter than the slot stride), allocated once
        self.sendflat = torch.zeros(self.P * self.body, dtype=torch.uint8, device=self.device)
        self.recvflat = torch.zeros(self.P * self.body, dtype=torch.uint8, device=self.device)
        self.streams = _Streams(self.device, overlap)
        self.ev_encoded, self.ev_gathered = _Event(self.cuda), _Event(self.cuda)

    def step(self, x_local, rng=None):
        S = self.streams
        _check_dtype(x_local, self.in_dtype)
        t = self.senders[0].step + 1
        # identity sends raw bodies every step, exactly like warmup (pl:89-97)
        warm = t <= self.warmup or cx.CompressorKind(self.codec.kind) == cx.CompressorKind.IDENTITY
        with _on(S.compute):
            if self.segmented:
                wire16 = self._encode_segmented(x_local, t, warm)
            else:
                for d in range(self.P):
                    chunk = x_local[:, d * self.cw:(d + 1) * self.cw].contiguous()
                    _, wire16, _ = self.engine.encode(self.senders[d], chunk, self.codec, self.sendbuf[d], rng)
            self.ev_encoded.record(S.compute)
        per = self.n * self.cw * (2 if wire16 else 4) if warm else body_bytes_for(self.codec, self.n, self.cw)
        with _on(S.comm):
            if S.comm is not None:
                self.ev_encoded.wait(S.comm)
            if self.P > 1 and not self.sim:
                # bodies are packed back to back at the step's wire size: slot d of the
                # send / receive staging is [d * per, (d + 1) * per)
                if per == self.body:
                    all_to_all_flat(self.recvbuf.view(-1), self.sendbuf.view(-1), group=self.group)
                else:
                    sflat = self.sendflat[:self.P * per]
                    sflat.view(self.P, per).copy_(self.sendbuf[:, :per])
                    rflat = self.recvflat[:self.P * per]
                    all_to_all_flat(rflat, sflat, group=self.group)
                    self.recvbuf[:, :per].copy_(rflat.view(self.P, per))
            else:  # loopback / single-GPU stand-in: the body of chunk d lands in slot d
                if per % 8 == 0 and self.recvbuf.shape[1] % 8 == 0:  # 8-byte words
                    self.recvbuf.view(torch.int64)[:, :per // 8].copy_(self.sendbuf.view(torch.int64)[:, :per // 8])
                else:
                    self.recvbuf[:, :per].copy_(self.sendbuf[:, :per])
            self.ev_gathered.record(S.comm)
        with _on(S.decode):
            if S.decode is not None:
                self.ev_gathered.wait(S.decode)
            for s in range(self.P):
                if self.recv_step[s] + 1 != t:
                    raise pl.ProtocolError(f"src {s}: step desynchronization")
            acc = _receiver_accumulate(self.codec, self.mode, self._canon_pending)
            self.engine.decode(self.codec, warm, wire16, acc, [self.n] * self.P, self.cw,
                               [self.recvbuf[s] for s in range(self.P)],
                               [self.out[s * self.n:(s + 1) * self.n] for s in range(self.P)])
            self._canon_pending = warm or (self._canon_pending and acc == 0)
            self.recv_step = [t] * self.P
        if S.decode is not None:
            torch.cuda.current_stream(self.device).wait_stream(S.decode)
        return self.out

    def _encode_segmented(self, x_local, t, warm):
        """All P chunk channels in one launch (see __init__); returns wire16."""
        lib = _lib.load()
        x = x_local if x_local.is_contiguous() else x_local.contiguous()
        if tuple(x.shape) != (self.n, self.C):
            raise pl.ShapeError(f"input shape {tuple(x.shape)} != {(self.n, self.C)}")
        mode = pl._MODE_CODE[self.mode]
        aux = None if self.mode == pl.PipelineMode.NAIVE else self.aux_full
        stream = _lib.stream_ptr()
        wire16 = x.dtype == torch.bfloat16
        if warm:
            # raw step (pl:89-97) on the full rows, then each chunk's raw body
            # (lossless bf16 for bf16 inputs) into its send slot
            esz = 2 if wire16 else 4
            tmp = cx._empty_body(self.n * self.C * esz)
            _lib.check(lib.cc_warmup_step(mode, self.n, self.C, _lib.ptr(x), cx.dtype_code(x),
                                          _lib.ptr(self.base_full), _lib.ptr(aux), _lib.ptr(tmp), cx.dtype_code(x),
                                          _lib.ptr(self.rec_seg), stream), "warmup")
            wdt = torch.bfloat16 if wire16 else torch.float32
            for d in range(self.P):
                dst = self.sendbuf[d, :self.n * self.cw * esz].view(wdt).view(self.n, self.cw)
                dst.copy_(x[:, d * self.cw:(d + 1) * self.cw])
        else:
            tag = cx._spec_tag(self.codec)
            ws = cx.workspace(_lib.check(lib.cc_workspace_bytes(tag, self.n, self.C, 0)))
            try:
                _lib.check(lib.cc_encode_step_segmented(
                    tag, mode, cx._SCALE_MODES[self.codec.scale_mode], self.n, self.C, self.P, _lib.ptr(x),
                    cx.dtype_code(x), _lib.ptr(self.base_full), _lib.ptr(aux), _lib.ptr(self.sendbuf), self.body,
                    _lib.ptr(ws), ws.numel(), _lib.ptr(self.rec_seg), stream), "segmented encode_step")
            except _lib.CudaError:
                # the persistent launch was refused (e.g. SMs held by another context):
                # encode every chunk channel on contiguous copies of its column slice
                # with the multi-kernel path — the same bytes, P launches instead of one
                self._encode_chunks_copied(x, t)
            wire16 = False
        for st in self.senders:
            st.step = t
        return wire16

    def _encode_chunks_copied(self, x, t):
        for d, st in enumerate(self.senders):
            sl = slice(d * self.cw, (d + 1) * self.cw)
            tmp = pl.LayerState.__new__(pl.LayerState)
            tmp.mode, tmp.warmup_steps, tmp.step, tmp._rec = self.mode, self.warmup, t - 1, None
            tmp.base = st.base.contiguous()
            tmp.feedback = st.feedback.contiguous() if st.feedback is not None else None
            tmp.ref = st.ref.contiguous() if st.ref is not None else None
            pl.encode_step(tmp, x[:, sl].contiguous(), self.codec, body_out=self.sendbuf[d])
            st.base.copy_(tmp.base)
            if st.feedback is not None:
                st.feedback.copy_(tmp.feedback)
            if st.ref is not None:
                st.ref.copy_(tmp.ref)


# ---------------------------------------------------------------------------
# The same exchanges through the C ABI (include/compactcomm.h "exchanges"): the
# whole layer step — K1, the NCCL collective, K2 — is one library call, with
# library-owned buffers; these classes only hold the handles.
# ---------------------------------------------------------------------------

class _DeviceArray:
    """A library-owned device buffer seen by torch (CUDA array interface)."""

    def __init__(self, ptr, shape, typestr="<f4"):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _as_tensor(ptr, shape, typestr="<f4"):
    return torch.as_tensor(_DeviceArray(ptr, shape, typestr), device="cuda")


class CComm:
    """cc_comm: adopts an NCCL communicator (a torch ProcessGroupNCCL's by default)
    or builds one from a unique id shared by the caller."""

    def __init__(self, handle):
        self.h = handle

    @staticmethod
    def from_process_group(group=None):
        dist = _dist()
        pg = group or dist.distributed_c10d._get_default_group()
        ptr = pg._get_backend(torch.device("cuda", torch.cuda.current_device()))._comm_ptr()
        h = ctypes.c_void_p()
        _lib.check(_lib.load().cc_comm_wrap(ctypes.c_void_p(ptr), ctypes.byref(h)), "cc_comm_wrap")
        return CComm(h)

    @staticmethod
    def unique_id():
        buf = (ctypes.c_uint8 * 128)()
        _lib.check(_lib.load().cc_comm_get_unique_id(buf), "cc_comm_get_unique_id")
        return bytes(buf)

    @staticmethod
    def init_rank(uid, nranks, rank):
        h = ctypes.c_void_p()
        _lib.check(_lib.load().cc_comm_init_rank((ctypes.c_uint8 * 128)(*uid), nranks, rank, ctypes.byref(h)),
                   "cc_comm_init_rank")
        return CComm(h)

    @property
    def rank(self):
        return _lib.load().cc_comm_rank(self.h)

    @property
    def size(self):
        return _lib.load().cc_comm_size(self.h)

    def destroy(self):
        if self.h:
            _lib.check(_lib.load().cc_comm_destroy(self.h), "cc_comm_destroy")
            self.h = None


def codec_spec_struct(codec):
    tag = codec_tag(codec)
    if cx.CompressorKind(codec.kind) == cx.CompressorKind.IDENTITY:
        tag = _lib.CC_RAW
    return _lib.CodecSpec(tag, cx._SCALE_MODES[getattr(codec, "scale_mode", "rank1")],
                          float(codec.keep_fraction or 0.0), int(codec.n or 0), int(codec.m or 0))


class CAllGather:
    """Patch-parallel compressed all-gather layer through the C ABI
    (cc_allgather_*): mesh.py:188-237 semantics, no Python on the step path."""

    def __init__(self, rows, cols, codec, mode="residual_with_feedback", warmup=1, in_dtype=torch.bfloat16,
                 comm=None):
        self.rows, self.cols, self.codec = int(rows), int(cols), codec
        self.comm = comm
        self.in_dtype = in_dtype
        spec = codec_spec_struct(codec)
        h = ctypes.c_void_p()
        _lib.check(_lib.load().cc_allgather_create(comm.h if comm else None, ctypes.byref(spec),
                                                   pl._MODE_CODE[pl.PipelineMode(mode)], self.rows, self.cols,
                                                   int(warmup), cx.dtype_code(torch.empty(0, dtype=in_dtype)),
                                                   ctypes.byref(h)), "cc_allgather_create")
        self.h = h
        lo, hi = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.load().cc_allgather_shard(h, ctypes.byref(lo), ctypes.byref(hi)))
        self.lo, self.hi = lo.value, hi.value

    def step(self, x_shard):
        _check_dtype(x_shard, self.in_dtype)
        if tuple(x_shard.shape) != (self.hi - self.lo, self.cols) or not x_shard.is_contiguous():
            raise pl.ShapeError(f"shard must be contiguous [{self.hi - self.lo}, {self.cols}]")
        _lib.check(_lib.load().cc_allgather_step(self.h, _lib.ptr(x_shard), _lib.stream_ptr()), "cc_allgather_step")
        return self.reconstruction()

    def reconstruction(self):
        return _as_tensor(_lib.load().cc_allgather_reconstruction(self.h), (self.rows, self.cols))

    def sender_base(self):
        return _as_tensor(_lib.load().cc_allgather_sender_base(self.h), (self.hi - self.lo, self.cols))

    def sender_aux(self):
        p = _lib.load().cc_allgather_sender_aux(self.h)
        return None if not p else _as_tensor(p, (self.hi - self.lo, self.cols))

    def body(self):
        nb = ctypes.c_int64()
        p = _lib.load().cc_allgather_body(self.h, ctypes.byref(nb))
        return _as_tensor(p, (max(nb.value, 1),), "|u1")[:nb.value]

    def record(self):
        return _as_tensor(_lib.load().cc_allgather_record(self.h), (2,), "<f8")

    def digest(self):
        torch.cuda.current_stream().synchronize()
        return hashlib.blake2b(self.reconstruction().cpu().numpy().tobytes(), digest_size=16).digest()

    def close(self):
        if self.h:
            _lib.check(_lib.load().cc_allgather_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class CAllToAll:
    """Ulysses compressed all-to-all layer through the C ABI (cc_alltoall_*)."""

    def __init__(self, n_local, cols, codec, mode="residual_with_feedback", warmup=1, in_dtype=torch.bfloat16,
                 comm=None):
        self.n, self.C = int(n_local), int(cols)
        self.P = comm.size if comm else 1
        self.in_dtype = in_dtype
        spec = codec_spec_struct(codec)
        h = ctypes.c_void_p()
        _lib.check(_lib.load().cc_alltoall_create(comm.h if comm else None, ctypes.byref(spec),
                                                  pl._MODE_CODE[pl.PipelineMode(mode)], self.n, self.C, int(warmup),
                                                  cx.dtype_code(torch.empty(0, dtype=in_dtype)), ctypes.byref(h)),
                   "cc_alltoall_create")
        self.h = h

    def step(self, x_local):
        _check_dtype(x_local, self.in_dtype)
        if tuple(x_local.shape) != (self.n, self.C) or not x_local.is_contiguous():
            raise pl.ShapeError(f"input must be contiguous [{self.n}, {self.C}]")
        _lib.check(_lib.load().cc_alltoall_step(self.h, _lib.ptr(x_local), _lib.stream_ptr()), "cc_alltoall_step")
        return self.output()

    def output(self):
        return _as_tensor(_lib.load().cc_alltoall_output(self.h), (self.P * self.n, self.C // self.P))

    def close(self):
        if self.h:
            _lib.check(_lib.load().cc_alltoall_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
