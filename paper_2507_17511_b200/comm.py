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
  * K1 writes its body straight into the per-layer NCCL send buffer; the
    collective runs on a dedicated comm stream, K2 (batched over all peers, one
    launch) on a decode stream, so layer l's exchange overlaps layer l+1's
    compression (`overlap=True`);
  * warmup steps move the raw activation in its own dtype (bf16 stays bf16 on
    the wire: lossless, half the bytes of the reference's f32 raw frame).

Without a process group (world size 1) the exchange runs a loopback receiver on
the same GPU: BASELINE config 1 (sender + receiver LayerState, pl:182-192).
"""

from __future__ import annotations

import hashlib

import torch

from . import _lib
from . import compressors as cx
from . import pipeline as pl


def shard_bounds(rows, devices):
    """Contiguous row shards; the last device takes the remainder (mesh:125-135)."""
    q = rows // devices
    if q == 0:
        raise ValueError(f"cannot shard {rows} rows across {devices} devices")
    return [(d * q, rows if d == devices - 1 else (d + 1) * q) for d in range(devices)]


def _codec_tag(spec):
    k = cx.CompressorKind(spec.kind)
    tag = cx._spec_tag(spec)
    if tag is None:
        if k == cx.CompressorKind.TOPK:
            return _lib.CC_TOPK
        if k == cx.CompressorKind.LOWRANK:
            return _lib.CC_LOWRANK4 if spec.int4_factors else _lib.CC_LOWRANK
        if k == cx.CompressorKind.IDENTITY:
            return _lib.CC_RAW
        raise NotImplementedError(k)
    return tag


def body_bytes_for(spec, rows, cols):
    lib = _lib.load()
    tag = _codec_tag(spec)
    if tag == _lib.CC_TOPK:
        return lib.cc_body_bytes(tag, rows, cols, cx.topk_count(rows, cols, spec.keep_fraction))
    if tag in (_lib.CC_LOWRANK, _lib.CC_LOWRANK4):
        return lib.cc_body_bytes(tag, rows, cols, spec.rank)
    if tag == _lib.CC_RAW:
        return 4 * rows * cols
    return lib.cc_body_bytes(tag, rows, cols, 0)


def _param(spec, rows, cols):
    tag = _codec_tag(spec)
    if tag == _lib.CC_TOPK:
        return cx.topk_count(rows, cols, spec.keep_fraction)
    if tag in (_lib.CC_LOWRANK, _lib.CC_LOWRANK4):
        return spec.rank
    return 0


class _Streams:
    def __init__(self, device, overlap):
        self.compute = torch.cuda.current_stream(device)
        if overlap:
            self.comm = torch.cuda.Stream(device)
            self.decode = torch.cuda.Stream(device)
        else:
            self.comm = self.decode = self.compute


class PatchParallelExchange:
    """Per-layer compressed all-gather of row shards (mesh:188-237).

    step(x_shard) encodes this rank's rows, all-gathers the packed bodies and
    reconstructs every peer's rows into `self.full` ([rows, cols] f32).  With no
    process group it is the world-size-1 loopback (sender + receiver).
    """

    def __init__(self, rows, cols, codec, mode="residual_with_feedback", warmup=1, group=None,
                 in_dtype=torch.bfloat16, overlap=True, streams=None, rng_seed=0):
        import torch.distributed as dist

        self.rows, self.cols, self.codec = int(rows), int(cols), codec
        self.mode = pl.PipelineMode(mode)
        self.warmup = int(warmup)
        self.group = group
        self.distributed = group is not None or (dist.is_available() and dist.is_initialized())
        if self.distributed:
            self.P = dist.get_world_size(group)
            self.rank = dist.get_rank(group)
        else:
            self.P, self.rank = 1, 0
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.bounds = shard_bounds(self.rows, self.P) if self.P > 1 else [(0, self.rows)]
        lo, hi = self.bounds[self.rank]
        self.lo, self.hi = lo, hi
        self.in_dtype = in_dtype
        self.streams = streams or _Streams(self.device, overlap)
        self.rng_seed = rng_seed

        self.full = torch.zeros(self.rows, self.cols, dtype=torch.float32, device=self.device)
        # sender state: base is a view of the full reconstruction (own shard = sender.base, mesh:233)
        self.sender = pl.LayerState(self.mode, self.warmup, torch.zeros(1, 1, device=self.device))
        self.sender.base = self.full[lo:hi]
        self.sender.feedback = torch.zeros(hi - lo, self.cols, device=self.device)
        if self.mode == pl.PipelineMode.RESIDUAL_NO_FEEDBACK:
            self.sender.ref = torch.zeros(hi - lo, self.cols, device=self.device)
        elif self.mode == pl.PipelineMode.NAIVE:
            pass
        # peers: receiver bases are views of `full`; only step counters on host
        self.peers = [p for p in range(self.P) if p != self.rank]
        self.peer_step = {p: 0 for p in self.peers}
        if self.P == 1:  # loopback receiver (config 1)
            self.loop_base = torch.zeros(self.rows, self.cols, dtype=torch.float32, device=self.device)
            self.loop_step = 0
        esz = 2 if in_dtype == torch.bfloat16 else 4
        shard_rows = [b[1] - b[0] for b in self.bounds]
        self.body_max = max(max(body_bytes_for(codec, r, self.cols) for r in shard_rows),
                            max(r * self.cols * esz for r in shard_rows))
        self.body_max = (self.body_max + 255) // 256 * 256
        self.sendbuf = torch.zeros(self.body_max, dtype=torch.uint8, device=self.device)
        self.recvbuf = torch.zeros(self.P, self.body_max, dtype=torch.uint8, device=self.device)
        self.ev_encoded = torch.cuda.Event()
        self.ev_gathered = torch.cuda.Event()
        self.ev_decoded = torch.cuda.Event()
        self.last_record = None
        self.last_nbytes = 0
        self.comm_bytes = 0

    # -- one step ---------------------------------------------------------------
    def step(self, x_shard, rng=None, skip_comm=False):
        """Returns the reconstruction tensor (valid on the decode stream)."""
        S = self.streams
        lib = _lib.load()
        t = self.sender.step + 1
        warm = t <= self.warmup or cx.CompressorKind(self.codec.kind) == cx.CompressorKind.IDENTITY
        with torch.cuda.stream(S.compute):
            # previous step's decode must not race this step's K1 on the shared `full`
            S.compute.wait_event(self.ev_decoded)
            payload, rec = pl.encode_step(self.sender, x_shard, self.codec, rng=rng, body_out=self.sendbuf)
            self.last_record = rec
            self.ev_encoded.record(S.compute)
        self.last_nbytes = payload.body.numel()
        # equal-size collective: every rank sends the largest shard's body size
        if warm:
            per = max((b[1] - b[0]) * self.cols for b in self.bounds) * (2 if payload.wire_dtype == torch.bfloat16 else 4)
        else:
            per = max(body_bytes_for(self.codec, b[1] - b[0], self.cols) for b in self.bounds)
        with torch.cuda.stream(S.comm):
            S.comm.wait_event(self.ev_encoded)
            if self.P > 1:
                if not skip_comm:
                    import torch.distributed as dist

                    out = self.recvbuf[:, :per].contiguous() if per != self.body_max else self.recvbuf
                    if per == self.body_max:
                        dist.all_gather_into_tensor(out.view(-1), self.sendbuf, group=self.group)
                    else:
                        flat = torch.empty(self.P * per, dtype=torch.uint8, device=self.device)
                        dist.all_gather_into_tensor(flat, self.sendbuf[:per], group=self.group)
                        self.recvbuf[:, :per].copy_(flat.view(self.P, per))
                self.comm_bytes = per * (self.P - 1)
            self.ev_gathered.record(S.comm)
        with torch.cuda.stream(S.decode):
            S.decode.wait_event(self.ev_gathered)
            if self.P == 1:
                self._loopback_decode(payload, t, warm)
            else:
                self._decode_peers(t, warm, per)
            self.ev_decoded.record(S.decode)
        return self.full if self.P > 1 else self.loop_base

    def _decode_peers(self, t, warm, per):
        lib = _lib.load()
        for p in self.peers:
            if self.peer_step[p] + 1 != t:
                raise pl.ProtocolError(f"peer {p}: step desynchronization")
        rows = [self.bounds[p][1] - self.bounds[p][0] for p in self.peers]
        if warm:
            tag, acc, dt = _lib.CC_RAW, 0, cx.dtype_code(torch.empty(0, dtype=self.in_dtype))
        else:
            tag, acc, dt = _codec_tag(self.codec), (0 if self.mode == pl.PipelineMode.NAIVE else 1), _lib.CC_F32
        param = _param(self.codec, rows[0], self.cols) if not warm else 0
        n = len(self.peers)
        import ctypes

        rows_arr = (ctypes.c_int64 * n)(*rows)
        bodies = (ctypes.c_void_p * n)(*[self.recvbuf[p].data_ptr() for p in self.peers])
        bases = (ctypes.c_void_p * n)(*[self.full[self.bounds[p][0]:self.bounds[p][1]].data_ptr()
                                        for p in self.peers])
        if tag in (_lib.CC_TOPK, _lib.CC_LOWRANK, _lib.CC_LOWRANK4) and len(set(rows)) > 1:
            for i, p in enumerate(self.peers):
                prm = _param(self.codec, rows[i], self.cols)
                _lib.check(lib.cc_decode_step(tag, acc, rows[i], self.cols, prm, ctypes.c_void_p(bodies[i]), dt,
                                              ctypes.c_void_p(bases[i]), _lib.stream_ptr()), "decode peer")
        else:
            _lib.check(lib.cc_decode_batched(tag, acc, n, rows_arr, self.cols, param, bodies, dt, bases,
                                             _lib.stream_ptr()), "decode peers")
        for p in self.peers:
            self.peer_step[p] = t

    def _loopback_decode(self, payload, t, warm):
        lib = _lib.load()
        if self.loop_step + 1 != t:
            raise pl.ProtocolError("loopback step desynchronization")
        replace = warm or self.mode == pl.PipelineMode.NAIVE
        _lib.check(lib.cc_decode_step(payload.tag, 0 if replace else 1, self.rows, self.cols, payload._param(),
                                      _lib.ptr(payload.body), payload._body_dtype(), _lib.ptr(self.loop_base),
                                      _lib.stream_ptr()), "loopback decode")
        self.loop_step = t

    def synchronize(self):
        torch.cuda.current_stream().wait_event(self.ev_decoded)

    def digest(self):
        """blake2b of the full reconstruction (mesh:237)."""
        self.synchronize()
        full = self.full if self.P > 1 else self.loop_base
        return hashlib.blake2b(full.cpu().numpy().tobytes(), digest_size=16).digest()


class UlyssesAllToAll:
    """Ulysses sequence-parallel exchange of compressed residuals (SPEC.md:473
    channel rule: every directed (src, dst) chunk is an independent LayerState).

    Rank r holds its sequence shard x[n_local, C] for all heads; the all-to-all
    sends column chunk d (heads of rank d, width C/P) to rank d, so rank d ends
    up with the full sequence for its heads: out[P * n_local, C/P].  Each of the
    P x P directed chunks is compressed through its own sender/receiver pair;
    bodies are fixed-size so `all_to_all_single` with equal splits suffices.
    """

    def __init__(self, n_local, cols, codec, mode="residual_with_feedback", warmup=1, group=None,
                 in_dtype=torch.bfloat16, overlap=True):
        import torch.distributed as dist

        self.group = group
        self.P = dist.get_world_size(group) if (dist.is_available() and dist.is_initialized()) else 1
        self.rank = dist.get_rank(group) if self.P > 1 else 0
        if cols % self.P:
            raise ValueError("cols must divide by world size (heads split evenly)")
        self.n, self.C, self.cw = int(n_local), int(cols), int(cols) // self.P
        self.codec, self.warmup = codec, int(warmup)
        self.mode = pl.PipelineMode(mode)
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.in_dtype = in_dtype
        z = torch.zeros(self.n, self.cw, device=self.device)
        self.senders = [pl.LayerState(self.mode, self.warmup, z) for _ in range(self.P)]
        # out[src] block: rows of rank src for our heads; receiver bases are views
        self.out = torch.zeros(self.P * self.n, self.cw, dtype=torch.float32, device=self.device)
        self.recv_step = [0] * self.P
        esz = 2 if in_dtype == torch.bfloat16 else 4
        self.body = max(body_bytes_for(codec, self.n, self.cw), self.n * self.cw * esz)
        self.body = (self.body + 255) // 256 * 256
        self.sendbuf = torch.zeros(self.P, self.body, dtype=torch.uint8, device=self.device)
        self.recvbuf = torch.zeros(self.P, self.body, dtype=torch.uint8, device=self.device)
        self.streams = _Streams(self.device, overlap)
        self.ev_encoded = torch.cuda.Event()
        self.ev_gathered = torch.cuda.Event()

    def step(self, x_local, rng=None):
        S = self.streams
        lib = _lib.load()
        t = self.senders[0].step + 1
        warm = t <= self.warmup
        with torch.cuda.stream(S.compute):
            for d in range(self.P):
                chunk = x_local[:, d * self.cw:(d + 1) * self.cw].contiguous()
                pl.encode_step(self.senders[d], chunk, self.codec, rng=rng, body_out=self.sendbuf[d])
            self.ev_encoded.record(S.compute)
        per = self.n * self.cw * (2 if self.in_dtype == torch.bfloat16 else 4) if warm else \
            body_bytes_for(self.codec, self.n, self.cw)
        with torch.cuda.stream(S.comm):
            S.comm.wait_event(self.ev_encoded)
            if self.P > 1:
                import torch.distributed as dist

                send = self.sendbuf[:, :per].contiguous()
                recv = torch.empty_like(send)
                dist.all_to_all_single(recv.view(-1), send.view(-1), group=self.group)
                self.recvbuf[:, :per].copy_(recv)
            else:
                self.recvbuf[:, :per].copy_(self.sendbuf[:, :per])
            self.ev_gathered.record(S.comm)
        with torch.cuda.stream(S.decode):
            S.decode.wait_event(self.ev_gathered)
            import ctypes

            if warm:
                tag, acc, dt = _lib.CC_RAW, 0, cx.dtype_code(torch.empty(0, dtype=self.in_dtype))
            else:
                tag, acc, dt = _codec_tag(self.codec), (0 if self.mode == pl.PipelineMode.NAIVE else 1), _lib.CC_F32
            rows = (ctypes.c_int64 * self.P)(*([self.n] * self.P))
            bodies = (ctypes.c_void_p * self.P)(*[self.recvbuf[s].data_ptr() for s in range(self.P)])
            bases = (ctypes.c_void_p * self.P)(*[self.out[s * self.n:(s + 1) * self.n].data_ptr()
                                                 for s in range(self.P)])
            _lib.check(lib.cc_decode_batched(tag, acc, self.P, rows, self.cw, _param(self.codec, self.n, self.cw),
                                             bodies, dt, bases, _lib.stream_ptr()), "ulysses decode")
            for s in range(self.P):
                self.recv_step[s] = t
        torch.cuda.current_stream().wait_stream(S.decode)
        return self.out
