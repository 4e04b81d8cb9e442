"""Test-only codec engine for the engine-agnostic exchange layer (comm.py).

It implements CudaEngine's interface with the numpy oracle on CPU tensors so
that the multi-process exchange logic (sharding, fixed-size framing, step
counters, reassembly, all-gather / all-to-all over the gloo backend) can be
tested without a GPU.  This is test infrastructure: the product never imports it.
"""

from __future__ import annotations

import numpy as np
import torch

from oracle import cc_oracle as O

_TAGS = {"sign1bit": O.SIGN1, "quant2bit": O.QUANT2, "topk": O.TOPK}


def _ocodec(codec):
    kind = getattr(codec.kind, "value", codec.kind)
    if kind == "topk":
        return O.Codec(O.TOPK, keep_fraction=codec.keep_fraction)
    if kind == "nm_block":
        return O.Codec(O.NMBLOCK, nm=(codec.n, codec.m))
    return O.Codec(_TAGS[kind])


class OracleEngine:
    device_type = "cpu"

    def encode(self, sender, x, codec, body_out, rng=None):
        mode = getattr(sender.mode, "value", sender.mode)
        ch = O.Channel(mode, sender.warmup_steps, sender.base.numpy().copy(),
                       fb=sender.feedback.numpy().copy(),
                       ref=sender.ref.numpy().copy() if sender.ref is not None else None, step=sender.step)
        xf = x.float().numpy()
        tag, body, rec = O.send(ch, xf, _ocodec(codec))
        sender.base.copy_(torch.from_numpy(ch.base))
        sender.feedback.copy_(torch.from_numpy(np.ascontiguousarray(ch.fb)))
        if sender.ref is not None:
            sender.ref.copy_(torch.from_numpy(np.ascontiguousarray(ch.ref)))
        sender.step = ch.step
        wire16 = tag == O.RAW and x.dtype == torch.bfloat16
        if wire16:
            body = x.contiguous().view(torch.uint8).numpy().tobytes()
        body_out[: len(body)].copy_(torch.frombuffer(bytearray(body), dtype=torch.uint8))
        return len(body), wire16, rec

    def decode(self, codec, warm, wire16, accumulate, rows, cols, bodies, bases):
        for r, b, base in zip(rows, bodies, bases):
            if warm:
                n = r * cols * (2 if wire16 else 4)
                raw = b[:n].clone()
                dec = (raw.view(torch.bfloat16).float() if wire16 else raw.view(torch.float32)).view(r, cols)
                base.copy_(dec)
                continue
            oc = _ocodec(codec)
            if oc.tag == O.TOPK:
                k = O.topk_count(r, cols, oc.keep_fraction)
                body = b[: 6 * k].numpy().tobytes()
            elif oc.tag == O.NMBLOCK:
                body = b[: O.body_bytes(oc.tag, r, cols, nm=oc.nm)].numpy().tobytes()
            else:
                body = b[: O.body_bytes(oc.tag, r, cols)].numpy().tobytes()
            dec = torch.from_numpy(O.decode_body(body, oc, r, cols))
            if accumulate == 0:
                base.copy_(dec)
            else:
                base.copy_(base + dec)
