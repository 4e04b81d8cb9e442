"""GPU parity for the north_star extensions the reference does not have: the 4-bit
element quantizer and per-token-only / per-channel-only scales (SURVEY §0 gaps 1
and 3).  Their definition lives in oracle/cc_oracle.py (quant_body, scales,
quant4_codes — "defined-by-repo parity"); the device path must match it bit for
bit (bodies, base, feedback) through encode_step / decode_step, on both the
persistent fused K1 (C % 128 == 0, C <= 3072) and the multi-kernel K1, in every
pipeline mode, including zero rows / columns (zero scales) and -0.0."""

import zlib

import numpy as np
import pytest
import torch

import synth
from oracle import cc_oracle as O

pytestmark = pytest.mark.gpu

TAGS = {"sign1bit": O.SIGN1, "quant2bit": O.QUANT2, "quant4bit": O.QUANT4}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)


@pytest.fixture
def quant_path():
    from paper_2507_17511_b200 import _lib

    lib = _lib.load()
    yield lib.cc_set_quant_path
    lib.cc_set_quant_path(-1)


def _inputs(n, c, key):
    rng = np.random.default_rng(zlib.crc32(key.encode()))
    xs = synth.flux_like(n, c, 5, seed=int(rng.integers(1 << 30)))
    xs[2][rng.random((n, c)) < 0.2] = 0.0   # exact zeros
    xs[2][n // 2] = 0.0                     # a zero row (per-token zero scale)
    xs[3][:, c // 3] = -0.0                 # a -0.0 column (per-channel zero scale)
    xs[4] = -xs[4]
    return xs


SHAPES = [(13, 136), (64, 3072), (100, 1000), (37, 384), (3, 1025)]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"{s[0]}x{s[1]}")
@pytest.mark.parametrize("codec", ["sign1bit", "quant2bit", "quant4bit"])
@pytest.mark.parametrize("scale_mode", ["rank1", "per_token", "per_channel"])
@pytest.mark.parametrize("mode", ["naive", "residual_with_feedback"])
@pytest.mark.parametrize("path", [-1, 0], ids=["auto", "multikernel"])
def test_extension_trajectories_vs_oracle(shape, codec, scale_mode, mode, path, quant_path):
    from paper_2507_17511_b200 import compressors as cx
    from paper_2507_17511_b200 import pipeline as pl

    if codec != "quant4bit" and scale_mode == "rank1":
        pytest.skip("reference codec: pinned to the reference goldens in test_gpu_parity.py")
    quant_path(path)
    n, c = shape
    spec = cx.CompressorSpec(cx.CompressorKind(codec), scale_mode=scale_mode)
    ocodec = O.Codec(TAGS[codec], scale_mode=scale_mode)
    xs = _inputs(n, c, f"{shape}|{codec}|{scale_mode}|{mode}")
    snd = pl.LayerState(mode, 1, torch.zeros(n, c, device="cuda"))
    rcv = pl.LayerState(mode, 1, torch.zeros(n, c, device="cuda"))
    och = O.Channel(mode, 1, np.zeros((n, c), np.float32))
    for t, x in enumerate(xs, start=1):
        p, rec = pl.encode_step(snd, torch.from_numpy(x).cuda(), spec)
        pl.decode_step(rcv, pl.device_message(t, 1, p))
        tag, body, orec = O.send(och, x, ocodec)
        assert p.tag == tag
        assert p.body_bytes() == body, f"body differs at step {t}"
        assert np.array_equal(snd.base.cpu().numpy(), och.base), f"base differs at step {t}"
        if mode == "residual_with_feedback":
            assert np.array_equal(snd.feedback.cpu().numpy(), och.fb), f"feedback differs at step {t}"
        assert torch.equal(rcv.base, snd.base)
        assert rec.compression_error == pytest.approx(orec["compression_error"], rel=1e-6, abs=1e-30)
        assert rec.bits == orec["bits"]


@pytest.mark.parametrize("codec", ["quant4bit", "quant2bit"])
@pytest.mark.parametrize("scale_mode", ["rank1", "per_token", "per_channel"])
def test_extension_codec_level_decode(codec, scale_mode):
    """Stateless compressors.encode / decode of the extensions (cx:459-481 shape)."""
    from paper_2507_17511_b200 import compressors as cx

    x = synth.flux_like(40, 384, 1, seed=5)[0]
    p = cx.encode(torch.from_numpy(x).cuda(), cx.CompressorSpec(cx.CompressorKind(codec), scale_mode=scale_mode))
    body = O.quant_body(x, TAGS[codec], scale_mode)
    assert p.body_bytes() == body
    dec = cx.decode(p)
    exp = O.decode_body(body, O.Codec(TAGS[codec]), 40, 384)
    assert np.array_equal(dec.cpu().numpy(), exp)


@pytest.mark.parametrize("scale_mode", ["per_token", "per_channel"])
@pytest.mark.parametrize("codec", ["sign1bit", "quant4bit"])
def test_segmented_extensions_vs_per_chunk_oracle(scale_mode, codec):
    """Ulysses segmented K1 with the extension codecs: every (src, dst) chunk channel
    matches its own oracle channel (SPEC.md:473 composition)."""
    from paper_2507_17511_b200 import compressors as cx
    from paper_2507_17511_b200.comm import UlyssesAllToAll

    P, n, C = 4, 48, 3072
    cw = C // P
    spec = cx.CompressorSpec(cx.CompressorKind(codec), scale_mode=scale_mode)
    ex = UlyssesAllToAll(n, C, spec, sim_world=(P, 0), in_dtype=torch.float32)
    assert ex.segmented
    chans = [O.Channel(O.WITH_FEEDBACK, 1, np.zeros((n, cw), np.float32)) for _ in range(P)]
    ocodec = O.Codec(TAGS[codec], scale_mode=scale_mode)
    for t, x in enumerate(_inputs(n, C, f"seg|{codec}|{scale_mode}"), start=1):
        out = ex.step(torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
        for d in range(P):
            _, body, _ = O.send(chans[d], x[:, d * cw:(d + 1) * cw], ocodec)
            if t > 1:
                assert ex.sendbuf[d, :len(body)].cpu().numpy().tobytes() == body, f"chunk {d} step {t}"
            assert np.array_equal(ex.senders[d].base.cpu().numpy(), chans[d].base)
        # sim_world loopback: slot d holds chunk d's body -> out rows [d n, (d+1) n) = chunk d's base
        for d in range(P):
            assert np.array_equal(out[d * n:(d + 1) * n].cpu().numpy(), chans[d].base)
