"""GPU parity of the top-k sparsifier (K4) against the reference goldens and the oracle."""

import zlib

import numpy as np
import pytest
import torch

import synth
from golden_fixtures import codec_arrays, manifest
from oracle import cc_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)


def _mods():
    from paper_2507_17511_b200 import compressors as cx
    from paper_2507_17511_b200 import pipeline as pl

    return cx, pl


@pytest.mark.parametrize("case", [c for c in manifest()["codec_cases"] if c["codec"].startswith("topk")],
                         ids=lambda c: f"{c['case']}|{c['codec']}")
def test_topk_body_vs_reference_golden(case):
    cx, _ = _mods()
    arr = codec_arrays()
    x = arr[f"x/{case['case']}"]
    p = cx.encode(torch.from_numpy(x).cuda(), cx.CompressorSpec(cx.CompressorKind.TOPK,
                                                                 keep_fraction=case["spec"]["keep_fraction"]))
    assert p.bit_size == case["bit_size"] and p.nominal_bits == case["nominal_bits"]
    assert p.body_bytes() == arr[f"body/{case['case']}|{case['codec']}"].tobytes()
    assert synth.digest(p.decode().cpu().numpy()) == case["dec_sha256"]
    blob = cx.to_bytes(p)
    assert cx.to_bytes(cx.from_bytes(blob)) == blob


@pytest.mark.parametrize("meta", manifest()["topk_digest"], ids=lambda m: str(m["keep_fraction"]))
def test_topk_flux_width_digest(meta):
    cx, _ = _mods()
    x = synth.flux_like(meta["rows"], meta["cols"], 1, meta["seed"])[0]
    p = cx.encode_topk(torch.from_numpy(x).cuda(), meta["keep_fraction"])
    assert p.k == meta["k"]
    assert synth.digest(p.body_bytes()) == meta["body_sha256"]


@pytest.mark.parametrize("shape", [(1, 1), (2, 3), (16, 16), (37, 101), (128, 384), (512, 3072), (1000, 999)])
@pytest.mark.parametrize("frac", [0.001, 0.01, 0.1, 0.5, 1.0])
@pytest.mark.parametrize("kind", ["gauss", "ties", "zeros"])
def test_topk_random_vs_oracle(shape, frac, kind):
    cx, _ = _mods()
    n, c = shape
    rng = np.random.default_rng(zlib.crc32(f"{n}x{c}{frac}{kind}".encode()))
    x = rng.standard_normal((n, c)).astype(np.float32)
    if kind == "ties":  # few distinct magnitudes -> massive ties at the threshold
        x = (np.round(x * 2) / 2).astype(np.float32)
    if kind == "zeros":
        x[rng.random((n, c)) < 0.9] = 0.0
        x[rng.random((n, c)) < 0.05] = -0.0
    p = cx.encode_topk(torch.from_numpy(x).cuda(), frac)
    assert p.body_bytes() == O.topk_body(x, frac)
    assert np.array_equal(p.decode().cpu().numpy(), O.topk_decode(p.body_bytes(), n, c))


@pytest.mark.parametrize("mode", ["naive", "residual_no_feedback", "residual_with_feedback"])
@pytest.mark.parametrize("frac", [0.01, 0.1])
@pytest.mark.parametrize("shape", [(64, 384), (512, 3072)])
def test_topk_protocol_vs_oracle(mode, frac, shape):
    cx, pl = _mods()
    n, c = shape
    xs = synth.flux_like(n, c, 5, seed=n + c)
    xs[1][0, :7] = -0.0  # exercise the dense `base + 0.0` semantics
    spec = cx.CompressorSpec(cx.CompressorKind.TOPK, keep_fraction=frac)
    snd = pl.LayerState(mode, 1, torch.zeros(n, c, device="cuda"))
    rcv = pl.LayerState(mode, 1, torch.zeros(n, c, device="cuda"))
    och = O.Channel(mode, 1, np.zeros((n, c), np.float32))
    for i, x in enumerate(xs):
        p, rec = pl.encode_step(snd, torch.from_numpy(x).cuda(), spec)
        tag, body, orec = O.send(och, x, O.Codec(O.TOPK, keep_fraction=frac))
        assert p.body_bytes() == body, f"step {i + 1}"
        assert snd.base.cpu().numpy().tobytes() == och.base.tobytes()
        if mode == "residual_with_feedback":
            assert snd.feedback.cpu().numpy().tobytes() == och.fb.tobytes()
        assert rec.compression_error == pytest.approx(orec["compression_error"], rel=1e-6, abs=1e-30)
        msg = pl.message_for(i + 1, 1, p) if i % 2 else pl.device_message(i + 1, 1, p)
        pl.decode_step(rcv, msg)
        assert rcv.base.cpu().numpy().tobytes() == snd.base.cpu().numpy().tobytes()


def test_topk_hand_example():  # T/test_compressors.py:231-233
    cx, _ = _mods()
    p = cx.encode_topk(torch.tensor([[3.0, 1.0], [-4.0, 0.0]], device="cuda"), 0.5)
    assert torch.equal(p.decode().cpu(), torch.tensor([[3.0, 0.0], [-4.0, 0.0]]))


def test_topk_delta_exceeds_fraction():  # T/test_compressors.py:236-240
    cx, _ = _mods()
    rng = np.random.default_rng(15)
    for frac in (0.1, 0.25, 0.5):
        x = torch.from_numpy(rng.standard_normal((32, 32)).astype(np.float32)).cuda()
        assert cx.empirical_delta(x, cx.encode_topk(x, frac)) >= frac
