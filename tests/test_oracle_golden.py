"""Pin the CPU oracle to the reference: oracle outputs must equal the golden
fixtures produced by running the reference itself (tests/golden/make_golden.py).
CPU only; also cross-checks against the live reference when /root/reference exists."""

import os
import sys

import numpy as np
import pytest

import synth
from golden_fixtures import codec_arrays, manifest, oracle_codec, traj_arrays, traj_nm_arrays
from oracle import cc_oracle as O

REF = "/root/reference/pkg/src"


def _rng17():
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(17)))


@pytest.mark.parametrize("case", manifest()["codec_cases"], ids=lambda c: f"{c['case']}|{c['codec']}")
def test_codec_body_matches_reference(case):
    arr = codec_arrays()
    x = arr[f"x/{case['case']}"]
    codec = oracle_codec(case["spec"])
    body = O.encode_body(x, codec, rng=_rng17())
    key = f"{case['case']}|{case['codec']}"
    assert len(body) == case["body_len"] == -(-case["bit_size"] // 8)
    assert body == arr[f"body/{key}"].tobytes()
    dec = O.decode_body(arr[f"body/{key}"].tobytes(), codec, case["rows"], case["cols"])
    assert synth.digest(dec) == case["dec_sha256"]
    n, c = case["rows"], case["cols"]
    kw = O._kw(codec, n, c, codec.tag)
    assert O.body_bits(codec.tag, n, c, **kw) == case["bit_size"]
    assert O.nominal_bits(codec.tag, n, c, **kw) == case["nominal_bits"]


@pytest.mark.parametrize("name", sorted({c["case"] for c in manifest()["codec_cases"]}))
def test_scale_estimate_matches_reference(name):
    arr = codec_arrays()
    u, v = O.rank1_scales(arr[f"x/{name}"])
    assert u.tobytes() == arr[f"u/{name}"].tobytes()
    assert v.tobytes() == arr[f"v/{name}"].tobytes()


def test_scale_kat_hand_values():
    u, v = O.rank1_scales(np.array([[1, -1], [2, -2]], np.float32))
    assert np.allclose(u, [2 / 3, 4 / 3], atol=1e-7) and np.allclose(v, [1.5, 1.5], atol=1e-7)


def _traj_inputs(meta):
    xs = synth.flux_like(meta["rows"], meta["cols"], meta["steps"], meta["seed"])
    assert synth.digest(np.stack(xs)) == meta["inputs_sha256"], "synthetic input generator drifted"
    return xs


@pytest.mark.parametrize("meta", manifest()["traj_small"], ids=lambda m: m["key"])
def test_protocol_trajectory_matches_reference(meta):
    arr = traj_arrays()
    xs = _traj_inputs(meta)
    codec = O.Codec(O.SIGN1 if meta["codec"] == "sign1bit" else O.QUANT2)
    n, c = meta["rows"], meta["cols"]
    snd = O.Channel(meta["mode"], meta["warmup"], np.zeros((n, c), np.float32))
    rcv = O.Channel(meta["mode"], meta["warmup"], np.zeros((n, c), np.float32))
    for i, x in enumerate(xs):
        tag, body, rec = O.send(snd, x, codec)
        exp = meta["records"][i]
        assert tag == exp["tag"]
        assert body == arr[f"body/{meta['key']}/{i}"].tobytes()
        assert synth.digest(snd.base) == exp["base_sha256"]
        assert synth.digest(snd.fb) == exp["fb_sha256"]
        assert rec["bits"] == exp["bits"]
        assert rec["compression_error"] == pytest.approx(exp["compression_error"], rel=1e-12, abs=1e-300)
        assert rec["delta_hat"] == pytest.approx(exp["delta_hat"], rel=1e-12)
        O.receive(rcv, i + 1, i + 1 <= meta["warmup"], tag, body, codec)
        assert np.array_equal(rcv.base, snd.base)
    assert np.array_equal(snd.base, arr[f"base/{meta['key']}"])
    assert np.array_equal(snd.fb, arr[f"fb/{meta['key']}"])


@pytest.mark.parametrize("meta", manifest()["traj_nm"], ids=lambda m: m["key"])
def test_nm_trajectory_matches_reference(meta):
    arr = traj_nm_arrays()
    xs = _traj_inputs(meta)
    codec = oracle_codec(meta["spec"])
    n, c = meta["rows"], meta["cols"]
    snd = O.Channel(meta["mode"], meta["warmup"], np.zeros((n, c), np.float32))
    rcv = O.Channel(meta["mode"], meta["warmup"], np.zeros((n, c), np.float32))
    for i, x in enumerate(xs):
        tag, body, rec = O.send(snd, x, codec)
        exp = meta["records"][i]
        assert tag == exp["tag"]
        assert body == arr[f"body/{meta['key']}/{i}"].tobytes()
        assert synth.digest(snd.base) == exp["base_sha256"]
        assert synth.digest(snd.fb) == exp["fb_sha256"]
        assert rec["bits"] == exp["bits"]
        assert rec["compression_error"] == pytest.approx(exp["compression_error"], rel=1e-12, abs=1e-300)
        O.receive(rcv, i + 1, i + 1 <= meta["warmup"], tag, body, codec)
        assert np.array_equal(rcv.base, snd.base)
    assert np.array_equal(snd.base, arr[f"base/{meta['key']}"])


@pytest.mark.parametrize("meta", manifest()["nm_digest"], ids=lambda m: m["key"])
def test_nm_flux_width_digests(meta):
    xs = _traj_inputs(meta)
    codec = oracle_codec(meta["spec"])
    snd = O.Channel(meta["mode"], meta["warmup"], np.zeros((meta["rows"], meta["cols"]), np.float32))
    for i, x in enumerate(xs):
        _, body, rec = O.send(snd, x, codec)
        assert synth.digest(body) == meta["body_sha256"][i]
        assert synth.digest(snd.base) == meta["base_sha256"][i]
        assert synth.digest(snd.fb) == meta["fb_sha256"][i]


@pytest.mark.parametrize("meta", manifest()["traj_digest"], ids=lambda m: m["key"])
def test_flux_width_trajectory_digests(meta):
    xs = _traj_inputs(meta)
    codec = O.Codec(O.SIGN1 if meta["codec"] == "sign1bit" else O.QUANT2)
    n, c = meta["rows"], meta["cols"]
    snd = O.Channel(meta["mode"], meta["warmup"], np.zeros((n, c), np.float32))
    for i, x in enumerate(xs):
        _, body, rec = O.send(snd, x, codec)
        assert synth.digest(body) == meta["body_sha256"][i]
        assert synth.digest(snd.base) == meta["base_sha256"][i]
        assert synth.digest(snd.fb) == meta["fb_sha256"][i]


@pytest.mark.parametrize("meta", manifest()["topk_digest"], ids=lambda m: str(m["keep_fraction"]))
def test_topk_digest(meta):
    x = synth.flux_like(meta["rows"], meta["cols"], 1, meta["seed"])[0]
    body = O.topk_body(x, meta["keep_fraction"])
    assert len(body) == 6 * meta["k"]
    assert synth.digest(body) == meta["body_sha256"]


@pytest.mark.parametrize("meta", [m for m in manifest()["lowrank"] if m["rows"] <= 64],
                         ids=lambda m: f"r{m['rank']}T{m['iterations']}{'i4' if m['int4'] else ''}")
def test_lowrank_reconstruction_error(meta):
    x = synth.flux_like(meta["rows"], meta["cols"], 1, meta["seed"])[0]
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(entropy=meta["seed"], spawn_key=(5, 2))))
    body = O.lowrank_body(x, meta["rank"], meta["iterations"], rng, int4=meta["int4"])
    assert len(body) == meta["body_len"]
    dec = O.lowrank_decode(body, meta["rows"], meta["cols"], meta["rank"], meta["int4"])
    err = np.sqrt(O.sqnorm(dec.astype(np.float64) - x) / O.sqnorm(x))
    assert err == pytest.approx(meta["rel_err"], rel=1e-9)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted (GPU box)")
def test_oracle_vs_live_reference_random():
    """Extra: fresh random shapes straight against the mounted reference."""
    sys.path.insert(0, REF)
    from compactcomm import compressors as cx
    from compactcomm import linalg

    rng = np.random.Generator(np.random.PCG64(1234))
    for trial in range(30):
        r, c = int(rng.integers(1, 70)), int(rng.integers(1, 300))
        x = (rng.standard_normal((r, c)) * rng.lognormal(0, 2)).astype(np.float32)
        if trial % 5 == 0:
            x[rng.random((r, c)) < 0.3] = 0.0
        xm = linalg.as_matrix(x)
        for tag, fn in ((O.SIGN1, cx.encode_sign1bit), (O.QUANT2, cx.encode_quant2bit)):
            ref = cx.to_bytes(fn(xm))[9:]
            assert O.encode_body(x, O.Codec(tag)) == ref
        f = float(rng.choice([0.01, 0.1, 0.5, 1.0]))
        assert O.topk_body(x, f) == cx.to_bytes(cx.encode_topk(xm, f))[13:]
