"""GPU parity of the N:M block sparsifier (K5, csrc/nm.cu) against the reference.

Anchors: golden bodies / decodes / trajectories produced by the reference itself
(tests/golden/make_golden.py: codec_cases "nm*", traj_nm, nm_digest) and the
oracle (oracle/cc_oracle.py nm_body / nm_decode, cx:429-443) on random shapes.
Bar: bit-exact bodies, base and feedback; records within rel 1e-6.
"""

import zlib

import numpy as np
import pytest
import torch

import synth
from golden_fixtures import codec_arrays, manifest, oracle_codec, traj_nm_arrays
from oracle import cc_oracle as O

pytestmark = pytest.mark.gpu

MODES = ["naive", "residual_no_feedback", "residual_with_feedback"]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)


def _mods():
    from paper_2507_17511_b200 import compressors as cx
    from paper_2507_17511_b200 import pipeline as pl

    return cx, pl


def _spec(n, m):
    cx, _ = _mods()
    return cx.CompressorSpec(cx.CompressorKind.NM_BLOCK, n=n, m=m)


@pytest.mark.parametrize("case", [c for c in manifest()["codec_cases"] if c["codec"].startswith("nm")],
                         ids=lambda c: f"{c['case']}|{c['codec']}")
def test_nm_body_vs_reference_golden(case):
    cx, _ = _mods()
    arr = codec_arrays()
    x = arr[f"x/{case['case']}"]
    s = case["spec"]
    p = cx.encode(torch.from_numpy(x).cuda(), _spec(s["n"], s["m"]))
    key = f"{case['case']}|{case['codec']}"
    assert p.bit_size == case["bit_size"]
    assert p.nominal_bits == case["nominal_bits"]
    assert p.payload_only_bits == case["payload_only_bits"]
    assert p.body_bytes() == arr[f"body/{key}"].tobytes()
    dec = p.decode().cpu().numpy()
    assert synth.digest(dec) == case["dec_sha256"]
    blob = cx.to_bytes(p)
    q = cx.from_bytes(blob)
    assert cx.to_bytes(q) == blob
    assert torch.equal(q.decode(), p.decode())


def _run_nm_traj(meta, bodies=None, in_dtype=torch.float32, bytes_msgs=False, offset=0):
    cx, pl = _mods()
    xs = synth.flux_like(meta["rows"], meta["cols"], meta["steps"], meta["seed"])
    assert synth.digest(np.stack(xs)) == meta["inputs_sha256"]
    n, c = meta["rows"], meta["cols"]
    snd = pl.LayerState(meta["mode"], meta["warmup"], torch.zeros(n, c, device="cuda"))
    rcv = pl.LayerState(meta["mode"], meta["warmup"], torch.zeros(n, c, device="cuda"))
    spec = _spec(meta["spec"]["n"], meta["spec"]["m"])
    for i, x in enumerate(xs):
        xd = torch.from_numpy(x).cuda().to(in_dtype)
        if offset:  # misaligned view -> scalar path
            big = torch.zeros(n * c + offset, device="cuda", dtype=in_dtype)
            big[offset:] = xd.reshape(-1)
            xd = big[offset:].view(n, c)
        payload, rec = pl.encode_step(snd, xd, spec)
        exp = meta["records"][i]
        assert payload.tag == exp["tag"]
        body = payload.body_bytes()
        if bodies is not None:
            assert body == bodies[i], f"step {i + 1}: body differs from reference"
        else:
            assert synth.digest(body) == meta["body_sha256"][i]
        assert synth.digest(snd.base.cpu().numpy()) == (exp.get("base_sha256") or meta["base_sha256"][i])
        if meta["mode"] == "residual_with_feedback":
            assert synth.digest(snd.feedback.cpu().numpy()) == (exp.get("fb_sha256") or meta["fb_sha256"][i])
        assert rec.bits == exp["bits"]
        assert rec.compression_error == pytest.approx(exp["compression_error"], rel=1e-6, abs=1e-30)
        assert rec.delta_hat == pytest.approx(exp["delta_hat"], rel=1e-6, abs=1e-9)
        msg = pl.message_for(i + 1, meta["warmup"], payload) if bytes_msgs else \
            pl.device_message(i + 1, meta["warmup"], payload)
        pl.decode_step(rcv, msg)
        assert torch.equal(rcv.base, snd.base)
    return snd


@pytest.mark.parametrize("meta", manifest()["traj_nm"], ids=lambda m: m["key"])
@pytest.mark.parametrize("variant", ["f32", "bf16", "bytes", "misaligned"])
def test_nm_trajectory_vs_reference_golden(meta, variant):
    arr = traj_nm_arrays()
    bodies = [arr[f"body/{meta['key']}/{i}"].tobytes() for i in range(meta["steps"])]
    snd = _run_nm_traj(meta, bodies, in_dtype=torch.bfloat16 if variant == "bf16" else torch.float32,
                       bytes_msgs=(variant == "bytes"), offset=(1 if variant == "misaligned" else 0))
    assert np.array_equal(snd.base.cpu().numpy(), arr[f"base/{meta['key']}"])


@pytest.mark.parametrize("meta", manifest()["nm_digest"], ids=lambda m: m["key"])
def test_nm_flux_width_vs_reference_digests(meta):
    _run_nm_traj(meta, None, in_dtype=torch.bfloat16)


NM_CASES = [(1, 2), (2, 4), (1, 4), (3, 4), (4, 8), (2, 8), (8, 16), (4, 16), (16, 32), (1, 32), (3, 5), (2, 3),
            (7, 40), (10, 64), (1, 1)]
SHAPES = [(1, 8), (5, 24), (13, 136), (64, 384), (3, 1025), (17, 3072), (31, 7), (129, 130)]


@pytest.mark.parametrize("nm", NM_CASES, ids=lambda v: f"{v[0]}:{v[1]}")
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"{s[0]}x{s[1]}")
def test_nm_stateless_vs_oracle(nm, shape):
    cx, _ = _mods()
    n, m = nm
    rows, cols = shape
    rng = np.random.default_rng(zlib.crc32(f"{rows}x{cols}|{n}:{m}".encode()))
    x = synth.flux_like(rows, cols, 1, seed=int(rng.integers(1 << 30)))[0]
    x[rng.random((rows, cols)) < 0.15] = 0.0
    x[rng.random((rows, cols)) < 0.05] = -0.0
    x[rng.random((rows, cols)) < 0.1] = 1.5  # exact magnitude ties
    dec = torch.empty(rows, cols, device="cuda")
    p = cx.encode_nm_block(torch.from_numpy(x).cuda(), n, m, decoded=dec)
    body = O.nm_body(x, n, m)
    assert p.body_bytes() == body
    ref = O.nm_decode(body, rows, cols, n, m)
    assert np.array_equal(p.decode().cpu().numpy(), ref)
    assert np.array_equal(dec.cpu().numpy(), ref)


@pytest.mark.parametrize("nm", [(2, 4), (4, 16), (3, 5), (7, 40)], ids=lambda v: f"{v[0]}:{v[1]}")
@pytest.mark.parametrize("shape", [(13, 136), (3, 1025), (64, 384)], ids=lambda s: f"{s[0]}x{s[1]}")
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_nm_random_trajectories_vs_oracle(nm, shape, mode, dtype):
    cx, pl = _mods()
    n, m = nm
    rows, cols = shape
    rng = np.random.default_rng(zlib.crc32(f"{rows}x{cols}|{n}:{m}|{mode}|{dtype}".encode()))
    xs = synth.flux_like(rows, cols, 5, seed=int(rng.integers(1 << 30)))
    xs[2][rng.random((rows, cols)) < 0.2] = 0.0
    xs[3] = -xs[3]
    if dtype == "bf16":
        xs = [synth.bf16_round(x) for x in xs]
    snd = pl.LayerState(mode, 1, torch.zeros(rows, cols, device="cuda"))
    rcv = pl.LayerState(mode, 1, torch.zeros(rows, cols, device="cuda"))
    och = O.Channel(mode, 1, np.zeros((rows, cols), np.float32))
    td = torch.bfloat16 if dtype == "bf16" else torch.float32
    for i, x in enumerate(xs):
        p, rec = pl.encode_step(snd, torch.from_numpy(x).cuda().to(td), _spec(n, m))
        tag, body, orec = O.send(och, x, O.Codec(O.NMBLOCK, nm=(n, m)))
        assert p.body_bytes() == body, f"step {i + 1}"
        assert np.array_equal(snd.base.cpu().numpy(), och.base)
        if mode == "residual_with_feedback":
            assert np.array_equal(snd.feedback.cpu().numpy(), och.fb)
        if mode == "residual_no_feedback":
            assert np.array_equal(snd.ref.cpu().numpy(), och.ref)
        assert rec.compression_error == pytest.approx(orec["compression_error"], rel=1e-6, abs=1e-30)
        pl.decode_step(rcv, pl.device_message(i + 1, 1, p))
        assert torch.equal(rcv.base, snd.base)


@pytest.mark.parametrize("nm", [(2, 4), (3, 5), (8, 16)], ids=lambda v: f"{v[0]}:{v[1]}")
def test_nm_edge_values_vs_oracle(nm):
    cx, _ = _mods()
    n, m = nm
    cases = [
        np.zeros((4, 16), np.float32),
        np.full((4, 16), 7.0, np.float32),
        np.array([[-0.0, 0.0, -1.0, 2.0] * 4, [0.0, -0.0, 0.0, 0.0] * 4], np.float32),
        np.array([[1e-38, -2e-39, 3e-45, 0.0] * 4, [1e-40, 0.0, -1e-44, 5e-45] * 4], np.float32),
        np.array([[1e30, -3e29, 7e4, 1.0] * 4, [-7.1e4, 6.6e4, 1.0, -2.0] * 4], np.float32),  # f16 overflow -> inf
    ]
    for x in cases:
        p = cx.encode(torch.from_numpy(x).cuda(), _spec(n, m))
        assert p.body_bytes() == O.nm_body(x, n, m)
        assert np.array_equal(p.decode().cpu().numpy(), O.nm_decode(p.body_bytes(), *x.shape, n, m))


@pytest.mark.parametrize("nm", [(2, 4), (3, 5)], ids=lambda v: f"{v[0]}:{v[1]}")
def test_nm_batched_decode_ragged_peers(nm):
    """One K2 launch over peers with different shard heights (mesh:125-135)."""
    import ctypes

    from paper_2507_17511_b200 import _lib

    cx, _ = _mods()
    n, m = nm
    cols = 130
    rows = [7, 7, 9]
    xs = [synth.flux_like(r, cols, 1, seed=50 + i)[0] for i, r in enumerate(rows)]
    ps = [cx.encode_nm_block(torch.from_numpy(x).cuda(), n, m) for x in xs]
    bases = [torch.from_numpy(synth.gaussian(r, cols, 60 + i)).cuda() for i, r in enumerate(rows)]
    expect = [b.cpu().numpy() + O.nm_decode(O.nm_body(x, n, m), r, cols, n, m)
              for b, x, r in zip(bases, xs, rows)]
    lib = _lib.load()
    k = len(rows)
    _lib.check(lib.cc_decode_batched(_lib.CC_NMBLOCK, 1, k, (ctypes.c_int64 * k)(*rows), cols, _lib.nm_param(n, m),
                                     (ctypes.c_void_p * k)(*[p.body.data_ptr() for p in ps]), _lib.CC_F32,
                                     (ctypes.c_void_p * k)(*[b.data_ptr() for b in bases]), _lib.stream_ptr()))
    for b, e in zip(bases, expect):
        assert np.array_equal(b.cpu().numpy(), e)


def test_nm_from_bytes_validation():  # cx:658-674
    cx, _ = _mods()
    x = synth.gaussian(6, 10, 3)
    blob = cx.to_bytes(cx.encode(torch.from_numpy(x).cuda(), _spec(2, 4)))
    with pytest.raises(cx.PayloadError):
        cx.from_bytes(blob[:-1])  # truncated values
    with pytest.raises(cx.PayloadError):
        cx.from_bytes(blob[:11])  # missing meta
    bad = bytearray(blob)
    bad[9:13] = (5).to_bytes(2, "little") + (4).to_bytes(2, "little")  # n > m
    with pytest.raises(cx.PayloadError):
        cx.from_bytes(bytes(bad))
    bad = bytearray(blob)
    bad[13] ^= 0x01  # flip one mask bit -> popcount mismatch
    with pytest.raises(cx.PayloadError):
        cx.from_bytes(bytes(bad))
    # total popcount preserved but uneven per block: block 0 keeps 3, block 1 keeps 1
    bad = bytearray(blob)
    masks = np.unpackbits(np.frombuffer(bytes(bad[13:14]), np.uint8), bitorder="little")
    b0, b1 = masks[:4].copy(), masks[4:8].copy()
    b0[np.flatnonzero(b0 == 0)[0]] = 1
    b1[np.flatnonzero(b1 == 1)[0]] = 0
    bad[13] = int(np.packbits(np.concatenate([b0, b1]), bitorder="little")[0])
    with pytest.raises(cx.PayloadError):
        cx.from_bytes(bytes(bad))


def test_nm_exchange_loopback():
    """PatchParallelExchange (world 1) carries N:M bodies end to end."""
    from paper_2507_17511_b200 import comm

    cx, pl = _mods()
    rows, cols = 64, 384
    ex = comm.PatchParallelExchange(rows, cols, _spec(2, 4), in_dtype=torch.float32)
    och = O.Channel("residual_with_feedback", 1, np.zeros((rows, cols), np.float32))
    for t, x in enumerate(synth.flux_like(rows, cols, 4, seed=77), start=1):
        full = ex.step(torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
        O.send(och, x, O.Codec(O.NMBLOCK, nm=(2, 4)))
        assert np.array_equal(full.cpu().numpy(), och.base)
