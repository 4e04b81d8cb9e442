"""GPU parity: the sm_100a path (through the C ABI, via the host mirror) against
the reference-generated golden fixtures and the CPU oracle, bit for bit on
codes / scales / bodies / base / feedback; StepRecord floats within rel 1e-6."""

import zlib

import numpy as np
import pytest
import torch

import synth
from golden_fixtures import codec_arrays, manifest, traj_arrays
from oracle import cc_oracle as O

pytestmark = pytest.mark.gpu

QUANT_CODECS = ("sign1bit", "quant2bit")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2507_17511_b200 import _lib

    _lib.load()
    torch.cuda.set_device(0)


def _mods():
    from paper_2507_17511_b200 import compressors as cx
    from paper_2507_17511_b200 import pipeline as pl

    return cx, pl


def _spec(name):
    cx, _ = _mods()
    return cx.CompressorSpec(cx.CompressorKind(name))


def _otag(name):
    return {"sign1bit": O.SIGN1, "quant2bit": O.QUANT2}[name]


# --------------------------------------------------------------------------
# codec level: golden bodies from the reference
# --------------------------------------------------------------------------

@pytest.mark.parametrize("case", [c for c in manifest()["codec_cases"] if c["codec"] in QUANT_CODECS],
                         ids=lambda c: f"{c['case']}|{c['codec']}")
def test_codec_body_vs_reference_golden(case):
    cx, _ = _mods()
    arr = codec_arrays()
    x = arr[f"x/{case['case']}"]
    p = cx.encode(torch.from_numpy(x).cuda(), _spec(case["codec"]))
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


@pytest.mark.parametrize("name", sorted({c["case"] for c in manifest()["codec_cases"]}))
def test_scale_estimate_vs_reference_golden(name):
    cx, _ = _mods()
    arr = codec_arrays()
    sp = cx.scale_estimate(torch.from_numpy(arr[f"x/{name}"]).cuda())
    assert sp.u.cpu().numpy().tobytes() == arr[f"u/{name}"].tobytes()
    assert sp.v.cpu().numpy().tobytes() == arr[f"v/{name}"].tobytes()


# --------------------------------------------------------------------------
# protocol level: golden trajectories (sender + receiver, all modes)
# --------------------------------------------------------------------------

def _run_traj_check(meta, bodies=None, in_dtype=torch.float32, bytes_msgs=False, offset=0):
    cx, pl = _mods()
    xs = synth.flux_like(meta["rows"], meta["cols"], meta["steps"], meta["seed"])
    assert synth.digest(np.stack(xs)) == meta["inputs_sha256"]
    n, c = meta["rows"], meta["cols"]
    zero = torch.zeros(n, c, device="cuda")
    snd = pl.LayerState(meta["mode"], meta["warmup"], zero)
    rcv = pl.LayerState(meta["mode"], meta["warmup"], zero)
    spec = _spec(meta["codec"])
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


@pytest.mark.parametrize("meta", manifest()["traj_small"], ids=lambda m: m["key"])
@pytest.mark.parametrize("variant", ["f32", "bf16", "bytes", "misaligned"])
def test_protocol_trajectory_vs_reference_golden(meta, variant):
    arr = traj_arrays()
    bodies = [arr[f"body/{meta['key']}/{i}"].tobytes() for i in range(meta["steps"])]
    snd = _run_traj_check(meta, bodies, in_dtype=torch.bfloat16 if variant == "bf16" else torch.float32,
                          bytes_msgs=(variant == "bytes"), offset=(1 if variant == "misaligned" else 0))
    assert np.array_equal(snd.base.cpu().numpy(), arr[f"base/{meta['key']}"])


@pytest.mark.parametrize("meta", manifest()["traj_digest"], ids=lambda m: m["key"])
def test_flux_width_trajectory_vs_reference_digests(meta):
    m = dict(meta)
    m["records"] = [dict(r, tag=(0 if i < meta["warmup"] else _otag(meta["codec"])))
                    for i, r in enumerate(meta["records"])]
    _run_traj_check(m, None, in_dtype=torch.bfloat16)


# --------------------------------------------------------------------------
# random shapes vs the oracle (vector path, scalar path, all modes, both dtypes)
# --------------------------------------------------------------------------

SHAPES = [(1, 8), (2, 2), (5, 24), (13, 136), (64, 384), (100, 1000), (3, 1025), (17, 3072), (31, 7), (129, 130)]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"{s[0]}x{s[1]}")
@pytest.mark.parametrize("codec", QUANT_CODECS)
@pytest.mark.parametrize("mode", ["naive", "residual_no_feedback", "residual_with_feedback"])
def test_random_trajectories_vs_oracle(shape, codec, mode):
    cx, pl = _mods()
    n, c = shape
    rng = np.random.default_rng(zlib.crc32(f"{n}x{c}|{codec}|{mode}".encode()))
    xs = synth.flux_like(n, c, 5, seed=int(rng.integers(1 << 30)))
    xs[2][rng.random((n, c)) < 0.2] = 0.0  # sprinkle exact zeros / sign-of-zero cases
    xs[3] = -xs[3]
    snd = pl.LayerState(mode, 1, torch.zeros(n, c, device="cuda"))
    och = O.Channel(mode, 1, np.zeros((n, c), np.float32))
    for i, x in enumerate(xs):
        p, rec = pl.encode_step(snd, torch.from_numpy(x).cuda(), _spec(codec))
        tag, body, orec = O.send(och, x, O.Codec(_otag(codec)))
        assert p.body_bytes() == body, f"step {i + 1}"
        assert np.array_equal(snd.base.cpu().numpy(), och.base)
        if mode == "residual_with_feedback":
            assert np.array_equal(snd.feedback.cpu().numpy(), och.fb)
        assert rec.compression_error == pytest.approx(orec["compression_error"], rel=1e-6, abs=1e-30)


@pytest.mark.parametrize("codec", QUANT_CODECS)
def test_edge_values_vs_oracle(codec):
    """zeros, -0.0, subnormals, huge values, zero rows / columns, constant input."""
    cx, _ = _mods()
    cases = [
        np.zeros((4, 16), np.float32),
        np.full((4, 16), 7.0, np.float32),
        np.array([[-0.0, 0.0, -1.0, 2.0] * 2, [0.0, -0.0, 0.0, 0.0] * 2], np.float32),
        np.array([[1e-38, -2e-39, 3e-45, 0.0] * 2, [1e-40, 0.0, -1e-44, 5e-45] * 2], np.float32),
        np.array([[1e30, -3e29, 7e4, 1.0] * 2, [-7.1e4, 6.6e4, 1.0, -2.0] * 2], np.float32),
    ]
    z = synth.gaussian(16, 64, 9)
    z[3] = 0.0
    z[:, 5] = 0.0
    cases.append(z)
    for x in cases:
        p = cx.encode(torch.from_numpy(x).cuda(), _spec(codec))
        assert p.body_bytes() == O.encode_body(x, O.Codec(_otag(codec)))
        assert np.array_equal(p.decode().cpu().numpy(), O.decode_body(p.body_bytes(), O.Codec(_otag(codec)), *x.shape))


# --------------------------------------------------------------------------
# full FLUX size: bit-exact vs oracle for a few steps, properties for 28
# --------------------------------------------------------------------------

def _flux_torch(rows, cols, steps, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.empty(rows, 1, device="cuda").log_normal_(0.0, 0.25, generator=g)
    c = torch.empty(1, cols, device="cuda").log_normal_(0.0, 1.0, generator=g)
    x = (a * c * torch.randn(rows, cols, device="cuda", generator=g)).to(torch.bfloat16)
    out = [x]
    for _ in range(1, steps):
        x = (x.float() + 0.1 * a * c * torch.randn(rows, cols, device="cuda", generator=g)).to(torch.bfloat16)
        out.append(x)
    return out


@pytest.mark.parametrize("codec", QUANT_CODECS)
def test_full_flux_shape_bit_exact_vs_oracle(codec):
    cx, pl = _mods()
    rows, cols = 4096, 3072
    xs = _flux_torch(rows, cols, 3, seed=77)
    snd = pl.LayerState("residual_with_feedback", 1, torch.zeros(rows, cols, device="cuda"))
    och = O.Channel(O.WITH_FEEDBACK, 1, np.zeros((rows, cols), np.float32))
    for x in xs:
        p, _ = pl.encode_step(snd, x, _spec(codec))
        _, body, _ = O.send(och, x.float().cpu().numpy(), O.Codec(_otag(codec)))
        assert p.body_bytes() == body
        assert np.array_equal(snd.base.cpu().numpy(), och.base)
        assert np.array_equal(snd.feedback.cpu().numpy(), och.fb)


@pytest.mark.parametrize("codec", QUANT_CODECS)
def test_full_flux_28_step_properties(codec):
    """Size-independent properties at BASELINE config 1 (28 steps, [4096,3072]):
    feedback conservation fb == t - decode(payload) exactly, sender == receiver
    bit-exact, payload length == ceil(bit_size/8), bounded reconstruction error."""
    cx, pl = _mods()
    rows, cols = 4096, 3072
    xs = _flux_torch(rows, cols, 28, seed=78)
    zero = torch.zeros(rows, cols, device="cuda")
    snd = pl.LayerState("residual_with_feedback", 1, zero)
    rcv = pl.LayerState("residual_with_feedback", 1, zero)
    for t, x in enumerate(xs, start=1):
        base0, fb0 = snd.base.clone(), snd.feedback.clone()
        p, rec = pl.encode_step(snd, x, _spec(codec))
        if t > 1:
            assert p.body.numel() == -(-p.bit_size // 8)
            target = (x.float() - base0) + fb0
            dec = p.decode()
            assert torch.equal(snd.feedback, target - dec)
            assert torch.equal(snd.base, base0 + dec)
            assert rec.delta_hat > 0.0
        pl.decode_step(rcv, pl.device_message(t, 1, p))
        assert torch.equal(rcv.base, snd.base)
        rel = (snd.base - x.float()).norm() / x.float().norm()
        assert rel < (0.5 if codec == "quant2bit" else 0.8)


# --------------------------------------------------------------------------
# ports of the reference's protocol tests (T/test_pipeline.py)
# --------------------------------------------------------------------------

def test_warmup_transmits_exactly():  # T/test_pipeline.py:22-30
    cx, pl = _mods()
    a = torch.from_numpy(synth.gaussian(4, 4, 1)).cuda()
    st = pl.LayerState("naive", 2, torch.zeros(4, 4, device="cuda"))
    p, rec = pl.encode_step(st, a, _spec("sign1bit"))
    assert p.tag == cx.TAG_RAW
    assert torch.equal(st.base, a)
    assert rec.compression_error == 0.0 and rec.delta_hat == 1.0


def test_step_counter_desync_and_corruption_leave_state_unchanged():  # :84-111
    cx, pl = _mods()
    xs = synth.flux_like(16, 16, 3, 3)
    snd = pl.LayerState("naive", 1, torch.zeros(16, 16, device="cuda"))
    rcv = pl.LayerState("naive", 1, torch.zeros(16, 16, device="cuda"))
    p1, _ = pl.encode_step(snd, xs[0], _spec("sign1bit"))
    m1 = pl.message_for(1, 1, p1)
    pl.decode_step(rcv, m1)
    p2, _ = pl.encode_step(snd, xs[1], _spec("sign1bit"))
    m2 = pl.message_for(2, 1, p2)
    with pytest.raises(pl.ProtocolError):
        pl.decode_step(rcv, m1)
    before = rcv.base.clone()
    with pytest.raises(pl.ProtocolError):
        pl.decode_step(rcv, pl.message_for(3, 1, p2))
    with pytest.raises(cx.PayloadError):
        pl.decode_step(rcv, m2[:-4])
    assert torch.equal(rcv.base, before) and rcv.step == 1
    pl.decode_step(rcv, m2)
    assert torch.equal(rcv.base, snd.base)


def test_feedback_mode_beats_naive():  # :128-133 (desk-scale, slowly varying stream)
    cx, pl = _mods()
    xs = synth.flux_like(64, 256, 20, 4, drift=0.05)
    errs = {}
    for mode in ("naive", "residual_with_feedback"):
        st = pl.LayerState(mode, 1, torch.zeros(64, 256, device="cuda"))
        e = []
        for x in xs:
            _, rec = pl.encode_step(st, x, _spec("sign1bit"))
            e.append(rec.compression_error)
        errs[mode] = np.mean(e[1:])
    assert errs["residual_with_feedback"] * 10.0 <= errs["naive"]


def test_constant_input_with_feedback_stays_exact():  # :72-81
    cx, pl = _mods()
    a = torch.from_numpy(synth.gaussian(6, 8, 5)).cuda()
    st = pl.LayerState("residual_with_feedback", 1, torch.zeros(6, 8, device="cuda"))
    errs = []
    for _ in range(11):
        pl.encode_step(st, a, _spec("sign1bit"))
        errs.append(float(((st.base - a).double() ** 2).sum()))
    assert errs[0] == 0.0
    for prev, cur in zip(errs, errs[1:]):
        assert cur <= prev + 1e-12


def test_payload_ratios():  # T/test_compressors.py:67-70, :90-93
    cx, _ = _mods()
    x = torch.from_numpy(synth.gaussian(32, 48, 0)).cuda()
    p = cx.encode_sign1bit(x)
    assert cx.payload_only_ratio(p) == 16.0 and p.bit_size == 32 * 48 + 32 * (32 + 48)
    q = cx.encode_quant2bit(x)
    assert cx.payload_only_ratio(q) == 8.0 and q.bit_size == 2 * 32 * 48 + 32 * (32 + 48)
    r = cx.encode_raw(x)
    assert cx.payload_only_ratio(r) == 1.0 and cx.overhead_ratio(r) == 1.0 and r.bit_size == 32 * 32 * 48


def test_quant_energy_bound_property():  # T/test_compressors.py:96-108 (1000 trials)
    cx, _ = _mods()
    rng = np.random.default_rng(77)
    wins = {"sign1bit": 0, "quant2bit": 0}
    for _ in range(1000):
        x = torch.from_numpy(rng.standard_normal((12, 12)).astype(np.float32)).cuda()
        for k in wins:
            if cx.empirical_delta(x, cx.encode(x, _spec(k))) > 0:
                wins[k] += 1
    assert all(v >= 990 for v in wins.values())


def test_kernels_really_launch():
    """Evidence counter: the CUDA library, not a host path, did the work."""
    from paper_2507_17511_b200 import _lib

    cx, pl = _mods()
    n0 = _lib.load().cc_launch_count()
    cx.encode_quant2bit(torch.randn(64, 256, device="cuda"))
    assert _lib.load().cc_launch_count() - n0 >= 1


# --------------------------------------------------------------------------
# the persistent fused K1 (C % 1024 == 0) against the multi-kernel K1 and the oracle
# --------------------------------------------------------------------------

@pytest.fixture
def quant_path():
    from paper_2507_17511_b200 import _lib

    lib = _lib.load()
    yield lib.cc_set_quant_path
    lib.cc_set_quant_path(-1)


@pytest.mark.parametrize("shape", [(1, 1024), (3, 2048), (64, 3072), (513, 3072), (2048, 3072), (7, 4096)],
                         ids=lambda s: f"{s[0]}x{s[1]}")
@pytest.mark.parametrize("codec", QUANT_CODECS + ("quant4bit",))
@pytest.mark.parametrize("mode", ["naive", "residual_no_feedback", "residual_with_feedback"])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32], ids=["bf16", "f32"])
def test_fused_k1_matches_multikernel_and_oracle(shape, codec, mode, dtype, quant_path):
    cx, pl = _mods()
    n, c = shape
    xs = _flux_torch(n, c, 4, seed=n * 7 + c)
    states = {}
    bodies = {}
    for path in (0, 1):
        quant_path(path)
        st = pl.LayerState(mode, 1, torch.zeros(n, c, device="cuda"))
        bl = []
        for x in xs:
            p, rec = pl.encode_step(st, x.to(dtype), _spec(codec))
            bl.append((p.body_bytes(), rec.compression_error))
        states[path] = st
        bodies[path] = bl
    for (b0, e0), (b1, e1) in zip(bodies[0], bodies[1]):
        assert b0 == b1
        assert e1 == pytest.approx(e0, rel=1e-6, abs=1e-30)
    assert torch.equal(states[0].base, states[1].base)
    if mode == "residual_with_feedback":
        assert torch.equal(states[0].feedback, states[1].feedback)
    if codec != "quant4bit" and n <= 513:
        och = O.Channel(mode, 1, np.zeros((n, c), np.float32))
        for x, (b1, _) in zip(xs, bodies[1]):
            _, body, _ = O.send(och, x.to(dtype).float().cpu().numpy(), O.Codec(_otag(codec)))
            assert b1 == body
        assert np.array_equal(states[1].base.cpu().numpy(), och.base)


@pytest.mark.parametrize("shape", [(5, 128), (40, 384), (300, 768), (9, 1536), (33, 2560)],
                         ids=lambda s: f"{s[0]}x{s[1]}")
@pytest.mark.parametrize("codec", QUANT_CODECS)
@pytest.mark.parametrize("mode", ["naive", "residual_with_feedback"])
def test_fused_k1_narrow_widths(shape, codec, mode, quant_path):
    """Row-group mapping of the persistent K1 (C < 3072, e.g. Ulysses chunks)."""
    cx, pl = _mods()
    n, c = shape
    xs = _flux_torch(n, c, 4, seed=n + 3 * c)
    res = {}
    for path in (0, 1):
        quant_path(path)
        st = pl.LayerState(mode, 1, torch.zeros(n, c, device="cuda"))
        res[path] = ([pl.encode_step(st, x, _spec(codec))[0].body_bytes() for x in xs], st.base.clone())
    assert res[0][0] == res[1][0]
    assert torch.equal(res[0][1], res[1][1])
    och = O.Channel(mode, 1, np.zeros((n, c), np.float32))
    for x, b in zip(xs, res[1][0]):
        assert O.send(och, x.float().cpu().numpy(), O.Codec(_otag(codec)))[1] == b


def test_pdl_launches_give_identical_results():
    """Programmatic dependent launch (cc_set_pdl) only changes launch scheduling:
    a K1 + K2 trajectory must be bit-identical with it on and off."""
    from paper_2507_17511_b200 import _lib

    cx, pl = _mods()
    lib = _lib.load()
    n, c = 96, 3072
    xs = synth.flux_like(n, c, 4, seed=23)
    outs = []
    try:
        for pdl in (0, 1):
            lib.cc_set_pdl(pdl)
            snd = pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda"))
            rcv = pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda"))
            bodies = []
            for t, x in enumerate(xs, start=1):
                payload, _ = pl.encode_step(snd, torch.from_numpy(x).cuda().to(torch.bfloat16), _spec("quant2bit"))
                pl.decode_step(rcv, pl.device_message(t, 1, payload))
                bodies.append(payload.body.clone())
            torch.cuda.synchronize()
            outs.append((bodies, snd.base.clone(), snd.feedback.clone(), rcv.base.clone()))
    finally:
        lib.cc_set_pdl(0)
    for a, b in zip(outs[0][0], outs[1][0]):
        assert torch.equal(a, b)
    for i in (1, 2, 3):
        assert torch.equal(outs[0][i], outs[1][i])
