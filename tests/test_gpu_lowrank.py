"""GPU parity of the low-rank compressor (K3).

The reference accumulates its projections in f64 BLAS (la:49-58) and orthogonalizes
with CGS2 (la:77-112); the device path accumulates in f64 in a different order and
orthogonalizes with CholQR2, so parity is stated as a tolerance on the
reconstruction error: |relerr_device - relerr_reference| <= 1e-4,
plus the reference's own property tests (T/test_compressors.py:114-177)."""

import numpy as np
import pytest
import torch

import synth
from golden_fixtures import codec_arrays, manifest
from oracle import cc_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)


def _mods():
    from paper_2507_17511_b200 import compressors as cx
    from paper_2507_17511_b200 import linalg
    from paper_2507_17511_b200 import pipeline as pl

    return cx, pl, linalg


def _spec(rank, iters=2, int4=False):
    cx, _, _ = _mods()
    return cx.CompressorSpec(cx.CompressorKind.LOWRANK, rank=rank, iterations=iters, int4_factors=int4)


def _relerr(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.sqrt(((a - b) ** 2).sum() / (b ** 2).sum()))


@pytest.mark.parametrize("meta", manifest()["lowrank"],
                         ids=lambda m: f"{m['rows']}x{m['cols']}-r{m['rank']}T{m['iterations']}{'i4' if m['int4'] else ''}")
def test_lowrank_error_vs_reference(meta):
    cx, _, linalg = _mods()
    x = synth.flux_like(meta["rows"], meta["cols"], 1, meta["seed"])[0]
    rng = linalg.spawn_rng(meta["seed"], 5, 2)  # same stream as the golden run -> same Q0 draw
    p = cx.encode_lowrank(torch.from_numpy(x).cuda(), _spec(meta["rank"], meta["iterations"], meta["int4"]), rng)
    assert p.body.numel() == meta["body_len"] and p.bit_size == meta["bit_size"]
    err = _relerr(p.decode().cpu().numpy(), x)
    assert abs(err - meta["rel_err"]) <= TOL, (err, meta["rel_err"])


@pytest.mark.parametrize("case", [c for c in manifest()["codec_cases"] if c["codec"].startswith("lowrank")],
                         ids=lambda c: f"{c['case']}|{c['codec']}")
def test_lowrank_codec_cases_vs_reference(case):
    cx, _, linalg = _mods()
    arr = codec_arrays()
    x = arr[f"x/{case['case']}"]
    s = case["spec"]
    p = cx.encode(torch.from_numpy(x).cuda(), _spec(s["rank"], s["iterations"], s["int4_factors"]),
                  rng=linalg.make_rng(17))
    assert p.bit_size == case["bit_size"] and p.body.numel() == case["body_len"]
    key = f"{case['case']}|{case['codec']}"
    ref_dec = O.decode_body(arr[f"body/{key}"].tobytes(),
                            O.Codec(O.LOWRANK4 if s["int4_factors"] else O.LOWRANK, rank=s["rank"]),
                            case["rows"], case["cols"])
    if np.sum(x.astype(np.float64) ** 2) == 0:
        assert np.allclose(p.decode().cpu().numpy(), 0.0)
        return
    e_dev = _relerr(p.decode().cpu().numpy(), x)
    e_ref = _relerr(ref_dec, x)
    assert abs(e_dev - e_ref) <= 5e-3 * max(1.0, e_ref), (e_dev, e_ref)
    blob = cx.to_bytes(p)
    assert cx.to_bytes(cx.from_bytes(blob)) == blob


def test_exact_rank_recovery():  # T/test_compressors.py:114-120
    cx, _, linalg = _mods()
    rng = np.random.default_rng(3)
    a = (rng.standard_normal((40, 6)) @ rng.standard_normal((6, 32))).astype(np.float32)
    p = cx.encode_lowrank(torch.from_numpy(a).cuda(), _spec(6), linalg.make_rng(3))
    # f16 factors bound the reconstruction at ~1e-3 relative
    assert _relerr(p.decode().cpu().numpy(), a) < 2e-3


def test_near_optimal_vs_svd():  # :123-131 (<= 1.10x the optimal rank-r error)
    cx, _, linalg = _mods()
    rng = np.random.default_rng(5)
    for r in (4, 8, 16):
        a = rng.standard_normal((64, 64)).astype(np.float32)
        p = cx.encode_lowrank(torch.from_numpy(a).cuda(), _spec(r), linalg.make_rng(r))
        err = np.sqrt(((p.decode().cpu().numpy().astype(np.float64) - a) ** 2).sum())
        s = np.linalg.svd(a.astype(np.float64), compute_uv=False)
        optimal = np.sqrt((s[r:] ** 2).sum())
        assert err <= 1.10 * optimal


def test_error_non_increasing_in_iterations():  # :134-141
    cx, _, linalg = _mods()
    a = torch.from_numpy(np.random.default_rng(8).standard_normal((64, 64)).astype(np.float32)).cuda()

    def err(t):
        p = cx.encode_lowrank(a, _spec(8, t), linalg.make_rng(99))
        return float(((p.decode().double() - a.double()) ** 2).sum().sqrt())

    assert err(10) <= err(2) * 1.01


def test_rank_deficient_input_uses_replacement():  # :144-149
    cx, _, linalg = _mods()
    rng = np.random.default_rng(13)
    a = (rng.standard_normal((24, 2)) @ rng.standard_normal((2, 24))).astype(np.float32)
    p = cx.encode_lowrank(torch.from_numpy(a).cuda(), _spec(5), linalg.make_rng(13))
    assert _relerr(p.decode().cpu().numpy(), a) < 2e-3


def test_rank1_near_exact():  # :152-158
    cx, _, linalg = _mods()
    a = np.outer([1.0, 2.0, 3.0], [4.0, 5.0, 6.0, 7.0]).astype(np.float32)
    p = cx.encode_lowrank(torch.from_numpy(a).cuda(), _spec(1), linalg.make_rng(2))
    assert _relerr(p.decode().cpu().numpy(), a) < 5e-3


def test_bit_budget_and_int4_beats_rank8():  # :161-177
    cx, _, linalg = _mods()
    rng = np.random.default_rng(4)
    a = torch.from_numpy(rng.standard_normal((64, 96)).astype(np.float32)).cuda()
    p32 = cx.encode_lowrank(a, _spec(32, 2, True), linalg.make_rng(4))
    p8 = cx.encode_lowrank(a, _spec(8), linalg.make_rng(4))
    assert p32.payload_only_bits == p8.payload_only_bits == 128 * (64 + 96)
    assert p32.bit_size == 4 * 32 * (64 + 96) + 32 * 2 * 32 and p8.bit_size == 16 * 8 * (64 + 96)
    b = torch.from_numpy(np.random.default_rng(6).standard_normal((128, 512)).astype(np.float32)).cuda()
    e32 = _relerr(cx.encode_lowrank(b, _spec(32, 2, True), linalg.make_rng(7)).decode().cpu().numpy(), b.cpu().numpy())
    e8 = _relerr(cx.encode_lowrank(b, _spec(8), linalg.make_rng(7)).decode().cpu().numpy(), b.cpu().numpy())
    assert e32 < e8


@pytest.mark.parametrize("int4", [False, True])
def test_lowrank_protocol_sender_receiver_identical(int4):
    cx, pl, linalg = _mods()
    xs = synth.flux_like(128, 384, 5, seed=11)
    spec = _spec(8, 2, int4)
    snd = pl.LayerState("residual_with_feedback", 1, torch.zeros(128, 384, device="cuda"))
    rcv = pl.LayerState("residual_with_feedback", 1, torch.zeros(128, 384, device="cuda"))
    och = O.Channel(O.WITH_FEEDBACK, 1, np.zeros((128, 384), np.float32))
    for t, x in enumerate(xs, start=1):
        base0, fb0 = snd.base.clone(), snd.feedback.clone()
        p, rec = pl.encode_step(snd, x, spec, rng=linalg.spawn_rng(11, 5, t))
        if t > 1:
            dec = p.decode()
            target = (torch.from_numpy(x).cuda() - base0) + fb0
            assert torch.equal(snd.feedback, target - dec)  # feedback conservation, bit-exact
            assert torch.equal(snd.base, base0 + dec)
        msg = pl.message_for(t, 1, p) if t % 2 else pl.device_message(t, 1, p)
        pl.decode_step(rcv, msg)
        assert torch.equal(rcv.base, snd.base)
        O.send(och, x, O.Codec(O.LOWRANK4 if int4 else O.LOWRANK, rank=8, iters=2),
               rng=linalg.spawn_rng(11, 5, t))
    # trajectory-level agreement with the reference algorithm (tolerance)
    assert _relerr(snd.base.cpu().numpy(), och.base) < 2e-2


@pytest.mark.parametrize("shape", [(64, 384), (200, 1000), (1024, 3072), (4096, 3072)], ids=lambda s: f"{s[0]}x{s[1]}")
@pytest.mark.parametrize("r", [4, 8, 16, 32])
def test_tcgen05_backend_matches_f64_backend(shape, r):
    """The tcgen05 3xTF32 projections vs the f64 CUDA-core projections: same
    subspace, reconstruction errors equal to ~1e-6 relative."""
    from paper_2507_17511_b200 import _lib

    cx, _, linalg = _mods()
    n, c = shape
    x = torch.from_numpy(synth.flux_like(n, c, 1, seed=n + r)[0]).cuda()
    lib = _lib.load()
    errs = {}
    try:
        for backend in (0, 1):
            lib.cc_set_lowrank_backend(backend)
            p = cx.encode_lowrank(x, _spec(r), linalg.make_rng(r))
            errs[backend] = _relerr(p.decode().cpu().numpy(), x.cpu().numpy())
    finally:
        lib.cc_set_lowrank_backend(1)
    assert abs(errs[0] - errs[1]) <= 1e-5 * max(1.0, errs[0]), errs


@pytest.mark.parametrize("shape", [(1024, 3072), (4096, 3072), (64, 384)], ids=lambda s: f"{s[0]}x{s[1]}")
@pytest.mark.parametrize("r", [4, 16, 32])
def test_tma_staged_projections_equal_register_staged(shape, r):
    """The TMA-staged tcgen05 projection kernel (2-D tensor map, 4-deep raw ring) and
    the register-staged one use the same split-K plan: identical payload bytes."""
    from paper_2507_17511_b200 import _lib

    cx, _, linalg = _mods()
    n, c = shape
    x = torch.from_numpy(synth.flux_like(n, c, 1, seed=n + 7 * r)[0]).cuda()
    lib = _lib.load()
    bodies = []
    try:
        for tma in (0, 1, 1, 2):
            lib.cc_debug_lowrank_tma(tma, 0)
            bodies.append(cx.encode_lowrank(x, _spec(r), linalg.make_rng(r)).body.cpu())
    finally:
        lib.cc_debug_lowrank_tma(2, 0)
    assert all(torch.equal(bodies[0], b) for b in bodies[1:])


@pytest.mark.parametrize("mode", ["residual_with_feedback", "residual_no_feedback", "naive"])
@pytest.mark.parametrize("int4", [False, True])
def test_fused_step_device_key_equals_host_rng(mode, int4):
    """cc_lowrank_encode_step with the start block drawn on the device (DeviceKey,
    advancing step word) is bit-identical to the same step with the host draw from
    spawn_rng(seed, 5, t) (pl:190), and the receiver mirrors the sender."""
    cx, pl, linalg = _mods()
    n, c = 256, 3072
    xs = synth.flux_like(n, c, 5, seed=21)
    spec = _spec(8, 2, int4)
    a = pl.LayerState(mode, 1, torch.zeros(n, c, device="cuda"))
    b = pl.LayerState(mode, 1, torch.zeros(n, c, device="cuda"))
    rcv = pl.LayerState(mode, 1, torch.zeros(n, c, device="cuda"))
    key = linalg.DeviceKey(9, 5, 2, advance=True)  # the first compressed step is t = 2
    for t, x in enumerate(xs, start=1):
        xd = torch.from_numpy(x).cuda().to(torch.bfloat16)
        pa, ra = pl.encode_step(a, xd, spec, rng=linalg.spawn_rng(9, 5, t))
        pb, rb = pl.encode_step(b, xd, spec, rng=key)
        assert pa.body_bytes() == pb.body_bytes(), f"step {t}"
        assert torch.equal(a.base, b.base) and torch.equal(a.feedback, b.feedback)
        assert ra.compression_error == rb.compression_error
        pl.decode_step(rcv, pl.device_message(t, 1, pb))
        assert torch.equal(rcv.base, b.base)


def test_lowrank_exchange_graph_replay_equals_eager():
    """The low-rank patch-parallel step (sim_world P=4, rank 0) captured in ONE CUDA graph
    with an advancing device key (start blocks drawn one step ahead on a side stream) and
    replayed three times: every replay equals the matching eager step bit for bit (the
    key advances on the device, the drawn-ahead block is handed over in stream order)."""
    cx, pl, linalg = _mods()
    from paper_2507_17511_b200.comm import PatchParallelExchange

    rows, cols, P = 1024, 3072, 4
    spec = _spec(8, 2)
    xs = [torch.from_numpy(x).cuda().to(torch.bfloat16)[: rows // P].contiguous()
          for x in synth.flux_like(rows, cols, 4, seed=5)]
    ea = PatchParallelExchange(rows, cols, spec, sim_world=(P, 0))
    eb = PatchParallelExchange(rows, cols, spec, sim_world=(P, 0))
    ka = linalg.DeviceKey(3, 6, 0, 2, advance=True)
    kb = linalg.DeviceKey(3, 6, 0, 2, advance=True)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for e, k in ((ea, ka), (eb, kb)):
            for i in range(3):
                e.step(xs[i], rng=k)
        ref = []
        for _ in range(3):  # eager: steps 4, 5, 6 on the same input
            ea.step(xs[3], rng=ka)
            ref.append(ea.reconstruction().clone())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            eb.step(xs[3], rng=kb)
            s.wait_stream(eb.streams.decode)
        eb.after_capture()
        got = []
        for _ in range(3):
            g.replay()
            s.synchronize()
            got.append(eb.reconstruction().clone())
    torch.cuda.synchronize()
    for i in range(3):
        assert torch.equal(got[i], ref[i]), f"replay {i + 1}"


@pytest.mark.parametrize("shape", [(256, 3072), (1024, 3072), (4096, 3072), (100, 999)], ids=lambda s: f"{s[0]}x{s[1]}")
@pytest.mark.parametrize("r", [4, 8, 16])
def test_orth_forms_agree(shape, r):
    """The cluster CholQR2 (default) and the single-CTA / grid forms give the same
    subspace: reconstruction errors agree to 1e-6 relative and both stay within the
    reference tolerance of each other (different f64 summation orders only)."""
    cx, _, linalg = _mods()
    from paper_2507_17511_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(r + shape[0])
    a = torch.from_numpy((rng.standard_normal(shape) * rng.random((1, shape[1])) * 2).astype(np.float32)).cuda()
    errs = []
    for cl in (1, 0):
        lib.cc_debug_orth_cluster(cl)
        try:
            p = cx.encode_lowrank(a, _spec(r, 2), linalg.spawn_rng(4, 5, 2))
        finally:
            lib.cc_debug_orth_cluster(1)
        errs.append(_relerr(p.decode().cpu().numpy(), a.cpu().numpy()))
    assert abs(errs[0] - errs[1]) <= 1e-6 * max(1.0, errs[1])


# ---------------------------------------------------------------------------
# The fused single-launch step (lr_step.cu): used by encode_step whenever the shard
# is large enough for its cluster grid (n >= 8 x clusters, C % 256 == 0, r <= 8, f16
# factors).  Checked against the multi-kernel step (same algorithm, different
# summation orders), the reference oracle channel, the receiver, and graph replay.
# ---------------------------------------------------------------------------
def _lib_handle():
    from paper_2507_17511_b200 import _lib

    return _lib.load()


def _run_steps(mode, xs, spec, key_seed, fused, dtype=torch.bfloat16):
    _, pl, linalg = _mods()
    lib = _lib_handle()
    n, c = xs[0].shape
    lib.cc_debug_lowrank_fused(fused)
    n0 = lib.cc_debug_lowrank_fused_count()
    try:
        snd = pl.LayerState(mode, 1, torch.zeros(n, c, device="cuda"))
        rcv = pl.LayerState(mode, 1, torch.zeros(n, c, device="cuda"))
        key = linalg.DeviceKey(key_seed, 5, 2, advance=True)
        out = []
        for t, x in enumerate(xs, start=1):
            xd = torch.from_numpy(x).cuda().to(dtype)
            base0, aux0 = snd.base.clone(), snd._aux().clone() if snd._aux() is not None else None
            p, rec = pl.encode_step(snd, xd, spec, rng=key)
            if t > 1:
                dec = p.decode()
                if mode == "residual_with_feedback":
                    target = (xd.float() - base0) + aux0
                    assert torch.equal(snd.feedback, target - dec)  # feedback conservation
                    assert torch.equal(snd.base, base0 + dec)
                elif mode == "naive":
                    assert torch.equal(snd.base, dec)
            pl.decode_step(rcv, pl.device_message(t, 1, p))
            assert torch.equal(rcv.base, snd.base)
            out.append((_relerr(snd.base.cpu().numpy(), x), rec.compression_error))
        used = lib.cc_debug_lowrank_fused_count() - n0
    finally:
        lib.cc_debug_lowrank_fused(1)
    return out, used


@pytest.mark.parametrize("case", [
    ((1024, 3072), 8, 2, "residual_with_feedback", torch.bfloat16, False),
    ((512, 3072), 4, 1, "residual_no_feedback", torch.float32, False),
    ((768, 2048), 8, 3, "naive", torch.bfloat16, False),
    ((1000, 1024), 6, 2, "residual_with_feedback", torch.float32, False),
    ((1024, 3072), 8, 2, "residual_with_feedback", torch.bfloat16, True),
    ((522, 2048), 5, 1, "naive", torch.float32, True),
], ids=lambda c: f"{c[0][0]}x{c[0][1]}-r{c[1]}T{c[2]}-{c[3]}{'-int4' if c[5] else ''}")
def test_fused_step_matches_multikernel(case):
    shape, r, iters, mode, dtype, int4 = case
    xs = synth.flux_like(shape[0], shape[1], 5, seed=r + iters)
    spec = _spec(r, iters, int4)
    fused, used = _run_steps(mode, xs, spec, 17, 1, dtype)
    multi, used0 = _run_steps(mode, xs, spec, 17, 0, dtype)
    assert used == len(xs) - 1 and used0 == 0  # the fused kernel ran every compressed step
    # INT4: a code can flip between two levels when the f64 orders differ (one level is 2/15
    # of the column range), so the agreement is looser than for f16 factors
    tol = 1e-3 if int4 else 1e-4
    for t, ((ef, cf), (em, cm)) in enumerate(zip(fused, multi)):
        assert abs(ef - em) <= tol * max(1.0, em), (t, ef, em)
        assert abs(cf - cm) <= tol * max(1.0, cm), (t, cf, cm)


def test_fused_step_vs_reference_channel():
    """Trajectory of the fused step against the oracle's restatement of the reference
    channel (pl:84-121 with cx:394-426, host PCG64 Q0 from the same keys)."""
    cx, pl, linalg = _mods()
    lib = _lib_handle()
    n, c = 1024, 3072
    xs = synth.flux_like(n, c, 4, seed=3)
    spec = _spec(8, 2)
    snd = pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda"))
    och = O.Channel(O.WITH_FEEDBACK, 1, np.zeros((n, c), np.float32))
    n0 = lib.cc_debug_lowrank_fused_count()
    for t, x in enumerate(xs, start=1):
        pl.encode_step(snd, x, spec, rng=linalg.spawn_rng(11, 5, t))
        O.send(och, x, O.Codec(O.LOWRANK, rank=8, iters=2), rng=linalg.spawn_rng(11, 5, t))
        assert _relerr(snd.base.cpu().numpy(), och.base) < 1e-3, t
    assert lib.cc_debug_lowrank_fused_count() - n0 == len(xs) - 1


@pytest.mark.parametrize("int4", [False, True])
def test_fused_step_device_key_equals_host_rng_at_shard_shape(int4):
    """[1024, 3072] (the P = 4 shard): the fused kernel with the device-drawn start
    block equals the fused kernel with the host draw of the same key, bit for bit."""
    cx, pl, linalg = _mods()
    n, c = 1024, 3072
    xs = synth.flux_like(n, c, 4, seed=8)
    spec = _spec(8, 2, int4)
    a = pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda"))
    b = pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda"))
    key = linalg.DeviceKey(9, 5, 2, advance=True)
    for t, x in enumerate(xs, start=1):
        xd = torch.from_numpy(x).cuda().to(torch.bfloat16)
        pa, ra = pl.encode_step(a, xd, spec, rng=linalg.spawn_rng(9, 5, t))
        pb, rb = pl.encode_step(b, xd, spec, rng=key)
        assert pa.body_bytes() == pb.body_bytes(), f"step {t}"
        assert torch.equal(a.base, b.base) and torch.equal(a.feedback, b.feedback)
        assert ra.compression_error == rb.compression_error


def test_fused_step_rank_deficient_uses_replacement():
    """A rank-3 residual with r = 8: the Gram of A^T A Q is singular, every CTA sees the
    same degenerate pivot and CTA 0's CGS2 with replacement columns takes over inside
    the launch; the rank-3 part is still recovered (cx:402-404, T/test_compressors.py:144)."""
    cx, pl, linalg = _mods()
    lib = _lib_handle()
    g = np.random.default_rng(2)
    n, c = 1024, 3072
    a = (g.standard_normal((n, 3)) @ g.standard_normal((3, c))).astype(np.float32)
    snd = pl.LayerState("naive", 1, torch.zeros(n, c, device="cuda"))
    pl.encode_step(snd, a, _spec(8, 2), rng=linalg.spawn_rng(1, 5, 1))  # warmup (raw)
    n0 = lib.cc_debug_lowrank_fused_count()
    pl.encode_step(snd, a, _spec(8, 2), rng=linalg.spawn_rng(1, 5, 2))
    assert lib.cc_debug_lowrank_fused_count() - n0 == 1
    assert _relerr(snd.base.cpu().numpy(), a) < 2e-3


@pytest.mark.parametrize("fused", [1, 0])
def test_fused_exchange_graph_replay_equals_eager(fused):
    """The P = 4 patch-parallel low-rank step at the benchmarked shard ([1024, 3072]:
    the fused kernel) captured in one CUDA graph and replayed three times equals the
    matching eager steps bit for bit."""
    cx, pl, linalg = _mods()
    from paper_2507_17511_b200.comm import PatchParallelExchange

    lib = _lib_handle()
    lib.cc_debug_lowrank_fused(fused)
    rows, cols, P = 4096, 3072, 4
    spec = _spec(8, 2)
    xs = [torch.from_numpy(x).cuda().to(torch.bfloat16)[: rows // P].contiguous()
          for x in synth.flux_like(rows, cols, 4, seed=6)]
    ea = PatchParallelExchange(rows, cols, spec, sim_world=(P, 0))
    eb = PatchParallelExchange(rows, cols, spec, sim_world=(P, 0))
    ka = linalg.DeviceKey(3, 6, 0, 2, advance=True)
    kb = linalg.DeviceKey(3, 6, 0, 2, advance=True)
    n0 = lib.cc_debug_lowrank_fused_count()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for e, k in ((ea, ka), (eb, kb)):
            for i in range(3):
                e.step(xs[i], rng=k)
        ref = []
        for _ in range(3):  # eager: steps 4, 5, 6 on the same input
            ea.step(xs[3], rng=ka)
            ref.append(ea.reconstruction().clone())
        g = torch.cuda.CUDAGraph()  # one step per graph (the exchange's documented capture unit)
        with torch.cuda.graph(g, stream=s):
            eb.step(xs[3], rng=kb)
            s.wait_stream(eb.streams.decode)
        eb.after_capture()
        got = []
        for _ in range(3):
            g.replay()
            s.synchronize()
            got.append(eb.reconstruction().clone())
    torch.cuda.synchronize()
    lib.cc_debug_lowrank_fused(1)
    assert (lib.cc_debug_lowrank_fused_count() - n0 >= 8) == bool(fused)  # 4 warm + 3 eager + 1 captured
    for i in range(3):
        assert torch.equal(got[i], ref[i]), f"replay {i + 1}"


@pytest.mark.parametrize("n", [256, 1024], ids=["multi-kernel", "fused"])
def test_cabi_step_with_device_key_equals_host_rng(n):
    """cc_lowrank_encode_step called through the C ABI with a device key (the start
    block drawn inside the call, the key's step word advanced on the device) equals
    the step with the host draw of the same key, bit for bit, on both step forms."""
    cx, pl, linalg = _mods()
    from paper_2507_17511_b200 import _lib

    lib = _lib.load()
    c, r = 3072, 8
    xs = synth.flux_like(n, c, 3, seed=2)
    spec = _spec(r, 2)
    a = pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda"))
    b = pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda"))
    key = linalg.DeviceKey(9, 5, 2, advance=True)
    ws = torch.empty(lib.cc_lowrank_step_workspace_bytes(n, c, r), dtype=torch.uint8, device="cuda")
    body = torch.empty(lib.cc_body_bytes(_lib.CC_LOWRANK, n, c, r), dtype=torch.uint8, device="cuda")
    rec = torch.empty(2, dtype=torch.float64, device="cuda")
    n0 = lib.cc_debug_lowrank_fused_count()
    for t, x in enumerate(xs, start=1):
        xd = torch.from_numpy(x).cuda().to(torch.bfloat16)
        pa, ra = pl.encode_step(a, xd, spec, rng=linalg.spawn_rng(9, 5, t))
        if t == 1:
            pl.encode_step(b, xd, spec)  # warmup: raw
            continue
        _lib.check(lib.cc_lowrank_encode_step(2, n, c, r, 2, 0, _lib.ptr(xd), cx.dtype_code(xd), _lib.ptr(b.base),
                                              _lib.ptr(b.feedback), None, _lib.ptr(key.words), key.nwords,
                                              key.step_word, _lib.ptr(body), _lib.ptr(ws), ws.numel(),
                                              _lib.ptr(rec), _lib.stream_ptr()), "step")
        b.step = t
        torch.cuda.synchronize()
        assert body.cpu().numpy().tobytes() == pa.body_bytes(), f"step {t}"
        assert torch.equal(a.base, b.base) and torch.equal(a.feedback, b.feedback)
        assert float(rec[0]) == ra.compression_error
    assert (lib.cc_debug_lowrank_fused_count() - n0 > 0) == (n == 1024)
