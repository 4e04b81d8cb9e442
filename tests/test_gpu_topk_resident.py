"""GPU parity of the shard-resident top-k encode_step (csrc/topk_resident.cu) against
the oracle (compressors.py:446-456, pipeline.py:84-121) and against the multi-kernel
radix select (topk.cu), which it replaces whenever the persistent grid can launch."""

import zlib

import numpy as np
import pytest
import torch

import synth
from oracle import cc_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)


def _mods():
    from paper_2507_17511_b200 import _lib
    from paper_2507_17511_b200 import compressors as cx
    from paper_2507_17511_b200 import pipeline as pl

    return _lib.load(), cx, pl


def _inputs(n, c, steps, kind, seed):
    rng = np.random.default_rng(seed)
    if kind == "flux":
        xs = synth.flux_like(n, c, steps, seed=seed)
    else:
        xs = [rng.standard_normal((n, c)).astype(np.float32) for _ in range(steps)]
    if kind == "ties":  # few distinct magnitudes: massive ties at the threshold
        xs = [(np.round(x * 2) / 2).astype(np.float32) for x in xs]
    if kind == "zeros":
        for x in xs:
            x[rng.random((n, c)) < 0.9] = 0.0
            x[rng.random((n, c)) < 0.05] = -0.0
    if kind == "huge":  # f16 overflow -> inf values, subnormal f16 values
        for x in xs:
            x[rng.random((n, c)) < 0.01] *= 1e5
            x[rng.random((n, c)) < 0.1] *= 1e-6
    xs[min(1, steps - 1)].reshape(-1)[:7] = -0.0  # dense `base + 0.0` semantics
    return xs


def _run(lib, cx, pl, xs, mode, frac, dtype, resident):
    lib.cc_debug_topk_resident(1 if resident else 0)
    try:
        n, c = xs[0].shape
        spec = cx.CompressorSpec(cx.CompressorKind.TOPK, keep_fraction=frac)
        st = pl.LayerState(mode, 1, torch.zeros(n, c, device="cuda"))
        out = []
        c0 = lib.cc_debug_topk_resident_count()
        for x in xs:
            xd = torch.from_numpy(x).cuda().to(dtype)
            p, rec = pl.encode_step(st, xd, spec)
            out.append((p.body_bytes(), st.base.cpu().numpy().tobytes(), st.feedback.cpu().numpy().tobytes()
                        if mode == "residual_with_feedback" else b"", rec.compression_error))
        used = lib.cc_debug_topk_resident_count() - c0
    finally:
        lib.cc_debug_topk_resident(1)
    return out, used


SHAPES = [(1, 1), (2, 3), (37, 101), (64, 384), (512, 3072), (1000, 999)]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"{s[0]}x{s[1]}")
@pytest.mark.parametrize("frac", [0.001, 0.01, 0.1, 1.0])
@pytest.mark.parametrize("kind", ["gauss", "ties", "zeros", "huge"])
def test_resident_vs_oracle(shape, frac, kind):
    lib, cx, pl = _mods()
    n, c = shape
    # huge: one compressed step (an inf decode makes the next step's state NaN, whose
    # bit pattern numpy and the device spell differently)
    xs = _inputs(n, c, 2 if kind == "huge" else 3, kind, zlib.crc32(f"{n}x{c}{frac}{kind}".encode()))
    mode = "residual_with_feedback"
    got, used = _run(lib, cx, pl, xs, mode, frac, torch.float32, True)
    assert used == len(xs) - 1  # every post-warmup step ran the persistent kernel
    och = O.Channel(mode, 1, np.zeros((n, c), np.float32))
    for i, x in enumerate(xs):
        _, body, orec = O.send(och, x, O.Codec(O.TOPK, keep_fraction=frac))
        assert got[i][0] == body, f"body step {i + 1}"
        assert got[i][1] == och.base.tobytes(), f"base step {i + 1}"
        assert got[i][2] == och.fb.tobytes(), f"feedback step {i + 1}"
        assert got[i][3] == pytest.approx(orec["compression_error"], rel=1e-6, abs=1e-30)


@pytest.mark.parametrize("mode", ["naive", "residual_no_feedback", "residual_with_feedback"])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32], ids=["bf16", "f32"])
@pytest.mark.parametrize("shape", [(512, 3072), (1024, 3072), (2048, 3072), (4096, 3072)],
                         ids=lambda s: f"{s[0]}x{s[1]}")
def test_resident_vs_multikernel(mode, dtype, shape):
    """Bit-identical bodies, states and records to the multi-kernel path: shards whose
    x / aux / base fit on chip (TMA-staged), shards where only t fits (register
    loads), and [4096, 3072], which the resident kernel declines (t does not fit)."""
    lib, cx, pl = _mods()
    n, c = shape
    xs = _inputs(n, c, 4, "flux", n + c)
    xs = [torch.from_numpy(x).to(dtype).float().numpy() for x in xs]  # exact inputs for both dtypes
    a, used = _run(lib, cx, pl, xs, mode, 0.01, dtype, True)
    b, used_b = _run(lib, cx, pl, xs, mode, 0.01, dtype, False)
    assert used == (0 if n == 4096 else len(xs) - 1) and used_b == 0
    for i, (ra, rb) in enumerate(zip(a, b)):
        assert ra[0] == rb[0] and ra[1] == rb[1] and ra[2] == rb[2], f"step {i + 1}"
        assert ra[3] == pytest.approx(rb[3], rel=1e-9, abs=1e-30)


@pytest.mark.parametrize("frac", [0.01, 0.1])
def test_resident_p2_shape_vs_oracle(frac):
    """[2048, 3072] (P = 2): t on chip, x / base streamed through registers."""
    lib, cx, pl = _mods()
    n, c = 2048, 3072
    xs = _inputs(n, c, 3, "flux", 7)
    got, used = _run(lib, cx, pl, xs, "residual_with_feedback", frac, torch.float32, True)
    assert used == 2
    och = O.Channel("residual_with_feedback", 1, np.zeros((n, c), np.float32))
    for i, x in enumerate(xs):
        _, body, _ = O.send(och, x, O.Codec(O.TOPK, keep_fraction=frac))
        assert got[i][0] == body and got[i][1] == och.base.tobytes() and got[i][2] == och.fb.tobytes()


def test_resident_graph_replay():
    """Captured in a CUDA graph and replayed: the slab words left zeroed by every
    launch make replays independent (same result as eager steps)."""
    lib, cx, pl = _mods()
    n, c = 512, 3072
    xs = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in _inputs(n, c, 2, "flux", 3)]
    spec = cx.CompressorSpec(cx.CompressorKind.TOPK, keep_fraction=0.01)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ea = pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda"))
        eb = pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda"))
        pl.encode_step(ea, xs[0], spec)
        pl.encode_step(eb, xs[0], spec)
        body = torch.empty(6 * cx.topk_count(n, c, 0.01), dtype=torch.uint8, device="cuda")
        p, _ = pl.encode_step(ea, xs[1], spec, body_out=body)  # warm the slab / workspace outside capture
        ref = [p.body_bytes()]
        for _ in range(3):
            p, _ = pl.encode_step(ea, xs[1], spec, body_out=body)
            ref.append(p.body_bytes())
        pl.encode_step(eb, xs[1], spec, body_out=body)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            pl.encode_step(eb, xs[1], spec, body_out=body)
        got = [body.cpu().numpy().tobytes()]
        for _ in range(3):
            g.replay()
            s.synchronize()
            got.append(body.cpu().numpy().tobytes())
    assert got == ref
    assert torch.equal(ea.base, eb.base) and torch.equal(ea.feedback, eb.feedback)
