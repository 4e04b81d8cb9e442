"""The shard-resident single-pass K1 (csrc/k1_resident.cu) against the streaming
K1 and the oracle: identical bodies / base / feedback / ref / records, bit for bit,
for every codec, mode, input dtype and scale mode, at the per-rank shard shapes
where it is used (patch P = 2 / 4 / 8, Ulysses senders) and at ragged row counts
(fewer rows than SMs, uneven rows per CTA)."""

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
def lib():
    from paper_2507_17511_b200 import _lib

    lib = _lib.load()
    yield lib
    lib.cc_debug_k1_resident(1)


def _traj(n, c, steps, seed):
    xs = synth.flux_like(n, c, steps, seed=seed)
    rng = np.random.default_rng(seed)
    xs[2][rng.random((n, c)) < 0.1] = 0.0
    xs[2][n // 3] = 0.0
    return xs


def _run(lib, resident, n, c, codec, mode, dtype, scale_mode="rank1", steps=4, seed=1):
    from paper_2507_17511_b200 import compressors as cx
    from paper_2507_17511_b200 import pipeline as pl

    lib.cc_debug_k1_resident(1 if resident else 0)
    spec = cx.CompressorSpec(cx.CompressorKind(codec), scale_mode=scale_mode)
    st = pl.LayerState(mode, 1, torch.zeros(n, c, device="cuda"))
    xs = _traj(n, c, steps, seed)
    c0 = lib.cc_debug_k1_resident_count()
    out = []
    for x in xs:
        p, rec = pl.encode_step(st, torch.from_numpy(x).cuda().to(dtype), spec)
        out.append((p.body_bytes(), rec.compression_error, rec.target_sqnorm))
    torch.cuda.synchronize()
    used = lib.cc_debug_k1_resident_count() - c0
    aux = st.feedback if mode == "residual_with_feedback" else st.ref
    return out, st.base.clone(), None if aux is None else aux.clone(), used, xs


# 512 / 1024: t + base in shared memory; 2048: t in shared memory; 4096 / 4500: t in
# shared + tensor memory; 100 / 149: fewer rows than SMs / uneven rows per CTA
SHAPES = [(512, 3072), (1024, 3072), (2048, 3072), (4096, 3072), (4500, 3072), (100, 3072), (149, 3072),
          (1000, 2048), (300, 2560), (2900, 2048)]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"{s[0]}x{s[1]}")
@pytest.mark.parametrize("codec", ["sign1bit", "quant2bit", "quant4bit"])
@pytest.mark.parametrize("mode", ["naive", "residual_no_feedback", "residual_with_feedback"])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32], ids=["bf16", "f32"])
def test_resident_matches_streaming_kernel(lib, shape, codec, mode, dtype):
    n, c = shape
    a = _run(lib, True, n, c, codec, mode, dtype, seed=n + c)
    b = _run(lib, False, n, c, codec, mode, dtype, seed=n + c)
    assert a[3] == 3, "resident kernel did not run for the compressed steps"
    assert b[3] == 0
    for (ba, ea, ta), (bb, eb, tb) in zip(a[0], b[0]):
        assert ba == bb
        # f64 record sums over a different row-to-CTA partition: equal up to rounding
        assert ea == pytest.approx(eb, rel=1e-12, abs=1e-300) and ta == pytest.approx(tb, rel=1e-12, abs=1e-300)
    assert torch.equal(a[1], b[1])
    if a[2] is not None:
        assert torch.equal(a[2], b[2])


@pytest.mark.parametrize("shape", [(512, 3072), (149, 3072), (4096, 3072)], ids=lambda s: f"{s[0]}x{s[1]}")
@pytest.mark.parametrize("codec", ["sign1bit", "quant2bit", "quant4bit"])
@pytest.mark.parametrize("scale_mode", ["rank1", "per_token", "per_channel"])
def test_resident_vs_oracle(lib, shape, codec, scale_mode):
    if shape[0] == 4096 and (codec, scale_mode) not in (("quant2bit", "rank1"), ("sign1bit", "per_token")):
        pytest.skip("full-shard oracle runs are slow on the host: two representative cases")
    n, c = shape
    mode = "residual_with_feedback"
    out, base, fb, used, xs = _run(lib, True, n, c, codec, mode, torch.float32, scale_mode, steps=4, seed=7)
    assert used == 3
    och = O.Channel(mode, 1, np.zeros((n, c), np.float32))
    oc = O.Codec(TAGS[codec], scale_mode=scale_mode)
    for (body, err, _), x in zip(out, xs):
        _, obody, orec = O.send(och, x, oc)
        assert body == obody
        assert err == pytest.approx(orec["compression_error"], rel=1e-6, abs=1e-30)
    assert np.array_equal(base.cpu().numpy(), och.base)
    assert np.array_equal(fb.cpu().numpy(), och.fb)


def test_too_tall_shard_takes_the_streaming_kernel(lib):
    """Shards taller than shared + tensor memory hold fall back to the streaming K1."""
    out, _, _, used, _ = _run(lib, True, 7000, 3072, "quant2bit", "residual_with_feedback", torch.bfloat16, steps=3)
    assert used == 0


@pytest.mark.parametrize("P,codec", [(8, "sign1bit"), (4, "quant2bit"), (8, "quant4bit")])
def test_resident_segmented_matches_streaming(lib, P, codec):
    """Ulysses senders: P column-segment channels in one resident launch."""
    from paper_2507_17511_b200 import compressors as cx
    from paper_2507_17511_b200.comm import UlyssesAllToAll

    n, C = 512, 3072
    spec = cx.CompressorSpec(cx.CompressorKind(codec))
    xs = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in _traj(n, C, 4, 5)]
    res = []
    for resident in (1, 0):
        lib.cc_debug_k1_resident(resident)
        ex = UlyssesAllToAll(n, C, spec, sim_world=(P, 0))
        assert ex.segmented
        c0 = lib.cc_debug_k1_resident_count()
        bodies = []
        for x in xs:
            ex.step(x)
            bodies.append(ex.sendbuf.clone())
        torch.cuda.synchronize()
        res.append((bodies, ex.base_full.clone(), ex.aux_full.clone(), ex.out.clone(),
                    lib.cc_debug_k1_resident_count() - c0))
    assert res[0][4] == 3 and res[1][4] == 0
    for a, b in zip(res[0][0], res[1][0]):
        assert torch.equal(a, b)
    for i in (1, 2, 3):
        assert torch.equal(res[0][i], res[1][i])


def test_resident_exchange_graph_replay(lib):
    """Patch P=4 rank shard under CUDA-graph replay (the bench's mode): the
    resident K1 keeps its control words zeroed across replays."""
    from paper_2507_17511_b200 import comm
    from paper_2507_17511_b200 import compressors as cx

    rows, cols, P = 4096, 3072, 4
    spec = cx.CompressorSpec(cx.CompressorKind.QUANT2BIT)
    xs = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in _traj(rows // P, cols, 6, 9)]
    eager = comm.PatchParallelExchange(rows, cols, spec, sim_world=(P, 0))
    graphed = comm.PatchParallelExchange(rows, cols, spec, sim_world=(P, 0))
    for t in range(3):
        eager.step(xs[t])
        graphed.step(xs[t])
    torch.cuda.synchronize()
    inp = torch.empty_like(xs[0])
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        graphed.step(inp)
        torch.cuda.current_stream().wait_stream(graphed.streams.decode)
    graphed.after_capture()
    c0 = lib.cc_debug_k1_resident_count()
    for t in range(3, 6):
        eager.step(xs[t])
        eager.synchronize()
        inp.copy_(xs[t])
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(eager.full, graphed.full), f"step {t}"
        assert torch.equal(eager.sender.feedback, graphed.sender.feedback), f"step {t}"
    assert lib.cc_debug_k1_resident_count() - c0 == 3  # the eager steps (replays are not counted)
