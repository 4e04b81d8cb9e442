"""Patch-parallel exchange in its single-GPU rank simulation (sim_world): every
peer slot receives this rank's own body, so every peer's reconstructed rows must
equal the sender's own base bit for bit after every step (sender == receiver,
pl:193-194, mesh:232-237) — for every codec, including the odd-sized top-k and
N:M bodies whose receive slots are padded to 16 bytes."""

import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)


SPECS = [("sign1bit", {}), ("quant2bit", {}), ("quant4bit", {}), ("topk", {"keep_fraction": 0.013}),
         ("topk", {"keep_fraction": 0.1}), ("nm_block", {"n": 2, "m": 4}), ("lowrank", {"rank": 4, "iterations": 2})]


@pytest.mark.parametrize("codec,kw", SPECS, ids=lambda v: str(v))
@pytest.mark.parametrize("P", [2, 4, 8])
def test_sim_exchange_peers_equal_sender(codec, kw, P):
    from paper_2507_17511_b200 import comm
    from paper_2507_17511_b200 import compressors as cx
    from paper_2507_17511_b200 import linalg as la

    rows, cols = 40 * P, 384
    spec = cx.CompressorSpec(cx.CompressorKind(codec), **kw)
    ex = comm.PatchParallelExchange(rows, cols, spec, sim_world=(P, 0))
    lo, hi = ex.lo, ex.hi
    for t, x in enumerate(synth.flux_like(hi - lo, cols, 4, seed=P), start=1):
        xd = torch.from_numpy(x).cuda().to(torch.bfloat16)
        full = ex.step(xd, rng=la.make_rng(t) if codec == "lowrank" else None)
        ex.synchronize()
        torch.cuda.synchronize()
        own = ex.sender.base.clone()
        for p in range(1, P):
            b0, b1 = ex.bounds[p]
            assert torch.equal(full[b0:b1], own), f"peer {p} differs at step {t}"


@pytest.mark.parametrize("codec,kw", [("quant2bit", {}), ("topk", {"keep_fraction": 0.02})], ids=lambda v: str(v))
def test_graph_replayed_exchange_matches_eager(codec, kw):
    """bench.py replays CUDA-graph-captured exchange steps: a captured step replayed
    must give exactly the state an eager step gives (K1's stream control slot is
    bound at capture time; the replay runs on another stream)."""
    from paper_2507_17511_b200 import comm
    from paper_2507_17511_b200 import compressors as cx

    rows, cols, P = 96, 3072, 4
    spec = cx.CompressorSpec(cx.CompressorKind(codec), **kw)
    xs = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in synth.flux_like(rows // P, cols, 6, seed=31)]
    eager = comm.PatchParallelExchange(rows, cols, spec, sim_world=(P, 0))
    graphed = comm.PatchParallelExchange(rows, cols, spec, sim_world=(P, 0))
    for t in range(3):  # warmup step + two compressed steps, eagerly on both
        eager.step(xs[t])
        graphed.step(xs[t])
    torch.cuda.synchronize()
    inp = torch.empty_like(xs[0])
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        graphed.step(inp)
        torch.cuda.current_stream().wait_stream(graphed.streams.decode)
    graphed.after_capture()
    for t in range(3, 6):
        eager.step(xs[t])
        eager.synchronize()
        inp.copy_(xs[t])
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(eager.full, graphed.full), f"step {t}"
        assert torch.equal(eager.sender.feedback, graphed.sender.feedback), f"step {t}"
