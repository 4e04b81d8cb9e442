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
