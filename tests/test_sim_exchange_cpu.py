"""Host logic of the single-GPU rank simulation (sim_world) on CPU with the oracle
engine: every peer slot holds this rank's own body, so every peer's rows must equal
the sender's base after every step; receive slots are 16-byte aligned for every
codec's body size (top-k bodies are 6k bytes)."""

import pytest
import torch

import synth
from oracle_engine import OracleEngine


def _spec(codec, **kw):
    from paper_2507_17511_b200 import compressors as cx

    return cx.CompressorSpec(cx.CompressorKind(codec), **kw)


@pytest.mark.parametrize("codec,kw", [("quant2bit", {}), ("sign1bit", {}), ("topk", {"keep_fraction": 0.013})])
@pytest.mark.parametrize("P", [2, 4])
def test_sim_patch_exchange_peers_equal_sender(codec, kw, P):
    from paper_2507_17511_b200 import comm

    rows, cols = 12 * P, 40
    ex = comm.PatchParallelExchange(rows, cols, _spec(codec, **kw), engine=OracleEngine(), device="cpu",
                                    sim_world=(P, 0))
    assert ex.P == P and ex.rank == 0 and ex.sim
    for t, x in enumerate(synth.flux_like(ex.hi - ex.lo, cols, 3, seed=P), start=1):
        full = ex.step(torch.from_numpy(x).to(torch.bfloat16))
        assert ex._per % 16 == 0, "receive slots must stay 16-byte aligned"
        own = ex.sender.base
        for p in range(1, P):
            b0, b1 = ex.bounds[p]
            assert torch.equal(full[b0:b1], own), f"peer {p} step {t}"


def test_wire_bytes_padded_to_16():
    from paper_2507_17511_b200 import comm

    ex = comm.PatchParallelExchange(64, 40, _spec("topk", keep_fraction=0.013), engine=OracleEngine(),
                                    device="cpu", sim_world=(4, 0))
    for warm in (True, False):
        assert ex.wire_bytes(warm, True) % 16 == 0
    assert ex.wire_bytes(False, True) >= comm.body_bytes_for(ex.codec, 16, 40)
