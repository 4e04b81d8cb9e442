"""Segmented K1 (cc_encode_step_segmented, the Ulysses sender): P column chunks of
one [n, C] activation, each an independent (src, dst) LayerState channel
(SPEC.md:473), encoded in ONE persistent launch.  Every chunk's body, base and
feedback must equal the CPU oracle's per-chunk channel (oracle.send on the
contiguous chunk, pl:84-121) bit for bit; the records within rel 1e-6."""

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
    from paper_2507_17511_b200 import _lib

    _lib.load()
    torch.cuda.set_device(0)


OTAG = {"sign1bit": O.SIGN1, "quant2bit": O.QUANT2}
OMODE = {"residual_with_feedback": O.WITH_FEEDBACK, "residual_no_feedback": O.NO_FEEDBACK, "naive": O.NAIVE}


def _run(n, C, P, codec, mode, steps, dtype, seed):
    from paper_2507_17511_b200 import _lib
    from paper_2507_17511_b200 import compressors as cx
    from paper_2507_17511_b200 import pipeline as pl

    lib = _lib.load()
    spec = cx.CompressorSpec(cx.CompressorKind(codec))
    tag = cx._spec_tag(spec)
    cw = C // P
    body_n = lib.cc_body_bytes(tag, n, cw, 0)
    stride = (body_n + 255) // 256 * 256
    xs = synth.flux_like(n, C, steps, seed=seed)
    base = torch.zeros(n, C, device="cuda")
    aux = torch.zeros(n, C, device="cuda")
    body = torch.zeros(P * stride, dtype=torch.uint8, device="cuda")
    rec = torch.zeros(2 * P, dtype=torch.float64, device="cuda")
    ws = torch.empty(lib.cc_workspace_bytes(tag, n, C, 0), dtype=torch.uint8, device="cuda")
    och = [O.Channel(OMODE[mode], 1, np.zeros((n, cw), np.float32)) for _ in range(P)]
    m = pl._MODE_CODE[pl.PipelineMode(mode)]
    for t, x in enumerate(xs, start=1):
        xd = torch.from_numpy(x).cuda().to(dtype)
        xo = xd.float().cpu().numpy()  # the exact values the device sees
        if t == 1:  # warmup (raw) step: base = x, aux = 0 / x
            _lib.check(lib.cc_warmup_step(m, n, C, _lib.ptr(xd), cx.dtype_code(xd), _lib.ptr(base),
                                          _lib.ptr(None if mode == "naive" else aux),
                                          _lib.ptr(torch.empty(n * C * 4, dtype=torch.uint8, device="cuda")),
                                          _lib.CC_F32, _lib.ptr(rec), _lib.stream_ptr()))
            for d in range(P):
                O.send(och[d], np.ascontiguousarray(xo[:, d * cw:(d + 1) * cw]), O.Codec(O.RAW))
            continue
        _lib.check(lib.cc_encode_step_segmented(
            tag, m, _lib.CC_SCALE_RANK1, n, C, P, _lib.ptr(xd), cx.dtype_code(xd), _lib.ptr(base),
            _lib.ptr(None if mode == "naive" else aux), _lib.ptr(body), stride, _lib.ptr(ws), ws.numel(),
            _lib.ptr(rec), _lib.stream_ptr()), "segmented")
        torch.cuda.synchronize()
        bh, ah, rh, by = base.cpu().numpy(), aux.cpu().numpy(), rec.cpu().numpy(), body.cpu().numpy()
        for d in range(P):
            tg, ob, orec = O.send(och[d], np.ascontiguousarray(xo[:, d * cw:(d + 1) * cw]), O.Codec(OTAG[codec]))
            assert by[d * stride:d * stride + body_n].tobytes() == ob, f"body chunk {d} step {t}"
            assert np.array_equal(bh[:, d * cw:(d + 1) * cw], och[d].base), f"base chunk {d} step {t}"
            if mode == "residual_with_feedback":
                assert np.array_equal(ah[:, d * cw:(d + 1) * cw], och[d].fb), f"feedback chunk {d} step {t}"
            elif mode == "residual_no_feedback":
                assert np.array_equal(ah[:, d * cw:(d + 1) * cw], och[d].ref), f"ref chunk {d} step {t}"
            assert rh[2 * d] == pytest.approx(orec["compression_error"], rel=1e-6, abs=1e-30)


@pytest.mark.parametrize("n,C,P", [(64, 3072, 8), (48, 3072, 4), (96, 3072, 2), (37, 2048, 4), (40, 1536, 3),
                                   (16, 1024, 8), (8, 512, 4)])
@pytest.mark.parametrize("codec", ["quant2bit", "sign1bit"])
def test_segmented_matches_per_chunk_oracle(n, C, P, codec):
    _run(n, C, P, codec, "residual_with_feedback", 4, torch.bfloat16, seed=n + C + P)


@pytest.mark.parametrize("mode", ["residual_no_feedback", "naive"])
def test_segmented_modes(mode):
    _run(32, 3072, 8, "quant2bit", mode, 3, torch.bfloat16, seed=3)


def test_segmented_f32_input():
    _run(24, 3072, 4, "quant2bit", "residual_with_feedback", 3, torch.float32, seed=5)


def test_segmented_flux_ulysses_shape():
    """Config 3's per-rank shape: [512, 3072] in 8 chunks of [512, 384]."""
    _run(512, 3072, 8, "sign1bit", "residual_with_feedback", 3, torch.bfloat16, seed=11)


def test_segmented_rejects_unsupported():
    from paper_2507_17511_b200 import _lib

    lib = _lib.load()
    x = torch.zeros(8, 3072, dtype=torch.bfloat16, device="cuda")
    b = torch.zeros(8, 3072, device="cuda")
    body = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    rec = torch.zeros(64, dtype=torch.float64, device="cuda")
    ws = torch.empty(lib.cc_workspace_bytes(_lib.CC_QUANT2, 8, 3072, 0), dtype=torch.uint8, device="cuda")
    # 3072 / 16 = 192 columns per chunk: not a multiple of 128
    st = lib.cc_encode_step_segmented(_lib.CC_QUANT2, _lib.CC_WITH_FEEDBACK, 0, 8, 3072, 16, _lib.ptr(x),
                                      _lib.CC_BF16, _lib.ptr(b), _lib.ptr(b), _lib.ptr(body), 65536, _lib.ptr(ws),
                                      ws.numel(), _lib.ptr(rec), _lib.stream_ptr())
    assert st == _lib.CC_ERR_UNSUPPORTED
    st = lib.cc_encode_step_segmented(_lib.CC_QUANT2, _lib.CC_WITH_FEEDBACK, 0, 8, 3072, 5, _lib.ptr(x),
                                      _lib.CC_BF16, _lib.ptr(b), _lib.ptr(b), _lib.ptr(body), 65536, _lib.ptr(ws),
                                      ws.numel(), _lib.ptr(rec), _lib.stream_ptr())
    assert st == _lib.CC_ERR_SHAPE


def test_ulysses_exchange_segmented_equals_chunked():
    """UlyssesAllToAll (sim rank 0 of 8): segmented path vs forced per-chunk path,
    identical bodies and reconstructions over a warmup + 3 compressed steps."""
    from paper_2507_17511_b200 import comm
    from paper_2507_17511_b200 import compressors as cx

    spec = cx.CompressorSpec(cx.CompressorKind.SIGN1BIT)
    n, C, P = 64, 3072, 8
    a = comm.UlyssesAllToAll(n, C, spec, sim_world=(P, 0))
    b = comm.UlyssesAllToAll(n, C, spec, sim_world=(P, 0))
    assert a.segmented
    b.segmented = False
    for d, st in enumerate(b.senders):  # contiguous per-chunk states for the chunked path
        st.base, st.feedback = torch.zeros(n, C // P, device="cuda"), torch.zeros(n, C // P, device="cuda")
    for x in synth.flux_like(n, C, 4, seed=9):
        xd = torch.from_numpy(x).cuda().to(torch.bfloat16)
        oa, ob = a.step(xd).clone(), b.step(xd).clone()
        torch.cuda.synchronize()
        assert torch.equal(a.sendbuf, b.sendbuf)
        assert torch.equal(oa, ob)
