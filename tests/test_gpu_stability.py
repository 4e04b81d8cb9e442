"""Closed-loop error-stability harness on the GPU path (pl:168-199,
proc:250-291, th:54-95).

run_trajectory's loop (pl:168-199) driven through the device encode_step /
decode_step: in the closed-loop modes a*_t = f_t(base) is evaluated on the shared
reconstruction, the no-feedback mode consumes the uncompressed states; the
receiver must equal the sender bit for bit every step (pl:193-194).  The synthetic
process is the oracle's restatement of the reference's make_process, pinned to the
reference by tests/test_process_oracle.py.

Checks: the whole closed-loop trajectory (every step's total error) equals the CPU
oracle's bit for bit (the codes are bit-exact, so the loop is); and the paper's
error-feedback properties hold on the device path — criterion 3 (no-feedback error
grows at (1 - delta)·sigma_delta^2 per step, feedback error flat), criterion 4
(Fig. 4 ordering feedback < no-feedback < naive), criterion 9 (warmup 2 does not
increase the error) and bounded feedback error across L in {0.3, 0.5, 0.7}.
"""

import numpy as np
import pytest
import torch

from oracle import cc_oracle as O
from oracle import process_oracle as PO

pytestmark = pytest.mark.gpu

MODES = {"residual_with_feedback": O.WITH_FEEDBACK, "residual_no_feedback": O.NO_FEEDBACK, "naive": O.NAIVE}
OTAG = {"sign1bit": O.SIGN1, "quant2bit": O.QUANT2}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2507_17511_b200 import _lib

    _lib.load()
    torch.cuda.set_device(0)


@pytest.fixture(scope="module")
def standard():  # SPEC.md / T/test_process.py:8 standard run
    return PO.Process(64, 64, 0.5, 100.0, 1.0, 200, seed=7)


def gpu_trajectory(proc, codec, mode, warmup=1):
    """pl:168-199 on the device path; returns per-step (total_error, delta_hat)."""
    from paper_2507_17511_b200 import compressors as cx
    from paper_2507_17511_b200 import pipeline as pl

    spec = cx.CompressorSpec(cx.CompressorKind(codec))
    init = torch.from_numpy(np.ascontiguousarray(proc.initial)).cuda()
    snd = pl.LayerState(mode, warmup, init)
    rcv = pl.LayerState(mode, warmup, init)
    out = []
    for t in range(1, len(proc.states) + 1):
        if mode == "residual_no_feedback":
            a_star = proc.states[t - 1]
        else:
            a_star = proc.step_map(t).apply(snd.base.cpu().numpy())
        payload, rec = pl.encode_step(snd, torch.from_numpy(np.ascontiguousarray(a_star)).cuda(), spec)
        pl.decode_step(rcv, pl.device_message(t, warmup, payload))
        recon = rcv.base.cpu().numpy()
        assert np.array_equal(recon, snd.base.cpu().numpy()), f"sender/receiver diverged at step {t}"
        out.append((PO.sqnorm(recon.astype(np.float64) - proc.states[t - 1].astype(np.float64)), rec.delta_hat))
    return out


def oracle_trajectory(proc, codec, mode, warmup=1):
    snd = O.Channel(MODES[mode], warmup, proc.initial.copy())
    out = []
    for t in range(1, len(proc.states) + 1):
        a_star = proc.states[t - 1] if mode == "residual_no_feedback" else proc.step_map(t).apply(snd.base)
        _, _, rec = O.send(snd, a_star, O.Codec(OTAG[codec]))
        out.append((PO.sqnorm(snd.base.astype(np.float64) - proc.states[t - 1].astype(np.float64)),
                    rec["delta_hat"]))
    return out


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("codec", list(OTAG))
def test_closed_loop_trajectory_bit_exact_vs_oracle(standard, codec, mode):
    g = gpu_trajectory(standard, codec, mode)
    o = oracle_trajectory(standard, codec, mode)
    assert [e for e, _ in g] == [e for e, _ in o]  # every step's total error, bit for bit
    for (_, dg), (_, do) in zip(g[1:], o[1:]):
        assert dg == pytest.approx(do, rel=1e-6)


def test_no_feedback_divergence_criterion_3(standard):
    nf = gpu_trajectory(standard, "sign1bit", "residual_no_feedback")
    fb = gpu_trajectory(standard, "sign1bit", "residual_with_feedback")
    te_nf = np.array([e for e, _ in nf])
    te_fb = np.array([e for e, _ in fb])
    slope_nf = np.polyfit(np.arange(len(te_nf)), te_nf, 1)[0]
    delta = float(np.mean([d for _, d in nf[1:]]))
    _, _, d_sq = standard.measure()
    predicted = PO.no_feedback_growth(delta, d_sq, 1)
    assert slope_nf > 0 and abs(slope_nf - predicted) <= 0.25 * predicted, (slope_nf, predicted)
    slope_fb = np.polyfit(np.arange(50), te_fb[-50:], 1)[0]
    assert abs(slope_fb) < 0.10 * slope_nf, (slope_fb, slope_nf)


def test_fig4_ordering_criterion_4(standard):
    m = {mode: np.mean([e for e, _ in gpu_trajectory(standard, "sign1bit", mode)]) for mode in MODES}
    assert m["residual_with_feedback"] < m["residual_no_feedback"] < m["naive"], m


@pytest.mark.parametrize("codec", list(OTAG))
def test_warmup_sensitivity_criterion_9(standard, codec):
    m1, m2 = (np.mean([e for e, _ in gpu_trajectory(standard, codec, "residual_with_feedback", warmup=w)])
              for w in (1, 2))
    assert m2 <= m1, (m1, m2)


@pytest.mark.parametrize("L", [0.3, 0.5, 0.7])
@pytest.mark.parametrize("codec", list(OTAG))
def test_feedback_error_bounded(codec, L):
    """Error feedback keeps the closed-loop error bounded and far below naive
    compression on every seed (Props. 2-3 regime), across contraction rates."""
    for seed in range(3):
        proc = PO.Process(64, 64, L, 100.0, 1.0, 120, seed=100 + seed)
        fb = np.array([e for e, _ in gpu_trajectory(proc, codec, "residual_with_feedback")])
        nv = np.array([e for e, _ in gpu_trajectory(proc, codec, "naive")])
        assert np.all(np.isfinite(fb))
        late_fb, early_fb = fb[-30:].mean(), fb[10:40].mean()
        assert late_fb <= 1.5 * early_fb + 1e-9, (late_fb, early_fb)  # no growth
        assert late_fb * 5.0 <= nv[-30:].mean(), (late_fb, nv[-30:].mean())
