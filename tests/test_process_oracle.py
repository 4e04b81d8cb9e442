"""The stability-harness oracle (oracle/process_oracle.py) against the reference:
the synthetic process bit for bit against digests of the reference's own
make_process (tests/golden/process_digests.json), the closed-form bounds against
the reference's theory KATs (T/test_theory.py:12-60), and SPEC.md:598 criterion 2
(ratio identity over 10^4 random stable draws)."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import process_oracle as PO

HERE = os.path.dirname(os.path.abspath(__file__))


def _digest(arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a, dtype="<f4").tobytes())
    return h.hexdigest()


CASES = json.load(open(os.path.join(HERE, "golden", "process_digests.json")))


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['spec']['drift']}-{c['spec']['rows']}x{c['spec']['cols']}")
def test_process_matches_reference_digests(case):
    d = case["spec"]
    p = PO.Process(d["rows"], d["cols"], d["lipschitz"], d["sigma_a_sq"], d["sigma_delta_sq"], d["steps"],
                   d["seed"], d["drift"])
    assert _digest([p.initial]) == case["initial"]
    assert _digest(p.states) == case["states"]
    assert list(p.measure()) == case["stats"]


def test_states_follow_maps():  # T/test_process.py:34-40
    p = PO.Process(16, 16, 0.5, 100.0, 1.0, 12, seed=3)
    prev = p.initial
    for t in range(1, 13):
        assert np.array_equal(p.step_map(t).apply(prev), p.states[t - 1])
        prev = p.states[t - 1]


def test_theory_hand_values():  # T/test_theory.py:12-60
    assert PO.v_naive(0.9, 0.5, 100.0) == pytest.approx(10.0 / 0.75)
    assert PO.v_residual(0.9, 0.5, 1.0) == pytest.approx(0.16)
    assert PO.bound_ratio(0.9, 0.5, 100.0, 1.0) == pytest.approx(0.01 * 0.75 / 0.625)
    assert PO.bound_ratio(1.0, 0.5, 100.0, 100.0) == 0.0
    assert PO.stability_threshold(0.5) == pytest.approx(0.4)
    assert PO.stability_threshold(0.0) == 0.0
    assert PO.no_feedback_growth(0.9, 1.0, 0) == 0.0
    with pytest.raises(ValueError):
        PO.v_residual(0.3, 0.5, 1.0)


def test_ratio_identity_criterion_2():
    """bound_ratio == v_residual / v_naive to 1e-12 relative, 10^4 draws."""
    rng = np.random.default_rng(0)
    n = 0
    while n < 10_000:
        L = rng.uniform(0.01, 0.99)
        delta = rng.uniform(PO.stability_threshold(L), 1.0)
        sa = rng.uniform(0.1, 1e3)
        sd = rng.uniform(1e-3, 1.0) * sa
        if delta >= 1.0 or (1.0 - L * L) - (1.0 - delta) * (L * L + 1.0) <= 1e-9:
            continue
        r = PO.bound_ratio(delta, L, sa, sd)
        direct = PO.v_residual(delta, L, sd) / PO.v_naive(delta, L, sa)
        assert abs(r - direct) <= 1e-12 * abs(direct)
        n += 1
