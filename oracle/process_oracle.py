"""Test infrastructure (never imported by the product): numpy restatement of the
reference's synthetic contractive process (process.py) and its closed-form error
bounds (theory.py), for the closed-loop error-stability harness of SURVEY §8f
row 4 (pl:168-199, proc:250-291, th:54-95; acceptance criteria SPEC.md:596-608).

The process is pinned to the reference: tests/golden/process_digests.json holds
digests of trajectories made by the reference's own make_process in the build
container (tests/golden/make_golden.py), and tests/test_oracle_golden.py checks
this restatement reproduces them bit for bit (same PCG64 streams, same draw order).

Step map (proc:1-8): x_t = L * P_t(x_{t-1} - c_{t-1}) + c_t + d_t with P_t the
identity ("walk", "smooth") or a fresh signed entry permutation ("scrambled"), an
anchor c_t moving on its energy sphere and Gaussian noise d_t; the anchor, drift and
noise energies are calibrated until the measured activation / drift energies land
within 10 % of (sigma_a^2, sigma_delta^2) (proc:250-282).
"""

from __future__ import annotations

import numpy as np

BURN_IN = 200            # proc:45
CAL_WINDOW = 200         # proc:46
CAL_ROUNDS = 8           # proc:47
BAND = 0.15              # proc:48
ANCHOR_SHARE = 0.8       # proc:49
MOMENTUM = 0.9           # proc:50


def stream(seed, *key):
    """la:24-26 spawn_rng: PCG64 keyed by (seed, key...)."""
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(entropy=seed, spawn_key=tuple(key))))


def sqnorm(m):
    d = np.asarray(m, dtype=np.float64).ravel()
    return float(np.dot(d, d))  # la:61-64


class Step:
    """One affine map (proc:107-121); `apply` returns f32 like the reference."""

    __slots__ = ("L", "perm", "signs", "c_prev", "offset")

    def __init__(self, L, perm, signs, c_prev, offset):
        self.L, self.perm, self.signs, self.c_prev, self.offset = L, perm, signs, c_prev, offset

    def apply(self, x):
        y = np.asarray(x, dtype=np.float64) - self.c_prev
        if self.perm is not None:
            y = (y.ravel()[self.perm] * self.signs).reshape(np.shape(x))
        return (self.L * y + self.offset).astype(np.float32)


class Process:
    """make_process(spec) result: initial state, states a_1..a_T, step maps."""

    def __init__(self, rows, cols, L, sigma_a_sq, sigma_delta_sq, steps, seed, drift="walk"):
        if not 0.0 <= L < 1.0:
            raise ValueError("lipschitz must be in [0, 1)")
        if not 0.0 <= sigma_delta_sq <= sigma_a_sq or sigma_a_sq <= 0.0:
            raise ValueError("need 0 <= sigma_delta_sq <= sigma_a_sq, sigma_a_sq > 0")
        self.rows, self.cols, self.L, self.steps, self.seed, self.drift = rows, cols, L, steps, seed, drift
        self.sa, self.sd = sigma_a_sq, sigma_delta_sq
        anchor_sq, noise_sq, drift_sq = self._knobs0()
        dirn = stream(seed, 1).standard_normal((rows, cols))
        dirn /= np.sqrt(np.sum(dirn * dirn))
        for rnd in range(CAL_ROUNDS):  # proc:262-282
            start, window, _ = self._run(anchor_sq, noise_sq, drift_sq, dirn, stream(seed, 2, rnd), CAL_WINDOW, False)
            a_sq, d_sq = _energies([start] + window)
            if abs(a_sq - self.sa) <= 0.10 * self.sa and (self.sd == 0.0 or abs(d_sq - self.sd) <= 0.10 * self.sd):
                break
            if self.sd > 0.0 and d_sq > 0.0:
                gain = self.sd / d_sq
                noise_sq, drift_sq = noise_sq * gain, drift_sq * gain
            anchor_sq = self.sa - max(a_sq - anchor_sq, 0.0)
            if anchor_sq <= 0.0:
                raise ValueError("calibration failed: drift floor exceeds sigma_a_sq")
        else:
            raise ValueError("calibration did not converge")
        self.initial, self.states, self.maps = self._run(anchor_sq, noise_sq, drift_sq, dirn, stream(seed, 3),
                                                        steps, True)

    def _knobs0(self):  # proc:139-153
        l2 = self.L * self.L
        share = ANCHOR_SHARE if (self.sd > 0.0 and self.rows >= 2) else 0.0
        noise_sq = (1.0 - share) * self.sd * (1.0 - l2) / 2.0
        anchor_sq = self.sa - (noise_sq / (1.0 - l2) if noise_sq > 0 else 0.0)
        if anchor_sq <= 0.0:
            raise ValueError("infeasible process statistics")
        return anchor_sq, noise_sq, share * self.sd

    def _run(self, anchor_sq, noise_sq, drift_sq, dirn, rng, steps, keep):  # proc:243-248
        rows, cols = self.rows, self.cols
        c = dirn * np.sqrt(anchor_sq)
        radius = np.sqrt(anchor_sq)
        mom = np.zeros_like(c)
        state = c.astype(np.float32)
        noise = np.sqrt(noise_sq / (rows * cols)) if noise_sq > 0 else 0.0

        def move(c, mom):  # proc:177-205: next anchor on the sphere
            if drift_sq <= 0.0:
                return c, mom
            if self.drift == "smooth":
                g = rng.standard_normal(c.shape)
                mom = MOMENTUM * mom + np.sqrt(drift_sq * (1.0 - MOMENTUM ** 2) / c.size) * g
                nc = c + mom
                return nc * (radius / np.sqrt(np.sum(nc * nc))), mom
            omc = min(drift_sq * rows / (4.0 * anchor_sq), 1.5)
            u, w = _plane(rng, rows)
            cos_t = 1.0 - omc
            sin_t = np.sqrt(max(1.0 - cos_t * cos_t, 0.0))
            p, q = u @ c, w @ c
            return c + (cos_t - 1.0) * (np.outer(u, p) + np.outer(w, q)) + sin_t * (np.outer(w, p) - np.outer(u, q)), mom

        def roll(state, c, mom, n, keep_maps):  # proc:208-228
            out, maps = [], []
            for _ in range(n):
                if self.drift == "scrambled":
                    perm = rng.permutation(rows * cols)
                    signs = np.where(rng.integers(0, 2, rows * cols) == 1, 1.0, -1.0)
                else:
                    perm = signs = None
                prev = c
                c, mom = move(c, mom)
                off = c + rng.standard_normal((rows, cols)) * noise if noise > 0.0 else c
                m = Step(self.L, perm, signs, prev, off)
                state = m.apply(state)
                out.append(state)
                if keep_maps:
                    maps.append(m)
            return out, maps, c, mom

        warm, _, c, mom = roll(state, c, mom, BURN_IN, False)
        states, maps, _, _ = roll(warm[-1], c, mom, steps, keep)
        return warm[-1], states, maps

    def step_map(self, t):
        return self.maps[t - 1]

    def measure(self, probes=8):
        """proc:294-312 measure_stats: (L_hat, sigma_a_sq_hat, sigma_delta_sq_hat)."""
        a_sq, d_sq = _energies([self.initial] + self.states)
        rng = stream(self.seed, 4)
        ratios = []
        for i in range(probes):
            m = self.maps[i % len(self.maps)]
            x = (rng.standard_normal((self.rows, self.cols), dtype=np.float64)).astype(np.float32)
            y = (rng.standard_normal((self.rows, self.cols), dtype=np.float64)).astype(np.float32)
            num = sqnorm(m.apply(x).astype(np.float64) - m.apply(y).astype(np.float64))
            ratios.append(np.sqrt(num / sqnorm(x.astype(np.float64) - y.astype(np.float64))))
        return float(np.mean(ratios)), a_sq, d_sq


def _plane(rng, rows):  # proc:156-165
    while True:
        u = rng.standard_normal(rows)
        u /= np.linalg.norm(u)
        w = rng.standard_normal(rows)
        w -= np.dot(u, w) * u
        nw = np.linalg.norm(w)
        if nw >= 1e-12:
            return u, w / nw


def _energies(states):  # proc:231-236
    a_sq = float(np.mean([sqnorm(s) for s in states]))
    d_sq = float(np.mean([sqnorm(b - a) for a, b in zip(states[:-1], states[1:])]))  # f32 differences
    return a_sq, d_sq


# ---- closed-form bounds (th:54-95) ------------------------------------------

def stability_threshold(L):
    l2 = L * L
    return 1.0 - (1.0 - l2) / (l2 + 1.0)  # th:54-59


def v_naive(delta, L, sigma_a_sq):
    return (1.0 - delta) * sigma_a_sq / (1.0 - L * L)  # th:62-66


def v_residual(delta, L, sigma_delta_sq):
    margin = (1.0 - L * L) - (1.0 - delta) * (L * L + 1.0)  # th:48-51, 69-77
    if margin <= 0.0:
        raise ValueError("residual bound requires delta above the stability threshold")
    return (1.0 - delta) * sigma_delta_sq / margin


def bound_ratio(delta, L, sigma_a_sq, sigma_delta_sq):
    if delta == 1.0:
        return 0.0  # th:80-88
    l2 = L * L
    margin = (1.0 - l2) - (1.0 - delta) * (l2 + 1.0)
    if margin <= 0.0:
        raise ValueError("ratio undefined below the stability threshold")
    return (sigma_delta_sq / sigma_a_sq) * (1.0 - l2) / margin


def no_feedback_growth(delta, sigma_delta_sq, t):
    return t * (1.0 - delta) * sigma_delta_sq  # th:91-95
