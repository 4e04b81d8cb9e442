"""Golden digests of the REFERENCE synthetic process (process.make_process) for the
closed-loop stability harness oracle (oracle/process_oracle.py).  Run in the build
container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_process_golden.py

Writes tests/golden/process_digests.json: per spec, sha256 of the initial state and of
all recorded states (f32 LE bytes), the first state's first entries, and measure_stats.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from compactcomm import process  # noqa: E402

SPECS = [
    dict(rows=64, cols=64, lipschitz=0.5, sigma_a_sq=100.0, sigma_delta_sq=1.0, steps=200, seed=7, drift="walk"),
    dict(rows=16, cols=16, lipschitz=0.5, sigma_a_sq=100.0, sigma_delta_sq=1.0, steps=40, seed=3, drift="walk"),
    dict(rows=32, cols=24, lipschitz=0.3, sigma_a_sq=50.0, sigma_delta_sq=2.0, steps=30, seed=11, drift="smooth"),
    dict(rows=16, cols=8, lipschitz=0.7, sigma_a_sq=10.0, sigma_delta_sq=0.5, steps=20, seed=5, drift="scrambled"),
]


def digest(arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a, dtype="<f4").tobytes())
    return h.hexdigest()


def main():
    out = []
    for d in SPECS:
        tr = process.make_process(process.ProcessSpec(**d))
        l_hat, a_sq, d_sq = process.measure_stats(tr)
        out.append({"spec": d, "initial": digest([tr.initial]), "states": digest(tr.states),
                    "head": [float(v) for v in np.asarray(tr.states[0]).ravel()[:4]],
                    "stats": [l_hat, a_sq, d_sq]})
    with open(os.path.join(HERE, "process_digests.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", len(out), "process digests")


if __name__ == "__main__":
    main()
