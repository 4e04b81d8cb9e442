"""Short driver for ncu captures of the config-1 path: `--reps` rounds of K1
encode_step + K2 loopback decode_step, rotating over `--layers` layer channels
(inputs L2-cold).  Not a benchmark: run it under ncu.

    ncu --set full -k regex:k1_fused -s 4 -c 1 -o gpurun_out/k1 python scripts/profile_path.py
"""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2507_17511_b200 import _lib  # noqa: E402
from paper_2507_17511_b200 import compressors as cx  # noqa: E402
from paper_2507_17511_b200 import pipeline as pl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=4096)
    ap.add_argument("--cols", type=int, default=3072)
    ap.add_argument("--layers", type=int, default=6)
    ap.add_argument("--reps", type=int, default=8)
    ap.add_argument("--codec", default="quant2bit")
    a = ap.parse_args()
    lib = _lib.load()
    n, c, L = a.rows, a.cols, a.layers
    spec = cx.CompressorSpec(cx.CompressorKind(a.codec))
    g = torch.Generator(device="cuda").manual_seed(0)
    xs = [(torch.randn(n, c, device="cuda", generator=g) * torch.rand(1, c, device="cuda", generator=g) * 3)
          .to(torch.bfloat16) for _ in range(2 * L)]
    snd = [pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda")) for _ in range(L)]
    rcv = [pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda")) for _ in range(L)]
    step = 0
    for r in range(a.reps):
        for i in range(L):
            payload, _ = pl.encode_step(snd[i], xs[2 * i + (r % 2)], spec)
            pl.decode_step(rcv[i], pl.device_message(snd[i].step, snd[i].warmup_steps, payload))
            step += 1
    torch.cuda.synchronize()
    print(f"profile_path: {step} encode_step launches, codec {a.codec}, [{n}x{c}]")


if __name__ == "__main__":
    main()
