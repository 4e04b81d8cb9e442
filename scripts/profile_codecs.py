"""encode_step of the non-quantizer codecs at a per-rank shard shape, for ncu
launch lists (per-kernel durations of the low-rank / top-k / N:M paths).

python scripts/profile_codecs.py --rows 1024 --codec lowrank --rank 8 --reps 3
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2507_17511_b200 import compressors as cx  # noqa: E402
from paper_2507_17511_b200 import linalg as la  # noqa: E402
from paper_2507_17511_b200 import pipeline as pl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1024)
    ap.add_argument("--cols", type=int, default=3072)
    ap.add_argument("--codec", default="lowrank")
    ap.add_argument("--rank", type=int, default=8)
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--keep", type=float, default=0.01)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--time", action="store_true", help="print CUDA-event µs per step instead of profiling")
    ap.add_argument("--device-key", action="store_true", help="low-rank: draw Q0 on the device (linalg.DeviceKey)")
    a = ap.parse_args()
    n, c = a.rows, a.cols
    kind = cx.CompressorKind(a.codec)
    if kind in (cx.CompressorKind.LOWRANK,):
        spec = cx.CompressorSpec(kind, rank=a.rank, iterations=a.iters)
    elif kind == cx.CompressorKind.TOPK:
        spec = cx.CompressorSpec(kind, keep_fraction=a.keep)
    elif kind == cx.CompressorKind.NM_BLOCK:
        spec = cx.CompressorSpec(kind, n=2, m=4)
    else:
        spec = cx.CompressorSpec(kind)
    g = torch.Generator(device="cuda").manual_seed(0)
    xs = [(torch.randn(n, c, device="cuda", generator=g) * torch.rand(1, c, device="cuda", generator=g) * 3)
          .to(torch.bfloat16) for _ in range(2)]
    st = pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda"))
    key = la.DeviceKey(7, 6, 0, 1, advance=True) if a.device_key else None
    pl.encode_step(st, xs[0], spec, rng=key or la.make_rng(0))
    pl.encode_step(st, xs[1], spec, rng=key or la.make_rng(1))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(a.reps):
        pl.encode_step(st, xs[i % 2], spec, rng=key or la.make_rng(2 + i))
    e1.record()
    torch.cuda.synchronize()
    if a.time:
        print(f"{a.codec} [{n}x{c}] {e0.elapsed_time(e1) * 1e3 / a.reps:.1f} us/step")


if __name__ == "__main__":
    main()
