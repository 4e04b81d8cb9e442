"""Stress: persistent K1 vs multi-kernel K1, bit-for-bit over many full-shape steps."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2507_17511_b200 import _lib, compressors as cx, pipeline as pl
lib = _lib.load()
n, c = int(sys.argv[1]), 3072
steps = int(sys.argv[2])
spec = cx.CompressorSpec(cx.CompressorKind.QUANT2BIT)
g = torch.Generator(device="cuda").manual_seed(1)
x0 = torch.randn(n, c, device="cuda", generator=g) * torch.rand(1, c, device="cuda", generator=g) * 3
sa = pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda"))
sb = pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda"))
bad = 0
for t in range(steps):
    x = (x0 + 0.1 * t * torch.randn(n, c, device="cuda", generator=g)).to(torch.bfloat16)
    lib.cc_set_quant_path(-1)
    pa, _ = pl.encode_step(sa, x, spec)
    lib.cc_set_quant_path(0)
    pb, _ = pl.encode_step(sb, x, spec)
    lib.cc_set_quant_path(-1)
    same = torch.equal(pa.body, pb.body) and torch.equal(sa.base, sb.base) and torch.equal(sa.feedback, sb.feedback)
    if not same:
        bad += 1
        sb.base.copy_(sa.base); sb.feedback.copy_(sa.feedback)
print(f"rows {n}: {steps} steps, mismatching steps: {bad}")
