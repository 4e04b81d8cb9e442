"""One low-rank encode (r=8, T=2) and one top-k encode_step at [1024, 3072] for kernel traces."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_17511_b200 import compressors as cx, pipeline as pl, linalg as la
n, c = 1024, 3072
x = (torch.randn(n, c, device="cuda") * torch.rand(1, c, device="cuda")).to(torch.bfloat16)
x2 = (x.float() + 0.1 * torch.randn(n, c, device="cuda")).to(torch.bfloat16)
sp = cx.CompressorSpec(cx.CompressorKind.LOWRANK, rank=8, iterations=2)
for i in range(2):
    cx.encode_lowrank(x.float(), sp, la.make_rng(i))
st = pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda"))
tk = cx.CompressorSpec(cx.CompressorKind.TOPK, keep_fraction=0.01)
pl.encode_step(st, x, tk)
for i in range(2):
    pl.encode_step(st, x2 if i % 2 == 0 else x, tk)
torch.cuda.synchronize()
