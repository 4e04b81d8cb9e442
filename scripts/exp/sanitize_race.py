import os, sys
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import torch, synth
from paper_2507_17511_b200 import _lib, compressors as cx, pipeline as pl, linalg as la
which = sys.argv[1]
spec = {"q2": cx.CompressorSpec(cx.CompressorKind.QUANT2BIT),
        "lr": cx.CompressorSpec(cx.CompressorKind.LOWRANK, rank=4, iterations=1),
        "tk": cx.CompressorSpec(cx.CompressorKind.TOPK, keep_fraction=0.05)}[which]
n, c = (256, 3072) if which != "lr" else (256, 1024)
snd = pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda"))
for t, x in enumerate(synth.flux_like(n, c, 2, seed=1), start=1):
    pl.encode_step(snd, torch.from_numpy(x).cuda().to(torch.bfloat16), spec, rng=la.make_rng(t))
torch.cuda.synchronize()
print("ok", which)
