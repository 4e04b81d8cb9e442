"""One K1 shard-resident step at [4096, 3072] (tensor-memory form) for compute-sanitizer."""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2507_17511_b200 import compressors as cx, pipeline as pl, linalg as la  # noqa: E402

spec = cx.CompressorSpec(cx.CompressorKind.QUANT2BIT)
snd = pl.LayerState("residual_with_feedback", 1, torch.zeros(4096, 3072, device="cuda"))
for t, x in enumerate(synth.flux_like(4096, 3072, 2, seed=1), start=1):
    pl.encode_step(snd, torch.from_numpy(x).cuda().to(torch.bfloat16), spec, rng=la.make_rng(t))
torch.cuda.synchronize()
print("ok")
