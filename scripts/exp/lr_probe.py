"""A few fused low-rank encode_steps on a fresh state ([1024, 3072] r8 T2, drifting
inputs): the driver for ncu captures of lrs::k_lr_step."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_2507_17511_b200 import compressors as cx  # noqa: E402
from paper_2507_17511_b200 import linalg as la  # noqa: E402
from paper_2507_17511_b200 import pipeline as pl  # noqa: E402

rows, cols = int(sys.argv[1]) if len(sys.argv) > 1 else 1024, 3072
torch.manual_seed(0)
scale = torch.rand(1, cols, device="cuda") * 3 + 0.1
lowr = torch.randn(rows, 12, device="cuda") @ torch.randn(12, cols, device="cuda")
xs = [((lowr * (1 + 0.05 * t) + 0.3 * torch.randn(rows, cols, device="cuda")) * scale).to(torch.bfloat16)
      for t in range(8)]
spec = cx.CompressorSpec(cx.CompressorKind.LOWRANK, rank=8, iterations=2)
snd = pl.LayerState(pl.PipelineMode.RESIDUAL_WITH_FEEDBACK, 1, torch.zeros(rows, cols, device="cuda"))
key = la.DeviceKey(5, 6, 0, 2, advance=True)
for t in range(6):
    pl.encode_step(snd, xs[t], spec, rng=key)
torch.cuda.synchronize()
