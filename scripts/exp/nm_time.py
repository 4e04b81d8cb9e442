"""Graph-replayed N:M (2:4) encode_step (16 layer states, L2-cold rotation) at a shard shape."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_2507_17511_b200 import compressors as cx  # noqa: E402
from paper_2507_17511_b200 import pipeline as pl  # noqa: E402

L = 16
for rows in (4096, 512):
    for keep in (0,):
        spec = cx.CompressorSpec(cx.CompressorKind.NM_BLOCK, n=2, m=4)
        g = torch.Generator(device="cuda").manual_seed(0)
        xs = [(torch.randn(rows, 3072, device="cuda", generator=g) * torch.rand(1, 3072, device="cuda", generator=g)
               * 3).to(torch.bfloat16) for _ in range(L)]
        sts = [pl.LayerState("residual_with_feedback", 1, torch.zeros(rows, 3072, device="cuda")) for _ in range(L)]
        for _ in range(2):
            for s, x in zip(sts, xs):
                pl.encode_step(s, x, spec)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for s, x in zip(sts, xs):
                pl.encode_step(s, x, spec)
        gr.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            gr.replay()
        b.record()
        torch.cuda.synchronize()
        print(f"nm2:4 {rows}x3072: {1e3 * a.elapsed_time(b) / (10 * L):.1f} us/step")
