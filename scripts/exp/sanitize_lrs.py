"""compute-sanitizer driver for the fused low-rank step (lr_step.cu) and the batched
low-rank decode: a few steps at shard shapes that take the fused kernel (modes, dtypes,
ranks, a rank-deficient input for the in-kernel CGS2 fallback).  Prints the number of
fused launches so a silent fallback is visible."""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2507_17511_b200 import _lib, compressors as cx, pipeline as pl, linalg as la  # noqa: E402

lib = _lib.load()
n0 = lib.cc_debug_lowrank_fused_count()
for (n, c), r, it, mode, dt, i4 in (((1024, 3072), 8, 2, "residual_with_feedback", torch.bfloat16, False),
                                    ((520, 2048), 5, 1, "residual_no_feedback", torch.float32, False),
                                    ((300, 1024), 8, 3, "naive", torch.bfloat16, False),
                                    ((1024, 3072), 8, 2, "residual_with_feedback", torch.bfloat16, True),
                                    ((522, 2048), 3, 1, "naive", torch.float32, True)):
    spec = cx.CompressorSpec(cx.CompressorKind.LOWRANK, rank=r, iterations=it, int4_factors=i4)
    snd = pl.LayerState(mode, 1, torch.zeros(n, c, device="cuda"))
    rcv = pl.LayerState(mode, 1, torch.zeros(n, c, device="cuda"))
    key = la.DeviceKey(3, 5, 2, advance=True)
    for t, x in enumerate(synth.flux_like(n, c, 3, seed=r), start=1):
        p, _ = pl.encode_step(snd, torch.from_numpy(x).cuda().to(dt), spec, rng=key)
        pl.decode_step(rcv, pl.device_message(t, 1, p))
    torch.cuda.synchronize()
    print("ok", n, c, r, it, mode, "int4" if i4 else "f16", flush=True)
g = np.random.default_rng(2)
a = (g.standard_normal((1024, 3)) @ g.standard_normal((3, 3072))).astype(np.float32)
snd = pl.LayerState("naive", 1, torch.zeros(1024, 3072, device="cuda"))
spec = cx.CompressorSpec(cx.CompressorKind.LOWRANK, rank=8, iterations=2)
for t in (1, 2):
    pl.encode_step(snd, a, spec, rng=la.spawn_rng(1, 5, t))
torch.cuda.synchronize()
print("ok rank-deficient; fused launches:", lib.cc_debug_lowrank_fused_count() - n0, flush=True)
