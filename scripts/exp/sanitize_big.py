"""compute-sanitizer driver at shard shapes that take the persistent kernels: K1
shard-resident ([512 / 1024 / 4096, 3072]), the resident top-k ([512, 3072]), N:M, and
the batched decodes (2 steps each)."""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2507_17511_b200 import _lib, compressors as cx, pipeline as pl, linalg as la  # noqa: E402

lib = _lib.load()
k1 = lib.cc_debug_k1_resident_count()
tk = lib.cc_debug_topk_resident_count()
cases = [("quant2bit", {}, n) for n in (512, 1024, 4096)] + [("topk", {"keep_fraction": 0.01}, 512),
                                                               ("nm_block", {"n": 2, "m": 4}, 1024)]
for codec, kw, n in cases:
    spec = cx.CompressorSpec(cx.CompressorKind(codec), **kw)
    snd = pl.LayerState("residual_with_feedback", 1, torch.zeros(n, 3072, device="cuda"))
    rcv = pl.LayerState("residual_with_feedback", 1, torch.zeros(n, 3072, device="cuda"))
    for t, x in enumerate(synth.flux_like(n, 3072, 3, seed=1), start=1):
        p, _ = pl.encode_step(snd, torch.from_numpy(x).cuda().to(torch.bfloat16), spec, rng=la.make_rng(t))
        pl.decode_step(rcv, pl.device_message(t, 1, p))
    torch.cuda.synchronize()
    print("ok", codec, kw, n, flush=True)
print("k1 resident launches", lib.cc_debug_k1_resident_count() - k1, "topk resident launches",
      lib.cc_debug_topk_resident_count() - tk, flush=True)
