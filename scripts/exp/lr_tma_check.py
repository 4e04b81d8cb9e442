"""TMA-staged vs register-staged tcgen05 projections must give identical payloads."""
import os, sys
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import torch, synth
from paper_2507_17511_b200 import _lib, compressors as cx, linalg as la
lib = _lib.load()
for (n, c) in ((1024, 3072), (4096, 3072), (200, 1000), (64, 384)):
    x = torch.from_numpy(synth.flux_like(n, c, 1, seed=n)[0]).cuda()
    for r in (4, 8, 16, 32):
        sp = cx.CompressorSpec(cx.CompressorKind.LOWRANK, rank=r, iterations=2)
        out = []
        for tma in (0, 1, 1):
            lib.cc_debug_lowrank_tma(tma, 0)
            p = cx.encode_lowrank(x, sp, la.make_rng(r))
            out.append(p.body.cpu())
        print(n, c, r, "tma==reg:", torch.equal(out[0], out[1]), "tma deterministic:", torch.equal(out[1], out[2]),
              "max|diff| f16:", float((out[0].view(torch.float16).float() - out[1].view(torch.float16).float()).abs().max()) if out[0].numel() % 2 == 0 else None)
lib.cc_debug_lowrank_tma(2, 0)
