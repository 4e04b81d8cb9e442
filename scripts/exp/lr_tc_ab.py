"""A/B of the low-rank tcgen05 projection variants (TMA-staged vs register-staged)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2507_17511_b200 import _lib, compressors as cx, linalg as la
lib = _lib.load()
for n in (1024, 4096):
    t = torch.randn(n, 3072, device="cuda")
    for r in (8, 16):
        sp = cx.CompressorSpec(cx.CompressorKind.LOWRANK, rank=r, iterations=2)
        res = {}
        for name, tma, waves in (("reg", 0, 0), ("tma1", 1, 1), ("tma2", 1, 2), ("tma4", 1, 4)):
            lib.cc_debug_lowrank_tma(tma, waves)
            p = cx.encode_lowrank(t, sp, la.make_rng(0))
            err = float(((p.decode() - t).norm() / t.norm()).item())
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(10):
                cx.encode_lowrank(t, sp, la.make_rng(i))
            e1.record()
            torch.cuda.synchronize()
            res[name] = (round(e0.elapsed_time(e1) * 100, 1), round(err, 7))
        print(n, r, res, flush=True)
lib.cc_debug_lowrank_tma(1, 1)
