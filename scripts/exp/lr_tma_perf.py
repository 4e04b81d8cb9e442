"""Per-kernel time of the tcgen05 projections, TMA-staged vs register-staged (ncu launch list)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2507_17511_b200 import _lib, compressors as cx, linalg as la
lib = _lib.load()
tma = int(sys.argv[1]); n = int(sys.argv[2])
lib.cc_debug_lowrank_tma(tma, 0)
t = torch.randn(n, 3072, device="cuda")
sp = cx.CompressorSpec(cx.CompressorKind.LOWRANK, rank=8, iterations=2)
for i in range(2):
    cx.encode_lowrank(t, sp, la.make_rng(i))
torch.cuda.synchronize()
