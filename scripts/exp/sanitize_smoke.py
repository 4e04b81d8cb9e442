"""Small runs of every device path for compute-sanitizer memcheck."""
import os, sys
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import torch, synth
from paper_2507_17511_b200 import _lib, comm, compressors as cx, pipeline as pl, linalg as la
lib = _lib.load()
for codec, kw in (("quant2bit", {}), ("sign1bit", {}), ("quant4bit", {}), ("topk", {"keep_fraction": 0.05}),
                  ("nm_block", {"n": 2, "m": 4}), ("nm_block", {"n": 3, "m": 6}), ("lowrank", {"rank": 4, "iterations": 2})):
    spec = cx.CompressorSpec(cx.CompressorKind(codec), **kw)
    for n, c in ((64, 3072), (40, 384), (7, 1000)):
        snd = pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda"))
        rcv = pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda"))
        for t, x in enumerate(synth.flux_like(n, c, 3, seed=1), start=1):
            p, _ = pl.encode_step(snd, torch.from_numpy(x).cuda().to(torch.bfloat16), spec, rng=la.make_rng(t))
            pl.decode_step(rcv, pl.device_message(t, 1, p))
        torch.cuda.synchronize()
    print("ok", codec, kw, flush=True)
# segmented (Ulysses) and the rank simulation
spec = cx.CompressorSpec(cx.CompressorKind.SIGN1BIT)
u = comm.UlyssesAllToAll(32, 3072, spec, sim_world=(8, 0))
for x in synth.flux_like(32, 3072, 3, seed=2):
    u.step(torch.from_numpy(x).cuda().to(torch.bfloat16))
torch.cuda.synchronize()
print("ok ulysses segmented")
