import time, sys, os
sys.path.insert(0, os.getcwd())
import torch, cProfile, pstats
from paper_2507_17511_b200 import compressors as cx, pipeline as pl, linalg as la
n, c = 1024, 3072
spec = cx.CompressorSpec(cx.CompressorKind.LOWRANK, rank=8, iterations=2)
xs = [torch.randn(n, c, device="cuda").to(torch.bfloat16) for _ in range(2)]
st = pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda"))
for i in range(3): pl.encode_step(st, xs[i % 2], spec, rng=la.make_rng(i))
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(20): pl.encode_step(st, xs[i % 2], spec, rng=la.make_rng(i))
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e6*(t1-t0)/20:.1f} us/step, total {1e6*(t2-t0)/20:.1f} us/step")
pr = cProfile.Profile(); pr.enable()
for i in range(20): pl.encode_step(st, xs[i % 2], spec, rng=la.make_rng(i))
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
