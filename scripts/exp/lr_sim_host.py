"""Host vs device time of one low-rank (r=8, T=2) patch-parallel exchange step at the
P=4 per-rank shape, eager: where the host time goes (cProfile) and the GPU-only time
(the same launches replayed with the Q0 draw hoisted out)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_2507_17511_b200 import compressors as cx  # noqa: E402
from paper_2507_17511_b200 import linalg as la  # noqa: E402
from paper_2507_17511_b200.comm import PatchParallelExchange  # noqa: E402

rows, cols, P, L = 4096, 3072, 4, 16
spec = cx.CompressorSpec(cx.CompressorKind.LOWRANK, rank=8, iterations=2)
exs = [PatchParallelExchange(rows, cols, spec, sim_world=(P, 0)) for _ in range(L)]
n = rows // P
xs = [torch.randn(n, cols, device="cuda").to(torch.bfloat16) for _ in range(2)]


def step(s):
    for i, e in enumerate(exs):
        e.step(xs[s % 2], rng=la.make_rng(1000 * i + s))


for s in range(4):
    step(s)
torch.cuda.synchronize()
t0 = time.perf_counter()
for s in range(5):
    step(s)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e6 * (t1 - t0) / (5 * L):.1f} us/layer, wall {1e6 * (t2 - t0) / (5 * L):.1f} us/layer")
t0 = time.perf_counter()
for i in range(100):
    la.gaussian_matrix(la.make_rng(i), cols, 8)
print(f"Q0 draw {1e6 * (time.perf_counter() - t0) / 100:.1f} us")
# eager GPU time: queue the steps behind a long spin so the host is far ahead of the GPU
for s in range(2):
    step(s)
torch.cuda.synchronize()
ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(int(4e8))
ea.record()
h0 = time.perf_counter()
for s in range(5):
    step(s)
h1 = time.perf_counter()
for e in exs:
    if e.streams.decode is not None:
        torch.cuda.current_stream().wait_stream(e.streams.decode)
eb.record()
torch.cuda.synchronize()
print(f"eager GPU time behind a spin: {1e3 * ea.elapsed_time(eb) / (5 * L):.1f} us/layer "
      f"(host enqueue {1e6 * (h1 - h0) / (5 * L):.1f} us/layer)")
pr = cProfile.Profile()
pr.enable()
for s in range(3):
    step(s)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)

# the same step with Q0 drawn once (host draw removed): eager, then CUDA-graph replay (GPU time)
_q = {}
_orig = cx.subspace_init
cx.subspace_init = lambda rng, c, r: _q[(c, r)] if (c, r) in _q else _q.setdefault((c, r), _orig(rng, c, r))
for s in range(3):
    step(s)
torch.cuda.synchronize()
t0 = time.perf_counter()
for s in range(5):
    step(s)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"no-draw eager: host enqueue {1e6 * (t1 - t0) / (5 * L):.1f} us/layer, wall {1e6 * (t2 - t0) / (5 * L):.1f}")
streams = exs[0].streams
for e in exs[1:]:
    e.streams = streams
step(0)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step(1)
    torch.cuda.current_stream().wait_stream(streams.decode)
for e in exs:
    e.after_capture()
g.replay()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    g.replay()
b.record()
torch.cuda.synchronize()
print(f"graph replay (GPU time): {1e3 * a.elapsed_time(b) / (5 * L):.1f} us/layer")
