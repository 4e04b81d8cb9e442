"""Fused low-rank encode_step (lr_step.cu, one cluster launch) vs the multi-kernel
step: reconstruction error per step on drifting activations, sender/receiver
agreement, graph-replayed step time, and the fused kernel's phase stamps.

    python scripts/exp/lr_fused_ab.py [rows] [cols] [rank] [iters]
"""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_17511_b200 import _lib  # noqa: E402
from paper_2507_17511_b200 import compressors as cx  # noqa: E402
from paper_2507_17511_b200 import linalg as la  # noqa: E402
from paper_2507_17511_b200 import pipeline as pl  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
cols = int(sys.argv[2]) if len(sys.argv) > 2 else 3072
rank = int(sys.argv[3]) if len(sys.argv) > 3 else 8
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 2
lib = _lib.load()
torch.manual_seed(0)
g = np.random.default_rng(0)
scale = torch.from_numpy((g.random((1, cols)) * 3 + 0.1).astype(np.float32)).cuda()
lowr = torch.randn(rows, 12, device="cuda") @ torch.randn(12, cols, device="cuda")
xs = [((lowr * (1 + 0.05 * t) + 0.3 * torch.randn(rows, cols, device="cuda")) * scale).to(torch.bfloat16)
      for t in range(8)]
spec = cx.CompressorSpec(cx.CompressorKind.LOWRANK, rank=rank, iterations=iters)
MODE = pl.PipelineMode.RESIDUAL_WITH_FEEDBACK


def fresh():
    return pl.LayerState(MODE, 1, torch.zeros(rows, cols, device="cuda"))


def run(fused, steps=6):
    lib.cc_debug_lowrank_fused(fused)
    n0 = lib.cc_debug_lowrank_fused_count()
    snd, rcv = fresh(), fresh()
    key = la.DeviceKey(5, 6, 0, 2, advance=True)
    out = []
    for t in range(steps):
        p, rec = pl.encode_step(snd, xs[t], spec, rng=key)
        pl.decode_step(rcv, pl.message_for(snd.step, 1, p))
        torch.cuda.synchronize()
        tgt = xs[t].float()
        rel = float((snd.base - tgt).norm() / tgt.norm())
        out.append((rel, rec.compression_error, bool(torch.equal(rcv.base, snd.base))))
    return out, lib.cc_debug_lowrank_fused_count() - n0


for fused in (1, 0):
    res, used = run(fused)
    print(f"fused={fused} (fused launches {used}):")
    for t, (rel, ce, same) in enumerate(res):
        print(f"   step {t}: relerr(base vs x) {rel:.6f}  record {ce:.10g}  receiver==sender {same}")


def graph_time(fn, reps=10):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn(0)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            for i in range(reps):
                fn(i)
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / reps


for fused in (1, 0):
    lib.cc_debug_lowrank_fused(fused)
    snd = fresh()
    key = la.DeviceKey(5, 6, 0, 2, advance=True)
    pl.encode_step(snd, xs[0], spec, rng=key)  # warmup step
    us = graph_time(lambda i: pl.encode_step(snd, xs[3 + i % 2], spec, rng=key), reps=6)
    print(f"graph-replayed encode_step [{rows}x{cols}] r{rank} T{iters} fused={fused}: {us:.1f} us")

lib.cc_debug_lowrank_fused(1)
st = torch.zeros(48, dtype=torch.int64, device="cuda")
snd = fresh()
key = la.DeviceKey(5, 6, 0, 2, advance=True)
pl.encode_step(snd, xs[0], spec, rng=key)
pl.encode_step(snd, xs[1], spec, rng=key)
torch.cuda.synchronize()
lib.cc_debug_lowrank_fused_stamps(_lib.ptr(st))
pl.encode_step(snd, xs[2], spec, rng=key)
torch.cuda.synchronize()
lib.cc_debug_lowrank_fused_stamps(None)
v = [x for x in st.cpu().tolist() if x]
print("   stamp deltas (us):", " ".join(f"{(v[k] - v[k - 1]) / 1000:.2f}" for k in range(1, len(v))))
print(f"   total (CTA 0): {(v[-1] - v[0]) / 1000:.2f} us")
