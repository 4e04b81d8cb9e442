"""Experiment: config-1 step graph instantiated with per-node priorities
(cudaGraphInstantiateFlagUseNodePriority): K1 captured from a high-priority compute
stream, K2 from a low-priority decode stream, so when both become ready the K1's CTAs
are dispatched first and the decode fills the SMs K1 leaves free.
python scripts/exp/prio_ab.py <use_priority 0|1>"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402
from cuda.bindings import runtime as rt  # noqa: E402

import bench  # noqa: E402
from paper_2507_17511_b200 import comm  # noqa: E402
from paper_2507_17511_b200 import compressors as cx  # noqa: E402


def main():
    prio = int(sys.argv[1])
    L, rows, cols = 57, 4096, 3072
    dev = torch.device("cuda", 0)
    lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -5)
    cap_stream = torch.cuda.Stream(priority=-5 if prio else 0)
    spec = cx.CompressorSpec(cx.CompressorKind.QUANT2BIT)
    exs = [comm.PatchParallelExchange(rows, cols, spec) for _ in range(L)]
    for e in exs[1:]:
        e.streams = exs[0].streams
    S = exs[0].streams
    S._decode = torch.cuda.Stream(priority=0)
    S._comm = torch.cuda.Stream(priority=-5 if prio else 0)
    inputs = [bench.flux_inputs(rows, cols, 0, rows, l, dev) for l in range(L)]

    def one(par):
        for l, e in enumerate(exs):
            e.step(inputs[l][par])

    with torch.cuda.stream(cap_stream):
        one(0)
        for s in range(3):
            one((s + 1) % 2)
    torch.cuda.synchronize()
    execs = []
    graphs = []
    for p in (0, 1):
        g = torch.cuda.CUDAGraph(keep_graph=True)
        with torch.cuda.graph(g, stream=cap_stream):
            one(p)
            torch.cuda.current_stream().wait_stream(S.decode)
        graphs.append(g)
        raw = g.raw_cuda_graph()
        flags = rt.cudaGraphInstantiateFlags.cudaGraphInstantiateFlagUseNodePriority if prio else 0
        err, ex = rt.cudaGraphInstantiateWithFlags(raw, flags)
        assert err == rt.cudaError_t.cudaSuccess, err
        execs.append(ex)
    for e in exs:
        e.after_capture()
    run_stream = torch.cuda.Stream(priority=-5 if prio else 0)
    for k in range(4):
        rt.cudaGraphLaunch(execs[k % 2], run_stream.cuda_stream)
    torch.cuda.synchronize()
    K = 10
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(run_stream)
    for k in range(K):
        rt.cudaGraphLaunch(execs[k % 2], run_stream.cuda_stream)
    b.record(run_stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / K
    print({"node_priority": prio, "us_per_layer": round(ms / L * 1e3, 2),
           "GBs": round(L * 2 * rows * cols / (ms / 1e3) / 1e9, 1)}, flush=True)


if __name__ == "__main__":
    main()
