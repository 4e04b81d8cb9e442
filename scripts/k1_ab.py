"""A/B of the K1 kernels: shard-resident (k1_resident.cu) vs streaming
(k1_fused_impl.cuh) encode_step at the per-rank shard heights, CUDA-graph replay
over L layer channels (L2-cold: the layers' state far exceeds L2 at the larger
shapes), mean µs per K1 and algorithmic GB/s (18 + b/8 B per element + scales).

python scripts/k1_ab.py [--rows 512,1024,2048,4096] [--layers 16] [--codec quant2bit]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2507_17511_b200 import _lib  # noqa: E402
from paper_2507_17511_b200 import compressors as cx  # noqa: E402
from paper_2507_17511_b200 import pipeline as pl  # noqa: E402


def graph_time(fn, reps):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.current_stream()):
        for i in range(reps):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = None
    for _ in range(3):
        s.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) * 1e3 / reps
        best = us if best is None else min(best, us)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", default="512,1024,2048,4096")
    ap.add_argument("--cols", type=int, default=3072)
    ap.add_argument("--layers", type=int, default=16)
    ap.add_argument("--codec", default="quant2bit")
    ap.add_argument("--mode", default="residual_with_feedback")
    ap.add_argument("--per-sm", action="store_true")
    ap.add_argument("--policies", default="", type=lambda v: [int(x) for x in v.split(",") if x])
    a = ap.parse_args()
    lib = _lib.load()
    torch.cuda.set_stream(torch.cuda.Stream())
    spec = cx.CompressorSpec(cx.CompressorKind(a.codec))
    bits = {"sign1bit": 1, "quant2bit": 2, "quant4bit": 4}[a.codec]
    mode = pl._MODE_CODE[pl.PipelineMode(a.mode)]
    tag = cx._spec_tag(spec)
    out = []
    for n in [int(r) for r in a.rows.split(",")]:
        c, L = a.cols, a.layers
        xs = [(torch.randn(n, c, device="cuda") * torch.rand(1, c, device="cuda") * 3).to(torch.bfloat16)
              for _ in range(2 * L)]
        sts = [pl.LayerState(a.mode, 1, torch.zeros(n, c, device="cuda")) for _ in range(L)]
        for i, st in enumerate(sts):
            pl.encode_step(st, xs[2 * i], spec)
            pl.encode_step(st, xs[2 * i + 1], spec)
        wsb = lib.cc_workspace_bytes(tag, n, c, 0)
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        body = torch.empty(lib.cc_body_bytes(tag, n, c, 0) + 64, dtype=torch.uint8, device="cuda")
        rec = torch.zeros(2, dtype=torch.float64, device="cuda")
        stream = _lib.stream_ptr()

        def enc(i):
            st = sts[i % L]
            _lib.check(lib.cc_encode_step(tag, mode, 0, n, c, _lib.ptr(xs[2 * (i % L) + (i // L) % 2]), _lib.CC_BF16,
                                          _lib.ptr(st.base), _lib.ptr(st._aux()), _lib.ptr(body), _lib.ptr(ws), wsb,
                                          _lib.ptr(rec), stream))

        algo = n * c * (18 + bits / 8) + 4 * (n + c)
        row = {"rows": n, "cols": c, "codec": a.codec, "algo_MB": round(algo / 1e6, 2)}
        for name, flag in (("resident", 1), ("streaming", 0)):
            lib.cc_debug_k1_resident(flag)
            c0 = lib.cc_debug_k1_resident_count()
            enc(0)
            torch.cuda.synchronize()
            used = lib.cc_debug_k1_resident_count() - c0
            us = graph_time(enc, 2 * L)
            row[name] = {"us": round(us, 2), "GBs": round(algo / us / 1e3, 1), "resident_ran": bool(used)}
        # per-phase timeline of the resident launch (globaltimer stamps per CTA, last of
        # 2L back-to-back eager launches), [min, max] over CTAs in µs from the first start
        lib.cc_debug_k1_resident(1)
        tbuf = torch.zeros(1024 * 16, dtype=torch.int64, device="cuda")
        lib.cc_debug_fused_timer(_lib.ptr(tbuf))
        for i in range(2 * L):
            enc(i)
        torch.cuda.synchronize()
        lib.cc_debug_fused_timer(None)
        tb = tbuf.view(1024, 16).cpu()
        g = int((tb[:, 0] > 0).sum())
        tb = tb[:g].double()
        t0 = tb[:, 0].min()
        names = ["start", "first_data", "A_done", "sync1", "F_done", "sync2", "B_done", "end", "smid", "colpart_done", "pre_arrive", "arrived", "rec_part", "ticket"]
        row["resident_timeline_us"] = {nm: [round(float((tb[:, i] - t0).min()) / 1e3, 2),
                                            round(float((tb[:, i] - t0).max()) / 1e3, 2)]
                                       for i, nm in enumerate(names) if nm != "smid"}
        if a.per_sm:  # phase-A end per SM id (imbalance map)
            sm = tb[:, 8].long()
            ad = (tb[:, 2] - t0) / 1e3
            order = torch.argsort(sm)
            row["A_done_by_smid"] = [[int(sm[i]), round(float(ad[i]), 2)] for i in order.tolist()]
        for pol in a.policies:
            lib.cc_debug_fused_policy(pol)
            enc(0)
            row[f"resident_policy{pol}_us"] = round(graph_time(enc, 2 * L), 2)
        lib.cc_debug_fused_policy(0)
        print(json.dumps(row), flush=True)
        out.append(row)
        del xs, sts
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
