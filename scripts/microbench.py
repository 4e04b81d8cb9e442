"""Kernel microbenchmarks (CUDA events, warm, L2-cold by rotating over layers).

python scripts/microbench.py [--rows 4096] [--cols 3072] [--layers 16] [--codec quant2bit]
Prints one line per kernel variant: mean µs and GB/s of algorithmic bytes.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2507_17511_b200 import _lib  # noqa: E402
from paper_2507_17511_b200 import compressors as cx  # noqa: E402
from paper_2507_17511_b200 import pipeline as pl  # noqa: E402


def timed(fn, reps, graph=True):
    """Mean µs per call.  graph=True captures the `reps` calls into one CUDA graph
    and times a replay, so host launch overhead never leaves the GPU idle."""
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=torch.cuda.current_stream()):
            for i in range(reps):
                fn(i)
        g.replay()
        torch.cuda.synchronize()
        s.record()
        g.replay()
        e.record()
    else:
        s.record()
        for i in range(reps):
            fn(i)
        e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=4096)
    ap.add_argument("--cols", type=int, default=3072)
    ap.add_argument("--layers", type=int, default=16)
    ap.add_argument("--codec", default="quant2bit")
    ap.add_argument("--reps", type=int, default=48)
    a = ap.parse_args()
    lib = _lib.load()
    torch.cuda.set_stream(torch.cuda.Stream())  # a capturable (non-legacy) stream for every launch
    n, c, L = a.rows, a.cols, a.layers
    spec = cx.CompressorSpec(cx.CompressorKind(a.codec))
    bits = {"sign1bit": 1, "quant2bit": 2, "quant4bit": 4}[a.codec]
    # two alternating activations per layer (as in bench.py): nonzero residuals every step
    xs = [(torch.randn(n, c, device="cuda") * torch.rand(1, c, device="cuda") * 3).to(torch.bfloat16)
          for _ in range(2 * L)]
    sts = [pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda")) for _ in range(L)]
    for i, st in enumerate(sts):  # warmup protocol step + one compressed step
        pl.encode_step(st, xs[2 * i], spec)
        pl.encode_step(st, xs[2 * i + 1], spec)
    tag = cx._spec_tag(spec)
    wsb = lib.cc_workspace_bytes(tag, n, c, 0)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    body = torch.empty(lib.cc_body_bytes(tag, n, c, 0) + 64, dtype=torch.uint8, device="cuda")
    rec = torch.zeros(2, dtype=torch.float64, device="cuda")
    stream = _lib.stream_ptr()

    def enc(i):
        st = sts[i % L]
        lib.cc_encode_step(tag, 2, 0, n, c, _lib.ptr(xs[2 * (i % L) + (i // L) % 2]), _lib.CC_BF16, _lib.ptr(st.base),
                           _lib.ptr(st.feedback), _lib.ptr(body), _lib.ptr(ws), wsb, _lib.ptr(rec), stream)

    out = {}
    alg = n * c * (18 + bits / 8)
    for name, path, stop in (("k1_multikernel", 0, 0), ("k1_fused", -1, 0), ("k1_fused_phaseA", -1, 1),
                             ("k1_fused_phaseA+F", -1, 2)):
        lib.cc_set_quant_path(path)
        lib.cc_debug_fused_stop(stop)
        for i in range(L):
            enc(i)
        us = timed(enc, a.reps)
        out[name] = {"us": round(us, 2), "alg_GBps": round(alg / us / 1e3, 1)}
    lib.cc_set_quant_path(-1)
    lib.cc_debug_fused_stop(0)
    # experiment bits (k1_fused.cu Params::policy): 1 = phase-B stores without L2 hint,
    # 2 = phase-B loads evict_first, 4 = phase-A loads evict_normal, 8 = phase-A
    # consumers skip the math, 16 = skip row finishing, 32 = control words in the workspace
    for pol, stop in ((1, 0), (2, 0), (4, 0), (32, 0), (128, 0), (15 << 8, 0), (5 << 8, 0), (6 << 8, 0), (7 << 8, 0), (8 << 8, 0), (0, 1), (8, 1), (0, 3)):
        lib.cc_debug_fused_policy(pol)
        lib.cc_debug_fused_stop(stop)
        for i in range(L):
            enc(i)
        us = timed(enc, a.reps)
        out[f"k1_fused_policy{pol}{'_stop%d' % stop if stop else ''}"] = {"us": round(us, 2)}
    lib.cc_debug_fused_policy(0)
    lib.cc_debug_fused_stop(0)
    for si, so in ((6, 1), (4, 2), (3, 3), (2, 4), (7, 1)):
        lib.cc_debug_fused_rings(si, so)
        for i in range(L):
            enc(i)
        us = timed(enc, a.reps)
        out[f"k1_fused_rings{si}_{so}"] = {"us": round(us, 2), "alg_GBps": round(alg / us / 1e3, 1)}
    lib.cc_debug_fused_rings(0, 0)
    # phase-A tile height / ring depth sweep (phase A only and full step)
    for ra, sa in ((1, 2), (1, 4), (1, 8), (2, 2), (2, 3), (2, 4), (2, 8), (3, 2), (4, 2)):
        lib.cc_debug_fused_phase_a(ra, sa)
        for stop in (1, 0):
            lib.cc_debug_fused_stop(stop)
            for i in range(L):
                enc(i)
            us = timed(enc, a.reps)
            out[f"k1_fused_A{ra}x{sa}{'_phaseA' if stop else ''}"] = {"us": round(us, 2)}
    lib.cc_debug_fused_phase_a(0, 0)
    lib.cc_debug_fused_stop(0)
    # per-phase timeline of one fused launch (globaltimer stamps per CTA)
    tbuf = torch.zeros(1024 * 16, dtype=torch.int64, device="cuda")
    for pol in (0, 8 | 64):  # 8|64: data movement only (both phases skip the math)
        lib.cc_debug_fused_policy(pol)
        lib.cc_debug_fused_timer(_lib.ptr(tbuf))
        for i in range(2 * L):  # steady state: the previous launch's dirty lines drain during this one
            enc(i)
        torch.cuda.synchronize()
        lib.cc_debug_fused_timer(None)
        tb = tbuf.view(1024, 16).cpu()
        g = int((tb[:, 0] > 0).sum())
        tb = tb[:g].double()
        t0 = tb[:, 0].min()
        names = ["start", "A_done", "sync1", "F_done", "sync2", "B_done", "end", "F_cols", "A_first_data", "A_cons_done", "A_loader_drained"]
        out[f"fused_timeline_us{'_movement_only' if pol else ''}"] = {
            nm: [round(float((tb[:, i] - t0).min()) / 1e3, 2), round(float((tb[:, i] - t0).max()) / 1e3, 2)]
            for i, nm in enumerate(names)}
        out["fused_grid"] = g
    lib.cc_debug_fused_policy(8 | 64)
    for i in range(L):
        enc(i)
    out["k1_fused_movement_only"] = {"us": round(timed(enc, a.reps), 2)}
    lib.cc_debug_fused_policy(0)
    for pol, nm in ((16384, "static"), (0, "hybrid"), (32768, "dynamic"), (16384, "static"), (0, "hybrid"),
                    (32768, "dynamic")):  # tile schedules (see Params::static_sched)
        lib.cc_debug_fused_policy(pol)
        for i in range(L):
            enc(i)
        out.setdefault(f"k1_fused_sched_{nm}", {"us": []})["us"].append(round(timed(enc, a.reps), 2))
    lib.cc_debug_fused_policy(0)
    for mult, keep in ((-1, 1), (2, 2)):  # phase-B end-game
        lib.cc_debug_fused_tail(mult, keep)
        for i in range(L):
            enc(i)
        out[f"k1_fused_tail{mult}_{keep}"] = {"us": round(timed(enc, a.reps), 2)}
    lib.cc_debug_fused_tail(0, 0)
    if os.environ.get("MB_K1_ONLY"):
        print(json.dumps({"shape": [n, c], "codec": a.codec, **out}))
        return
    # K2: accumulate decode of the last body into each layer's base
    bases = [st.base for st in sts]

    def dec(i):
        lib.cc_decode_step(tag, 1, n, c, 0, _lib.ptr(body), _lib.CC_F32, _lib.ptr(bases[i % L]), stream)

    us = timed(dec, a.reps)
    out["k2_decode"] = {"us": round(us, 2), "alg_GBps": round(n * c * (8 + bits / 8) / us / 1e3, 1)}
    # K2 batched over 7 peers of n/8 rows each (P=8 patch-parallel receive)
    if n % 8 == 0:
        import ctypes
        rows8 = n // 8
        peers = [torch.zeros(rows8, c, device="cuda") for _ in range(7)]
        bod = torch.empty(lib.cc_body_bytes(tag, rows8, c, 0) + 64, dtype=torch.uint8, device="cuda")
        st8 = pl.LayerState("naive", 1, torch.zeros(rows8, c, device="cuda"))
        pl.encode_step(st8, xs[0][:rows8], spec)
        pl.encode_step(st8, xs[1][:rows8], spec, body_out=bod)
        ra = (ctypes.c_int64 * 7)(*([rows8] * 7))
        ba = (ctypes.c_void_p * 7)(*([bod.data_ptr()] * 7))
        pa = (ctypes.c_void_p * 7)(*[q.data_ptr() for q in peers])

        def dec7(i):
            lib.cc_decode_batched(tag, 1, 7, ra, c, 0, ba, _lib.CC_F32, pa, stream)

        us = timed(dec7, a.reps)
        out["k2_decode_7peers_P8"] = {"us": round(us, 2),
                                      "alg_GBps": round(7 * rows8 * c * (8 + bits / 8) / us / 1e3, 1)}
    # low-rank encode (T=2) on this shard: tensor-core vs f64 CUDA-core projections
    from paper_2507_17511_b200 import linalg as la
    xt = xs[0].float()
    for r in (8, 16):
        sp = cx.CompressorSpec(cx.CompressorKind.LOWRANK, rank=r, iterations=2)
        for backend in (1, 0):
            lib.cc_set_lowrank_backend(backend)
            cx.encode_lowrank(xt, sp, la.make_rng(0))
            us = timed(lambda i: cx.encode_lowrank(xt, sp, la.make_rng(i)), 5, graph=False)
            out[f"lowrank_r{r}_{'tc' if backend else 'f64'}"] = {"us": round(us, 1)}
    lib.cc_set_lowrank_backend(1)
    # top-k encode_step (residual + select + ordered write + sparse update)
    for f in (0.01, 0.1):
        sp = cx.CompressorSpec(cx.CompressorKind.TOPK, keep_fraction=f)
        st = pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda"))
        pl.encode_step(st, xs[0], sp)
        pl.encode_step(st, xs[1], sp)
        us = timed(lambda i: pl.encode_step(st, xs[i % 2], sp), 10, graph=False)
        out[f"topk_step_{f}"] = {"us": round(us, 1)}
    # N:M encode_step (one fused pass) and its K2 decode, L2-cold layer rotation
    for (nn, mm) in ((2, 4), (1, 4), (4, 8), (8, 16), (16, 32), (3, 5)):
        prm = _lib.nm_param(nn, mm)
        nb = lib.cc_body_bytes(_lib.CC_NMBLOCK, n, c, prm)
        nbody = torch.empty(nb + 64, dtype=torch.uint8, device="cuda")
        nws_b = lib.cc_workspace_bytes(_lib.CC_NMBLOCK, n, c, prm)
        nws = torch.empty(max(nws_b, 1), dtype=torch.uint8, device="cuda")

        def nenc(i, nn=nn, mm=mm, nbody=nbody, nws=nws, nws_b=nws_b):
            st = sts[i % L]
            lib.cc_nm_encode_step(2, n, c, nn, mm, _lib.ptr(xs[2 * (i % L) + (i // L) % 2]), _lib.CC_BF16,
                                  _lib.ptr(st.base), _lib.ptr(st.feedback), _lib.ptr(nbody), _lib.ptr(nws), nws_b,
                                  _lib.ptr(rec), stream)

        for i in range(L):
            nenc(i)
        us = timed(nenc, a.reps)
        alg_nm = n * c * 18 + nb
        out[f"nm{nn}:{mm}_step"] = {"us": round(us, 2), "alg_GBps": round(alg_nm / us / 1e3, 1)}

        def ndec(i, prm=prm, nbody=nbody):
            lib.cc_decode_step(_lib.CC_NMBLOCK, 1, n, c, prm, _lib.ptr(nbody), _lib.CC_F32,
                               _lib.ptr(bases[i % L]), stream)

        us = timed(ndec, a.reps)
        out[f"nm{nn}:{mm}_decode"] = {"us": round(us, 2), "alg_GBps": round((n * c * 8 + nb) / us / 1e3, 1)}
    # plain copy roofline reference: base -> feedback of another layer
    def cp(i):
        sts[(i + 1) % L].feedback.copy_(sts[i % L].base)

    us = timed(cp, a.reps)
    out["torch_copy_f32"] = {"us": round(us, 2), "GBps": round(2 * n * c * 4 / us / 1e3, 1)}
    print(json.dumps({"shape": [n, c], "codec": a.codec, **out}))


if __name__ == "__main__":
    main()
