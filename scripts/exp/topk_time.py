"""Graph-replayed top-k encode_step (16 layer states, L2-cold rotation) at a shard shape."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_2507_17511_b200 import compressors as cx  # noqa: E402
from paper_2507_17511_b200 import _lib  # noqa: E402
from paper_2507_17511_b200 import pipeline as pl  # noqa: E402

L = 16
lib = _lib.load()
for rows, keep, res in ([] if os.environ.get('TK_TIMELINE_ONLY') else [(r, k, s) for r in (4096, 1024, 512) for k in (0.01, 0.1) for s in ((2, 1, 0) if r == 4096 else (1, 0))]):
        lib.cc_debug_topk_resident(res)
        c0 = lib.cc_debug_topk_resident_count()
        spec = cx.CompressorSpec(cx.CompressorKind.TOPK, keep_fraction=keep)
        g = torch.Generator(device="cuda").manual_seed(0)
        xs = [(torch.randn(rows, 3072, device="cuda", generator=g) * torch.rand(1, 3072, device="cuda", generator=g)
               * 3).to(torch.bfloat16) for _ in range(L)]
        sts = [pl.LayerState("residual_with_feedback", 1, torch.zeros(rows, 3072, device="cuda")) for _ in range(L)]
        for _ in range(2):
            for s, x in zip(sts, xs):
                pl.encode_step(s, x, spec)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for s, x in zip(sts, xs):
                pl.encode_step(s, x, spec)
        gr.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            gr.replay()
        b.record()
        torch.cuda.synchronize()
        used = lib.cc_debug_topk_resident_count() - c0
        print(f"topk {rows}x3072 keep {keep} resident={res} (ran {used}): {1e3 * a.elapsed_time(b) / (10 * L):.1f} us/step",
              flush=True)
        del xs, sts, gr

# per-phase timeline of the resident kernel (globaltimer stamps per CTA)
import json  # noqa: E402
names = ["start", "A_done", "bar1", "find1", "bar2", "list_ready", "warp_counts", "lvl_a", "lvl_b", "selected", "write", "end"]
import bench  # noqa: E402  (FLUX-like inputs of the benchmark)
rows_list = [int(r) for r in os.environ.get("TK_ROWS", "512,1024,2048").split(",")]
for rows, data, keep in [(r, d, k) for r in rows_list for d in ("randscale", "flux") for k in (0.01, 0.1)]:
    lib.cc_debug_topk_resident(2 if rows >= 4096 else 1)
    spec = cx.CompressorSpec(cx.CompressorKind.TOPK, keep_fraction=keep)
    g = torch.Generator(device="cuda").manual_seed(0)
    if data == "flux":  # two consecutive denoising steps per layer, alternated
        pairs = [bench.flux_inputs(rows * 8, 3072, 0, rows, layer, torch.device("cuda")) for layer in range(L)]
    else:
        pairs = [[(torch.randn(rows, 3072, device="cuda", generator=g) * torch.rand(1, 3072, device="cuda", generator=g)
                   * 3).to(torch.bfloat16) for _ in range(2)] for _ in range(L)]
    sts = [pl.LayerState("residual_with_feedback", 1, torch.zeros(rows, 3072, device="cuda")) for _ in range(L)]
    for step in range(4):
        for s, pr in zip(sts, pairs):
            pl.encode_step(s, pr[step % 2], spec)
    tbuf = torch.zeros(1024 * 16, dtype=torch.int64, device="cuda")
    lib.cc_debug_topk_timer(_lib.ptr(tbuf))
    for s, pr in zip(sts, pairs):
        pl.encode_step(s, pr[0], spec)
    torch.cuda.synchronize()
    lib.cc_debug_topk_timer(None)
    tb = tbuf.view(1024, 16).cpu()
    G = int((tb[:, 0] > 0).sum())
    tb = tb[:G].double()
    t0 = tb[:, 0].min()
    print(json.dumps({"rows": rows, "data": data, "keep": keep, "grid": G, "in_b1": int(tb[0, 12]), "list_path": int(tb[0, 13]), "timeline_us": {
        nm: [round(float((tb[:, i] - t0).min()) / 1e3, 2), round(float((tb[:, i] - t0).max()) / 1e3, 2)]
        for i, nm in enumerate(names) if nm}}), flush=True)
