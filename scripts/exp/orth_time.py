"""Phase stamps (clock64, block 0) of the single-CTA CholQR2 inside one low-rank encode."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_2507_17511_b200 import _lib  # noqa: E402
from paper_2507_17511_b200 import compressors as cx  # noqa: E402
from paper_2507_17511_b200 import linalg as la  # noqa: E402

lib = _lib.load()
lib.cc_debug_orth_cluster(0)  # the single-CTA form carries the stamps
for n in (1024, 3072):
    a = torch.randn(n, 3072, device="cuda")
    spec = cx.CompressorSpec(cx.CompressorKind.LOWRANK, rank=8, iterations=2)
    cx.encode_lowrank(a, spec, la.make_rng(0))
    st = torch.zeros(16, dtype=torch.int64, device="cuda")
    lib.cc_debug_orth_stamps(_lib.ptr(st))
    cx.encode_lowrank(a, spec, la.make_rng(1))  # the last orth of the encode stamps last
    torch.cuda.synchronize()
    lib.cc_debug_orth_stamps(None)
    v = st.cpu().tolist()
    names = ["load", "gram1", "G1", "chol1", "apply1", "gram2", "G2", "chol2", "apply2", "store"]
    print(n, {nm: v[i + 1] - v[i] for i, nm in enumerate(names) if nm != "-" and v[i + 1] and v[i]}, "bad", v[11],
          "total", v[10] - v[0])

# cluster form vs single CTA: low-rank encode time (graph replay of one encode)
import time  # noqa: E402
for n in (1024, 4096):
    a = torch.randn(n, 3072, device="cuda")
    spec = cx.CompressorSpec(cx.CompressorKind.LOWRANK, rank=8, iterations=2)
    key = la.DeviceKey(1, 6, 0, 2, advance=True)
    for cl in (1, 0):
        lib.cc_debug_orth_cluster(cl)
        cx.encode_lowrank(a, spec, key)
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            cx.encode_lowrank(a, spec, key)
            with torch.cuda.graph(g, stream=s):
                for _ in range(10):
                    cx.encode_lowrank(a, spec, key)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        print(f"encode_lowrank [{n}x3072] r8 T2 cluster={cl}: {e0.elapsed_time(e1) * 100:.1f} us")
    lib.cc_debug_orth_cluster(1)
