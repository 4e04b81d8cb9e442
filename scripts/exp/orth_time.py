"""Phase stamps (clock64, block 0) of the single-CTA CholQR2 inside one low-rank encode."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_2507_17511_b200 import _lib  # noqa: E402
from paper_2507_17511_b200 import compressors as cx  # noqa: E402
from paper_2507_17511_b200 import linalg as la  # noqa: E402

lib = _lib.load()
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
