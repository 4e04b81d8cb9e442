"""K1 launches under debug knobs, for ncu launch lists (pure kernel durations).

python scripts/k1_variants.py "pol,stop" ...   e.g.  0,0 0,1 0,3 24,3
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2507_17511_b200 import _lib  # noqa: E402
from paper_2507_17511_b200 import compressors as cx  # noqa: E402
from paper_2507_17511_b200 import pipeline as pl  # noqa: E402

lib = _lib.load()
n, c, L = 4096, 3072, 4
spec = cx.CompressorSpec(cx.CompressorKind.QUANT2BIT)
xs = [(torch.randn(n, c, device="cuda") * torch.rand(1, c, device="cuda") * 3).to(torch.bfloat16) for _ in range(2 * L)]
sts = [pl.LayerState("residual_with_feedback", 1, torch.zeros(n, c, device="cuda")) for _ in range(L)]
for i, st in enumerate(sts):
    pl.encode_step(st, xs[2 * i], spec)
    pl.encode_step(st, xs[2 * i + 1], spec)
tag = cx._spec_tag(spec)
wsb = lib.cc_workspace_bytes(tag, n, c, 0)
ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
body = torch.empty(lib.cc_body_bytes(tag, n, c, 0) + 64, dtype=torch.uint8, device="cuda")
rec = torch.zeros(2, dtype=torch.float64, device="cuda")
stream = _lib.stream_ptr()
torch.cuda.synchronize()
for arg in sys.argv[1:]:
    pol, stop = (int(v) for v in arg.split(","))
    lib.cc_debug_fused_policy(pol)
    lib.cc_debug_fused_stop(stop)
    for i in range(2 * L):
        st = sts[i % L]
        lib.cc_encode_step(tag, 2, 0, n, c, _lib.ptr(xs[2 * (i % L) + (i // L) % 2]), _lib.CC_BF16, _lib.ptr(st.base),
                           _lib.ptr(st.feedback), _lib.ptr(body), _lib.ptr(ws), wsb, _lib.ptr(rec), stream)
    torch.cuda.synchronize()
print("done")
