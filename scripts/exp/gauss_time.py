"""Phase stamps (%globaltimer) of the device Gaussian draw (cc_gaussian_keyed) at [3072, 8]."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_2507_17511_b200 import _lib  # noqa: E402
from paper_2507_17511_b200 import linalg as la  # noqa: E402

lib = _lib.load()
rows, cols = 3072, 8
out = torch.empty(rows, cols, device="cuda")
ws = torch.empty(lib.cc_gaussian_workspace_bytes(rows, cols), dtype=torch.uint8, device="cuda")
key = la.DeviceKey(3, 6, 0, 2, advance=True)
st = torch.zeros(16, dtype=torch.int64, device="cuda")
for i in range(4):
    if i == 3:
        lib.cc_debug_gauss_stamps(_lib.ptr(st))
    _lib.check(lib.cc_gaussian_keyed(rows, cols, _lib.ptr(key.words), key.nwords, key.step_word, _lib.ptr(out),
                                     _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "g")
torch.cuda.synchronize()
lib.cc_debug_gauss_stamps(None)
v = st.cpu().tolist()
names = ["seed", "generate", "list+ticket", "gather", "evaluate", "resolve", "scan", "->out kernel", "outputs"]
print({nm: round((v[i + 1] - v[i]) / 1e3, 2) for i, nm in enumerate(names)}, "total", round((v[9] - v[0]) / 1e3, 2))
