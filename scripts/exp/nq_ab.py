"""Per-rank patch / Ulysses step (bench.sim_rank_measure, graph replay, overlapped
decode stream) with the resident K1 at 24 consumer warps (NQ=1) vs 12 register-capped
warps (NQ=2, leaves room for the decode kernel on the SM)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
from paper_2507_17511_b200 import _lib  # noqa: E402

lib = _lib.load()
for nq in (1, 2, 1, 2):
    lib.cc_debug_k1_resident_nq(nq)
    out = {f"patch{P}": bench.sim_rank_measure("patch", P, "quant2bit", 57, 4096, 3072)["ms_per_layer"] * 1e3
           for P in (2, 4, 8)}
    out["ulysses8"] = bench.sim_rank_measure("ulysses", 8, "sign1bit", 57, 4096, 3072)["ms_per_layer"] * 1e3
    print("nq", nq, {k: round(v, 2) for k, v in out.items()}, flush=True)
lib.cc_debug_k1_resident_nq(1)
