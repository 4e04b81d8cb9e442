"""Per-rank low-rank step (bench.sim_rank_measure, graph replay) with the projection
staging variants of cc_debug_lowrank_tma: 2 (default), 1, 0."""
import os
import sys

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
from paper_2507_17511_b200 import _lib  # noqa: E402

lib = _lib.load()
for v in (2, 1, 0, 2):
    lib.cc_debug_lowrank_tma(v, 0)
    r = bench.sim_rank_measure("patch", 4, "lowrank", 8, 4096, 3072, steps=5, warmup=3,
                               spec_kw={"rank": 8, "iterations": 2})
    print("tma", v, r["ms_per_layer"] * 1e3, flush=True)
lib.cc_debug_lowrank_tma(2, 0)
