"""Per-rank top-k sims of bench.py under the current environment (A/B of knobs)."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402

out = {"reserve": os.environ.get("CC_TOPK_RESIDENT_RESERVE", "0")}
for f in (0.01, 0.1):
    r = bench.sim_rank_measure("patch", 8, "topk", 57, 4096, 3072, spec_kw={"keep_fraction": f})
    out[f"topk{f}"] = round(r["ms_per_layer"] * 1e3, 2)
print(json.dumps(out), flush=True)
