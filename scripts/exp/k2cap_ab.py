"""A/B of the capped K2 grid (CC_K2_CTAS_PER_SM) on the per-rank sims of bench.py.
python scripts/exp/k2cap_ab.py   (run once per env setting)"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402

out = {"cap": os.environ.get("CC_K2_CTAS_PER_SM", "0")}
for name, kind, P, codec, kw in [("patch4", "patch", 4, "quant2bit", None), ("patch8", "patch", 8, "quant2bit", None),
                                 ("patch2", "patch", 2, "quant2bit", None), ("ulysses8", "ulysses", 8, "sign1bit", None),
                                 ("topk1pct_patch8", "patch", 8, "topk", {"keep_fraction": 0.01})]:
    r = bench.sim_rank_measure(kind, P, codec, 57, 4096, 3072, spec_kw=kw)
    out[name] = round(r["ms_per_layer"] * 1e3, 2)
print(json.dumps(out), flush=True)
