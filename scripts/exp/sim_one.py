"""One per-rank sim config of bench.sim_rank_measure (for ncu launch lists):
python scripts/exp/sim_one.py topk 8 0.01 | lowrank 4"""
import os
import sys

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402

codec, P = sys.argv[1], int(sys.argv[2])
kw = ({"keep_fraction": float(sys.argv[3])} if codec == "topk"
      else {"rank": 8, "iterations": 2} if codec == "lowrank" else None)
print(bench.sim_rank_measure("patch", P, codec, 4, 4096, 3072, steps=2, warmup=3, spec_kw=kw))
